#!/bin/bash
# Time library variants (.variants/libesdp_*.so) with one bench configuration each (diagnostic):
# tools/variants.sh "<bench args>" -> one line per variant with ms_per_step and ms_per_part
cp paper_2511_15629_b200/libesdp.so /tmp/libesdp_orig.so
for v in .variants/libesdp_*.so; do
  cp "$v" paper_2511_15629_b200/libesdp.so
  python bench.py $1 --no-cpu-baseline 2>/dev/null | tail -1 > /tmp/v.json
  python -c "import json,sys; d=json.load(open('/tmp/v.json')); print(sys.argv[1], round(d['ms_per_step'],4), d.get('ms_per_part'))" "$v"
done
cp /tmp/libesdp_orig.so paper_2511_15629_b200/libesdp.so
