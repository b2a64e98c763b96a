#!/bin/bash
# tools/ktime4.py for every library variant in .variants/ (diagnostic)
cp paper_2511_15629_b200/libesdp.so /tmp/libesdp_orig.so
for v in .variants/libesdp_*.so; do
  cp "$v" paper_2511_15629_b200/libesdp.so
  echo "$v $(python tools/ktime4.py 2>&1 | tail -1)"
done
cp /tmp/libesdp_orig.so paper_2511_15629_b200/libesdp.so
