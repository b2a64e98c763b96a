#!/bin/bash
# tools/ktime4.py (cfg4-shaped chain, warm contract launch) for every dmma3 variant in .variants/ (diagnostic)
cp paper_2511_15629_b200/libesdp.so /tmp/libesdp_orig.so
for v in .variants/libesdp_d3_*.so; do
  cp "$v" paper_2511_15629_b200/libesdp.so
  echo "$v $(ESDP_DMMA3=1 python tools/ktime4.py 2>&1 | tail -1)"
done
cp /tmp/libesdp_orig.so paper_2511_15629_b200/libesdp.so
if [ "$1" = "cfg5" ]; then
  for v in .variants/libesdp_d3_*.so; do
    cp "$v" paper_2511_15629_b200/libesdp.so
    echo "$v cfg5 $(ESDP_DMMA3=1 python bench.py --config cfg5 --instances 64 --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-190)"
  done
  cp /tmp/libesdp_orig.so paper_2511_15629_b200/libesdp.so
fi
