#!/bin/bash
# tools/ktime.py (cfg2 chain, warm contract launch) for every dmma3 variant in .variants/, forced on (diagnostic)
cp paper_2511_15629_b200/libesdp.so /tmp/libesdp_orig.so
for v in .variants/libesdp_d3_*.so; do
  cp "$v" paper_2511_15629_b200/libesdp.so
  echo "$v $(ESDP_DMMA3=1 python tools/ktime.py 2>&1 | head -1)"
done
cp /tmp/libesdp_orig.so paper_2511_15629_b200/libesdp.so
