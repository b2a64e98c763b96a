#!/bin/bash
# bench lines of every configuration (run on the GPU box from the repo root) -> gpurun_out/cfgs/
O=gpurun_out/cfgs; mkdir -p $O
for c in cfg2-rank1 cfg3 table1; do timeout 300 python bench.py --config $c > $O/$c.log 2>&1; tail -1 $O/$c.log > $O/$c.json; done
timeout 300 python bench.py --config cfg3 --stencil brute > $O/cfg3-brute.log 2>&1; tail -1 $O/cfg3-brute.log > $O/cfg3-brute.json
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 > $O/cfg4.log 2>&1; tail -1 $O/cfg4.log > $O/cfg4.json
for n in 16 64 128; do timeout 600 python bench.py --config cfg5 --instances $n --steps 5 --warmup 3 > $O/cfg5_$n.log 2>&1; tail -1 $O/cfg5_$n.log > $O/cfg5_$n.json; done
timeout 600 python bench.py --config cfg5 --contract ozaki --steps 5 --warmup 3 --no-cpu-baseline > $O/cfg5_ozaki.log 2>&1; tail -1 $O/cfg5_ozaki.log > $O/cfg5_ozaki.json
rm -f $O/table3_rows.jsonl
for hd in "4 0.1" "20 0.1" "100 0.1" "4 0.01" "20 0.01" "100 0.01"; do set -- $hd
  timeout 600 python bench.py --config table3 --t3-hours $1 --t3-delta $2 --steps 3 --warmup 3 > $O/t3.log 2>&1; tail -1 $O/t3.log >> $O/table3_rows.jsonl; done
