#!/bin/bash
# One profiling pass for profiles/ (run on the GPU box from the repo root): bench lines, the launch list of
# the bench command, full captures of the two stage kernels, and the DRAM bytes of one cfg2 backward.
set -x
O=gpurun_out/prof; mkdir -p $O
timeout 300 python bench.py > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
timeout 600 python bench.py --impl reference > $O/ref.log 2>&1; tail -1 $O/ref.log > $O/bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 > $O/ncu_launches.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches_summary.txt
timeout 400 ncu --set full --import-source on --clock-control none -k regex:window_stencil -s 100 -c 1 -o $O/window \
  python bench.py --steps 1 --warmup 3 > $O/ncu_w.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:contract_dmma3 -s 100 -c 1 -o $O/dmma3 \
  python bench.py --steps 1 --warmup 3 > $O/ncu_d.log 2>&1
timeout 400 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
  --clock-control none -s 1152 -c 576 --csv --log-file $O/traffic.csv python tools/traffic.py > $O/ncu_t.log 2>&1
python tools/traffic_sum.py $O/traffic.csv > $O/traffic_sum.json
