#!/bin/bash
# One profiling pass for profiles/ (run on the GPU box from the repo root): bench lines, the launch list of
# the bench command, full captures of the stage kernels (cfg2, cfg4, cfg5 batch), and the FP64 metric names.
# Every command runs once without ncu (exit 0) before its ncu capture (B200_PROFILING.md).
set -x
O=gpurun_out/prof; mkdir -p $O
ncu --query-metrics 2>/dev/null | grep -iE "fp64|dmma|dfma|dadd|dmul" > $O/fp64_metric_names.txt
timeout 300 python bench.py > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
timeout 600 python bench.py --impl reference > $O/ref.log 2>&1; tail -1 $O/ref.log > $O/bench_reference.json
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_l.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches_summary.txt
timeout 300 python tools/stagetime.py cfg2 > $O/plain_s.log 2>&1 && \
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"window_stencil|contract_dmma3" -s 200 -c 2 \
  -o $O/cfg2_stage python tools/stagetime.py cfg2 > $O/ncu_s.log 2>&1
timeout 300 python tools/batchrun.py > $O/plain_b.log 2>&1 && \
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"window_batch|contract_dmma3" -s 300 -c 2 \
  -o $O/cfg5_stage python tools/batchrun.py > $O/ncu_b.log 2>&1
echo done
