#!/bin/bash
# One profiling pass for profiles/ (run on the GPU box from the repo root): bench lines (cfg2 main, cfg5
# sweep, reference arm), the launch list of the bench command, per-launch ncu counts of the stage kernels
# (cfg2, cfg4, cfg5 batch) for bench.py's roofline fields, and full captures of the window kernels.
# Every command runs once without ncu (exit 0) before its ncu capture (B200_PROFILING.md).
set -x
O=gpurun_out/prof; mkdir -p $O
M=smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum
timeout 300 python tools/stagetime.py cfg2 > $O/plain_s2.log 2>&1 && \
  timeout 400 ncu --metrics $M --clock-control none -k regex:"window_stencil|contract_dmma3" -s 200 -c 8 --csv \
  --log-file $O/k_cfg2.csv python tools/stagetime.py cfg2 > $O/ncu_k2.log 2>&1
timeout 300 python tools/stagetime.py cfg4 > $O/plain_s4.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none -k regex:"window_stencil|contract_dmma3" -s 200 -c 8 --csv \
  --log-file $O/k_cfg4.csv python tools/stagetime.py cfg4 > $O/ncu_k4.log 2>&1
timeout 300 python tools/batchrun.py > $O/plain_b.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none -k regex:"window_batch|contract_dmma3|contract_pres" -s 300 -c 8 --csv \
  --log-file $O/k_cfg5.csv python tools/batchrun.py > $O/ncu_k5.log 2>&1
python tools/stage_kernels.py $O/r02_stage_kernels.json cfg2=$O/k_cfg2.csv cfg4=$O/k_cfg4.csv cfg5=$O/k_cfg5.csv \
  > $O/stage_kernels.log 2>&1
timeout 300 python bench.py > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
timeout 600 python bench.py --config cfg5 > $O/bench5.log 2>&1; tail -1 $O/bench5.log > $O/bench_cfg5.json
timeout 600 python bench.py --impl reference > $O/ref.log 2>&1; tail -1 $O/ref.log > $O/bench_reference.json
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_l.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
python tools/launches.py $O/launches.csv > $O/launches_summary.txt
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"window_stencil|contract_dmma3" -s 200 -c 2 \
  -o $O/cfg2_stage python tools/stagetime.py cfg2 > $O/ncu_s.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"window_batch|contract_dmma3|contract_pres" -s 300 -c 2 \
  -o $O/cfg5_stage python tools/batchrun.py > $O/ncu_b.log 2>&1
echo done
