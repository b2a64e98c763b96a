O=gpurun_out/prof5; mkdir -p $O
M=smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum,gpu__time_duration.sum
timeout 300 python tools/batchrun.py > $O/plain_b.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none -k regex:"window_batch|contract_dmma3|contract_pres" -s 300 -c 8 --csv \
  --log-file $O/k_cfg5.csv python tools/batchrun.py > $O/ncu_k5.log 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"window_batch|contract_dmma3|contract_pres" -s 300 -c 2 \
  -o $O/cfg5_stage python tools/batchrun.py > $O/ncu_b.log 2>&1
echo done
