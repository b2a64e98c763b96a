for cv in -1 def; do
  if [ $cv = def ]; then unset ESDP_CARVEOUT; else export ESDP_CARVEOUT=$cv; fi
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c.log 2>&1; tail -1 gpurun_out/c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cv', '$cv', 'cfg2', round(d['ms_per_step'],4), round(d['e2e']['value']/1e12,3))"
  for c in cfg2-rank1 cfg3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/c.log 2>&1; tail -1 gpurun_out/c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cv', '$cv', '$c', round(d['ms_per_step'],4))"; done
  timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c.log 2>&1; tail -1 gpurun_out/c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cv', '$cv', 'cfg4', round(d['ms_per_step'],3))"
  timeout 600 python bench.py --config cfg5 --no-cpu-baseline > gpurun_out/c.log 2>&1; tail -1 gpurun_out/c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cv', '$cv', 'cfg5', round(d['ms_per_step'],3))"
  timeout 600 python bench.py --config table3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c.log 2>&1; tail -1 gpurun_out/c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cv', '$cv', 'table3', round(d['ms_per_step'],3))"
  timeout 600 python bench.py --config table3 --t3-hours 4 --t3-delta 0.1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c.log 2>&1; tail -1 gpurun_out/c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cv', '$cv', 'table3-small', round(d['ms_per_step'],3))"
done
