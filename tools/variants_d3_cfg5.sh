#!/bin/bash
# DMMA expectation tilings on the cfg5 batch GEMM and cfg4 (large-output tiling, ESDP_D3_MT/NT/WC/KC/NS):
# bash tools/variants_d3_cfg5.sh > gpurun_out/d3_cfg5.log
VARIANTS=${VARIANTS:-"2,2,4,16,4 2,4,2,16,4 2,2,4,16,3 2,2,4,32,3 4,2,2,16,4 2,2,8,16,3 1,4,4,16,4 2,4,4,16,2 4,4,2,16,2"}
for w in $VARIANTS; do
  v=${w//,/ }
  set -- $v
  make clean > /dev/null
  make EXTRA="-DESDP_D3_MT=$1 -DESDP_D3_NT=$2 -DESDP_D3_WC=$3 -DESDP_D3_KC=$4 -DESDP_D3_NS=$5" all > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "MT NT WC KC NS = $v: $(python tools/batchrun.py 128 | sed 's/.*expectation/expectation/') | cfg4 $(python tools/stagetime.py cfg4 | sed 's/.*contract/contract/' | cut -c1-22)"
done
make clean > /dev/null; make all > /dev/null 2>&1
