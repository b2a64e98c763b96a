#!/bin/bash
# Small (latency-regime) DMMA tilings on cfg2 (ESDP_D3S_MT/NT/WC/KC/NS): bash tools/variants_d3s.sh
VARIANTS=${VARIANTS:-"1,2,2,16,4 2,1,2,16,4 2,2,1,16,4 2,1,1,16,4 2,2,2,16,4 2,1,2,32,2 2,1,2,16,2 2,1,4,16,4"}
for w in $VARIANTS; do
  set -- ${w//,/ }
  make clean > /dev/null
  make EXTRA="-DESDP_D3S_MT=$1 -DESDP_D3S_NT=$2 -DESDP_D3S_WC=$3 -DESDP_D3S_KC=$4 -DESDP_D3S_NS=$5" all > /dev/null 2>&1 || { echo "build failed $w"; continue; }
  echo "MT NT WC KC NS = $w: $(python tools/stagetime.py cfg2 | sed 's/^cfg2 kind=[0-9]*: //' | cut -c1-80)"
done
make clean > /dev/null; make all > /dev/null 2>&1
