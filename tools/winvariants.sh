#!/bin/bash
# Window-stencil variants (outputs per thread, fast vs generic queries) on cfg2, cfg4 and a cfg5 batch:
# bash tools/winvariants.sh > gpurun_out/winvariants.log
for g in 0 1; do
  for o in 1 2; do ESDP_WIN_GENERIC=$g ESDP_WIN_OPT=$o python tools/stagetime.py cfg2 | sed "s/^/generic=$g opt=$o /"; done
  for o in 2 4; do ESDP_WIN_GENERIC=$g ESDP_WIN_OPT=$o python tools/stagetime.py cfg4 | sed "s/^/generic=$g opt=$o /"; done
  for o in 2 4; do ESDP_WIN_GENERIC=$g ESDP_WIN_OPT=$o python tools/batchrun.py 128 | sed "s/^/generic=$g opt=$o /"; done
done
