#!/bin/bash
# A/B of the tapered work-list tail (LTGP_TAPER) on the config-3 batch.
# Usage: gpurun -- 'bash tools/taper_sweep.sh > gpurun_out/taper.log 2>&1'
for rep in 1 2; do
for t in 0 "0.75,0.5,0.5" "1,1,1" "0.5,0.5,0.5" "1,0.5,0.25" "0.5,0.25,0" "1,0,0" "1.5,1,0.5" "0.5,0.5,1"; do
  echo "== LTGP_TAPER=$t"
  LTGP_TAPER=$t python tools/prof_c3.py 5 | tail -2
done
done
