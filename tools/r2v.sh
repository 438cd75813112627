#!/bin/bash
# branch-free spine combine: GPU suite, config 4 A/B (LTGP_COMBINE_BF), bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/r2v_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2v_test.log
for bf in 1 0; do
  echo "== LTGP_COMBINE_BF=$bf"; LTGP_COMBINE_BF=$bf timeout 600 python tools/c4.py --trees 48 --nodes 10000001 --check 6 --reps 3
done > gpurun_out/r2v_c4.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-evolution --no-cpu-baseline > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err
