#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over a
# reduced -m gpu parity suite: resident and streamed evaluation, chunked
# trees + spine combine, deep Remy trees (window spills), capacity-overflow
# re-runs, device extents + splice. Logs go to gpurun_out/sanitize_<tool>.log.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SEL="test_spec_genomes or test_config3_small_chunked or test_remy_deep_trees or test_adversarial or test_capacity_overflow_reruns or test_execute_generation_children or test_streamed_small_and_outputs or test_subtree_extents"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  echo "== $tool" > gpurun_out/sanitize_$tool.log
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --error-exitcode 7 --target-processes all \
     --print-limit 50 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "$SEL" -p no:cacheprovider \
     >> gpurun_out/sanitize_$tool.log 2>&1
  echo "== rc $?" >> gpurun_out/sanitize_$tool.log
done
