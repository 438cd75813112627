#!/bin/bash
# e2e (streamed evaluate_packed) throughput of bench.py across slice counts / slice sizes
for cfg in "32 24" "40 20" "48 16" "56 14" "64 12" "64 8"; do
  set -- $cfg
  echo "slices<=$1 slice_mb=$2: $(LTGP_SLICES=$1 LTGP_SLICE_KB=$(( $2 * 1024 )) python bench.py --steps 8 --warmup 3 --no-evolution --no-cpu-baseline 2>/dev/null | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["e2e"]["value"]/1e12,3), "T e2e;", round(d["value"]/1e12,3), "T value")')"
done
