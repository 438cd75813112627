#!/bin/bash
# config-2 run wall time with the libraries of exp/<name>/ (both .so files)
for v in "$@"; do
  for i in 1 2; do
    echo "== $v: $(python - "$v" <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1902_09215_b200 as ltgp
v = sys.argv[1]
ltgp.CUDA_LIB_PATH = f"exp/{v}/libltgp_cuda.so"
ltgp.HOST_LIB_PATH = f"exp/{v}/libltgp_host.so"
with ltgp.Engine([0], node_limit=2**62) as e:
    t = time.perf_counter(); r = e.run(4000, 200, 2**62, 7, 1, None, 1); w = time.perf_counter() - t
print(f"wall {w:.3f} s eval {r['eval_seconds']:.3f} s")
PY
)"
  done
done
