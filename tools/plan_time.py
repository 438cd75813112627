import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1902_09215_b200 as ltgp
rec = np.zeros(4000, ltgp.RECORD_DTYPE)
rng = np.random.default_rng(0)
rec["fitness"] = rng.random(4000).astype(np.float32)
rec["size"] = rng.integers(1, 5000, 4000)
for _ in range(3): ltgp.plan_generation(1, rec, 7)
t = time.perf_counter()
for i in range(200): ltgp.plan_generation(i, rec, 7)
print(f"plan_generation M=4000 k=7: {(time.perf_counter()-t)/200*1e3:.3f} ms per call (incl. ctypes)")
