"""A/B of the streamed (e2e) evaluation: libraries given on the command line
(paths), each timed on the config-3 batch from pinned memory, interleaved."""
import os
import subprocess
import sys

CODE = r'''
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1902_09215_b200 as ltgp
ltgp.CUDA_LIB_PATH = sys.argv[1]
buf, offs, sizes = ltgp.corpus(1, 4000, 4.0, 6.0)
hb = torch.from_numpy(buf).pin_memory().numpy()
with ltgp.Engine([0], node_limit=2**62) as e:
    e.set_suite(*ltgp.make_suite(ltgp.suite_seed(1)))
    for _ in range(3): e.evaluate_packed(hb, offs, sizes)
    torch.cuda.synchronize()
    t = time.perf_counter(); n = 10
    for _ in range(n): e.evaluate_packed(hb, offs, sizes)
    dt = (time.perf_counter() - t) / n
    print(f"{sys.argv[1]}: {dt*1e3:.3f} ms per call, {int(sizes.sum())*48/dt/1e12:.3f} T GPops/s")
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        subprocess.run([sys.executable, "-c", CODE, lib], check=True)
