"""Streamed evaluation timeline of the config-3 batch (LTGP_TRACE=1 prints,
per slice, when its copy, plan and evaluation ended) at a given chunk length."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_09215_b200 as ltgp  # noqa: E402

if os.environ.get("LTGP_CUDA_LIB"):  # a variant from tools/build_variant.py
    ltgp.CUDA_LIB_PATH = os.environ["LTGP_CUDA_LIB"]

chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
buf, offs, sizes = ltgp.corpus(1, 4000, 4.0, 6.0)
hb = torch.from_numpy(buf).pin_memory().numpy()
suite = ltgp.make_suite(ltgp.suite_seed(1))
with ltgp.Engine([0], node_limit=2**62, chunk_nodes=chunk) as e:
    e.set_suite(*suite)
    for _ in range(3):
        e.evaluate_packed(hb, offs, sizes)
