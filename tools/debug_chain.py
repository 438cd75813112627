import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1902_09215_b200 as ltgp
from tests._oracle import load_oracle, same_bits
o = load_oracle()
suite = ltgp.make_suite(ltgp.suite_seed(1))
ADD, SUB, X = 0, 1, 4
gs = [np.array([ADD] * 8000 + [X] + [5 + 7] * 8000, np.uint8),
      np.array([SUB] * 5000 + [X] + [5 + (k % 250) for k in range(5000)], np.uint8),
      ltgp.remy_tree(43, 200001)]
for chunk in (0, 64, 4096, 16384):
    for sel in ([0], [1], [2], [0, 1, 2]):
        e = ltgp.Engine([0], node_limit=2**40, chunk_nodes=chunk)
        e.set_suite(*suite)
        e.upload_population([gs[i] for i in sel])
        try:
            rec, outs = e.evaluate_outputs()
            st = e.stats()
            ok = [same_bits(outs[k], o.eval_batch(gs[i], suite[0], suite[2])[0]) for k, i in enumerate(sel)]
            dep = [(int(rec["depth"][k]), o.depth(gs[i])) for k, i in enumerate(sel)]
            print(chunk, sel, "reruns", st["last_fallback_items"], "chunks", st["last_chunks"], "ok", ok, "depth", dep, flush=True)
        except Exception as ex:
            print(chunk, sel, "ERROR", ex, flush=True)
        e.close()
