"""Config 2 end to end under the current LTGP_DEVICE_GEN / LTGP_GEN_GRAPH
settings: a warm-up run, then a timed 200-generation run (pop 4000, k 7,
50/50 grow) with its generation dump written to the path given; prints one
JSON line. tools/devgen_ab.sh runs it for the host path, the device path
with plain launches and the device path as a CUDA graph, and compares dumps.
Usage: python tools/devgen_ab.py DUMP [GENS]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

dump = sys.argv[1]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 200
with ltgp.Engine([0], node_limit=2**62) as e:
    e.run(4000, G, 2**62, 7, 1, None, 1)
    t0 = time.perf_counter()
    r = e.run(4000, G, 2**62, 7, 1, None, 1)
    wall = time.perf_counter() - t0
    e.run(4000, G, 2**62, 7, 1, dump, 1)
print(json.dumps({"device_gen": os.environ.get("LTGP_DEVICE_GEN", "1"), "graph": os.environ.get("LTGP_GEN_GRAPH", "1"),
                  "generations": r["generations"], "nodes": r["nodes"], "wall_s": wall,
                  "eval_s": r["eval_seconds"], "e2e_gpops": r["nodes"] * 48 / wall,
                  "eval_gpops": r["nodes"] * 48 / r["eval_seconds"], "ms_per_gen": wall / G * 1e3}), flush=True)
