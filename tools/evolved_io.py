"""Evolved population to / from a file: `dump G path` runs config 2 for G
generations and writes the final genomes; `eval path [reps]` uploads them
and evaluates (an ncu target that contains only the evaluations)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

if os.environ.get("LTGP_CUDA_LIB"):
    ltgp.CUDA_LIB_PATH = os.environ["LTGP_CUDA_LIB"]

if sys.argv[1] == "dump":
    G, path = int(sys.argv[2]), sys.argv[3]
    with ltgp.Engine([0], node_limit=2**62) as e:
        e.run(4000, G, 2**62, 7, 1, None, 1)
        gs = [e.download_genome(k) for k in range(e.population_size())]
    sizes = np.array([g.size for g in gs], np.uint64)
    np.savez(path, buf=np.concatenate(gs), sizes=sizes)
    print("dumped", len(gs), int(sizes.sum()), "nodes")
else:
    path, reps = sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 2
    d = np.load(path)
    buf, sizes = d["buf"], d["sizes"]
    starts = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
    gs = [buf[int(s):int(s) + int(n)] for s, n in zip(starts, sizes)]
    with ltgp.Engine([0], node_limit=2**62) as e:
        e.set_suite(*ltgp.make_suite(ltgp.suite_seed(1)))
        e.upload_population(gs)
        for _ in range(reps):
            rec = e.evaluate_population()
            st = e.stats()
            print(f"{int(sizes.sum())} nodes: eval {st['eval_seconds']*1e3:.3f} ms (k_eval {st['keval_seconds']*1e3:.3f}, combine {st['combine_seconds']*1e3:.3f})", flush=True)
