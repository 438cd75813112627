"""Evaluate one evolved (config-2, generation G) population at several fixed
chunk lengths: how per-item overheads trade against parallelism on small
populations."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 200
suite = ltgp.make_suite(ltgp.suite_seed(1))
with ltgp.Engine([0], node_limit=2**62) as e:
    e.run(4000, G, 2**62, 7, 1, None, 1)
    genomes = [e.download_genome(i) for i in range(e.population_size())]
n = sum(g.size for g in genomes)
ref = None
for chunk in (0, 1024, 2048, 4096, 8192, 16384):
    with ltgp.Engine([0], node_limit=2**62, chunk_nodes=chunk) as e:
        e.set_suite(*suite)
        e.upload_population(genomes)
        best = 1e9
        for _ in range(5):
            rec = e.evaluate_population()
            st = e.stats()
            best = min(best, st["eval_seconds"])
        ref = rec if ref is None else ref
        assert rec.tobytes() == ref.tobytes()
        print(f"chunk {chunk or 'auto'}: {best * 1e3:.3f} ms ({n * 48 / best / 1e12:.3f} T GPops/s), "
              f"chunks {st['last_chunks']}, exits {st['last_exits']}", flush=True)
