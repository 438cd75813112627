"""Device crossover bandwidth: run the engine's run() for G generations (50/50
grow, so trees bloat), then time further generations driven from Python and
report the splice kernel's device time (ltgp_stats.splice_seconds) per
generation against the bytes the splice moves (children written + the same
bytes read from parents: 2 B/node)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
with ltgp.Engine([0], node_limit=2**62) as e:
    e.run(4000, G, 2**62, 7, 1, None, 1)
    rec = e.evaluate_population()
    for g in range(5):
        plans = ltgp.plan_generation(1000 + g, rec, 7)
        rec, hit = e.execute_generation(plans)
        assert not hit
        st = e.stats()
        n = int(rec["size"].sum())
        s = st["splice_seconds"]
        print(f"generation +{g}: children {n} nodes (mean {n / 4000:.0f}); splice {s * 1e3:.3f} ms: "
              f"{2 * n / s / 1e9:.0f} GB/s of 2 B/node; evaluation {st['eval_seconds'] * 1e3:.3f} ms", flush=True)
