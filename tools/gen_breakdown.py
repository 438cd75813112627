"""Per-generation time breakdown of a bloated config-2/5 population: run G
generations (50/50 grow, so trees bloat; node limit 15M as in config 5), then
time further execute_generation calls from Python: wall clock of the call,
device time of k_splice and of the evaluation, and the rest (extent scan,
host work, launches and synchronisation inside the call).
Usage: python tools/gen_breakdown.py [G] [extra_generations]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

if os.environ.get("LTGP_CUDA_LIB"):
    ltgp.CUDA_LIB_PATH = os.environ["LTGP_CUDA_LIB"]

G = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
X = int(sys.argv[2]) if len(sys.argv) > 2 else 6
with ltgp.Engine([0], node_limit=15_000_000) as e:
    t = time.perf_counter()
    r = e.run(4000, G, 15_000_000, 7, 1, None, 1)
    print(f"{r['generations']} generations in {time.perf_counter() - t:.1f} s (reason {r['reason']})", flush=True)
    rec = e.evaluate_population()
    for g in range(X):
        t0 = time.perf_counter()
        plans = ltgp.plan_generation(1000 + g, rec, 7)
        t1 = time.perf_counter()
        rec, hit = e.execute_generation(plans)
        t2 = time.perf_counter()
        if hit:
            print("size limit hit")
            break
        st = e.stats()
        n = int(rec["size"].sum())
        sp, ev = st["splice_seconds"], st["eval_seconds"]
        wall = t2 - t1
        print(f"+{g}: {n / 1e9:.3f} G nodes; plan {1e3 * (t1 - t0):.2f} ms; execute_generation {1e3 * wall:.2f} ms = "
              f"splice {1e3 * sp:.2f} ms ({2 * n / sp / 1e9:.0f} GB/s of 2 B/node) + evaluation "
              f"{1e3 * ev:.2f} ms ({n * 48 / ev / 1e12:.2f} T GPops/s) + other {1e3 * (wall - sp - ev):.2f} ms",
              flush=True)
