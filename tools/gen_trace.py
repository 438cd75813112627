import os, sys, time
sys.path.insert(0, "/root/repo")
import paper_1902_09215_b200 as ltgp
G = int(sys.argv[1])
with ltgp.Engine([0], node_limit=15_000_000) as e:
    e.run(4000, G, 15_000_000, 7, 1, None, 1)
    rec = e.evaluate_population()
    os.environ["LTGP_TRACE"] = "1"
    for g in range(3):
        plans = ltgp.plan_generation(1000 + g, rec, 7)
        t = time.perf_counter()
        rec, hit = e.execute_generation(plans)
        print(f"-- gen +{g}: {1e3*(time.perf_counter()-t):.3f} ms wall, eval {e.stats()['eval_seconds']*1e3:.3f} ms", file=sys.stderr, flush=True)
