"""The reference's bench mode (bench.hpp:33-35, driver.hpp:44-51) on the engine:
tree sizes 1001..1000001, >= 4M nodes per cell, best of 3, GPU counts given
on the command line (default 1). Prints one row per BenchCell."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

gpus = [int(x) for x in sys.argv[1:]] or [1]
cells = ltgp.run_bench([1001, 10001, 100001, 1000001], gpus, seed=1, min_corpus_nodes=4_000_000, repeats=3)
print(f"{'tree_size':>10} {'gpus':>5} {'nodes':>10} {'1-GPU GPops/s':>14} {'N-GPU GPops/s':>14} {'speedup':>8} counters")
for c in cells:
    print(f"{c['tree_size']:>10} {c['workers']:>5} {c['nodes']:>10} {c['batch_gpops']:>14.4g} {c['parallel_gpops']:>14.4g} "
          f"{c['parallel_speedup']:>8.2f} {'ok' if c['counters_consistent'] else 'INCONSISTENT'}")
