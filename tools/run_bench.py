"""The reference's bench mode (bench.hpp:17-35, driver.hpp:44-51) with every
BenchCell column: tree sizes 1001..1000001, >= 4M nodes per cell, best of 3.

GPU columns come from the engine's run_bench (include/ltgp_host.h): the
1-GPU throughput and the throughput with `workers` GPUs (the reference's
workers become GPUs; cells with more workers than visible GPUs are skipped).
The CPU columns the engine library cannot fill (it has no CPU interpreter:
no fallback) come from the CPU oracle (oracle/, the reference's eval_scalar /
eval_batch restated), timed here on the same trees:
  scalar_gpops    eval_scalar, one fitness case per call (eval.hpp:65-68)
  batch_gpops     eval_batch, all 48 lanes per node, one thread (eval.hpp:70-79)
  vector_speedup  batch / scalar (bench.hpp:21-24: > 1 at size >= 1e5)
  cpu_parallel    eval_batch on every host thread (the reference's workers)
Each CPU column is timed on a bounded sample (~0.3 s of work per column).

  python tools/run_bench.py [workers ...]      (default: 1 2 4 8)
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1902_09215_b200 as ltgp  # noqa: E402
from tests._oracle import load_oracle  # noqa: E402

SIZES = [1001, 10001, 100001, 1000001]
MIN_NODES = 4_000_000
SEED = 1


def cpu_columns(o, suite, n, budget_s=0.3):
    inputs, targets, consts = suite
    count = max(1, (MIN_NODES + n - 1) // n)
    trees = [o.random_tree_of_size(ltgp.tree_seed(SEED, i), n) for i in range(min(count, 64))]
    # scalar: one case per call
    t0, nodes_cases = time.perf_counter(), 0
    cp = consts.ctypes.data_as(C.c_void_p)
    k = 0
    while time.perf_counter() - t0 < budget_s:
        g = trees[k % len(trees)]
        for x in inputs[:8]:
            o.orc_eval_scalar(g.ctypes.data_as(C.c_void_p), g.size, float(x), cp)
        nodes_cases += g.size * 8
        k += 1
    scalar = nodes_cases / (time.perf_counter() - t0)
    # batch (one thread) and all threads, on whole trees
    stride = (n + 15) // 16 * 16
    buf = np.full(stride * len(trees) + 64, 0xFF, np.uint8)
    offs = np.arange(len(trees), dtype=np.uint64) * stride
    for j, g in enumerate(trees):
        buf[j * stride:j * stride + n] = g
    sizes = np.full(len(trees), n, np.uint64)
    res = {}
    for name, threads in (("batch", 1), ("parallel", os.cpu_count() or 1)):
        t0, done = time.perf_counter(), 0
        while time.perf_counter() - t0 < budget_s:
            o.evaluate_population(buf, offs, sizes, suite, threads=threads)
            done += 1
        res[name] = done * len(trees) * n * 48 / (time.perf_counter() - t0)
    return scalar, res["batch"], res["parallel"]


def main():
    workers = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
    import torch
    ngpu = torch.cuda.device_count()
    run = [w for w in workers if w <= ngpu]
    skipped = [w for w in workers if w > ngpu]
    cells = ltgp.run_bench(SIZES, run, seed=SEED, min_corpus_nodes=MIN_NODES, repeats=3)
    o = load_oracle()
    suite = ltgp.make_suite(ltgp.suite_seed(SEED))
    cpu = {n | 1: cpu_columns(o, suite, n | 1) for n in SIZES}
    print(f"host: {os.cpu_count()} threads; GPUs visible: {ngpu}; skipped worker counts (more than the GPUs): {skipped}")
    print(f"{'tree_size':>10} {'gpus':>5} {'nodes':>9} {'scalar':>10} {'batch(1t)':>10} {'vec_x':>6} "
          f"{'cpu_all':>10} {'1-GPU':>10} {'N-GPU':>10} {'N/1':>6} counters")
    rows = []
    for c in cells:
        sc, bt, par = cpu[int(c["tree_size"])]
        row = {"tree_size": int(c["tree_size"]), "workers": int(c["workers"]), "nodes": int(c["nodes"]),
               "scalar_gpops": sc, "batch_gpops": bt, "vector_speedup": bt / sc, "cpu_parallel_gpops": par,
               "gpu_batch_gpops": float(c["batch_gpops"]), "gpu_parallel_gpops": float(c["parallel_gpops"]),
               "parallel_speedup": float(c["parallel_speedup"]), "counters_consistent": bool(c["counters_consistent"])}
        rows.append(row)
        print(f"{row['tree_size']:>10} {row['workers']:>5} {row['nodes']:>9} {sc:>10.3g} {bt:>10.3g} {bt / sc:>6.1f} "
              f"{par:>10.3g} {row['gpu_batch_gpops']:>10.3g} {row['gpu_parallel_gpops']:>10.3g} "
              f"{row['parallel_speedup']:>6.2f} {'ok' if row['counters_consistent'] else 'INCONSISTENT'}")
    print(json.dumps({"cells": rows, "skipped_workers": skipped, "host_threads": os.cpu_count()}))


if __name__ == "__main__":
    main()
