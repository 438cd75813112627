"""Config 4 at configurable scale: T uniform-random (Remy) trees of N nodes,
evaluated as one population; checks `--check` trees against the oracle."""
import argparse
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

if os.environ.get("LTGP_CUDA_LIB"):  # a variant from tools/build_variant.py
    ltgp.CUDA_LIB_PATH = os.environ["LTGP_CUDA_LIB"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trees", type=int, default=48)
    ap.add_argument("--nodes", type=int, default=10_000_001)
    ap.add_argument("--check", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--chunks", default="", help="comma list of chunk lengths to time on the same trees (a sweep)")
    ap.add_argument("--ops", default="",
                    help="remap function opcodes (e.g. '0120': division -> add) to study the op mix")
    ap.add_argument("--cpu-trees", type=int, default=0,
                    help="time the CPU oracle (evaluate_population, all host threads) on this many trees")
    a = ap.parse_args()
    n = a.nodes | 1
    t = time.perf_counter()
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        trees = list(ex.map(lambda i: ltgp.remy_tree(7000 + i, n), range(a.trees)))
    print(f"generated {a.trees} x {n} nodes in {time.perf_counter() - t:.1f} s", flush=True)
    if a.ops:  # opcodes 0..3 -> the given ones (leaves unchanged)
        lut = np.arange(256, dtype=np.uint8)
        lut[:4] = [int(c) for c in a.ops]
        trees = [lut[g] for g in trees]
    suite = ltgp.make_suite(ltgp.suite_seed(1))
    for c in [int(x) for x in a.chunks.split(",") if x][:-1]:
        with ltgp.Engine([0], node_limit=2**62, chunk_nodes=c) as e:
            e.set_suite(*suite)
            e.upload_population(trees)
            for _ in range(a.reps):
                e.evaluate_population()
                st = e.stats()
                print(f"chunk {c}: eval {st['eval_seconds']*1e3:.1f} ms (k_eval {st['keval_seconds']*1e3:.1f}, combine "
                      f"{st['combine_seconds']*1e3:.1f}) {a.trees*n*48/st['eval_seconds']/1e12:.3f} T GPops/s, chunks "
                      f"{st['last_chunks']}, reruns {st['last_fallback_items']}, spine steps {st['last_spine_steps']}", flush=True)
    if a.chunks:
        a.chunk = int(a.chunks.split(",")[-1])
    with ltgp.Engine([0], node_limit=2**62, chunk_nodes=a.chunk) as e:
        e.set_suite(*suite)
        e.upload_population(trees)
        for _ in range(a.reps):
            rec, outs = e.evaluate_outputs()
            st = e.stats()
            tot = a.trees * n
            print(f"eval {st['eval_seconds']*1e3:.1f} ms (decode+plan+k_eval {st['eval_kernel_seconds']*1e3:.1f}, k_eval alone "
                  f"{st['keval_seconds']*1e3:.1f}, combine "
                  f"{st['combine_seconds']*1e3:.1f}) {tot*48/st['eval_seconds']/1e12:.3f} T GPops/s, chunks "
                  f"{st['last_chunks']}, reruns {st['last_fallback_items']}, exits {st['last_exits']}, "
                  f"adjusts {st['last_window_adjusts']}, spine steps {st['last_spine_steps']}", flush=True)
    if a.cpu_trees:  # the reference's CPU path (oracle port), one tree per thread as the reference does
        from tests._oracle import load_oracle
        o = load_oracle()
        k = min(a.cpu_trees, a.trees)
        offs = np.zeros(k, np.uint64)
        sizes = np.full(k, n, np.uint64)
        stride = (n + 15) // 16 * 16
        buf = np.full(stride * k + 64, 0xFF, np.uint8)
        for j in range(k):
            offs[j] = j * stride
            buf[j * stride:j * stride + n] = trees[j]
        t = time.perf_counter()
        o.evaluate_population(buf, offs, sizes, suite, threads=0)
        dt = time.perf_counter() - t
        print(f"cpu oracle: {k} trees x {n} nodes in {dt:.2f} s on {os.cpu_count()} threads: "
              f"{k * n * 48 / dt / 1e12:.4f} T GPops/s", flush=True)
    if a.check:
        # every checked tree: all 48 per-case outputs and the exact record
        # (fitness bits, hits, size, depth) against the oracle, trees checked
        # in parallel (ctypes releases the GIL inside the oracle)
        from tests._oracle import load_oracle, same_bits
        o = load_oracle()

        def check(k):
            out, _ = o.eval_batch(trees[k], suite[0], suite[2])
            fit = o.fitness(out, suite[1])
            ok = (same_bits(outs[k], out) and same_bits([rec["fitness"][k]], [fit])
                  and rec["hits"][k] == o.hits(out, suite[1]) and rec["size"][k] == trees[k].size
                  and rec["depth"][k] == o.depth(trees[k]))
            return k, ok
        t = time.perf_counter()
        with ThreadPoolExecutor(os.cpu_count()) as ex:
            res = list(ex.map(check, range(min(a.check, a.trees))))
        for k, ok in res:
            print(f"tree {k}: size {rec['size'][k]}, depth {rec['depth'][k]}, fitness {rec['fitness'][k]!r}, "
                  f"hits {rec['hits'][k]}: matches oracle: {ok}", flush=True)
        print(f"checked {len(res)} trees against the oracle in {time.perf_counter() - t:.1f} s: "
              f"{sum(ok for _, ok in res)} match", flush=True)


if __name__ == "__main__":
    main()
