"""Config 2: pop 4000, tournament 7, crossover only, no size limit, G
generations from ramped half-and-half, on the engine (C++ run loop through the
C ABI). Prints per-run totals; with --oracle also runs the CPU oracle's run()
and compares the generation dumps byte for byte."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pop", type=int, default=4000)
    ap.add_argument("--gens", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--limit", type=int, default=2**62)
    ap.add_argument("--shards", type=int, default=1)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--grow", type=int, default=1, help="0: SPEC grow (runs collapse), 1: 50/50 grow (runs bloat)")
    ap.add_argument("--dump", default="/tmp/c2_gpu.txt", help="generation dump path ('' for none)")
    ap.add_argument("--checkpoint", default="", help="checkpoint file (written every --every generations)")
    ap.add_argument("--every", type=int, default=0)
    ap.add_argument("--resume", default="", help="continue the run from this checkpoint")
    a = ap.parse_args()
    if a.oracle and not a.dump:
        ap.error("--oracle compares generation dumps: give --dump a path")
    with ltgp.Engine([0] * a.shards, node_limit=a.limit) as e:
        t = time.perf_counter()
        r = e.run(a.pop, a.gens, a.limit, 7, a.seed, a.dump or None, a.grow,
                  checkpoint=a.checkpoint or None, checkpoint_every=a.every, resume=a.resume or None)
        wall = time.perf_counter() - t
    print(f"engine: {r['generations']} gens, reason {r['reason']}, {r['nodes']} nodes, eval {r['eval_seconds']:.3f} s "
          f"({r['nodes'] * 48 / max(r['eval_seconds'], 1e-9) / 1e12:.3f} T GPops/s eval), wall {wall:.2f} s "
          f"({r['nodes'] * 48 / wall / 1e9:.1f} G GPops/s end to end, {r['generations'] / wall * 3600:.0f} generations/hour)",
          flush=True)
    if a.oracle:
        from tests._oracle import load_oracle
        o = load_oracle()
        t = time.perf_counter()
        ro = o.run(a.pop, a.gens, a.limit, 7, a.seed, 0, a.dump + ".oracle", a.grow)
        wo = time.perf_counter() - t
        same = open(a.dump, "rb").read() == open(a.dump + ".oracle", "rb").read()
        print(f"oracle: {ro['generations']} gens, {ro['nodes']} nodes, wall {wo:.2f} s "
              f"({ro['nodes'] * 48 / wo / 1e9:.1f} G GPops/s); dumps identical: {same}", flush=True)


if __name__ == "__main__":
    main()
