"""Regenerate the golden fixtures (run in the build container, where
/root/reference exists):

  ref_inline_kats.json  — known answers printed by oracle/_ref/ref_kat, which
                          is compiled from the REFERENCE's own headers
                          (rng.hpp, eval.hpp inline code; oracle/Makefile `ref`)
  oracle_golden.json    — frozen outputs of the oracle once it passes every
                          reference KAT and SPEC example (tests/test_oracle.py):
                          suites, a config-1 population evaluation, per-case
                          outputs of seeded config-3 trees.

    python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def ref_kats():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True, capture_output=True)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_kat")], check=True, capture_output=True,
                         text=True).stdout
    data = json.loads(out)
    with open(os.path.join(HERE, "ref_inline_kats.json"), "w") as f:
        json.dump(data, f)


def oracle_golden():
    from tests._oracle import load_oracle
    o = load_oracle()
    g = {"suites": {}, "c1": {}, "trees": []}
    for s in (1, 2, 3):
        i, t, c = o.make_suite(o.orc_suite_seed(s))
        g["suites"][str(s)] = {"inputs": i.view(np.uint32).tolist(), "targets": t.view(np.uint32).tolist(),
                               "constants": c.view(np.uint32).tolist()}
        pop = o.ramped(s, 48)
        sizes = np.array([p.size for p in pop], np.uint64)
        offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
        buf = np.concatenate(pop + [np.zeros(16, np.uint8)])
        rec = o.evaluate_population(buf, offs, sizes, (i, t, c), threads=1)
        g["c1"][str(s)] = {"genomes": [p.tolist() for p in pop],
                           "fitness_bits": rec["fitness"].view(np.uint32).tolist(),
                           "hits": rec["hits"].tolist(), "size": rec["size"].tolist(),
                           "depth": rec["depth"].tolist()}
    i, t, c = o.make_suite(o.orc_suite_seed(1))
    for k, n in enumerate([1, 3, 5, 63, 255, 1001, 4097, 20001]):
        tree = o.random_tree_of_size(1000 + k, n)
        out, _ = o.eval_batch(tree, i, c)
        g["trees"].append({"seed": 1000 + k, "n": n, "outputs_bits": out.view(np.uint32).tolist(),
                           "fitness_bits": int(np.float32(o.fitness(out, t)).view(np.uint32)),
                           "hits": o.hits(out, t), "depth": o.depth(tree)})
    with open(os.path.join(HERE, "oracle_golden.json"), "w") as f:
        json.dump(g, f)


if __name__ == "__main__":
    if os.path.isdir("/root/reference"):
        ref_kats()
    oracle_golden()
