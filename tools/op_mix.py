import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1902_09215_b200 as ltgp
def mix(trees, label):
    h = np.zeros(256, np.int64)
    pairs = np.zeros((5, 5), np.int64)
    for g in trees:
        h += np.bincount(g, minlength=256)
        c = np.minimum(g, 4)
        n = len(c) // 2 * 2
        r = c[::-1][:n]  # scan order
        np.add.at(pairs, (r[0::2], r[1::2]), 1)
    tot = h.sum()
    print(label, "nodes", tot, "ADD %.3f SUB %.3f MUL %.3f DIV %.3f X %.3f CONST %.3f" % tuple(
        [h[i] / tot for i in range(5)] + [h[5:].sum() / tot]))
    p = pairs / pairs.sum()
    print("  pairs LL %.3f FL+LF %.3f FF %.3f  div-in-pair %.3f" % (p[4, 4], p[4, :4].sum() + p[:4, 4].sum(), p[:4, :4].sum(), p[3, :].sum() + p[:, 3].sum()))
G = int(sys.argv[1])
with ltgp.Engine([0], node_limit=15_000_000) as e:
    e.run(4000, G, 15_000_000, 7, 1, None, 1)
    trees = [e.download_genome(i) for i in range(0, 4000, 4)]
mix(trees, f"evolved gen {G}")
buf, offs, sizes = ltgp.corpus(1, 200, 4.0, 6.0)
mix([buf[int(o):int(o) + int(s)] for o, s in zip(offs, sizes)], "config 3")
