import sys; sys.path.insert(0, "/root/repo")
import paper_1902_09215_b200 as ltgp
with ltgp.Engine([0], node_limit=2**62) as e:
    print(e.run(4000, 200, 2**62, 7, 1, None, 1))
