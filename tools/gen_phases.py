"""Per-generation host phases of config 2 (pop 4000, k 7, 50/50 grow, 200
generations) from LTGP_TRACE: the run loop's plan_generation and
execute_generation wall times and the engine's phase marks, averaged over a
second (warm) run. Usage: python tools/gen_phases.py [GENS]"""
import collections
import os
import re
import sys
import tempfile

os.environ["LTGP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 200
log = tempfile.NamedTemporaryFile(delete=False, suffix=".log").name
saved = os.dup(2)
with open(log, "w") as f:
    os.dup2(f.fileno(), 2)
    try:
        with ltgp.Engine([0], node_limit=2**62) as e:
            e.run(4000, G, 2**62, 7, 1, None, 1)
            sys.stderr.flush()
            print("=== timed run", file=sys.stderr, flush=True)
            e.run(4000, G, 2**62, 7, 1, None, 1)
    finally:
        sys.stderr.flush()
        os.dup2(saved, 2)
text = open(log).read().split("=== timed run", 1)[1]
sums, counts = collections.defaultdict(float), collections.defaultdict(int)
for m in re.finditer(r"gen \d+: plan_generation ([\d.]+) us, execute_generation ([\d.]+) us, (\d+) draws", text):
    for k, v in (("plan_generation", m.group(1)), ("execute_generation", m.group(2)), ("draws", m.group(3))):
        sums[k] += float(v)
        counts[k] += 1
for m in re.finditer(r"\[ltgp\] (\S[^\n]*?)\s+([\d.]+) us\n", text):
    k = m.group(1).strip()
    if k.startswith("gen "):
        continue
    sums[k] += float(m.group(2))
    counts[k] += 1
for k in sums:
    print(f"{k:24s} {sums[k] / max(counts[k], 1):9.1f} us avg over {counts[k]}")
