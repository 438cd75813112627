"""Config 2 (pop 4000, 200 generations, 50/50 grow) with LTGP_TRACE: host
plan_generation and execute_generation wall time per generation and the
engine's phase marks, averaged over the run (second run: buffers warm)."""
import os
import re
import subprocess
import sys

if os.environ.get("C2_CHILD"):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import time
    import paper_1902_09215_b200 as ltgp
    with ltgp.Engine([0], node_limit=2**62) as e:
        e.run(4000, 200, 2**62, 7, 1, None, 1)
        print("=== timed run", file=sys.stderr, flush=True)
        t = time.perf_counter()
        r = e.run(4000, 200, 2**62, 7, 1, None, 1)
        wall = time.perf_counter() - t
    print(f"=== wall {wall * 1e3:.1f} ms, {r['nodes'] * 48 / wall / 1e12:.3f} T GPops/s e2e, "
          f"eval {r['eval_seconds'] * 1e3:.1f} ms", file=sys.stderr, flush=True)
    sys.exit(0)

env = dict(os.environ, C2_CHILD="1", LTGP_TRACE="1")
p = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
err = p.stderr.split("=== timed run", 1)[-1]
sums, cnt = {}, {}
for line in err.splitlines():
    m = re.match(r"\[ltgp\] gen (\d+): plan_generation ([\d.]+) us, execute_generation ([\d.]+) us", line)
    if m:
        for k, v in (("plan_generation", m.group(2)), ("execute_generation", m.group(3))):
            sums[k] = sums.get(k, 0.0) + float(v)
            cnt[k] = cnt.get(k, 0) + 1
        continue
    m = re.match(r"\[ltgp\]\s+(.+?)\s+([\d.]+) us$", line)
    if m:
        k = m.group(1).strip()
        sums[k] = sums.get(k, 0.0) + float(m.group(2))
        cnt[k] = cnt.get(k, 0) + 1
for k in sums:
    print(f"{k:32s} {sums[k] / cnt[k]:9.1f} us avg over {cnt[k]}")
print([l for l in err.splitlines() if l.startswith("===")])
if p.returncode:
    print(p.stderr[-3000:])
