"""Evaluate an evolved (bloated) population: run config 2 (50/50 grow) for G
generations on the engine, then re-evaluate the final population a few times
and print device time, exits and window adjustments."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

if os.environ.get("LTGP_CUDA_LIB"):  # a variant from tools/build_variant.py
    ltgp.CUDA_LIB_PATH = os.environ["LTGP_CUDA_LIB"]

G = int(sys.argv[1]) if len(sys.argv) > 1 else 200
with ltgp.Engine([0], node_limit=2**62, chunk_nodes=int(os.environ.get("LTGP_CHUNK", "0"))) as e:
    e.run(4000, G, 2**62, 7, 1, None, 1)
    for _ in range(3):
        rec = e.evaluate_population()
        st = e.stats()
        n = int(rec["size"].sum())
        print(f"gen {G}: {n} nodes (mean {n/4000:.0f}, max depth {rec['depth'].max()}), eval {st['eval_seconds']*1e3:.3f} ms "
              f"(decode+plan+k_eval {st['eval_kernel_seconds']*1e3:.3f}, k_eval alone {st['keval_seconds']*1e3:.3f}), {n*48/st['eval_seconds']/1e12:.3f} T GPops/s, "
              f"combine {st['combine_seconds']*1e3:.3f} ms, chunks {st['last_chunks']}, spine steps {st['last_spine_steps']}, "
              f"exits {st['last_exits']}, adjusts {st['last_window_adjusts']}", flush=True)
