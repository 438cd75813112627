"""Profiling driver: evaluate the config-3 batch (bench.py workload) a few
times on cuda:0 so ncu can capture k_eval / k_combine. Not a bench."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1902_09215_b200 as ltgp  # noqa: E402

if os.environ.get("LTGP_CUDA_LIB"):  # a variant from tools/build_variant.py
    ltgp.CUDA_LIB_PATH = os.environ["LTGP_CUDA_LIB"]


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    trees = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
    buf, offs, sizes = ltgp.corpus(1, trees, 4.0, 6.0)
    with ltgp.Engine([0], chunk_nodes=int(os.environ.get("LTGP_CHUNK", "0"))) as e:
        e.set_suite(*ltgp.make_suite(ltgp.suite_seed(1)))
        e.upload_packed(buf, offs, sizes)
        for _ in range(reps):
            t = time.perf_counter()
            rec = e.evaluate_population()
            st = e.stats()
            print(f"{sizes.sum()} nodes: {st['eval_seconds']*1e3:.3f} ms device "
                  f"(decode+plan+k_eval {st['eval_kernel_seconds']*1e3:.3f} ms, k_eval alone {st['keval_seconds']*1e3:.3f} ms, combine {st['combine_seconds']*1e3:.3f} ms), "
                  f"{sizes.sum()*48/st['eval_seconds']/1e12:.3f} TGPops/s, wall {1e3*(time.perf_counter()-t):.1f} ms, "
                  f"chunks {st['last_chunks']}, exits {st['last_exits']}, window adjusts {st['last_window_adjusts']}", flush=True)
        assert rec["hits"].min() >= 0


if __name__ == "__main__":
    main()
