"""Debug helper: one streamed evaluation of a small config-3 corpus, with a
host traceback dump if it hangs (cross-slice k_eval bring-up)."""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(40, exit=True)
import paper_1902_09215_b200 as ltgp  # noqa: E402

if os.environ.get("LTGP_CUDA_LIB"):  # a variant from tools/build_variant.py
    ltgp.CUDA_LIB_PATH = os.environ["LTGP_CUDA_LIB"]

trees = int(sys.argv[1]) if len(sys.argv) > 1 else 200
buf, offs, sizes = ltgp.corpus(1, trees, 3.0, 5.0)
with ltgp.Engine([0], node_limit=2**62) as e:
    e.set_suite(*ltgp.make_suite(ltgp.suite_seed(1)))
    e.upload_packed(buf, offs, sizes)
    ref = e.evaluate_population()
    print("resident ok", flush=True)
    t = time.perf_counter()
    got = e.evaluate_packed(buf, offs, sizes)
    print("streamed", "identical" if got.tobytes() == ref.tobytes() else "DIFFERENT", f"{(time.perf_counter()-t)*1e3:.1f} ms", e.stats()["kernel_launches"], flush=True)
