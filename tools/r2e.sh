# streamed e2e: cross-slice k_eval A/B (every step under its own timeout)
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q -k "streamed or packed" > gpurun_out/r2e_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2e_test.log
grep -q "pytest exit 0" gpurun_out/r2e_test.log || exit 1
L=paper_1902_09215_b200/libltgp_cuda.so
timeout 120 python tools/prof_c3.py 3 > gpurun_out/r2e_res.log 2>&1
( echo "== per-slice k_eval"; LTGP_XSLICE=0 timeout 120 python tools/e2e_ab.py $L | tail -1
  for r in 6 12 20; do for n in 24 48; do echo "== xslice plan_sms $r slices $n"; LTGP_PLAN_SMS=$r LTGP_SLICES=$n timeout 120 python tools/e2e_ab.py $L | tail -1; done; done ) > gpurun_out/r2e_ab.log 2>&1
LTGP_TRACE=1 timeout 120 python tools/trace_streamed.py > gpurun_out/r2e_trace.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "randomized or error_behaviour" > gpurun_out/r2e_test2.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2e_test2.log
