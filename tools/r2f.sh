# cross-slice k_eval: e2e sweep (each step under its own timeout)
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q -k "streamed or packed" > gpurun_out/r2f_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2f_test.log
L=paper_1902_09215_b200/libltgp_cuda.so
( for n in 32 48 64; do for t in 15 12; do echo "== slices $n threads $t"; LTGP_PACK_THREADS=$t LTGP_SLICES=$n timeout 120 python tools/e2e_ab.py $L | tail -1; done; done ) > gpurun_out/r2f_ab.log 2>&1
LTGP_SLICES=48 LTGP_TRACE=1 timeout 120 python tools/trace_streamed.py > gpurun_out/r2f_trace.log 2>&1
