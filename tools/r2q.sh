cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2q_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2q_test.log
( for v in 0 1 0 1; do echo "== RXS=$v"; LTGP_RXS=$v timeout 120 python tools/prof_c3.py 3 | tail -1; LTGP_RXS=$v timeout 200 python tools/evolved_pop.py 3000 | tail -1; done ) > gpurun_out/r2q.log 2>&1
L=paper_1902_09215_b200/libltgp_cuda.so
timeout 120 python tools/e2e_ab.py $L | tail -1 >> gpurun_out/r2q.log
