cd $GRAFT_REPO_ROOT
timeout 300 python tools/evolved_io.py dump 3000 /tmp/evo3000.npz > gpurun_out/r2r.log 2>&1
for v in 0 1; do LTGP_RXS=$v timeout 120 python tools/evolved_io.py eval /tmp/evo3000.npz 3 >> gpurun_out/r2r.log 2>&1; done
for v in 0 1; do echo "== c3 RXS=$v" >> gpurun_out/r2r.log; LTGP_RXS=$v timeout 120 python tools/prof_c3.py 3 | tail -1 >> gpurun_out/r2r.log; done
timeout 120 python tools/e2e_ab.py paper_1902_09215_b200/libltgp_cuda.so | tail -1 >> gpurun_out/r2r.log
