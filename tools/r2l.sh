cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -x -q -k "streamed or packed" > gpurun_out/r2l_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2l_test.log
bash tools/pack_probe.sh > gpurun_out/r2l_probe.log 2>&1
for i in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-evolution --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench e2e', d['e2e']['value']/1e12, 'value', d['value']/1e12)"; done > gpurun_out/r2l.log 2>&1
L=paper_1902_09215_b200/libltgp_cuda.so
for t in 14 12; do echo "== threads $t" >> gpurun_out/r2l.log; LTGP_PACK_THREADS=$t timeout 120 python tools/e2e_ab.py $L | tail -1 >> gpurun_out/r2l.log; done
