cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests -m gpu -x -q -k "streamed or packed or randomized or error_behaviour or nccl" > gpurun_out/r2o_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2o_test.log
grep -q "pytest exit 0" gpurun_out/r2o_test.log || exit 1
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-evolution --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench e2e', d['e2e']['value']/1e12, 'value', d['value']/1e12)"; done > gpurun_out/r2o.log 2>&1
LTGP_TRACE=1 timeout 120 python tools/trace_streamed.py 2>&1 | grep "ltgp trace" | tail -1 >> gpurun_out/r2o.log
