# Round-2 final-build long runs: config 5 (10^4 generations, 15M cap) with a
# 2000-generation dump comparison against the oracle, and config 4 at full
# BASELINE scale with all 48 trees checked against the oracle.
cd $GRAFT_REPO_ROOT
( timeout 900 python tools/run_c2.py --gens 10000 --limit 15000000 --grow 1 --dump ""
  timeout 900 python tools/run_c2.py --gens 2000 --limit 15000000 --grow 1 --dump /tmp/c5.txt --oracle ) > gpurun_out/r2u_c5.log 2>&1
timeout 1500 python tools/c4.py --trees 48 --nodes 400000001 --reps 2 --check 48 > gpurun_out/r2u_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_c4.log
