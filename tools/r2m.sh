cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-evolution --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "exit $?" >> gpurun_out/ncu_launch.log
