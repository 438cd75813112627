#!/bin/bash
# Round measurement recipe (one B200): bench line, reference arm, launch
# list, one ncu --set full capture of k_eval. Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-evolution --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_eval" -s 2 -c 1 -o gpurun_out/keval_full \
    python tools/prof_c3.py 2 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"k_plan_warp|k_combine" -c 2 -o gpurun_out/plan_combine_full \
    python tools/prof_c3.py 1 > gpurun_out/ncu_full2.log 2>&1
echo done
