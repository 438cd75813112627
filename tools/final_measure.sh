#!/bin/bash
# Round measurement recipe (one B200): parity suite, bench line, reference
# arm, launch list, one ncu --set full capture of k_eval. Outputs in
# gpurun_out/. (Under ncu the streamed path uses per-slice launches: the
# engine turns the cross-slice launch off when CUDA_INJECTION64_PATH is set.)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_final.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
LTGP_TRACE=1 timeout 120 python tools/trace_streamed.py > gpurun_out/trace_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-evolution --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_eval" -s 1 -c 1 -o gpurun_out/keval_full \
    python tools/prof_c3.py 2 > gpurun_out/ncu_full.log 2>&1
echo done
