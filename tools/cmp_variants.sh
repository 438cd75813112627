#!/bin/bash
# Time kernel variants built by tools/build_variant.py (base = the product
# library): config 3 (prof_c3), an evolved population (evolved_pop 3000) and
# config 4 at 48 x 1e7 nodes (c4).   bash tools/cmp_variants.sh base v1 ...
for v in "$@"; do
  if [ "$v" = base ]; then L=paper_1902_09215_b200/libltgp_cuda.so; else L=exp/$v/libltgp_cuda.so; fi
  echo "== $v"
  LTGP_CUDA_LIB=$L python tools/prof_c3.py 3 | tail -1
  [ -n "$CMP_EVOLVED" ] && LTGP_CUDA_LIB=$L python tools/evolved_pop.py 3000 | tail -1
  [ -n "$CMP_EVO200" ] && LTGP_CUDA_LIB=$L python tools/evolved_pop.py 200 | tail -1
  [ -n "$CMP_C4" ] && LTGP_CUDA_LIB=$L python tools/c4.py --reps 2 --check 1 2>&1 | tail -2
done
