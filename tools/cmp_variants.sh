#!/bin/bash
# Time kernel variants built by tools/build_variant.py on the config-3 batch:
#   bash tools/cmp_variants.sh base v1 v2 ...   (base = the product library)
for v in "$@"; do
  if [ "$v" = base ]; then L=paper_1902_09215_b200/libltgp_cuda.so; else L=exp/$v/libltgp_cuda.so; fi
  echo "== $v"; LTGP_CUDA_LIB=$L python tools/prof_c3.py 3 | tail -1
done
