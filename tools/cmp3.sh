for v in "$@"; do
  if [ "$v" = base ]; then L=paper_1902_09215_b200/libltgp_cuda.so; else L=exp/$v/libltgp_cuda.so; fi
  echo "== $v"
  LTGP_CUDA_LIB=$L python tools/prof_c3.py 3 | tail -1 | cut -c1-140
  LTGP_CUDA_LIB=$L python tools/evolved_pop.py 3000 | tail -1 | cut -c60-190
  LTGP_CUDA_LIB=$L python tools/c4.py --reps 2 --check 0 2>&1 | grep "^eval" | tail -1 | cut -c1-110
done
