for v in base spec base spec; do
  if [ $v = base ]; then L=paper_1902_09215_b200/libltgp_cuda.so; else L=exp/$v/libltgp_cuda.so; fi
  echo "== $v"; LTGP_CUDA_LIB=$L python tools/prof_c3.py 4 | tail -2
done
