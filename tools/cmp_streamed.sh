for v in base xs6 xs8 base xs6 xs8; do
  if [ "$v" = base ]; then L=paper_1902_09215_b200/libltgp_cuda.so; else L=exp/$v/libltgp_cuda.so; fi
  echo "== $v $(LTGP_CUDA_LIB=$L LTGP_TRACE=1 python tools/trace_streamed.py 2>&1 | grep 'to the last record' | tail -2 | tr '\n' ' ')"
done
