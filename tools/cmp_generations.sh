for v in ${VARIANTS:-base p5}; do
  if [ "$v" = base ]; then L=paper_1902_09215_b200/libltgp_cuda.so; else L=exp/$v/libltgp_cuda.so; fi
  for g in 100 200 300 600 1000 2000; do echo "$v: $(LTGP_CUDA_LIB=$L python tools/evolved_pop.py $g | tail -1 | cut -c1-110)"; done
done
