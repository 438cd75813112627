# A/B timing of interpreter variants (tools/build_variant.py): bash tools/ab_run.sh v1 v2 ...
cd ${GRAFT_REPO_ROOT:-.}
for v in "$@"; do
  if [ "$v" = base ]; then L=paper_1902_09215_b200/libltgp_cuda.so; else L=exp/$v/libltgp_cuda.so; fi
  echo "== $v"
  LTGP_CUDA_LIB=$L python tools/prof_c3.py 3 | tail -1
  LTGP_CUDA_LIB=$L python tools/evolved_pop.py 3000 | tail -1
done
