#!/usr/bin/env python3
"""Experiment helper: compile the current csrc/ into exp/<name>/libltgp_cuda.so
(same flags as the product build) so several kernel variants can be timed in
one GPU call with tools/prof_c3.py (LTGP_CUDA_LIB=exp/<name>/libltgp_cuda.so)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1902_09215_b200 import build as B  # noqa: E402

name = sys.argv[1]
extra = sys.argv[2:]
out = os.path.join(ROOT, "exp", name)
os.makedirs(out, exist_ok=True)
B._run(["g++", *B.CXX_FLAGS, "-c", "-o", os.path.join(out, "ltgp_pack.o"), B.PACK_SRC])
B._run(["nvcc", *B.NVCC_FLAGS, *extra, "-shared", "-o", os.path.join(out, "libltgp_cuda.so"),
        os.path.join(B.CSRC, "ltgp_engine.cu"), os.path.join(out, "ltgp_pack.o")], log=os.path.join(out, "ptxas.log"))
B.patch_jump_tables(os.path.join(out, "libltgp_cuda.so"), verbose=True)
print("built", out)
