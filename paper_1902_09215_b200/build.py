"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  libltgp_cuda.so  — sm_100a kernels + the C ABI (include/ltgp_cuda.h)
  libltgp_host.so  — C++ host API mirroring the reference (include/ltgp_host.h)

The oracle (test infrastructure) is built by oracle/Makefile, see
__graft_entry__.build().
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")

CUDA_LIB = os.path.join(PKG, "libltgp_cuda.so")
# host packing of streamed slices (csrc/ltgp_pack.h): g++, linked into CUDA_LIB
PACK_SRC = os.path.join(CSRC, "ltgp_pack.cpp")
PACK_OBJ = os.path.join(CSRC, "ltgp_pack.o")
HOST_LIB = os.path.join(PKG, "libltgp_host.so")

# Bit-exactness flags: one IEEE RN op per node, no
# FMA contraction, IEEE division, denormals preserved.
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xptxas", "-v",
]
CXX_FLAGS = ["-std=c++20", "-O3", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall", "-pthread"]


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))
    return r


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps(dirname, exts):
    out = []
    for base, _, files in os.walk(dirname):
        for f in files:
            if f.endswith(exts):
                out.append(os.path.join(base, f))
    return out


def patch_jump_tables(lib: str, verbose: bool = False) -> None:
    """Post-build step on a freshly linked libltgp_cuda.so (patch_jt.py): fails
    the build if the interpreter's dispatch sites do not end up on one table."""
    if PKG not in sys.path:
        sys.path.insert(0, PKG)
    import patch_jt
    patch_jt.patch(lib, verbose=verbose)
    patch_jt.verify(lib)


def build(force: bool = False, verbose: bool = False) -> None:
    nvcc = os.environ.get("NVCC", "nvcc")
    cu_deps = _deps(CSRC, (".cu", ".cuh", ".h")) + [os.path.join(ROOT, "include", "ltgp_cuda.h")]
    cu_deps += [PACK_SRC, os.path.join(PKG, "patch_jt.py")]
    if force or _stale(CUDA_LIB, cu_deps):
        _run(["g++", *CXX_FLAGS, "-c", "-o", PACK_OBJ, PACK_SRC])
        _run([nvcc, *NVCC_FLAGS, "-shared", "-o", CUDA_LIB, os.path.join(CSRC, "ltgp_engine.cu"), PACK_OBJ],
             log=os.path.join(CSRC, "ptxas.log"))
        # the direct-threaded interpreter's jump-table copies become one (see patch_jt.py)
        patch_jump_tables(CUDA_LIB, verbose)
    host_deps = _deps(HOST, (".cpp", ".hpp")) + [os.path.join(ROOT, "include", "ltgp_host.h"), CUDA_LIB]
    if force or _stale(HOST_LIB, host_deps):
        _run(["g++", *CXX_FLAGS, "-shared", "-o", HOST_LIB, os.path.join(HOST, "ltgp_host.cpp"),
              "-L" + PKG, "-lltgp_cuda", "-Wl,-rpath,$ORIGIN"])
    build_refabi(force)
    if verbose:
        print("built", CUDA_LIB, HOST_LIB)


REF_INC = "/root/reference/proj/include"
REFABI_LIB = os.path.join(PKG, "libltgp_refabi.so")
REFABI_SRC = os.path.join(HOST, "evolve_cuda.cpp")
REF_RUN_SRC = os.path.join(ROOT, "tests", "refabi", "ref_run.cpp")
REF_RUN_BIN = os.path.join(ROOT, "tests", "refabi", "_bin", "ref_run")


def build_refabi(force: bool = False) -> bool:
    """libltgp_refabi.so: the reference-typed drop-in (evolve_cuda.cpp),
    compiled against the reference's unmodified headers where they lie, plus
    the reference-typed test harness tests/refabi/_bin/ref_run. Built only
    when /root/reference is present (this container); the built files travel
    to the GPU box like the other .so files. Returns whether they exist."""
    if not os.path.isdir(REF_INC):
        return os.path.exists(REFABI_LIB)
    inc = ["-I" + REF_INC, "-I" + os.path.join(ROOT, "include")]
    deps = [REFABI_SRC, os.path.join(ROOT, "include", "ltgp_refabi.h"), CUDA_LIB]
    if force or _stale(REFABI_LIB, deps):
        _run(["g++", *CXX_FLAGS, *inc, "-shared", "-o", REFABI_LIB, REFABI_SRC,
              "-L" + PKG, "-lltgp_cuda", "-Wl,-rpath,$ORIGIN"])
    oracle_lib = os.path.join(ROOT, "oracle", "libltgp_oracle.so")
    if os.path.exists(oracle_lib) and (force or _stale(REF_RUN_BIN, [REF_RUN_SRC, REFABI_LIB, oracle_lib])):
        os.makedirs(os.path.dirname(REF_RUN_BIN), exist_ok=True)
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-Wall", *inc, "-o", REF_RUN_BIN, REF_RUN_SRC,
              "-L" + PKG, "-lltgp_refabi", "-lltgp_cuda", "-L" + os.path.dirname(oracle_lib), "-lltgp_oracle",
              "-Wl,-rpath,$ORIGIN/../../../paper_1902_09215_b200:$ORIGIN/../../../oracle"])
    return True


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
