"""B200 fitness-evaluation engine for GPquick-style GP (arXiv 1902.09215).

Python view of the two native libraries built in-tree by ``build.py``:

* ``libltgp_cuda.so`` — the sm_100a engine behind the C ABI in
  ``include/ltgp_cuda.h`` (the drop-in for the reference's
  ``evaluate_population`` / ``execute_generation``,
  /root/reference/proj/include/ltgp/evolve.hpp:106-117).
* ``libltgp_host.so`` — the C++ host side that keeps the reference's RNG,
  tree construction, tournament and crossover planning
  (``include/ltgp_host.h``).

There is no CPU evaluation path here: if the CUDA library is missing or no
B200 is visible, engine construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# (LTGP_CUDA_LIB: a kernel variant from tools/build_variant.py, for experiments)
CUDA_LIB_PATH = os.environ.get("LTGP_CUDA_LIB") or os.path.join(_PKG, "libltgp_cuda.so")
HOST_LIB_PATH = os.path.join(_PKG, "libltgp_host.so")

LANES = 48
CONSTANTS = 250
MAX_SHARDS = 16

RECORD_DTYPE = np.dtype([("fitness", "<f4"), ("hits", "<i4"), ("size", "<u4"), ("depth", "<u4")])
GEN_STATS_DTYPE = np.dtype([("best_index", "<u4"), ("best_fitness", "<f4"), ("best_hits", "<i4"),
                            ("best_size", "<u4"), ("best_depth", "<u4"), ("convergence", "<u4"),
                            ("max_size", "<u4"), ("pad", "<u4"), ("sum_size", "<u8"), ("sum_depth", "<u8"),
                            ("sum_fitness", "<f8")])
PLAN_DTYPE = np.dtype([("mum_index", "<u4"), ("dad_index", "<u4"), ("mum_pt", "<u4"), ("dad_pt", "<u4")])
BENCH_CELL_DTYPE = np.dtype([("tree_size", "<u8"), ("workers", "<u4"), ("nodes", "<u8"), ("scalar_gpops", "<f8"),
                             ("batch_gpops", "<f8"), ("parallel_gpops", "<f8"), ("vector_speedup", "<f8"),
                             ("parallel_speedup", "<f8"), ("counters_consistent", "<i4")], align=True)


class EngineError(RuntimeError):
    pass


class _Config(C.Structure):
    _fields_ = [("n_shards", C.c_int), ("devices", C.c_int * MAX_SHARDS), ("node_limit", C.c_uint64),
                ("arena_bytes", C.c_uint64), ("chunk_nodes", C.c_uint32), ("use_nccl", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("nodes_evaluated", C.c_uint64), ("eval_seconds", C.c_double),
                ("eval_kernel_seconds", C.c_double), ("combine_seconds", C.c_double),
                ("splice_seconds", C.c_double), ("gather_seconds", C.c_double),
                ("arena_high_water", C.c_uint64), ("last_chunks", C.c_uint64),
                ("last_fallback_items", C.c_uint64), ("last_exits", C.c_uint64),
                ("last_window_adjusts", C.c_uint64), ("last_spine_steps", C.c_uint64),
                ("kernel_launches", C.c_uint32), ("gather_nccl", C.c_uint32), ("keval_seconds", C.c_double),
                ("live_genomes_high_water", C.c_uint64), ("arena_used_high_water", C.c_uint64),
                ("last_h2d_bytes", C.c_uint64)]


_cuda = None
_host = None

# every symbol include/ltgp_cuda.h declares, with its ctypes signature
_P = C.c_void_p
_CUDA_SIGS = {
    "ltgp_last_error": (C.c_char_p, []),
    "ltgp_version": (C.c_char_p, []),
    "ltgp_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ltgp_engine_create": (C.c_int, [C.POINTER(_Config), C.POINTER(_P)]),
    "ltgp_engine_destroy": (C.c_int, [_P]),
    "ltgp_set_suite": (C.c_int, [_P, _P, _P, _P]),
    "ltgp_set_memory_budget": (C.c_int, [_P, C.c_uint64]),
    "ltgp_set_streaming": (C.c_int, [_P, C.c_int, C.c_uint32]),
    "ltgp_generation_stats": (C.c_int, [_P, _P]),
    "ltgp_upload_population": (C.c_int, [_P, C.c_uint32, _P, _P]),
    "ltgp_upload_packed": (C.c_int, [_P, C.c_uint32, _P, C.c_uint64, _P, _P]),
    "ltgp_evaluate_packed": (C.c_int, [_P, C.c_uint32, _P, C.c_uint64, _P, _P, _P, _P]),
    "ltgp_evaluate_population": (C.c_int, [_P, _P, _P]),
    "ltgp_evaluate_outputs": (C.c_int, [_P, _P, _P]),
    "ltgp_evaluate_launch": (C.c_int, [_P]),
    "ltgp_evaluate_collect": (C.c_int, [_P, _P, _P]),
    "ltgp_execute_generation": (C.c_int, [_P, _P, C.c_uint32, _P, C.POINTER(C.c_int)]),
    "ltgp_execute_generation_launch": (C.c_int, [_P, _P, C.c_uint32]),
    "ltgp_execute_generation_finish": (C.c_int, [_P, _P, C.POINTER(C.c_int)]),
    "ltgp_download_genome": (C.c_int, [_P, C.c_uint32, _P, C.c_uint64, C.POINTER(C.c_uint64)]),
    "ltgp_eval_one": (C.c_int, [_P, _P, C.c_uint64, _P]),
    "ltgp_eval_one_record": (C.c_int, [_P, _P, C.c_uint64, _P, _P]),
    "ltgp_subtree_extents": (C.c_int, [_P, C.c_uint32, _P, _P, _P]),
    "ltgp_get_stats": (C.c_int, [_P, C.POINTER(_Stats)]),
    "ltgp_population_size": (C.c_uint32, [_P]),
    "ltgp_shard_records": (C.c_int, [_P, C.c_int, C.POINTER(_P), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint32), C.POINTER(_P)]),
    "ltgp_nccl_unique_id": (C.c_int, [_P]),
    "ltgp_nccl_attach": (C.c_int, [_P, _P, C.c_int, C.c_int]),
    "ltgp_gathered_records": (C.c_int, [_P, _P, C.c_uint32, C.POINTER(C.c_uint32)]),
    "ltgp_pack_bound": (C.c_uint64, [C.c_uint64]),
    "ltgp_pack_host": (C.c_uint64, [_P, C.c_uint64, _P, C.c_int]),
}
_HOST_SIGS = {
    "ltgp_host_splitmix64": (C.c_uint64, [C.c_uint64]),
    "ltgp_host_suite_seed": (C.c_uint64, [C.c_uint64]),
    "ltgp_host_make_suite": (None, [C.c_uint64, _P, _P, _P]),
    "ltgp_host_corpus": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_uint32, C.c_uint32,
                                      _P, _P, _P, C.c_int]),
    "ltgp_host_tree_seed": (C.c_uint64, [C.c_uint64, C.c_uint32]),
    "ltgp_host_rng_selftest": (C.c_int, []),
    "ltgp_host_random_tree_of_size": (C.c_int, [C.c_uint64, C.c_uint64, _P]),
    "ltgp_host_remy_tree": (C.c_int, [C.c_uint64, C.c_uint64, _P]),
    "ltgp_host_ramped": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.c_int, _P,
                                      C.c_uint64, _P]),
    "ltgp_host_plan_generation": (None, [C.c_uint64, C.c_uint32, _P, C.c_uint32, _P]),
    "ltgp_host_run": (C.c_int64, [_P, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.c_uint64,
                                  C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_double)]),
    "ltgp_host_run_bench": (C.c_int, [_P, C.c_uint32, _P, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, _P]),
    "ltgp_host_run_checkpointed": (C.c_int64, [_P, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                               C.c_int, C.c_uint64, C.c_char_p, C.c_char_p, C.c_uint32,
                                               C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_uint64),
                                               C.POINTER(C.c_double)]),
}


def _bind(lib, sigs):
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)  # AttributeError if the library lacks a declared symbol
        f.restype = res
        f.argtypes = args


def cuda_lib():
    """Load libltgp_cuda.so (RTLD_GLOBAL so libltgp_host.so resolves it)."""
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_LIB_PATH):
            raise EngineError(f"{CUDA_LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        lib = C.CDLL(CUDA_LIB_PATH, mode=C.RTLD_GLOBAL)
        _bind(lib, _CUDA_SIGS)
        _cuda = lib
    return _cuda


def host_lib():
    global _host
    if _host is None:
        cuda_lib()
        if not os.path.exists(HOST_LIB_PATH):
            raise EngineError(f"{HOST_LIB_PATH} is missing: run __graft_entry__.build()")
        lib = C.CDLL(HOST_LIB_PATH, mode=C.RTLD_GLOBAL)
        _bind(lib, _HOST_SIGS)
        _host = lib
    return _host


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _err():
    return cuda_lib().ltgp_last_error().decode(errors="replace")


def _check(status):
    if status != 0:
        raise EngineError(_err())


def nccl_unique_id() -> bytes:
    """A communicator id for Engine.nccl_attach (made on one rank, broadcast
    by the caller)."""
    buf = np.zeros(128, np.uint8)
    _check(cuda_lib().ltgp_nccl_unique_id(_ptr(buf)))
    return buf.tobytes()


def pack_host(buf: np.ndarray, threads: int = 1) -> np.ndarray:
    """The packed PCIe form of a byte range (ltgp_pack.h), as a streamed
    evaluation sends it: host code, no GPU needed."""
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    lib = cuda_lib()
    out = np.zeros(lib.ltgp_pack_bound(buf.nbytes), dtype=np.uint8)
    n = lib.ltgp_pack_host(_ptr(buf), buf.nbytes, _ptr(out), threads)
    if n == 0 and buf.nbytes:
        raise EngineError(_err())
    return out[:n]


# --------------------------------------------------------------------------
# host side (C++): rng / suite / generators / planning
# --------------------------------------------------------------------------
def splitmix64(x: int) -> int:
    return int(host_lib().ltgp_host_splitmix64(x))


def suite_seed(run_seed: int) -> int:
    return int(host_lib().ltgp_host_suite_seed(run_seed))


def make_suite(seed: int):
    """TestSuite (sextic.hpp:25-51): (inputs[48], targets[48], constants[250])."""
    i = np.zeros(LANES, np.float32)
    t = np.zeros(LANES, np.float32)
    c = np.zeros(CONSTANTS, np.float32)
    host_lib().ltgp_host_make_suite(seed, _ptr(i), _ptr(t), _ptr(c))
    return i, t, c


def corpus_sizes(seed: int, count: int, lg_lo: float = 4.0, lg_hi: float = 6.0) -> np.ndarray:
    """Tree sizes of the config-3 corpus (cheap: no trees are built)."""
    sizes = np.zeros(count, np.uint64)
    host_lib().ltgp_host_corpus(seed, count, lg_lo, lg_hi, 0, 0, None, None, _ptr(sizes), 0)
    return sizes


def corpus(seed: int, count: int, lg_lo: float = 4.0, lg_hi: float = 6.0, threads: int = 0, pinned=None,
           first: int = 0, n: int | None = None):
    """Config-3 style evaluation corpus: trees [first, first+n) of the
    ``count``-tree corpus. Returns (buf uint8, offsets u64, sizes u64) with
    offsets relative to buf (16-byte aligned) and sizes of the range.

    ``pinned``: optional callable(nbytes) -> writable uint8 array (e.g. a
    view of pinned host memory) to hold the packed buffer."""
    h = host_lib()
    n = count - first if n is None else n
    sizes = np.zeros(count, np.uint64)
    offs = np.zeros(max(n, 1), np.uint64)
    total = int(h.ltgp_host_corpus(seed, count, lg_lo, lg_hi, first, n, None, _ptr(offs), _ptr(sizes), threads))
    buf = pinned(total + 64) if pinned else np.empty(total + 64, np.uint8)
    h.ltgp_host_corpus(seed, count, lg_lo, lg_hi, first, n, _ptr(buf), _ptr(offs), _ptr(sizes), threads)
    return buf, offs[:n], sizes[first:first + n].copy()


def tree_seed(seed: int, i: int) -> int:
    return int(host_lib().ltgp_host_tree_seed(seed, i))


def random_tree_of_size(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint8)
    _check_host(host_lib().ltgp_host_random_tree_of_size(seed, n, _ptr(out)), "random_tree_of_size")
    return out


def remy_tree(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint8)
    _check_host(host_lib().ltgp_host_remy_tree(seed, n, _ptr(out)), "remy_tree")
    return out


def ramped_half_and_half(seed: int, count: int, capacity: int = 15_000_000, dmin: int = 2, dmax: int = 6):
    sizes = np.zeros(count, np.uint64)
    cap = count * 64 + 64
    out = np.empty(cap, np.uint8)
    total = int(host_lib().ltgp_host_ramped(seed, count, capacity, dmin, dmax, _ptr(out), cap, _ptr(sizes)))
    if total == 0:
        raise ValueError("ramped_half_and_half failed (capacity)")
    genomes, pos = [], 0
    for s in sizes:
        genomes.append(out[pos:pos + int(s)].copy())
        pos += int(s)
    return genomes


def plan_generation(seed: int, records: np.ndarray, k: int = 7) -> np.ndarray:
    records = np.ascontiguousarray(records, RECORD_DTYPE)
    out = np.zeros(len(records), PLAN_DTYPE)
    host_lib().ltgp_host_plan_generation(seed, len(records), _ptr(records), k, _ptr(out))
    return out


def run_bench(tree_sizes, worker_counts=(1,), seed: int = 1, min_corpus_nodes: int = 4_000_000,
              repeats: int = 3) -> np.ndarray:
    """run_bench (bench.hpp:33-35) on the engine: one BenchCell per (tree
    size, GPU count); see include/ltgp_host.h."""
    ts = np.ascontiguousarray(tree_sizes, np.uint64)
    wc = np.ascontiguousarray(worker_counts, np.uint32)
    out = np.zeros(ts.size * wc.size, BENCH_CELL_DTYPE)
    st = host_lib().ltgp_host_run_bench(_ptr(ts), ts.size, _ptr(wc), wc.size, seed, min_corpus_nodes, repeats,
                                        _ptr(out))
    if st != 0:
        raise EngineError(_err() or "ltgp_host_run_bench failed")
    return out


def _check_host(status, what):
    if status != 0:
        raise ValueError(f"{what} failed")


# --------------------------------------------------------------------------
# the engine (C ABI)
# --------------------------------------------------------------------------
class Engine:
    """One engine handle: population shards on ``devices`` (may repeat)."""

    def __init__(self, devices: Sequence[int] = (0,), node_limit: int = 15_000_000,
                 chunk_nodes: int = 0, use_nccl: bool = True):
        lib = cuda_lib()
        cfg = _Config()
        cfg.n_shards = len(devices)
        for i, d in enumerate(devices):
            cfg.devices[i] = d
        cfg.node_limit = node_limit
        cfg.arena_bytes = 0
        cfg.chunk_nodes = chunk_nodes
        cfg.use_nccl = 1 if use_nccl else 0
        h = _P()
        _check(lib.ltgp_engine_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._lib = lib
        self.devices = list(devices)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ltgp_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def set_suite(self, inputs, targets, constants):
        i = np.ascontiguousarray(inputs, np.float32)
        t = np.ascontiguousarray(targets, np.float32)
        c = np.ascontiguousarray(constants, np.float32)
        assert i.size == LANES and t.size == LANES and c.size == CONSTANTS
        _check(self._lib.ltgp_set_suite(self._h, _ptr(i), _ptr(t), _ptr(c)))

    def set_streaming(self, on: bool = True, wave: int = 0):
        """RunConfig::streaming_memory (evolve.hpp:45): children spliced in
        waves into the parents' arena, parents released after their last
        planned use (ltgp_set_streaming)."""
        _check(self._lib.ltgp_set_streaming(self._h, 1 if on else 0, wave))

    def set_memory_budget(self, nbytes: int):
        """RunConfig::memory_budget_bytes (evolve.hpp:44)."""
        _check(self._lib.ltgp_set_memory_budget(self._h, nbytes))

    def upload_population(self, genomes: Sequence[np.ndarray]):
        gs = [np.ascontiguousarray(g, np.uint8) for g in genomes]
        ptrs = (_P * max(len(gs), 1))(*[g.ctypes.data for g in gs])
        sizes = np.array([g.size for g in gs], np.uint64)
        self._keep = gs
        _check(self._lib.ltgp_upload_population(self._h, len(gs), ptrs, _ptr(sizes)))

    def upload_packed(self, buf: np.ndarray, offsets: np.ndarray, sizes: np.ndarray):
        offsets = np.ascontiguousarray(offsets, np.uint64)
        sizes = np.ascontiguousarray(sizes, np.uint64)
        _check(self._lib.ltgp_upload_packed(self._h, len(sizes), _ptr(buf), buf.nbytes, _ptr(offsets),
                                            _ptr(sizes)))

    def evaluate_packed(self, buf: np.ndarray, offsets: np.ndarray, sizes: np.ndarray, outputs: bool = False,
                        rec: np.ndarray | None = None):
        """evaluate_population on host genomes in one call: the packed buffer
        becomes the population and is evaluated while it uploads (slices
        overlap the copy; ``buf`` should be pinned). Returns records, or
        (records, outputs[M, 48]) with ``outputs``."""
        offsets = np.ascontiguousarray(offsets, np.uint64)
        sizes = np.ascontiguousarray(sizes, np.uint64)
        M = len(sizes)
        if rec is None:
            rec = np.zeros(M, RECORD_DTYPE)
        outs = np.zeros((M, LANES), np.float32) if outputs else None
        _check(self._lib.ltgp_evaluate_packed(self._h, M, _ptr(buf), buf.nbytes, _ptr(offsets), _ptr(sizes),
                                              _ptr(rec), _ptr(outs)))
        return (rec, outs) if outputs else rec

    def generation_stats(self) -> dict:
        """GenerationStats of the current population (stats.hpp:14-40), reduced
        on the device: best slot / fitness / hits / size / depth, convergence,
        max size, exact size and depth sums, fitness sum in slot order."""
        out = np.zeros(1, GEN_STATS_DTYPE)
        _check(self._lib.ltgp_generation_stats(self._h, _ptr(out)))
        return {k: out[k][0].item() for k in GEN_STATS_DTYPE.names if k != "pad"}

    def population_size(self) -> int:
        return int(self._lib.ltgp_population_size(self._h))

    def evaluate_population(self) -> np.ndarray:
        rec = np.zeros(self.population_size(), RECORD_DTYPE)
        n = C.c_uint64()
        _check(self._lib.ltgp_evaluate_population(self._h, _ptr(rec), C.byref(n)))
        return rec

    def evaluate_outputs(self):
        M = self.population_size()
        rec = np.zeros(M, RECORD_DTYPE)
        outs = np.zeros((M, LANES), np.float32)
        _check(self._lib.ltgp_evaluate_outputs(self._h, _ptr(rec), _ptr(outs)))
        return rec, outs

    def evaluate_launch(self):
        _check(self._lib.ltgp_evaluate_launch(self._h))

    def evaluate_collect(self, rec: np.ndarray | None = None) -> int:
        n = C.c_uint64()
        _check(self._lib.ltgp_evaluate_collect(self._h, _ptr(rec), C.byref(n)))
        return int(n.value)

    def execute_generation(self, plans: np.ndarray):
        plans = np.ascontiguousarray(plans, PLAN_DTYPE)
        rec = np.zeros(len(plans), RECORD_DTYPE)
        hit = C.c_int()
        _check(self._lib.ltgp_execute_generation(self._h, _ptr(plans), len(plans), _ptr(rec), C.byref(hit)))
        return rec, bool(hit.value)

    def execute_generation_launch(self, plans: np.ndarray):
        """First half of execute_generation: issues the generation, returns
        without waiting (see ltgp_execute_generation_launch)."""
        self._pending_plans = np.ascontiguousarray(plans, PLAN_DTYPE)
        _check(self._lib.ltgp_execute_generation_launch(self._h, _ptr(self._pending_plans),
                                                        len(self._pending_plans)))

    def execute_generation_finish(self):
        """Second half: waits; returns (records, outcome) with outcome 0,
        1 = SizeLimitHit or 2 = MemoryBudgetExceeded."""
        rec = np.zeros(len(self._pending_plans), RECORD_DTYPE)
        hit = C.c_int()
        _check(self._lib.ltgp_execute_generation_finish(self._h, _ptr(rec), C.byref(hit)))
        return rec, int(hit.value)

    def download_genome(self, idx: int) -> np.ndarray:
        n = C.c_uint64()
        _check(self._lib.ltgp_download_genome(self._h, idx, None, 0, C.byref(n)))
        out = np.empty(int(n.value), np.uint8)
        _check(self._lib.ltgp_download_genome(self._h, idx, _ptr(out), out.size, C.byref(n)))
        return out

    def eval_batch(self, genome: np.ndarray) -> np.ndarray:
        """eval_batch (eval.hpp:78-79): 48 per-case outputs of one genome."""
        g = np.ascontiguousarray(genome, np.uint8)
        out = np.zeros(LANES, np.float32)
        _check(self._lib.ltgp_eval_one(self._h, _ptr(g), g.size, _ptr(out)))
        return out

    def subtree_extents(self, slots, points) -> np.ndarray:
        s = np.ascontiguousarray(slots, np.uint32)
        p = np.ascontiguousarray(points, np.uint32)
        out = np.zeros((s.size, 2), np.uint64)
        _check(self._lib.ltgp_subtree_extents(self._h, s.size, _ptr(s), _ptr(p), _ptr(out)))
        return out

    def stats(self) -> dict:
        st = _Stats()
        _check(self._lib.ltgp_get_stats(self._h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in _Stats._fields_}

    def nccl_attach(self, uid: bytes, nranks: int, rank: int):
        """One process per GPU: join the ranks' NCCL communicator; every
        evaluation then all-gathers the ranks' records (gathered_records)."""
        ub = np.frombuffer(uid, np.uint8).copy()
        _check(self._lib.ltgp_nccl_attach(self._h, _ptr(ub), nranks, rank))

    def gathered_records(self) -> np.ndarray:
        n = C.c_uint32(0)
        _check(self._lib.ltgp_gathered_records(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, RECORD_DTYPE)
        _check(self._lib.ltgp_gathered_records(self._h, _ptr(out), n.value, C.byref(n)))
        return out

    def gather_mode(self) -> str:
        """How multi-shard records are all-gathered: "nccl" (distinct devices,
        one grouped ncclAllGather), "copies" (peer copies to shard 0: shards
        that repeat a device), "nccl-processes" (ltgp_nccl_attach: one
        process per GPU) or "none" (one shard)."""
        g = self.stats()["gather_nccl"]
        if g == 2:
            return "nccl-processes"
        if g:
            return "nccl"
        return "copies" if len(self.devices) > 1 else "none"

    def shard_records(self, s: int):
        p, f, n, st = _P(), C.c_uint32(), C.c_uint32(), _P()
        _check(self._lib.ltgp_shard_records(self._h, s, C.byref(p), C.byref(f), C.byref(n), C.byref(st)))
        return p.value, f.value, n.value, st.value

    def run(self, M: int, generations: int, node_limit: int, k: int = 7, seed: int = 1,
            dump_path: str | None = None, grow_mode: int = 0, memory_budget: int = 0,
            checkpoint: str | None = None, checkpoint_every: int = 0, resume: str | None = None):
        """run() (run.hpp:33-36) driven from C++ on this engine; reason 0
        MaxGenerations, 1 SizeLimitHit, 2 MemoryBudgetExceeded. With
        checkpoint_every > 0 the run state is written to `checkpoint` every
        that many generations; `resume` continues from such a file."""
        reason = C.c_int()
        nodes = C.c_uint64()
        secs = C.c_double()
        enc = lambda p: p.encode() if p else None  # noqa: E731
        done = host_lib().ltgp_host_run_checkpointed(self._h, M, generations, node_limit, k, seed, grow_mode,
                                                     memory_budget, enc(dump_path), enc(checkpoint),
                                                     checkpoint_every, enc(resume),
                                                     C.byref(reason), C.byref(nodes), C.byref(secs))
        if done < 0:
            raise EngineError(_err() or "ltgp_host_run failed")
        return {"generations": int(done), "reason": int(reason.value), "nodes": int(nodes.value),
                "eval_seconds": float(secs.value)}
