"""ctypes view of the CPU oracle (oracle/libltgp_oracle.so) — test
infrastructure only; the product never imports this module."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "libltgp_oracle.so")
P = C.c_void_p

REC = np.dtype([("fitness", "<f4"), ("hits", "<i4"), ("size", "<u4"), ("depth", "<u4")])
PLAN = np.dtype([("mum_index", "<u4"), ("dad_index", "<u4"), ("mum_pt", "<u4"), ("dad_pt", "<u4")])

SIGS = {
    "orc_splitmix64": (C.c_uint64, [C.c_uint64]),
    "orc_rng_below_seq": (None, [C.c_uint64, C.c_uint64, C.c_uint32, P]),
    "orc_rng_uniform_seq": (None, [C.c_uint64, C.c_uint32, P]),
    "orc_protected_div": (C.c_float, [C.c_float, C.c_float]),
    "orc_fitness_better": (C.c_int, [C.c_float, C.c_float]),
    "orc_fitness_tied": (C.c_int, [C.c_float, C.c_float]),
    "orc_flajolet_stack_bound": (C.c_double, [C.c_uint64, C.c_double]),
    "orc_validate": (C.c_int, [P, C.c_uint64]),
    "orc_depth": (C.c_uint64, [P, C.c_uint64]),
    "orc_subtree_extent": (C.c_int, [P, C.c_uint64, C.c_uint64, P, P]),
    "orc_crossover_child_size": (C.c_uint64, [P, C.c_uint64, P, C.c_uint64, C.c_uint64, C.c_uint64]),
    "orc_crossover": (C.c_uint64, [P, C.c_uint64, P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, P,
                                   C.c_uint64, P]),
    "orc_target": (C.c_float, [C.c_float]),
    "orc_suite_seed": (C.c_uint64, [C.c_uint64]),
    "orc_make_suite": (None, [C.c_uint64, P, P, P]),
    "orc_gen_full": (C.c_uint64, [P, C.c_int, C.c_uint64, P, C.c_uint64]),
    "orc_ramped_half_and_half": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.c_int, P,
                                              C.c_uint64, P]),
    "orc_random_tree_of_size": (C.c_int, [C.c_uint64, C.c_uint64, P]),
    "orc_corpus": (C.c_uint64, [C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_uint32, C.c_uint32,
                                P, P, P, C.c_int]),
    "orc_eval_scalar": (C.c_float, [P, C.c_uint64, C.c_float, P]),
    "orc_eval_batch": (C.c_int, [P, C.c_uint64, P, P, P, P]),
    "orc_fitness": (C.c_float, [P, P]),
    "orc_hits": (C.c_int32, [P, P, C.c_float]),
    "orc_evaluate_population": (C.c_uint64, [C.c_uint32, P, P, P, P, P, P, C.c_int, P]),
    "orc_tournament_seq": (C.c_uint32, [C.c_uint64, C.c_uint32, P, C.c_uint32, C.c_uint32, P]),
    "orc_plan_generation": (None, [C.c_uint64, C.c_uint32, P, C.c_uint32, P]),
    "orc_run": (C.c_int64, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_int, C.c_char_p,
                            C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.c_int, C.c_uint64]),
}


def _p(a):
    return None if a is None else a.ctypes.data_as(P)


class Oracle:
    def __init__(self, lib):
        self.lib = lib

    def __getattr__(self, name):
        return getattr(self.lib, name)

    # convenience wrappers -------------------------------------------------
    def make_suite(self, seed):
        i, t, c = np.zeros(48, np.float32), np.zeros(48, np.float32), np.zeros(250, np.float32)
        self.lib.orc_make_suite(seed, _p(i), _p(t), _p(c))
        return i, t, c

    def eval_scalar(self, g, x, consts):
        g = np.ascontiguousarray(g, np.uint8)
        return np.float32(self.lib.orc_eval_scalar(_p(g), g.size, float(x), _p(np.ascontiguousarray(consts, np.float32))))

    def eval_batch(self, g, inputs, consts):
        g = np.ascontiguousarray(g, np.uint8)
        out = np.zeros(48, np.float32)
        peak = C.c_uint64()
        r = self.lib.orc_eval_batch(_p(g), g.size, _p(np.ascontiguousarray(inputs, np.float32)),
                                    _p(np.ascontiguousarray(consts, np.float32)), _p(out), C.byref(peak))
        if r != 0:
            raise ValueError("malformed genome")
        return out, int(peak.value)

    def fitness(self, out, tgt):
        return np.float32(self.lib.orc_fitness(_p(np.ascontiguousarray(out, np.float32)),
                                               _p(np.ascontiguousarray(tgt, np.float32))))

    def hits(self, out, tgt, thr=0.01):
        return int(self.lib.orc_hits(_p(np.ascontiguousarray(out, np.float32)),
                                     _p(np.ascontiguousarray(tgt, np.float32)), thr))

    def depth(self, g):
        g = np.ascontiguousarray(g, np.uint8)
        return int(self.lib.orc_depth(_p(g), g.size))

    def validate(self, g):
        g = np.ascontiguousarray(g, np.uint8)
        return bool(self.lib.orc_validate(_p(g), g.size))

    def subtree_extent(self, g, idx):
        g = np.ascontiguousarray(g, np.uint8)
        s, e = C.c_uint64(), C.c_uint64()
        if self.lib.orc_subtree_extent(_p(g), g.size, idx, C.byref(s), C.byref(e)) != 0:
            raise IndexError("subtree_extent out of range")
        return int(s.value), int(e.value)

    def crossover(self, mum, dad, mp, dp, cap):
        mum = np.ascontiguousarray(mum, np.uint8)
        dad = np.ascontiguousarray(dad, np.uint8)
        out = np.zeros(mum.size + dad.size, np.uint8)
        hit = C.c_int()
        n = self.lib.orc_crossover(_p(mum), mum.size, _p(dad), dad.size, mp, dp, cap, _p(out), out.size,
                                   C.byref(hit))
        return (None if hit.value else out[:n].copy()), bool(hit.value), int(n)

    def random_tree_of_size(self, seed, n):
        out = np.zeros(n, np.uint8)
        assert self.lib.orc_random_tree_of_size(seed, n, _p(out)) == 0
        return out

    def ramped(self, seed, count, cap=15_000_000, dmin=2, dmax=6):
        out = np.zeros(count * 64 + 64, np.uint8)
        sizes = np.zeros(count, np.uint64)
        tot = self.lib.orc_ramped_half_and_half(seed, count, cap, dmin, dmax, _p(out), out.size, _p(sizes))
        assert tot > 0
        gs, pos = [], 0
        for s in sizes:
            gs.append(out[pos:pos + int(s)].copy())
            pos += int(s)
        return gs

    def corpus_sizes(self, seed, count, lg_lo=4.0, lg_hi=6.0):
        sizes = np.zeros(count, np.uint64)
        self.lib.orc_corpus(seed, count, lg_lo, lg_hi, 0, 0, None, None, _p(sizes), 0)
        return sizes

    def corpus(self, seed, count, lg_lo=4.0, lg_hi=6.0, first=0, n=None, threads=0):
        """Config-3 corpus trees [first, first+n): (buf, offsets, sizes)."""
        n = count - first if n is None else n
        sizes = np.zeros(count, np.uint64)
        offs = np.zeros(max(n, 1), np.uint64)
        total = int(self.lib.orc_corpus(seed, count, lg_lo, lg_hi, first, n, None, _p(offs), _p(sizes), threads))
        buf = np.empty(total + 64, np.uint8)
        self.lib.orc_corpus(seed, count, lg_lo, lg_hi, first, n, _p(buf), _p(offs), _p(sizes), threads)
        return buf, offs[:n], sizes[first:first + n].copy()

    def evaluate_population(self, buf, offsets, sizes, suite, threads=0):
        i, t, c = suite
        M = len(sizes)
        rec = np.zeros(M, REC)
        self.lib.orc_evaluate_population(M, _p(buf), _p(np.ascontiguousarray(offsets, np.uint64)),
                                         _p(np.ascontiguousarray(sizes, np.uint64)), _p(i), _p(t), _p(c),
                                         threads, _p(rec))
        return rec

    def plan_generation(self, seed, rec, k=7):
        out = np.zeros(len(rec), PLAN)
        self.lib.orc_plan_generation(seed, len(rec), _p(np.ascontiguousarray(rec, REC)), k, _p(out))
        return out

    def run(self, M, G, node_limit, k=7, seed=1, threads=0, dump=None, grow_mode=0, memory_budget=0):
        reason, nodes = C.c_int(), C.c_uint64()
        done = self.lib.orc_run(M, G, node_limit, k, seed, threads, dump.encode() if dump else None,
                                C.byref(reason), C.byref(nodes), grow_mode, memory_budget)
        return {"generations": int(done), "reason": int(reason.value), "nodes": int(nodes.value)}


_ORACLE = None


def load_oracle() -> Oracle:
    global _ORACLE
    if _ORACLE is None:
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(os.path.join(ORACLE_DIR, "ltgp_oracle.cpp")):
            subprocess.run(["make", "-C", ORACLE_DIR], check=True, capture_output=True)
        lib = C.CDLL(LIB)
        for name, (res, args) in SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _ORACLE = Oracle(lib)
    return _ORACLE


def same_bits(a, b):
    """Bit equality of float32 arrays with every NaN treated as equal (NaN
    payloads differ between x86 and the GPU)."""
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    return np.array_equal(a[~na].view(np.uint32), b[~nb].view(np.uint32))
