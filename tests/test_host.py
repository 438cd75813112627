"""The C++ host side (libltgp_host.so: Rng, suite, generators, tournament
and planning — the caller of the hot path) against the oracle (CPU only)."""
import numpy as np

import paper_1902_09215_b200 as ltgp
from tests._oracle import REC


def test_splitmix_and_suite_seed(oracle):
    for x in (0, 1, 2, 42, 2**63, 2**64 - 1):
        assert ltgp.splitmix64(x) == oracle.orc_splitmix64(x)
        assert ltgp.suite_seed(x) == oracle.orc_suite_seed(x)


def test_make_suite_matches_oracle(oracle):
    for s in (1, 2, 3, 99):
        a = ltgp.make_suite(ltgp.suite_seed(s))
        b = oracle.make_suite(oracle.orc_suite_seed(s))
        for x, y in zip(a, b):
            assert x.view(np.uint32).tolist() == y.view(np.uint32).tolist()
        i, t, c = a
        assert np.all(np.abs(i) <= 1) and len(set(c.tolist())) == 250 and np.all(np.diff(c) > 0)


def test_random_tree_of_size_matches_oracle(oracle):
    for k, n in enumerate((1, 3, 7, 999, 100001)):
        assert np.array_equal(ltgp.random_tree_of_size(50 + k, n), oracle.random_tree_of_size(50 + k, n))


def test_corpus_trees_match_oracle_generator(oracle):
    buf, offs, sizes = ltgp.corpus(11, 24, 2.0, 4.0)
    assert np.all(offs % 16 == 0) and np.all(sizes % 2 == 1)
    assert sizes.min() >= 100 and sizes.max() <= 10001
    for i in range(24):
        g = buf[int(offs[i]):int(offs[i]) + int(sizes[i])]
        assert np.array_equal(g, oracle.random_tree_of_size(ltgp.tree_seed(11, i), int(sizes[i])))


def test_oracle_corpus_is_the_product_corpus(oracle):
    # bench.py's reference arm builds the workload with the oracle alone
    # (orc_corpus): it must be byte-identical to the product's corpus
    for seed, M, lo, hi, first, n in ((1, 4000, 4.0, 6.0, 0, 3), (1, 4000, 4.0, 6.0, 3990, 10), (7, 50, 2.0, 4.0, 5, 20)):
        assert np.array_equal(oracle.corpus_sizes(seed, M, lo, hi), ltgp.corpus_sizes(seed, M, lo, hi))
        b1, o1, s1 = oracle.corpus(seed, M, lo, hi, first=first, n=n)
        b2, o2, s2 = ltgp.corpus(seed, M, lo, hi, first=first, n=n)
        assert np.array_equal(o1, o2) and np.array_equal(s1, s2)
        end = int(o1[-1] + (s1[-1] + 15) // 16 * 16)
        assert np.array_equal(b1[:end], b2[:end])


def test_remy_tree_valid(oracle):
    for n in (1, 3, 1001, 200001):
        g = ltgp.remy_tree(5, n)
        assert oracle.validate(g)
    # uniform random shapes are deep: depth ~ 2 sqrt(pi n / 2)
    g = ltgp.remy_tree(6, 200001)
    d = oracle.depth(g)
    assert 0.3 * 2 * np.sqrt(np.pi * 100000) < d < 3 * 2 * np.sqrt(np.pi * 100000)


def test_ramped_matches_oracle(oracle):
    for s in (1, 2, 3):
        a = ltgp.ramped_half_and_half(s, 48)
        b = oracle.ramped(s, 48)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_plan_generation_matches_oracle(oracle):
    rng = np.random.default_rng(3)
    rec = np.zeros(500, REC)
    rec["fitness"] = rng.choice([0.5, 0.25, 0.125, np.nan, 0.3], size=500).astype(np.float32)  # many ties
    rec["size"] = rng.integers(1, 1000, size=500) | 1
    for seed in (1, 7):
        a = ltgp.plan_generation(seed, rec.view(ltgp.RECORD_DTYPE), 7)
        b = oracle.plan_generation(seed, rec, 7)
        assert a.tobytes() == b.tobytes()
        assert np.all(a["mum_pt"] < rec["size"][a["mum_index"]])


def test_checkpoint_file_validation_without_gpu(tmp_path):
    """A resume file is validated before the engine is touched: missing,
    truncated or foreign files are refused (the run returns an error), so a
    damaged checkpoint can never half-restore a run."""
    import ctypes as C
    lib = ltgp.host_lib()
    reason, nodes, secs = C.c_int(), C.c_uint64(), C.c_double()

    def resume(path):
        return lib.ltgp_host_run_checkpointed(None, 48, 10, 10**9, 7, 1, 1, 0, None, None, 0, str(path).encode(),
                                              C.byref(reason), C.byref(nodes), C.byref(secs))

    assert resume(tmp_path / "missing.ckpt") == -1
    (tmp_path / "short.ckpt").write_bytes(b"LTGPCKP1")
    assert resume(tmp_path / "short.ckpt") == -1
    (tmp_path / "foreign.ckpt").write_bytes(b"NOTACKPT" + bytes(200))
    assert resume(tmp_path / "foreign.ckpt") == -1
    # ckpt_every without a path is a configuration error
    assert lib.ltgp_host_run_checkpointed(None, 48, 10, 10**9, 7, 1, 1, 0, None, None, 5, None,
                                          C.byref(reason), C.byref(nodes), C.byref(secs)) == -1


def test_run_bench_argument_validation_without_gpu():
    """run_bench (bench.hpp:33-35) rejects an empty grid and GPU counts of 0
    or above LTGP_MAX_SHARDS before creating any engine."""
    import pytest
    for sizes, workers in (([], [1]), ([1001], []), ([1001], [0]), ([1001], [17])):
        with pytest.raises(ltgp.EngineError):
            ltgp.run_bench(sizes, workers, min_corpus_nodes=1000, repeats=1)


def test_run_null_out_pointers_are_errors():
    """The C ABI reports null out-pointers as an error instead of crashing."""
    import ctypes as C
    lib = ltgp.host_lib()
    assert lib.ltgp_host_run_checkpointed(None, 48, 10, 10**9, 7, 1, 1, 0, None, None, 0, None,
                                          None, None, None) == -1


def test_bulk_mt64_engine_is_std_mt19937_64():
    # the host's Rng engine (rng.hpp:50 names std::mt19937_64) tempers a
    # whole twist at once; outputs and checkpoint text must be the standard's
    assert ltgp.host_lib().ltgp_host_rng_selftest() == 0
