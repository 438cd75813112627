"""Parity of the B200 engine with the CPU oracle (run on the GPU box: -m gpu).

Every test goes through the C ABI (include/ltgp_cuda.h) via the package's
ctypes binding. Tolerance: bit-exact per case (modulo NaN payload, which
differs between x86 and the GPU — SURVEY.md App. A #14) and bit-exact
fitness / hits / size / depth.
"""
import json
import os

import numpy as np
import pytest

import paper_1902_09215_b200 as ltgp
from tests._oracle import REC, same_bits

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ADD, SUB, MUL, DIV, X = 0, 1, 2, 3, 4


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.fixture(scope="module")
def suite():
    return ltgp.make_suite(ltgp.suite_seed(1))


def engine(suite, devices=(0,), chunk=0):
    e = ltgp.Engine(list(devices), node_limit=2**40, chunk_nodes=chunk)
    e.set_suite(*suite)
    return e


def pack(genomes):
    sizes = np.array([g.size for g in genomes], np.uint64)
    offs = np.zeros(len(genomes), np.uint64)
    o = 0
    for k, s in enumerate(sizes):
        offs[k] = o
        o += (int(s) + 15) // 16 * 16
    buf = np.full(o + 64, 0xFF, np.uint8)
    for k, g in enumerate(genomes):
        buf[int(offs[k]):int(offs[k]) + g.size] = g
    return buf, offs, sizes


def assert_records_equal(got, exp):
    assert same_bits(got["fitness"], exp["fitness"])
    assert np.array_equal(got["hits"], exp["hits"])
    assert np.array_equal(got["size"], exp["size"])
    assert np.array_equal(got["depth"], exp["depth"])


def check_population(oracle, suite, genomes, chunk=0, devices=(0,)):
    with engine(suite, devices, chunk) as e:
        e.upload_population(genomes)
        rec, outs = e.evaluate_outputs()
    buf, offs, sizes = pack(genomes)
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    for k, g in enumerate(genomes):
        o, _ = oracle.eval_batch(g, suite[0], suite[2])
        assert same_bits(outs[k], o), f"tree {k} (size {g.size}) per-case outputs differ"
    assert_records_equal(rec, exp)
    return rec


def test_spec_genomes(oracle, suite):
    i, t, c = suite
    with engine(suite) as e:
        assert same_bits(e.eval_batch(np.array([X], np.uint8)), i)
        assert same_bits(e.eval_batch(np.array([5 + 9], np.uint8)), np.full(48, c[9]))
        for g in ([ADD, X, X], [SUB, MUL, X, X, X], [DIV, X, SUB, X, X], [DIV, X, 5 + 0]):
            g = np.array(g, np.uint8)
            o, _ = oracle.eval_batch(g, i, c)
            assert same_bits(e.eval_batch(g), o), g


def test_golden_fixture_trees(suite):
    """Per-case outputs frozen from the oracle (tests/golden/oracle_golden.json)."""
    g = json.load(open(os.path.join(HERE, "golden", "oracle_golden.json")))
    with engine(suite) as e:
        for tr in g["trees"]:
            tree = ltgp.random_tree_of_size(tr["seed"], tr["n"])
            out = e.eval_batch(tree)
            assert out.view(np.uint32).tolist() == tr["outputs_bits"] or \
                same_bits(out, np.array(tr["outputs_bits"], np.uint32).view(np.float32))


def test_config1_population_golden(oracle):
    """Config 1: pop 48 ramped half-and-half, one evaluation; golden records."""
    g = json.load(open(os.path.join(HERE, "golden", "oracle_golden.json")))
    for s, d in g["c1"].items():
        suite = ltgp.make_suite(ltgp.suite_seed(int(s)))
        genomes = [np.array(x, np.uint8) for x in d["genomes"]]
        with engine(suite) as e:
            e.upload_population(genomes)
            rec = e.evaluate_population()
        assert rec["fitness"].view(np.uint32).tolist() == d["fitness_bits"]
        assert rec["hits"].tolist() == d["hits"]
        assert rec["size"].tolist() == d["size"]
        assert rec["depth"].tolist() == d["depth"]


@pytest.mark.parametrize("chunk", [64, 1024, 16384])
def test_config3_small_chunked(oracle, suite, chunk):
    """Config-3 trees (uniform prefix splits) across chunk sizes: chunk
    summaries + spine combine must reproduce the sequential scan bit for bit."""
    buf, offs, sizes = ltgp.corpus(5, 40, 1.0, 4.7)
    genomes = [buf[int(o):int(o) + int(n)].copy() for o, n in zip(offs, sizes)]
    check_population(oracle, suite, genomes, chunk=chunk)


@pytest.mark.parametrize("chunk", [256, 16384])
def test_remy_deep_trees(oracle, suite, chunk):
    """Uniform random shapes (config 4 generator): deep stacks exercise the
    shared-window spill/fill and long spines."""
    genomes = [ltgp.remy_tree(40 + k, n) for k, n in enumerate((1, 3, 1001, 20001, 200001))]
    check_population(oracle, suite, genomes, chunk=chunk)


def test_combine_many_chunks(oracle, suite):
    """Trees of more chunks than k_cpops's shared-memory segment stack holds
    (over 3072 chunks: its stack falls back to global memory) next to
    smaller chunked trees in the same launch."""
    genomes = [ltgp.remy_tree(90, 400001), ltgp.remy_tree(91, 5001), ltgp.random_tree_of_size(92, 250001)]
    check_population(oracle, suite, genomes, chunk=64)


def test_auto_chunk_wave_balance(oracle, suite):
    """Automatic chunk length with the wave balance: 100 trees of 3e5 nodes
    get 8192-node chunks from the power-of-two rule (3700 chunks, one part-
    full wave of the persistent grid), shortened to the shortest multiple of
    1024 that keeps one wave -- a length that is not a power of two."""
    import torch
    n, T = 300001, 100
    genomes = [ltgp.random_tree_of_size(500 + k, n) for k in range(T)]
    W = torch.cuda.get_device_properties(0).multi_processor_count * 32
    chunks = lambda c: T * -(-n // c)
    waves = -(-chunks(8192) // W)
    c = next(c for c in range(4096, 8193, 1024) if chunks(c) <= waves * W)
    with engine(suite) as e:
        e.upload_population(genomes)
        rec, outs = e.evaluate_outputs()
        assert e.stats()["last_chunks"] == chunks(c)
    assert c % 1024 == 0 and c & (c - 1)  # not a power of two on a 148-SM B200
    buf, offs, sizes = pack(genomes)
    assert_records_equal(rec, oracle.evaluate_population(buf, offs, sizes, suite, threads=0))
    for k in (0, T - 1):
        o, _ = oracle.eval_batch(genomes[k], suite[0], suite[2])
        assert same_bits(outs[k], o)


def test_adversarial(oracle, suite):
    c0 = 5 + int(np.argmin(np.abs(suite[2])))  # constant nearest 0 (may be 0.000)
    gs = []
    # left chain: DIV(DIV(...(X, c)...)) -> repeated division, underflow to subnormal / 0
    gs.append(np.array([DIV] * 3000 + [X] + [5 + 200] * 3000, np.uint8))
    # right chain of MUL: overflow to inf then inf*0 = NaN
    gs.append(np.array([MUL, 5 + 249] * 2000 + [X], np.uint8))
    # zero divisors everywhere: x / (x - x) and c / (c - c)
    gs.append(np.array([DIV, X, SUB, X, X], np.uint8))
    gs.append(np.array([ADD] * 50 + sum(([DIV, X, SUB, X, X] for _ in range(51)), []), np.uint8))
    gs.append(np.array([DIV, 5 + 1, c0], np.uint8))
    # subnormal arithmetic: (c*c*c*...)/x chains
    gs.append(np.array([SUB] + [MUL] * 40 + [5 + 3] * 41 + [DIV, 5 + 5, X], np.uint8))
    for chunk in (64, 0):
        check_population(oracle, suite, gs, chunk=chunk)


def test_capacity_overflow_reruns(oracle, suite):
    """Work items that outgrow a capacity are re-run with worst-case capacities,
    bit-exactly: whole-tree items whose stack outgrows the per-warp spill area
    (chunk 65536: a 16001-node left chain holds 8001 values), and chunks of
    4096 leaves (their stack outgrows the spill area and their summaries the
    sqrt(C)-sized summary pool). All-leaf 64-node chunks overflow only the
    pool's first estimate: the second evaluation sizes the pool from the
    first one's exact claims and needs no re-run."""
    gs = [np.array([ADD] * 8000 + [X] + [5 + 7] * 8000, np.uint8),
          np.array([SUB] * 5000 + [X] + [5 + (k % 250) for k in range(5000)], np.uint8)]
    for chunk, rerun in ((64, False), (4096, True), (65536, True)):
        with engine(suite, chunk=chunk) as e:
            e.upload_population(gs)
            rec, outs = e.evaluate_outputs()
            n = e.stats()["last_fallback_items"]
            assert n > 0 or not rerun, (chunk, n)
            rec2, outs2 = e.evaluate_outputs()
            n2 = e.stats()["last_fallback_items"]
            assert (n2 > 0) == rerun, (chunk, n2)
            assert rec2.tobytes() == rec.tobytes() and same_bits(outs2, outs)
        for k, g in enumerate(gs):
            o, _ = oracle.eval_batch(g, suite[0], suite[2])
            assert same_bits(outs[k], o)
            assert rec["depth"][k] == oracle.depth(g)


def test_streamed_capacity_overflow_reruns(oracle, suite, monkeypatch):
    """The cross-slice launch (ltgp_evaluate_packed, several slices) hands
    items that outgrow the spill area or the summary pool to the same re-run
    tiers as a resident evaluation: records and outputs equal the resident
    path's and the oracle's, with re-runs counted."""
    gs = [ltgp.random_tree_of_size(31, 4999),
          np.array([ADD] * 8000 + [X] + [5 + 7] * 8000, np.uint8),
          ltgp.remy_tree(32, 20001),
          np.array([SUB] * 5000 + [X] + [5 + (k % 250) for k in range(5000)], np.uint8),
          ltgp.random_tree_of_size(33, 2999)]
    buf, offs, sizes = pack(gs)
    monkeypatch.setenv("LTGP_SLICE_KB", "8")
    for chunk in (4096, 65536):
        with engine(suite, chunk=chunk) as e:
            rec, outs = e.evaluate_packed(buf, offs, sizes, outputs=True)
            n = e.stats()["last_fallback_items"]
            e.upload_packed(buf, offs, sizes)
            ref, refo = e.evaluate_outputs()
        assert n > 0, chunk
        assert rec.tobytes() == ref.tobytes() and same_bits(outs, refo)
        for k, g in enumerate(gs):
            o, _ = oracle.eval_batch(g, suite[0], suite[2])
            assert same_bits(outs[k], o)
            assert rec["depth"][k] == oracle.depth(g)


def test_subtree_extents(oracle, suite):
    genomes = [ltgp.remy_tree(7, 4001), ltgp.random_tree_of_size(8, 999), np.array([X], np.uint8)]
    with engine(suite) as e:
        e.upload_population(genomes)
        rng = np.random.default_rng(0)
        slots, pts = [], []
        for s, g in enumerate(genomes):
            for p in list(rng.integers(0, g.size, 200)) + [0, g.size - 1]:
                slots.append(s)
                pts.append(int(p))
        ext = e.subtree_extents(slots, pts)
    for (s, p), (a, b) in zip(zip(slots, pts), ext):
        assert (int(a), int(b)) == oracle.subtree_extent(genomes[s], p)


def test_execute_generation_children(oracle, suite):
    """Device splice vs the oracle's crossover, child by child, and records."""
    genomes = [ltgp.random_tree_of_size(100 + k, 2 * k + 1) for k in range(60)] + \
              [ltgp.remy_tree(300, 30001)]
    M = len(genomes)
    rng = np.random.default_rng(5)
    plans = np.zeros(M, ltgp.PLAN_DTYPE)
    plans["mum_index"] = rng.integers(0, M, M)
    plans["dad_index"] = rng.integers(0, M, M)
    plans["mum_pt"] = [rng.integers(0, genomes[m].size) for m in plans["mum_index"]]
    plans["dad_pt"] = [rng.integers(0, genomes[d].size) for d in plans["dad_index"]]
    for devices in ((0,), (0, 0, 0)):
        with engine(suite, devices, chunk=512) as e:
            e.upload_population(genomes)
            e.evaluate_population()
            rec, hit = e.execute_generation(plans)
            assert not hit
            children = [e.download_genome(c) for c in range(M)]
        for c in range(M):
            p = plans[c]
            exp, h, n = oracle.crossover(genomes[p["mum_index"]], genomes[p["dad_index"]], int(p["mum_pt"]),
                                         int(p["dad_pt"]), 2**40)
            assert np.array_equal(children[c], exp), c
        buf, offs, sizes = pack(children)
        assert_records_equal(rec, oracle.evaluate_population(buf, offs, sizes, suite))


def test_execute_generation_size_limit(suite):
    genomes = [ltgp.random_tree_of_size(1, 31), ltgp.random_tree_of_size(2, 63)]
    with ltgp.Engine([0], node_limit=63) as e:
        e.set_suite(*suite)
        e.upload_population(genomes)
        e.evaluate_population()
        plans = np.zeros(2, ltgp.PLAN_DTYPE)
        plans[0] = (0, 1, 0, 0)   # child = dad (63 nodes) -> reaches the limit
        plans[1] = (0, 0, 1, 1)
        rec, hit = e.execute_generation(plans)
        assert hit
        assert np.array_equal(e.download_genome(0), genomes[0])  # population unchanged


@pytest.mark.parametrize("seed,grow", [(1, 0), (2, 0), (3, 0), (1, 1), (2, 1)])
def test_run_dump_matches_oracle(oracle, tmp_path, seed, grow):
    """run() on the engine vs the oracle's run(): identical generation dumps
    (fitness bits, hits, size, depth of every individual, every generation),
    so selected parents are identical too. grow=1 runs bloat."""
    d_ref = tmp_path / "ref.txt"
    r = oracle.run(48, 40, 10**9, 7, seed, 0, str(d_ref), grow)
    for devices in ((0,), (0, 0)):
        d = tmp_path / f"gpu{len(devices)}.txt"
        with ltgp.Engine(list(devices), node_limit=10**9, chunk_nodes=256) as e:
            g = e.run(48, 40, 10**9, 7, seed, str(d), grow)
        assert g["generations"] == r["generations"] == 40
        assert d.read_bytes() == d_ref.read_bytes()


@pytest.mark.parametrize("shards", [1, 2])
def test_run_checkpoint_resume_matches_oracle(oracle, tmp_path, shards):
    """Checkpoint/resume: a run checkpointed every 7
    generations, stopped at generation 20 and resumed in a fresh engine to
    40, writes the same dump as the oracle's uninterrupted 40 generations;
    totals (generations, nodes) count the whole run. A checkpoint from a run
    with other parameters, or a damaged file, is refused."""
    ref = tmp_path / "ref.txt"
    r = oracle.run(48, 40, 10**9, 7, 2, 0, str(ref), 1)
    ck = tmp_path / "run.ckpt"
    d = tmp_path / "gpu.txt"
    with ltgp.Engine([0] * shards, node_limit=10**9, chunk_nodes=256) as e:
        g1 = e.run(48, 20, 10**9, 7, 2, str(d), 1, checkpoint=str(ck), checkpoint_every=7)
    assert g1["generations"] == 20 and ck.exists()
    with ltgp.Engine([0] * shards, node_limit=10**9) as e:
        g2 = e.run(48, 40, 10**9, 7, 2, str(d), 1, resume=str(ck))
    assert g2["generations"] == r["generations"] == 40
    assert d.read_bytes() == ref.read_bytes()
    with ltgp.Engine([0], node_limit=10**9) as e:
        full = e.run(48, 40, 10**9, 7, 2, None, 1)
    assert g2["nodes"] == full["nodes"]
    with ltgp.Engine([0], node_limit=10**9) as e:
        with pytest.raises(ltgp.EngineError):
            e.run(48, 40, 10**9, 7, 3, None, 1, resume=str(ck))  # other seed
        bad = tmp_path / "bad.ckpt"
        raw = bytearray(ck.read_bytes())
        raw[len(raw) // 2] ^= 1
        bad.write_bytes(bytes(raw))
        with pytest.raises(ltgp.EngineError):
            e.run(48, 40, 10**9, 7, 2, None, 1, resume=str(bad))


def test_resume_truncates_dump_after_crash(oracle, tmp_path):
    """A run that dies between checkpoints (checkpoint at generation 14, dump
    written through 17) resumes from generation 14: the dump is cut back to
    the checkpoint's length first, so it ends identical to an uninterrupted
    run's (the resumed run must not dump generations 15-17 twice)."""
    ref = tmp_path / "ref.txt"
    oracle.run(48, 30, 10**9, 7, 5, 0, str(ref), 1)
    ck = tmp_path / "run.ckpt"
    d = tmp_path / "gpu.txt"
    with ltgp.Engine([0], node_limit=10**9, chunk_nodes=256) as e:
        assert e.run(48, 14, 10**9, 7, 5, str(d), 1, checkpoint=str(ck), checkpoint_every=7)["generations"] == 14
    # the "crashed" continuation: generations 15-17 dumped, no checkpoint after 14
    with ltgp.Engine([0], node_limit=10**9, chunk_nodes=256) as e:
        assert e.run(48, 17, 10**9, 7, 5, str(d), 1, resume=str(ck))["generations"] == 17
    assert d.read_bytes().count(b"\n") == 18 * 48
    with ltgp.Engine([0], node_limit=10**9) as e:
        assert e.run(48, 30, 10**9, 7, 5, str(d), 1, resume=str(ck))["generations"] == 30
    assert d.read_bytes() == ref.read_bytes()


def test_run_size_limit_matches_oracle(oracle, tmp_path):
    # node_limit=63 -> SizeLimitHit within a few generations
    r = oracle.run(48, 300, 63, 7, 4, 0, str(tmp_path / "a"))
    with ltgp.Engine([0], node_limit=63) as e:
        g = e.run(48, 300, 63, 7, 4, str(tmp_path / "b"), 0)
    assert r["reason"] == g["reason"] == 1
    assert r["generations"] == g["generations"]
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()


def test_run_memory_budget_matches_oracle(oracle, tmp_path):
    """MemoryBudgetExceeded (evolve.hpp:44, :89-93): the engine's
    run refuses the same generation as the oracle's (planned bytes from the
    device's child sizes), with identical dumps, at 1 and 2 shards."""
    from tests.test_oracle import budget_case
    G = 40
    full = tmp_path / "full.txt"
    oracle.run(48, G, 10**9, 7, 1, 2, str(full), 1)
    budget, g0 = budget_case(full.read_text(), G)
    ref = tmp_path / "ref.txt"
    ro = oracle.run(48, G, 10**9, 7, 1, 2, str(ref), 1, memory_budget=budget)
    assert ro["reason"] == 2 and ro["generations"] == g0 - 1
    for shards in (1, 2):
        out = tmp_path / f"gpu{shards}.txt"
        with ltgp.Engine([0] * shards, node_limit=10**9) as e:
            r = e.run(48, G, 10**9, 7, 1, str(out), 1, memory_budget=budget)
        assert r["reason"] == 2 and r["generations"] == g0 - 1
        assert out.read_bytes() == ref.read_bytes()


def host_generation_stats(rec):
    """GenerationStats (stats.hpp:14-40) from records, on the host: best =
    first slot of the best fitness (NaN worst), convergence = bit-equal
    fitness, fitness summed in slot order in double."""
    f = rec["fitness"]
    order = sorted(range(len(f)), key=lambda i: (np.isnan(f[i]), f[i] if not np.isnan(f[i]) else 0.0, i))
    b = order[0]
    s = 0.0
    for v in f:
        s += float(v)
    return {"best_index": b, "best_fitness": float(f[b]), "best_hits": int(rec["hits"][b]),
            "best_size": int(rec["size"][b]), "best_depth": int(rec["depth"][b]),
            "convergence": int((f.view(np.uint32) == f[b:b + 1].view(np.uint32)[0]).sum()),
            "max_size": int(rec["size"].max()), "sum_size": int(rec["size"].astype(np.uint64).sum()),
            "sum_depth": int(rec["depth"].astype(np.uint64).sum()), "sum_fitness": s}


def test_generation_stats_on_device(oracle, suite):
    """ltgp_generation_stats equals the host reduction of the records: ties on
    the best fitness (duplicated genomes), NaN fitness, 1 and 2 shards."""
    gs = [np.array([MUL, 5 + 249] * 2000 + [X], np.uint8)] * 3            # NaN fitness
    gs += [np.array([SUB, MUL, X, X, X], np.uint8)] * 5                   # ties, convergence 5
    gs += [ltgp.random_tree_of_size(900 + k, 201 + 2 * k) for k in range(40)]
    gs += [np.array([SUB, MUL, X, X, X], np.uint8)] * 2
    for shards in (1, 2):
        with ltgp.Engine([0] * shards, node_limit=10**9) as e:
            e.set_suite(*suite)
            e.upload_population(gs)
            rec = e.evaluate_population()
            got = e.generation_stats()
        exp = host_generation_stats(rec)
        fit = got.pop("sum_fitness"), exp.pop("sum_fitness")
        assert got == exp or (np.isnan(got["best_fitness"]) and np.isnan(exp["best_fitness"]))
        assert fit[0] == fit[1] or (np.isnan(fit[0]) and np.isnan(fit[1]))
    # after a generation on device (children never leave the GPU)
    with ltgp.Engine([0], node_limit=10**9) as e:
        e.set_suite(*suite)
        e.upload_population(gs)
        rec0 = e.evaluate_population()
        plans = ltgp.plan_generation(3, rec0, 7)
        rec1, hit = e.execute_generation(plans)
        assert not hit
        got = e.generation_stats()
    exp = host_generation_stats(rec1)
    got.pop("sum_fitness"), exp.pop("sum_fitness")
    assert got == exp or np.isnan(exp["best_fitness"])


def test_config3_full_size_sampled(oracle, suite):
    """BASELINE config 3 at full size (4000 trees, 10^4..10^6 nodes): every
    record compared with the oracle (multi-threaded)."""
    buf, offs, sizes = ltgp.corpus(1, 4000, 4.0, 6.0)
    with engine(suite) as e:
        e.upload_packed(buf, offs, sizes)
        rec, outs = e.evaluate_outputs()
        rec2 = e.evaluate_population()
        chunks = e.stats()["last_chunks"]
    assert rec.tobytes() == rec2.tobytes()  # determinism across launches
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    assert_records_equal(rec, exp)
    # The work list's tapered tail (11 waves of the persistent grid: the
    # smallest chunked trees are cut into 8192/4096/2048-node chunks and run
    # last) is in effect: more chunks than 16384-node chunks alone give, and
    # the smallest chunked trees (the shortest chunks) match per case
    big = sizes[sizes > 16384]
    assert chunks > int(np.sum(-(-big.astype(np.int64) // 16384)))
    order = np.argsort(sizes)
    for k in order[sizes[order] > 16384][:3]:
        g = np.ascontiguousarray(buf[int(offs[k]):int(offs[k]) + int(sizes[k])])
        o, _ = oracle.eval_batch(g, suite[0], suite[2])
        assert same_bits(outs[k], o)


def test_streamed_evaluate_packed_matches_resident(oracle, suite):
    """ltgp_evaluate_packed (upload in ~32 MB slices overlapped with their
    evaluation; the full config-3 corpus is 16 slices) gives the same records
    as the resident path, on one shard and on two; and again on reuse (cached
    work list, arena reused while the previous call's data is still there)."""
    buf, offs, sizes = ltgp.corpus(1, 4000, 4.0, 6.0)
    with engine(suite) as e:
        e.upload_packed(buf, offs, sizes)
        exp = e.evaluate_population()
        got = e.evaluate_packed(buf, offs, sizes)
        assert got.tobytes() == exp.tobytes()
        got2 = e.evaluate_packed(buf, offs, sizes)
        assert got2.tobytes() == exp.tobytes()
        assert e.evaluate_population().tobytes() == exp.tobytes()  # population = the streamed one
    with engine(suite, devices=(0, 0)) as e:
        assert e.evaluate_packed(buf, offs, sizes).tobytes() == exp.tobytes()
    # three shards: the records come back through the engine's all-gather
    # (peer copies into shard 0's n x cmax array; NCCL on distinct devices)
    with engine(suite, devices=(0, 0, 0)) as e:
        e.upload_packed(buf, offs, sizes)
        assert e.evaluate_population().tobytes() == exp.tobytes()
        assert e.stats()["gather_seconds"] > 0
    # and against the oracle on a sample of slots
    idx = np.arange(0, 4000, 97)
    sub = [buf[int(offs[k]):int(offs[k]) + int(sizes[k])].copy() for k in idx]
    b2, o2, s2 = pack(sub)
    ref = oracle.evaluate_population(b2, o2, s2, suite, threads=0)
    assert_records_equal(got[idx], ref)


def test_streamed_packed_transfer(oracle, suite, monkeypatch):
    """The streamed path's packed PCIe form (ltgp_pack.h, k_decode_packed):
    records, per-case outputs and the rebuilt arena equal the raw-byte
    transfer (LTGP_PACK=0) and the oracle, with garbage (any byte value) in
    the gaps between trees, constants of every opcode 5..254, slices of every
    size down to one packet, and the scalar host encoder; the bytes sent are
    ~0.63 per node on a config-3 corpus."""
    rng = np.random.default_rng(5)
    genomes = [ltgp.remy_tree(900 + k, n) for k, n in enumerate((1, 3, 15, 17, 33, 255, 4097, 30001, 123457))]
    for g in genomes:  # every constant opcode
        leaves = g >= X
        g[leaves] = np.where(rng.random(leaves.sum()) < 0.3, X, rng.integers(5, 255, leaves.sum()))
    buf, offs, sizes = pack(genomes)
    for k in range(len(genomes)):  # garbage between trees: the arena keeps every byte
        end = int(offs[k]) + int(sizes[k])
        nxt = int(offs[k + 1]) if k + 1 < len(genomes) else buf.size
        buf[end:nxt] = rng.integers(0, 256, nxt - end)
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    results = []
    # (LTGP_XSLICE=0: per-slice launches, k_decode_packed / k_decode + k_plan_warp<false>,
    # the path a profiler or sanitizer gets)
    for env in ({"LTGP_PACK": "0"}, {}, {"LTGP_SLICES": "64", "LTGP_SLICE_KB": "1"}, {"LTGP_PACK_THREADS": "3"},
                {"LTGP_XSLICE": "0", "LTGP_SLICE_KB": "8"}, {"LTGP_XSLICE": "0", "LTGP_PACK": "0", "LTGP_SLICE_KB": "8"}):
        for k in ("LTGP_PACK", "LTGP_SLICES", "LTGP_SLICE_KB", "LTGP_PACK_THREADS", "LTGP_XSLICE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with engine(suite, chunk=1024) as e:
            rec, outs = e.evaluate_packed(buf, offs, sizes, outputs=True)
            arena = [e.download_genome(k) for k in range(len(genomes))]
            h2d = e.stats()["last_h2d_bytes"]
        assert_records_equal(rec, exp)
        for k, g in enumerate(genomes):
            assert np.array_equal(arena[k], g)
            o, _ = oracle.eval_batch(g, suite[0], suite[2])
            assert same_bits(outs[k], o)
        results.append((rec.tobytes(), outs.tobytes(), h2d))
    assert len({r[:2] for r in results}) == 1
    assert results[0][2] <= buf.size and results[1][2] < results[0][2]
    # config-3 corpus: ~0.63 bytes a node cross PCIe, records unchanged
    for k in ("LTGP_PACK", "LTGP_SLICES", "LTGP_SLICE_KB", "LTGP_PACK_THREADS", "LTGP_XSLICE"):
        monkeypatch.delenv(k, raising=False)
    cb, co, cs = ltgp.corpus(1, 400, 4.0, 5.0)
    with engine(suite) as e:
        e.upload_packed(cb, co, cs)
        ref = e.evaluate_population()
        assert e.evaluate_packed(cb, co, cs).tobytes() == ref.tobytes()
        assert e.stats()["last_h2d_bytes"] < 0.66 * cb.size


def test_streamed_small_and_outputs(oracle, suite):
    """A small population (one slice) with per-case outputs, from pageable memory."""
    genomes = [ltgp.remy_tree(70 + k, n) for k, n in enumerate((1, 3, 17, 1001, 20001, 70001))]
    buf, offs, sizes = pack(genomes)
    with engine(suite, chunk=1024) as e:
        rec, outs = e.evaluate_packed(buf, offs, sizes, outputs=True)
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    assert_records_equal(rec, exp)
    for k, g in enumerate(genomes):
        o, _ = oracle.eval_batch(g, suite[0], suite[2])
        assert same_bits(outs[k], o)


def test_streamed_slice_cap(oracle, suite, monkeypatch):
    """The streamed path at its slice-count cap (64 slices of ~9 KB, every
    slice with its own work queue), record- and output-identical to the
    oracle; then the defaults again on the same engine."""
    buf, offs, sizes = ltgp.corpus(31, 600, 2.0, 3.5)
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    with engine(suite, chunk=1024) as e:
        monkeypatch.setenv("LTGP_SLICES", "64")
        monkeypatch.setenv("LTGP_SLICE_KB", "8")
        rec, outs = e.evaluate_packed(buf, offs, sizes, outputs=True)
        assert_records_equal(rec, exp)
        for k in (0, 299, 599):
            g = buf[int(offs[k]):int(offs[k]) + int(sizes[k])]
            o, _ = oracle.eval_batch(g, suite[0], suite[2])
            assert same_bits(outs[k], o)
        monkeypatch.delenv("LTGP_SLICES")
        monkeypatch.delenv("LTGP_SLICE_KB")
        rec = e.evaluate_packed(buf, offs, sizes)
        assert_records_equal(rec, exp)


@pytest.mark.slow
def test_config2_bloating_run_matches_oracle(oracle, tmp_path):
    """Config 2 at its full BASELINE size: pop 4000, tournament 7, no size
    limit, all 200 generations with the bloating grow variant, at 1 and 2
    shards; generation dumps (sizes, depths, hits, fitness bits of every
    individual: the selected parents follow from them) identical to the
    oracle's run()."""
    r = oracle.run(4000, 200, 2**62, 7, 1, 0, str(tmp_path / "a"), 1)
    for shards in (1, 2):
        with ltgp.Engine([0] * shards, node_limit=2**62) as e:
            g = e.run(4000, 200, 2**62, 7, 1, str(tmp_path / "b"), 1)
        assert r["generations"] == g["generations"] == 200
        assert r["nodes"] == g["nodes"]
        assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()


@pytest.mark.slow
def test_config5_capped_run_matches_oracle(oracle, tmp_path):
    """Config 5's regime: pop 4000 capped at a 15M-node limit per individual
    (node_limit = 15e6), bloating grow, 300 generations on device splicing;
    the dump is identical to the oracle's."""
    r = oracle.run(4000, 300, 15_000_000, 7, 1, 0, str(tmp_path / "a"), 1)
    with ltgp.Engine([0], node_limit=15_000_000) as e:
        g = e.run(4000, 300, 15_000_000, 7, 1, str(tmp_path / "b"), 1)
    assert r["generations"] == g["generations"] and r["reason"] == g["reason"]
    assert r["nodes"] == g["nodes"]
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()


@pytest.mark.slow
def test_config4_regime_large_remy_trees(oracle, suite):
    """Config 4's regime: uniform random (Remy) trees of 4e7 nodes at the
    automatic chunk length (>= 2^18-node chunks, an 8 sqrt(C) spill area per
    warp, spine chains of thousands of steps): records and all 48 per-case
    outputs of both trees equal the oracle's."""
    from concurrent.futures import ThreadPoolExecutor
    n = 40_000_001
    with ThreadPoolExecutor(2) as ex:
        genomes = list(ex.map(lambda k: ltgp.remy_tree(7100 + k, n), range(2)))
    with engine(suite) as e:
        e.upload_population(genomes)
        rec, outs = e.evaluate_outputs()
        st = e.stats()
    assert st["last_chunks"] >= 2 * (n // 2**18)          # chunks of at most 2^18 nodes
    assert st["last_chunks"] <= 2 * (n // 2**17 + 1)      # ... and more than 2^17
    buf, offs, sizes = pack(genomes)
    assert_records_equal(rec, oracle.evaluate_population(buf, offs, sizes, suite, threads=0))
    for k, g in enumerate(genomes):
        o, _ = oracle.eval_batch(g, suite[0], suite[2])
        assert same_bits(outs[k], o)


@pytest.mark.parametrize("round_", range(int(os.environ.get("LTGP_FUZZ_ROUNDS", "3"))))
def test_randomized_populations(oracle, suite, round_, monkeypatch):
    """Randomized sweep: mixed shapes (Remy, uniform splits, ramped
    half-and-half, left/right chains), random sizes and chunk lengths, the
    resident and the streamed path (random slice sizes: one slice, or several
    through the cross-slice launch); every record and per-case output equal
    to the oracle's."""
    rng = np.random.default_rng(1000 + round_)
    genomes = []
    for k in range(60):
        kind = rng.integers(0, 5)
        n = int(rng.integers(1, 40000)) | 1
        if kind == 0:
            genomes.append(ltgp.remy_tree(int(rng.integers(1 << 30)), n))
        elif kind == 1:
            genomes.append(ltgp.random_tree_of_size(int(rng.integers(1 << 30)), n))
        elif kind == 2:
            genomes += ltgp.ramped_half_and_half(int(rng.integers(1 << 30)), 2)
        elif kind == 3:  # left chain: op op ... op leaf leaf ... leaf
            m = n // 2
            ops = rng.integers(0, 4, m).astype(np.uint8)
            leaves = rng.integers(4, 255, m + 1).astype(np.uint8)
            genomes.append(np.concatenate([ops, leaves]))
        else:  # right chain: op leaf op leaf ... leaf
            m = n // 2
            g = np.empty(2 * m + 1, np.uint8)
            g[0:2 * m:2] = rng.integers(0, 4, m)
            g[1:2 * m:2] = rng.integers(4, 255, m)
            g[-1] = 4
            genomes.append(g)
    chunk = int(rng.choice([0, 64, 256, 1024, 4096, 16384]))
    slice_kb = str(rng.choice(["", "16", "64", "256"]))
    if slice_kb:
        monkeypatch.setenv("LTGP_SLICE_KB", slice_kb)
    buf, offs, sizes = pack(genomes)
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    with engine(suite, chunk=chunk) as e:
        e.upload_population(genomes)
        rec, outs = e.evaluate_outputs()
        rec_s, outs_s = e.evaluate_packed(buf, offs, sizes, outputs=True)
    assert_records_equal(rec, exp)
    assert rec_s.tobytes() == rec.tobytes() and same_bits(outs_s, outs)
    for k, g in enumerate(genomes):
        o, _ = oracle.eval_batch(g, suite[0], suite[2])
        assert same_bits(outs[k], o), f"tree {k} (size {g.size}, chunk {chunk})"


def test_error_behaviour_and_edge_cases(oracle, suite):
    """The reference's error conventions through the ABI: malformed genomes
    (stack underflow / leftover values), out-of-range plans and crossover
    points, a missing suite and misaligned packed offsets are errors (status
    < 0 with a message, no crash); single-node trees and one-tree populations
    evaluate normally, including on the streamed path."""
    with engine(suite) as e:
        for bad in ([ADD, X], [X, X], [ADD, X, X, X], [DIV]):
            e.upload_population([np.array(bad, np.uint8)])
            with pytest.raises(ltgp.EngineError, match="malformed"):
                e.evaluate_population()
        big_bad = np.concatenate([ltgp.remy_tree(5, 30001), np.array([X], np.uint8)])  # a leftover value
        e.upload_population([big_bad])
        with pytest.raises(ltgp.EngineError, match="malformed"):
            e.evaluate_population()
        # opcode 255 (invalid, opcodes.hpp:8-15) inside a tree is malformed,
        # wherever it falls: a leaf slot of a small tree, the middle of a
        # full packet of a large one, a chunked tree's interior, and on the
        # streamed path
        g = ltgp.random_tree_of_size(3, 40001)
        leaves = np.flatnonzero(g >= 4)
        for pos in (leaves[0], leaves[len(leaves) // 2], leaves[-1]):
            bad = g.copy()
            bad[pos] = 255
            for chunk in (0, 1024):
                with ltgp.Engine([0], node_limit=10**9, chunk_nodes=chunk) as e2:
                    e2.set_suite(*suite)
                    e2.upload_population([bad])
                    with pytest.raises(ltgp.EngineError, match="malformed"):
                        e2.evaluate_population()
                    b3, o3, s3 = pack([g, bad])
                    with pytest.raises(ltgp.EngineError, match="malformed"):
                        e2.evaluate_packed(b3, o3, s3)
        e.upload_population([np.array([ADD, X, 255], np.uint8)])
        with pytest.raises(ltgp.EngineError, match="malformed"):
            e.evaluate_population()
        # engine still usable afterwards
        one = [np.array([5 + 17], np.uint8)]
        e.upload_population(one)
        rec = e.evaluate_population()
        assert rec["size"][0] == 1 and rec["depth"][0] == 1
        buf, offs, sizes = pack(one)
        assert e.evaluate_packed(buf, offs, sizes).tobytes() == rec.tobytes()
        # crossover plans
        gs = [ltgp.random_tree_of_size(k, 101) for k in range(4)]
        e.upload_population(gs)
        e.evaluate_population()
        plans = np.zeros(4, ltgp.PLAN_DTYPE)
        plans["mum_index"] = [0, 1, 2, 7]
        with pytest.raises(ltgp.EngineError, match="outside the population"):
            e.execute_generation(plans)
        plans["mum_index"] = [0, 1, 2, 3]
        plans["mum_pt"] = [0, 1, 2, 101]
        with pytest.raises(ltgp.EngineError, match="out of range"):
            e.execute_generation(plans)
        # misaligned packed offsets
        b2, o2, s2 = pack(gs)
        o2[1] += 1
        with pytest.raises(ltgp.EngineError, match="16-aligned"):
            e.evaluate_packed(b2, o2, s2)
    with ltgp.Engine([0], node_limit=10**6) as e:
        e.upload_population([np.array([X], np.uint8)])
        with pytest.raises(ltgp.EngineError, match="set_suite"):
            e.evaluate_population()


@pytest.mark.skipif("_gpus() < 2", reason="needs >= 2 GPUs")
def test_run_bench_cells_multi_gpu():
    """run_bench (bench.hpp:33-35) cells with workers > 1 = GPUs
    (driver.hpp:44-51 grid {1, 2, 4, 8}, as many as are visible)."""
    ws = [w for w in (1, 2, 4, 8) if w <= _gpus()]
    cells = ltgp.run_bench([1001, 100001], ws, seed=1, min_corpus_nodes=2_000_000, repeats=2)
    assert len(cells) == 2 * len(ws)
    assert all(c["counters_consistent"] for c in cells)
    assert all(c["parallel_gpops"] > 0 for c in cells)


def test_run_bench_cells():
    """run_bench (bench.hpp:33-35) on the engine: one cell per (size, GPU
    count) with consistent node counters and a positive device throughput."""
    cells = ltgp.run_bench([1001, 20000], [1], seed=1, min_corpus_nodes=200_000, repeats=2)
    assert cells["tree_size"].tolist() == [1001, 20001]
    assert cells["nodes"].tolist() == [1001 * 200, 20001 * 10]
    assert (cells["counters_consistent"] == 1).all()
    assert (cells["batch_gpops"] > 0).all() and (cells["parallel_gpops"] == cells["batch_gpops"]).all()
    assert (cells["scalar_gpops"] == 0).all()
    with pytest.raises(ltgp.EngineError):
        ltgp.run_bench([1001], [0])



def test_reference_kat_grid_on_gpu():
    """The GPU arithmetic against bits printed by the reference's OWN inline
    apply_op / protected_div (eval.hpp:54-63, compiled from the reference
    headers by oracle/_ref/ref_kat, frozen in tests/golden/ref_inline_kats.json):
    20 special values (+-0, +-1, subnormals, FLT_MAX, +-inf, NaN, ...) as the
    constant table, every `op Ci Cj`. Bare 3-node trees run on the checked
    per-node path; the same pair wrapped as MUL(...MUL(op Ci Cj, 1)..., 1)
    puts the op inside a full packet (the generated fast path, including the
    packed division's domain check and its IEEE slow block). NaN payloads
    differ between x86 and the GPU: NaN matches NaN."""
    kats = json.load(open(os.path.join(HERE, "golden", "ref_inline_kats.json")))
    vals = np.array(kats["values"], np.uint32)
    nv = len(vals)
    consts = np.zeros(250, np.float32)
    consts[:nv] = vals.view(np.float32)
    one = 5 + int(np.flatnonzero(vals == 0x3F800000)[0])
    inputs = np.linspace(-1, 1, 48).astype(np.float32)
    targets = np.zeros(48, np.float32)
    for wrap in (0, 10, 11):
        genomes, expect = [], []
        for op in range(4):
            for i in range(nv):
                for j in range(nv):
                    core = [op, 5 + i, 5 + j]
                    genomes.append(np.array([MUL] * wrap + core + [one] * wrap, np.uint8))
                    expect.append(kats["apply_op"][op][i * nv + j])
        with ltgp.Engine([0], node_limit=10**6) as e:
            e.set_suite(inputs, targets, consts)
            e.upload_population(genomes)
            _, outs = e.evaluate_outputs()
        exp = np.array(expect, np.uint32).view(np.float32)
        for lane in (0, 1, 23, 47):
            assert same_bits(outs[:, lane], exp), f"wrap {wrap}, lane {lane}"
    # protected_div's own table equals apply_op's DIV row (same function)
    assert kats["protected_div"] == kats["apply_op"][3]


@pytest.mark.slow
def test_depth_beyond_2_24(oracle, suite):
    """Depth is an integer (genome.hpp:46 returns std::size_t): a right-deep
    chain ADD/SUB x (... ) of 2^24 + 11 function nodes has depth 2^24 + 12,
    which float32 cannot represent (a float depth chain sticks at 2^24). The
    tree (33.6M nodes) is chunked at the automatic length, so the depth also
    crosses the spine combine."""
    k = 2**24 + 11
    g = np.empty(2 * k + 1, np.uint8)
    g[0:2 * k:2] = np.where(np.arange(k) % 2 == 0, ADD, SUB)
    g[1:2 * k:2] = np.where(np.arange(k) % 3 == 0, X, 5 + 17)
    g[-1] = X
    with engine(suite) as e:
        e.upload_population([g])
        rec, outs = e.evaluate_outputs()
        assert e.stats()["last_chunks"] > 1
    assert int(rec["depth"][0]) == k + 1 == oracle.depth(g)
    o, _ = oracle.eval_batch(g, suite[0], suite[2])
    assert same_bits(outs[0], o)
    buf, offs, sizes = pack([g])
    assert_records_equal(rec, oracle.evaluate_population(buf, offs, sizes, suite, threads=0))


@pytest.mark.skipif("_gpus() < 2", reason="needs >= 2 GPUs (distinct-device NCCL all-gather and P2P splice)")
@pytest.mark.parametrize("G", [2, 4, 8])
def test_distinct_devices_nccl_matches_one_shard(oracle, suite, tmp_path, G):
    """The multi-GPU product path: a population sharded over
    G distinct GPUs, records all-gathered by one grouped ncclAllGather over
    NVLink (use_nccl), children spliced from parents on peer GPUs. Records
    and run dumps are byte-identical to one shard and to the oracle
    (bit-identical for any worker count, evolve.hpp:111-117)."""
    if _gpus() < G:
        pytest.skip(f"needs {G} GPUs")
    devs = list(range(G))
    buf, offs, sizes = ltgp.corpus(3, 64, 3.0, 5.0)
    genomes = [buf[int(o):int(o) + int(n)].copy() for o, n in zip(offs, sizes)]
    with engine(suite, devs) as e:
        assert e.gather_mode() == "nccl"
        e.upload_population(genomes)
        rec, outs = e.evaluate_outputs()
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    assert_records_equal(rec, exp)
    ref = tmp_path / "ref.txt"
    r = oracle.run(400, 60, 10**9, 7, 3, 0, str(ref), 1)
    d = tmp_path / "gpu.txt"
    with ltgp.Engine(devs, node_limit=10**9) as e:
        g = e.run(400, 60, 10**9, 7, 3, str(d), 1)
    assert g["generations"] == r["generations"] and g["nodes"] == r["nodes"]
    assert d.read_bytes() == ref.read_bytes()


def _streaming_model(psizes, csizes, plans, W):
    """The engine's streaming placement (splice_streaming), restated: first
    fit into free arena intervals, children in plan order in waves of W, a
    parent's bytes released after the wave of its last planned use. Returns
    (live genome high water, live byte high water)."""
    c16 = lambda n: (int(n) + 15) // 16 * 16  # noqa: E731
    P, M = len(psizes), len(csizes)
    last = [-1] * P
    for c, p in enumerate(plans):
        last[int(p["mum_index"])] = c
        last[int(p["dad_index"])] = c
    live, live_b = P, sum(c16(n) for n in psizes)
    live_hw, bytes_hw = live, live_b
    retire = {}
    for p in range(P):
        retire.setdefault(0 if last[p] < 0 else last[p] // W + 1, []).append(p)
    for p in retire.get(0, []):
        live -= 1
        live_b -= c16(psizes[p])
    for w, w0 in enumerate(range(0, M, W), start=1):
        for c in range(w0, min(M, w0 + W)):
            live += 1
            live_b += c16(csizes[c])
        live_hw, bytes_hw = max(live_hw, live), max(bytes_hw, live_b)
        for p in retire.get(w, []):
            live -= 1
            live_b -= c16(psizes[p])
    return live_hw, bytes_hw


def test_streaming_memory_mode(oracle, suite, tmp_path):
    """RunConfig::streaming_memory (evolve.hpp:45, :111-114; SPEC.md:367,
    :387): children spliced in waves into the parents' own
    arena, a parent's bytes released after its last planned use. Records
    equal the double-buffered mode's; the live-genome and live-byte high
    waters equal a restated model of the policy and stay below 2M; a whole
    run's dump equals the oracle's."""
    gs = [ltgp.random_tree_of_size(300 + k, 2 * (k % 97) + 1) for k in range(500)]
    rec0 = np.zeros(len(gs), REC)
    with engine(suite) as e:
        e.upload_population(gs)
        rec0 = e.evaluate_population()
    plans = oracle.plan_generation(9, rec0)
    csizes = []
    for p in plans:
        mum, dad = gs[int(p["mum_index"])], gs[int(p["dad_index"])]
        ms, me = oracle.subtree_extent(mum, int(p["mum_pt"]))
        ds, de = oracle.subtree_extent(dad, int(p["dad_pt"]))
        csizes.append(mum.size - (me - ms) + (de - ds))
    results = {}
    for streaming in (False, True):
        with engine(suite) as e:
            if streaming:
                e.set_streaming(True, 64)
            e.upload_population(gs)
            e.evaluate_population()
            rec, hit = e.execute_generation(plans)
            assert not hit
            st = e.stats()
            kids = [e.download_genome(i) for i in range(0, len(gs), 37)]
            results[streaming] = (rec, st, kids)
    assert results[True][0].tobytes() == results[False][0].tobytes()
    assert all(np.array_equal(a, b) for a, b in zip(results[True][2], results[False][2]))
    live_hw, bytes_hw = _streaming_model([g.size for g in gs], csizes, plans, 64)
    st = results[True][1]
    assert st["live_genomes_high_water"] == live_hw < 2 * len(gs)
    assert st["arena_used_high_water"] == bytes_hw
    assert bytes_hw < sum((g.size + 15) // 16 * 16 for g in gs) + sum((n + 15) // 16 * 16 for n in csizes)
    # a whole bloating run in streaming mode (arena regrows keep the parents)
    ref = tmp_path / "ref.txt"
    r = oracle.run(400, 60, 10**9, 7, 6, 0, str(ref), 1)
    d = tmp_path / "gpu.txt"
    with ltgp.Engine([0], node_limit=10**9) as e:
        e.set_streaming(True, 32)
        g = e.run(400, 60, 10**9, 7, 6, str(d), 1)
        assert e.stats()["live_genomes_high_water"] < 2 * 400
    assert g["generations"] == r["generations"] and g["nodes"] == r["nodes"]
    assert d.read_bytes() == ref.read_bytes()


def test_nccl_attach_one_rank(oracle, suite):
    """One process per GPU (ltgp_nccl_attach, bench.py --gpus N): a
    single-rank communicator across processes; every evaluation all-gathers
    the records inside the engine, equal to the records."""
    buf, offs, sizes = ltgp.corpus(3, 60, 3.0, 4.5)
    uid = ltgp.nccl_unique_id()
    with engine(suite) as e:
        e.nccl_attach(uid, 1, 0)
        assert e.gather_mode() == "nccl-processes"
        e.upload_packed(buf, offs, sizes)
        rec = e.evaluate_population()
        assert e.gathered_records().tobytes() == rec.tobytes()
        rec2 = e.evaluate_packed(buf, offs, sizes)
        assert e.gathered_records().tobytes() == rec2.tobytes() == rec.tobytes()
        with pytest.raises(ltgp.EngineError):
            e.nccl_attach(uid, 1, 0)  # already attached
    assert_records_equal(rec, oracle.evaluate_population(buf, offs, sizes, suite, threads=0))


@pytest.mark.skipif("_gpus() < 2")
def test_bench_multi_gpu_engine_gather(tmp_path):
    """bench.py --gpus 2 under torchrun (the SCALE run's launch): each rank's
    engine all-gathers every rank's records through its own NCCL
    communicator, and each rank's block is its own records."""
    import subprocess
    import sys
    root = os.path.dirname(HERE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-evolution", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["collective"]["impl"] == "nccl-processes" and line["collective"]["own_block_matches"]
    assert "ncclCommInitRank nranks=2" in out.stderr
