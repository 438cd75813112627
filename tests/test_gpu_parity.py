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
        rec = e.evaluate_population()
        rec2 = e.evaluate_population()
    assert rec.tobytes() == rec2.tobytes()  # determinism across launches
    exp = oracle.evaluate_population(buf, offs, sizes, suite, threads=0)
    assert_records_equal(rec, exp)


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
    """Config 2 scale: pop 4000, tournament 7, no size limit, 100 generations
    with the bloating grow variant; 2 shards; dumps identical to the oracle."""
    r = oracle.run(4000, 100, 2**62, 7, 1, 0, str(tmp_path / "a"), 1)
    with ltgp.Engine([0, 0], node_limit=2**62) as e:
        g = e.run(4000, 100, 2**62, 7, 1, str(tmp_path / "b"), 1)
    assert r["generations"] == g["generations"] == 100
    assert r["nodes"] == g["nodes"]
    assert (tmp_path / "a").read_bytes() == (tmp_path / "b").read_bytes()


@pytest.mark.parametrize("round_", range(int(os.environ.get("LTGP_FUZZ_ROUNDS", "3"))))
def test_randomized_populations(oracle, suite, round_):
    """Randomized sweep: mixed shapes (Remy, uniform splits, ramped
    half-and-half, left/right chains), random sizes and chunk lengths, the
    resident and the streamed path; every record and per-case output equal
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

