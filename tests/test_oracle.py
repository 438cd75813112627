"""Pin the CPU oracle before trusting it (CPU only).

1. against known answers printed by the reference's OWN inline code
   (tests/golden/ref_inline_kats.json, made by oracle/_ref/ref_kat from
   /root/reference/proj/include/ltgp/{rng,eval,evolve}.hpp);
2. against every SPEC example for the path (SPEC.md line cited per test);
3. against the SPEC properties (oracle equivalence, stack discipline,
   reduction order, crossover size algebra).
"""
import json
import math
import os

import numpy as np
import pytest

from tests._oracle import same_bits

HERE = os.path.dirname(os.path.abspath(__file__))
KATS = json.load(open(os.path.join(HERE, "golden", "ref_inline_kats.json")))

ADD, SUB, MUL, DIV, X = 0, 1, 2, 3, 4


def f32(bits):
    return np.array([bits], np.uint32).view(np.float32)[0]


# --- 1. reference-pinned known answers ------------------------------------
def test_splitmix64_matches_reference(oracle):
    for x, y in KATS["splitmix64"]:
        assert oracle.orc_splitmix64(int(x)) == int(y)


def test_rng_below_matches_reference(oracle):
    for case in KATS["below"]:
        out = np.zeros(16, np.uint64)
        oracle.orc_rng_below_seq(case["seed"], int(case["n"]), 16, out.ctypes.data)
        assert [int(v) for v in out] == [int(v) for v in case["v"]], case


def test_rng_uniform_matches_reference(oracle):
    for case in KATS["uniform_pm1"]:
        out = np.zeros(48, np.float32)
        oracle.orc_rng_uniform_seq(case["seed"], 48, out.ctypes.data)
        assert out.view(np.uint32).tolist() == case["bits"]


def test_survey_appendix_b_rng(oracle):
    # SURVEY.md App. B (computed from rng.hpp): Rng(1) below(255) x5
    out = np.zeros(5, np.uint64)
    oracle.orc_rng_below_seq(1, 255, 5, out.ctypes.data)
    assert out.tolist() == [135, 227, 227, 141, 28]
    assert oracle.orc_splitmix64(42) == 0xbdd732262feb6e95


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_apply_op_and_protected_div_match_reference(oracle):
    vals = [f32(b) for b in KATS["values"]]
    n = len(vals)
    for op in range(4):
        exp = KATS["apply_op"][op]
        for i in range(n):
            for j in range(n):
                if op < 3:
                    got = {0: np.float32(vals[i] + vals[j]), 1: np.float32(vals[i] - vals[j]),
                           2: np.float32(vals[i] * vals[j])}[op]
                else:
                    got = np.float32(oracle.orc_protected_div(vals[i], vals[j]))
                assert same_bits([got], [f32(exp[i * n + j])]), (op, i, j)
    for k, b in enumerate(KATS["protected_div"]):
        got = np.float32(oracle.orc_protected_div(vals[k // n], vals[k % n]))
        assert same_bits([got], [f32(b)])


def test_fitness_order_matches_reference(oracle):
    vals = [f32(b) for b in KATS["values"]]
    n = len(vals)
    for k in range(n * n):
        a, b = vals[k // n], vals[k % n]
        assert oracle.orc_fitness_better(a, b) == KATS["fitness_better"][k]
        assert oracle.orc_fitness_tied(a, b) == KATS["fitness_tied"][k]


def test_abi_layout_matches_reference():
    from paper_1902_09215_b200 import PLAN_DTYPE
    lay = KATS["layout"]
    assert PLAN_DTYPE.itemsize == lay["CrossoverPlan"][0]
    assert [PLAN_DTYPE.fields[f][1] for f in PLAN_DTYPE.names] == lay["CrossoverPlan"][1:]
    assert lay["kLaneWidth"] == 48 and lay["kConstantCount"] == 250


# --- 2. SPEC examples -------------------------------------------------------
def test_protected_div_spec(oracle):
    # SPEC.md:179-181, 557
    for a in (0.0, 1.0, -3.5, math.inf):
        assert oracle.orc_protected_div(a, 0.0) == 1.0
    assert oracle.orc_protected_div(1.0, -0.0) == 1.0
    assert oracle.orc_protected_div(6.0, 3.0) == 2.0


def test_eval_scalar_spec(oracle):
    c = np.zeros(250, np.float32)
    assert oracle.eval_scalar([X], 0.25, c) == np.float32(0.25)
    assert oracle.eval_scalar([ADD, X, X], 0.25, c) == np.float32(0.5)
    assert oracle.eval_scalar([SUB, MUL, X, X, X], 0.5, c) == np.float32(-0.25)


def test_eval_batch_spec(oracle):
    i, t, c = oracle.make_suite(oracle.orc_suite_seed(1))
    out, _ = oracle.eval_batch([X], i, c)
    assert same_bits(out, i)
    out, _ = oracle.eval_batch([5 + 17], i, c)
    assert same_bits(out, np.full(48, c[17], np.float32))


def test_target_spec(oracle):
    assert oracle.orc_target(0.5) == np.float32(0.140625)
    for x in (0.0, 1.0, -1.0):
        assert oracle.orc_target(x) == 0.0


def test_fitness_hits_spec(oracle):
    t = np.linspace(-0.5, 0.5, 48).astype(np.float32)
    assert oracle.fitness(t, t) == 0.0
    assert oracle.hits(t, t) == 48
    assert oracle.hits(t + np.float32(0.02), t) == 0
    off = (t + np.float32(0.01)).astype(np.float32)
    s = np.float32(0)
    for k in range(48):
        s = np.float32(s + np.float32(abs(np.float32(off[k] - t[k]))))
    assert oracle.fitness(off, t) == np.float32(s / np.float32(48))       # SPEC.md:207 (sequential)


def test_flajolet_spec(oracle):
    assert abs(oracle.orc_flajolet_stack_bound(2, 1.0) - 3.5449) < 1e-4
    # SPEC.md:225 quotes "~9708.4"; the formula it states gives 9708.13
    assert abs(oracle.orc_flajolet_stack_bound(15_000_000, 1.0) - 9708.4) < 0.5
    assert abs(oracle.orc_flajolet_stack_bound(15_000_000, 1.0) - 2 * math.sqrt(math.pi * 7_500_000)) < 1e-9


def test_genome_spec(oracle):
    assert oracle.depth([X]) == 1 and oracle.depth([ADD, X, X]) == 2
    assert oracle.depth([ADD, ADD, X, X, X]) == 3
    assert oracle.subtree_extent([ADD, X, X], 0) == (0, 3)
    assert oracle.subtree_extent([ADD, X, X], 1) == (1, 2)
    assert oracle.subtree_extent([ADD, MUL, X, X, X], 1) == (1, 4)
    with pytest.raises(IndexError):
        oracle.subtree_extent([ADD, X, X], 3)
    assert oracle.validate([ADD, X, X])
    assert not oracle.validate([ADD, X])
    assert not oracle.validate([X, X])
    child, hit, n = oracle.crossover([ADD, X, X], [X], 0, 0, 100)
    assert child.tolist() == [X] and not hit
    child, hit, n = oracle.crossover([ADD, X, X], [MUL, X, X], 1, 0, 100)
    assert child.tolist() == [ADD, MUL, X, X, X] and n == 5
    _, hit, n = oracle.crossover([ADD, X, X], [MUL, X, X], 1, 0, 5)      # SPEC.md:140 (>= limit)
    assert hit and n == 5


def test_gen_full_spec(oracle):
    import ctypes
    for d, n in ((1, 1), (3, 7), (6, 63)):
        seed = ctypes.c_uint64(5)
        out = np.zeros(64, np.uint8)
        assert oracle.orc_gen_full(ctypes.byref(seed), d, 1000, out.ctypes.data, 64) == n
        assert oracle.depth(out[:n]) == d


def test_ramped_spec(oracle):
    pop = oracle.ramped(3, 10)
    assert all(oracle.validate(g) for g in pop)
    depths = [oracle.depth(g) for g in pop]
    assert max(depths) <= 6
    assert [depths[i] for i in range(0, 10, 2)] == [2, 3, 4, 5, 6]        # full trees: exact depth


# --- 3. properties ----------------------------------------------------------
def test_eval_batch_equals_eval_scalar(oracle):
    # SPEC.md:199, 229, 555 (oracle equivalence, bit-identical per lane)
    i, t, c = oracle.make_suite(oracle.orc_suite_seed(2))
    rng = np.random.default_rng(0)
    for k in range(300):
        n = int(rng.integers(0, 2000)) * 2 + 1
        g = oracle.random_tree_of_size(7000 + k, n)
        out, peak = oracle.eval_batch(g, i, c)
        ref = np.array([oracle.eval_scalar(g, x, c) for x in i], np.float32)
        assert same_bits(out, ref)                                        # all 48 lanes
        assert peak <= oracle.depth(g)


def test_eval_batch_equals_eval_scalar_adversarial(oracle):
    i, t, c = oracle.make_suite(oracle.orc_suite_seed(3))
    # deep left chain DIV(DIV(...X...)...) and MUL chains (overflow to inf / NaN)
    chain = [DIV] * 200 + [X] + [5 + 3] * 200
    g = np.array(chain, np.uint8)
    out, _ = oracle.eval_batch(g, i, c)
    ref = np.array([oracle.eval_scalar(g, x, c) for x in i], np.float32)
    assert same_bits(out, ref)
    # x / (x - x): zero divisor in every lane
    g = np.array([DIV, X, SUB, X, X], np.uint8)
    out, _ = oracle.eval_batch(g, i, c)
    assert np.all(out == 1.0)


def test_fitness_not_reassociated(oracle):
    # SPEC.md:232 (reduction-order mutation check): 1e8 followed by 47 ones.
    # Left to right every +1 is absorbed (ulp(1e8) = 8): the sum is 1e8.
    # Any other order that adds the ones first gives 1e8 + 48 (a reversed
    # sum, a pairwise tree): the MAE must be the left-to-right one.
    t = np.zeros(48, np.float32)
    out = np.array([1e8] + [1.0] * 47, np.float32)
    s = np.float32(0)
    for v in out:
        s = np.float32(s + np.float32(abs(v)))
    assert s == np.float32(1e8)
    assert oracle.fitness(out, t) == np.float32(s / np.float32(48))
    rev = np.float32(0)
    for v in out[::-1]:
        rev = np.float32(rev + np.float32(abs(v)))
    pairwise = np.float32(np.float32(np.abs(out[:24]).sum(dtype=np.float32)) +
                          np.float32(np.abs(out[24:]).sum(dtype=np.float32)))
    assert rev != s and pairwise != s
    assert oracle.fitness(out, t) != np.float32(rev / np.float32(48))
    assert oracle.fitness(out, t) != np.float32(pairwise / np.float32(48))


def test_crossover_size_algebra(oracle):
    # size(child) = size(mum) - |extent_mum| + |extent_dad|
    rng = np.random.default_rng(1)
    for k in range(300):
        mum = oracle.random_tree_of_size(100 + k, int(rng.integers(0, 200)) * 2 + 1)
        dad = oracle.random_tree_of_size(900 + k, int(rng.integers(0, 200)) * 2 + 1)
        mp, dp = int(rng.integers(0, mum.size)), int(rng.integers(0, dad.size))
        child, hit, n = oracle.crossover(mum, dad, mp, dp, 10**9)
        ms, me = oracle.subtree_extent(mum, mp)
        ds, de = oracle.subtree_extent(dad, dp)
        assert n == mum.size - (me - ms) + (de - ds)
        assert oracle.validate(child)
        assert child.tolist() == mum[:ms].tolist() + dad[ds:de].tolist() + mum[me:].tolist()


def test_random_tree_of_size_shapes(oracle):
    for n in (1, 3, 5, 101, 10001):
        g = oracle.random_tree_of_size(n, n)
        assert g.size == n and oracle.validate(g)


def test_oracle_golden_frozen(oracle):
    """The frozen oracle outputs (tests/golden/oracle_golden.json) still hold."""
    g = json.load(open(os.path.join(HERE, "golden", "oracle_golden.json")))
    for s, d in g["suites"].items():
        i, t, c = oracle.make_suite(oracle.orc_suite_seed(int(s)))
        assert i.view(np.uint32).tolist() == d["inputs"]
        assert t.view(np.uint32).tolist() == d["targets"]
        assert c.view(np.uint32).tolist() == d["constants"]
    i, t, c = oracle.make_suite(oracle.orc_suite_seed(1))
    for tr in g["trees"]:
        tree = oracle.random_tree_of_size(tr["seed"], tr["n"])
        out, _ = oracle.eval_batch(tree, i, c)
        assert out.view(np.uint32).tolist() == tr["outputs_bits"]


def test_run_determinism_thread_invariance(oracle, tmp_path):
    # seeds x workers give byte-identical dumps (small scale)
    for seed in (1, 2):
        dumps = []
        for threads in (1, 2, 8):
            p = tmp_path / f"d{seed}_{threads}.txt"
            r = oracle.run(48, 15, 10**9, 7, seed, threads, str(p), 1)
            assert r["generations"] == 15
            dumps.append(p.read_bytes())
        assert dumps[0] == dumps[1] == dumps[2]


def test_run_size_limit(oracle):
    # node_limit=63, bloating run terminates with SizeLimitHit
    r = oracle.run(48, 500, 63, 7, 1, 1, None)
    assert r["reason"] == 1 and r["generations"] < 500


def budget_case(dump_text, gens):
    """From an unbudgeted run's dump: per-generation genome bytes T[g] and a
    memory budget under which generation g0 is the first refused (its planned
    bytes T[g0-1] + T[g0] exceed the budget, every earlier one fits)."""
    T = [0] * (gens + 1)
    for line in dump_text.splitlines():
        g, _, size = line.split()[:3]
        T[int(g)] += int(size)
    planned = [T[g - 1] + T[g] for g in range(1, gens + 1)]
    # the last generation (after the first) whose planned bytes set a new record
    records = [g for g in range(2, gens + 1) if planned[g - 1] > max(planned[: g - 1])]
    assert records, "no generation plans more bytes than all before it (the run does not bloat)"
    g0 = records[-1]
    return max(planned[: g0 - 1]), g0


def test_run_memory_budget(oracle, tmp_path):
    # SPEC.md:376, :395 / evolve.hpp:44, :89-93: with a memory budget the run
    # stops with MemoryBudgetExceeded before materializing the first
    # generation whose planned bytes (parents + children) exceed it; the
    # generations before are unchanged
    G = 40
    full = tmp_path / "full.txt"
    r = oracle.run(48, G, 10**9, 7, 1, 2, str(full), 1)
    assert r["reason"] == 0 and r["generations"] == G
    budget, g0 = budget_case(full.read_text(), G)
    assert g0 > 1
    cut = tmp_path / "cut.txt"
    rb = oracle.run(48, G, 10**9, 7, 1, 2, str(cut), 1, memory_budget=budget)
    assert rb["reason"] == 2 and rb["generations"] == g0 - 1
    lines = full.read_text().splitlines()
    assert cut.read_text().splitlines() == lines[: 48 * g0]
    # budget 0 disables the check
    assert oracle.run(48, G, 10**9, 7, 1, 2, None, 1, memory_budget=0)["reason"] == 0
