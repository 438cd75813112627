"""The reference-typed drop-in (libltgp_refabi.so, host/evolve_cuda.cpp).

The reference's own declarations (/root/reference/proj/include/ltgp/
evolve.hpp:106-117, eval.hpp:27-79) are defined on the engine by a file that
includes the reference's UNMODIFIED headers. CPU tests: the library exports
exactly the reference's mangled signatures, and (where /root/reference is
present) it compiles from scratch against those headers together with a
reference-typed run loop. GPU tests: that run loop (tests/refabi/ref_run.cpp,
the reference's run.hpp:33-36 order on the reference's types) writes a
generation dump byte-identical to the CPU oracle's run().
"""
import os
import subprocess

import pytest

from paper_1902_09215_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# the reference declarations libltgp_refabi.so must define (demangled)
REFERENCE_SYMBOLS = [
    "ltgp::evaluate_population(std::vector<ltgp::Individual, std::allocator<ltgp::Individual> >&, ltgp::ExecContext)",
    "ltgp::execute_generation(std::span<ltgp::CrossoverPlan const, 18446744073709551615ul>, "
    "std::vector<ltgp::Individual, std::allocator<ltgp::Individual> >&, "
    "std::vector<ltgp::Individual, std::allocator<ltgp::Individual> >&, ltgp::ExecContext)",
    "ltgp::evaluate_individual(ltgp::Individual&, ltgp::TestSuite const&, ltgp::WorkerState&)",
    "ltgp::eval_batch_raw(ltgp::Genome const&, float const*, std::span<float const, 18446744073709551615ul>, "
    "ltgp::EvalStack&, ltgp::GpopsCounter*)",
    "ltgp::eval_batch(ltgp::Genome const&, std::array<float, 48ul> const&, "
    "std::span<float const, 18446744073709551615ul>, ltgp::EvalStack&, ltgp::GpopsCounter*)",
    "ltgp::EvalStack::reserve_frames(unsigned long)",
    "ltgp::EvalStack::grow(unsigned long, unsigned long)",
]


def _defined(lib):
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    return {line.split(" ", 2)[2] for line in out.splitlines() if line.count(" ") >= 2}


def test_refabi_exports_the_reference_signatures():
    assert B.build_refabi(), "libltgp_refabi.so missing (build it where /root/reference exists)"
    syms = _defined(B.REFABI_LIB)
    for s in REFERENCE_SYMBOLS:
        assert s in syms, s
    for s in ("ltgp_ref_bind_engine", "ltgp_ref_unbind", "ltgp_ref_engine"):
        assert s in syms


@pytest.mark.skipif(not os.path.isdir(B.REF_INC), reason="needs the reference headers (/root/reference)")
def test_refabi_compiles_against_unmodified_reference_headers(tmp_path):
    """A fresh compile of the adapter and of the reference-typed harness with
    -I/root/reference/proj/include and nothing of the repo's own C++ type
    mirror: the definitions match the reference's declarations, and the
    harness links (every reference function it calls is defined)."""
    inc = ["-I" + B.REF_INC, "-I" + os.path.join(ROOT, "include")]
    lib = tmp_path / "libltgp_refabi.so"
    subprocess.run(["g++", *B.CXX_FLAGS, "-Werror", *inc, "-shared", "-o", str(lib), B.REFABI_SRC,
                    "-L" + B.PKG, "-lltgp_cuda"], check=True)
    oracle_dir = os.path.join(ROOT, "oracle")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Werror", *inc, "-o", str(tmp_path / "ref_run"),
                    B.REF_RUN_SRC, "-L" + str(tmp_path), "-lltgp_refabi", "-L" + B.PKG, "-lltgp_cuda",
                    "-L" + oracle_dir, "-lltgp_oracle", "-Wl,--no-undefined"], check=True)
    for s in REFERENCE_SYMBOLS:
        assert s in _defined(str(lib))


def _ref_run(tmp_path, M, G, limit, seed, grow, mode):
    d = tmp_path / f"refabi_{mode}.txt"
    r = subprocess.run([B.REF_RUN_BIN, str(M), str(G), str(limit), "7", str(seed), str(grow), str(d), mode],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    f = r.stdout.split()
    return d, dict(zip(f[0::2], f[1::2]))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["0", "1", "default"])
def test_reference_typed_run_matches_oracle(oracle, tmp_path, mode):
    """The reference's loop on the reference's types, with the engine behind
    evaluate_population / execute_generation: children device-resident
    (mode 0), children genomes copied back into Individual::genome (mode 1),
    or an engine the adapter creates itself (default). The dump equals the
    oracle's run(); the GpopsCounter of the worker pool counts every node."""
    ref = tmp_path / "oracle.txt"
    r = oracle.run(48, 40, 10**9, 7, 2, 0, str(ref), 1)
    d, out = _ref_run(tmp_path, 48, 40, 10**9, 2, 1, mode)
    assert int(out["generations"]) == r["generations"] == 40
    assert int(out["nodes"]) == r["nodes"]
    assert float(out["elapsed"]) > 0
    assert d.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
def test_reference_typed_run_size_limit(oracle, tmp_path):
    """SizeLimitHit through the reference's ExecOutcome (evolve.hpp:102-104):
    node_limit 63 stops the run at the same generation as the oracle's."""
    ref = tmp_path / "oracle.txt"
    r = oracle.run(48, 300, 63, 7, 4, 0, str(ref))
    d, out = _ref_run(tmp_path, 48, 300, 63, 4, 0, "0")
    assert r["reason"] == 1 and int(out["reason"]) == 1
    assert int(out["generations"]) == r["generations"]
    assert d.read_bytes() == ref.read_bytes()


@pytest.mark.gpu
def test_reference_typed_single_genome_entry_points(oracle):
    """evaluate_individual (evolve.hpp:106), eval_batch_raw and eval_batch
    (eval.hpp:73-79) of libltgp_refabi.so, called on the reference's own
    types (Individual, TestSuite, WorkerState, Genome, EvalStack,
    GpopsCounter): record and all 48 outputs equal the oracle's, eval_batch
    equals eval_batch_raw, and the GpopsCounter counts every node."""
    import numpy as np
    from tests._oracle import same_bits
    r = subprocess.run([B.REF_RUN_BIN, "eval", "3", "24"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    suite = oracle.make_suite(int(oracle.orc_suite_seed(3)))
    total = 0
    for head, gl in zip(lines[0:-1:2], lines[1:-1:2]):
        f = head.split()
        g = np.frombuffer(bytes.fromhex(gl[1:]), np.uint8)
        n, fit_bits, hits, size, depth = int(f[0]), int(f[1], 16), int(f[2]), int(f[3]), int(f[4])
        outs = np.array([int(x, 16) for x in f[5:53]], np.uint32).view(np.float32)
        assert f[53] == "1" and g.size == n == size
        o, _ = oracle.eval_batch(g, suite[0], suite[2])
        assert same_bits(outs, o)
        assert same_bits(np.array([fit_bits], np.uint32).view(np.float32), [oracle.fitness(o, suite[1])])
        assert hits == oracle.hits(o, suite[1]) and depth == oracle.depth(g)
        total += n
    counter = lines[-1].split()
    assert counter[0] == "counter" and int(counter[1]) == total and float(counter[2]) > 0
