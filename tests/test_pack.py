"""The packed PCIe form of a streamed evaluation (csrc/ltgp_pack.h), on the
CPU: packing is lossless for every byte value and length, independent of
the thread count and of the encoder (AVX-512 or scalar), and its layout is
what k_decode_packed reads. The GPU side (k_decode_packed rebuilding the
arena) is covered by the streamed-path parity tests in test_gpu_parity.py."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1902_09215_b200 as ltgp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ceil16(x):
    return (x + 15) & ~15


def unpack(pk: np.ndarray, n: int) -> np.ndarray:
    """Restatement of the format: three 16-bit code planes per 16-byte
    packet, block literal bases, literals in byte order."""
    npk = (n + 15) // 16
    nblk = (npk + 255) // 256
    plane = nblk * 512   # whole blocks of 256 packets
    base_off = 3 * plane
    lit_off = base_off + (nblk * 4 + 63) // 64 * 64
    planes = [pk[j * plane: j * plane + 2 * npk].view(np.uint16) for j in range(3)]
    bits = np.arange(16, dtype=np.uint16)
    code = sum(((planes[j][:, None] >> bits) & 1).astype(np.uint8) << j for j in range(3)).reshape(-1)
    lit = code == 5
    out = np.where(code == 6, 0xFF, code).astype(np.uint8)
    nlit = int(lit.sum())
    assert pk.size == lit_off + nlit, "packed size = header + literals"
    out[lit] = pk[lit_off: lit_off + nlit]
    # block bases: literals before each block of 256 packets
    base = pk[base_off: base_off + 4 * nblk].view(np.uint32)
    if nblk:
        per_block = np.add.reduceat(lit.astype(np.int64), np.arange(0, npk * 16, 256 * 16))
        assert np.array_equal(base, np.concatenate([[0], np.cumsum(per_block)[:-1]]).astype(np.uint32))
    assert (code[n:] == 6).all(), "bytes past the end read as padding"
    for j in range(3):  # the last block's unused packets encode 0xFF bytes
        pad = pk[j * plane + 2 * npk: (j + 1) * plane].view(np.uint16)
        assert (pad == (0 if j == 0 else 0xFFFF)).all()
    return out[:n]


def corpus_bytes(n):
    rng = np.random.default_rng(7)
    u = rng.integers(0, 256, n)
    return np.where(u < 128, u & 3, np.where(u < 192, 4, 5 + (u * 7) % 250)).astype(np.uint8)


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 63, 64, 65, 4095, 4096, 4097, 70_001, 1 << 20])
def test_round_trip_every_byte_value(n):
    rng = np.random.default_rng(n)
    buf = rng.integers(0, 256, n, dtype=np.uint8)
    pk = ltgp.pack_host(buf, 3)
    assert np.array_equal(unpack(pk, n), buf)


def test_corpus_ratio_and_threads():
    buf = corpus_bytes(5_000_003)
    one = ltgp.pack_host(buf, 1)
    assert np.array_equal(unpack(one, buf.size), buf)
    for t in (2, 7, 16):
        assert np.array_equal(ltgp.pack_host(buf, t), one)
    # 3 bits a byte plus a literal per constant (a quarter of the bytes here)
    assert abs(one.size / buf.size - 0.625) < 0.01


def test_config3_corpus_round_trip():
    buf, offs, sizes = ltgp.corpus(1, 40, 3.0, 4.0)
    pk = ltgp.pack_host(buf, 4)
    assert np.array_equal(unpack(pk, buf.size), buf)
    assert pk.size < 0.7 * buf.size


def test_scalar_encoder_matches_simd():
    code = ("import numpy as np, paper_1902_09215_b200 as ltgp, sys;"
            "b=np.random.default_rng(3).integers(0,256,300_017,dtype=np.uint8);"
            "sys.stdout.buffer.write(ltgp.pack_host(b, 4).tobytes())")
    outs = []
    for scalar in (False, True):
        env = dict(os.environ, PYTHONPATH=ROOT)
        env.pop("LTGP_PACK_SCALAR", None)
        if scalar:
            env["LTGP_PACK_SCALAR"] = "1"
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, check=True).stdout)
    assert outs[0] == outs[1] and len(outs[0]) > 0
