"""Pins for oracle.quant (GPTQ asymmetric grid; readings D14-D17)."""
import numpy as np
import pytest
import torch

from oracle import quant
from oracle.bf16 import round_bf16
from golden_util import load_golden
import synthetic

Q = load_golden("quant_examples.json")


@pytest.mark.parametrize("case", Q["cases"])
def test_worked_examples(case):
    w = np.array([case["w"]], np.float32)
    q, s, z = quant.quantize_groups(w, case["bits"], case["group"])
    assert q[0].tolist() == case["codes"]
    assert int(z[0, 0]) == case["zero"]
    if "scale" in case:
        assert float(s[0, 0]) == case["scale"]
    if "inv" in case:
        assert float(np.float32(1) / s[0, 0]) == case["inv"]
    if "max_err" in case:
        err = np.abs(w[0].astype(np.float64) - (q[0].astype(np.float64) - z[0, 0]) * float(s[0, 0]))
        assert err.max() == pytest.approx(case["max_err"], rel=1e-6)


def test_pack_layout():
    p = Q["pack"]
    words = quant.pack(np.array([p["codes"]], np.uint8), p["bits"])
    assert "%08x" % int(words[0, 0]) == p["word_hex"]
    w2 = quant.pack(np.array([[3, 0, 1, 2] * 4], np.uint8), 2)
    assert int(w2[0, 0]) == sum(c << (2 * i) for i, c in enumerate([3, 0, 1, 2] * 4))
    w8 = quant.pack(np.array([[0x11, 0x22, 0x33, 0xff]], np.uint8), 8)
    assert int(w8[0, 0]) == 0xff332211


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_pack_roundtrip(bits):
    rng = np.random.default_rng(bits)
    q = rng.integers(0, 2 ** bits, size=(7, 256)).astype(np.uint8)
    assert np.array_equal(quant.unpack(quant.pack(q, bits), bits, 256), q)


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_grid_aligned_roundtrip_exact(bits):
    # w = (q - z) * s with s a power of two, group containing both grid ends -> exact
    maxq = 2 ** bits - 1
    rng = np.random.default_rng(10 + bits)
    G = 128
    rows = []
    for r in range(16):
        s = 2.0 ** int(rng.integers(-8, 0))
        z = int(rng.integers(1, maxq))
        q = rng.integers(0, maxq + 1, size=G)
        q[0], q[1] = 0, maxq
        rows.append((q - z) * s)
    w = np.array(rows, np.float32)
    assert (round_bf16(w) == w).all()
    q, s, z = quant.quantize_groups(w, bits, G)
    recon = (q.astype(np.float64) - z.astype(np.float64)) * s.astype(np.float64)
    assert np.array_equal(recon, w.astype(np.float64))


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("kind", ["normal", "positive", "negative", "zeros", "tiny", "mixed"])
def test_error_bound_and_brute_force(bits, kind):
    w = synthetic.random_matrix_bf16(8, 512, seed=bits, kind=kind).float().numpy()
    q, s, z = quant.quantize_groups(w, bits, 128)
    maxq = 2 ** bits - 1
    assert q.max() <= maxq and z.max() <= maxq
    wg = w.reshape(8, 4, 128).astype(np.float64)
    s64 = s.astype(np.float64)[:, :, None]
    qz = q.reshape(8, 4, 128).astype(np.float64) - z.astype(np.float64)[:, :, None]
    err = np.abs(wg - qz * s64)
    # |w - (q - z) s| <= s/2 up to the float32 rounding of w * inv
    assert (err <= s64 * (0.5 + 1e-5)).all()
    # brute force: q is the nearest grid point among all 2**b candidates (up to ties
    # decided within float32 rounding of w*inv)
    cand = (np.arange(maxq + 1)[None, None, None, :] - z[:, :, None, None]) * s64[..., None]
    d = np.abs(wg[..., None] - cand)
    best = d.min(-1)
    mine = np.take_along_axis(d, q.reshape(8, 4, 128, 1).astype(np.int64), -1)[..., 0]
    assert (mine <= best + s64 * 1e-5).all()
    # the grid contains 0 exactly (GPTQ widens min/max to include 0): z in [0, maxq]
    assert ((0 - z.astype(np.int64)) <= 0).all()


def test_division_vs_reciprocal_reading():
    # D16: the contract uses rint(w * (1/s)); rint(w / s) differs on rare groups.  Here we
    # only check the reciprocal form is what the oracle computes, on a case where they differ.
    rng = np.random.default_rng(0)
    found = False
    for _ in range(200):
        w = (rng.standard_normal((64, 128)) * 0.02).astype(np.float32)
        w = round_bf16(w).astype(np.float32)
        q, s, z = quant.quantize_groups(w, 8, 128)
        inv = (np.float32(1) / s).astype(np.float32)
        q_div = np.clip(np.rint(w / s.repeat(128, 1)) + z.repeat(128, 1), 0, 255)
        q_rec = np.clip(np.rint((w * inv.repeat(128, 1)).astype(np.float32)) + z.repeat(128, 1), 0, 255)
        assert np.array_equal(q, q_rec.astype(np.uint8))
        if not np.array_equal(q_div, q_rec):
            found = True
            break
    assert found


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_dequant_is_exact_product_rounded_once(bits):
    w = synthetic.random_matrix_bf16(4, 256, seed=3).float().numpy()
    codes, s, z = quant.quantize(w, bits, 128)
    d = quant.dequant(codes, s, z, bits, 256, 128)
    q = quant.unpack(codes, bits, 256).astype(np.int64)
    # independent evaluation with torch: (q - z) exact in bf16 for |q - z| <= 255 ... the
    # product of two 8-bit significands is exact in fp32, and fp32 -> bf16 is one RNE.
    sb = torch.from_numpy(s).to(torch.bfloat16).to(torch.float32)
    qz = torch.from_numpy((q.reshape(4, 2, 128) - z.astype(np.int64)[:, :, None]).astype(np.float32))
    ref = (qz * sb[:, :, None]).to(torch.bfloat16).to(torch.float64).reshape(4, 256).numpy()
    assert np.array_equal(d, ref)
    assert (round_bf16(d) == d).all()


def test_bytes_per_weight():
    assert quant.bytes_per_weight(4) == pytest.approx(0.5 + 5 / 128)
    assert quant.bytes_per_weight(16) == 2.0 and quant.bytes_per_weight(0) == 0.0
    # a Mixtral expert (3 * 4096 * 14336 weights) at Int4 is 95.0 MB
    assert 3 * 4096 * 14336 * quant.bytes_per_weight(4) / 1e6 == pytest.approx(95.0, abs=0.1)
