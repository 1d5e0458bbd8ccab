"""Pins for oracle.bf16.round_bf16 (RNE onto the bfloat16 grid)."""
import numpy as np
import torch

from oracle.bf16 import round_bf16, is_bf16


def test_hand_ties_to_even():
    # spacing in [1, 2) is 2**-7
    assert round_bf16(1 + 2.0 ** -8) == 1.0                       # tie -> even mantissa 0
    assert round_bf16(1 + 3 * 2.0 ** -8) == 1 + 2.0 ** -6          # tie between odd 1 and even 2
    assert round_bf16(1 + 2.0 ** -8 + 2.0 ** -30) == 1 + 2.0 ** -7  # just above the tie
    assert round_bf16(-(1 + 2.0 ** -8)) == -1.0
    assert round_bf16(255.0) == 255.0 and round_bf16(257.0) == 256.0 and round_bf16(259.0) == 260.0
    assert round_bf16(0.0) == 0.0


def test_subnormals_and_boundaries():
    step = 2.0 ** -133
    assert round_bf16(1.5 * step) == 2 * step                     # tie -> even multiple
    assert round_bf16(2.5 * step) == 2 * step
    assert round_bf16(0.4 * step) == 0.0
    assert round_bf16(2.0 ** -126) == 2.0 ** -126
    assert np.isinf(round_bf16(3.5e38))


def test_matches_torch_float32_cast():
    # torch's float32 -> bfloat16 cast is RNE; on float32 inputs both must agree bit for bit
    g = torch.Generator().manual_seed(0)
    x = torch.randn(200000, generator=g) * torch.exp(torch.randn(200000, generator=g) * 20)
    x = torch.cat([x, torch.randn(1000, generator=g) * 1e-39])
    ref = x.to(torch.bfloat16).to(torch.float64).numpy()
    got = round_bf16(x.to(torch.float64).numpy())
    assert np.array_equal(ref, got)
    assert is_bf16(got).all()
