"""Pins for oracle/attention.py (f3): closed form for uniform attention (harmonic tails), every
query row distributes exactly one unit of mass, and a hand-worked 3-token case."""
import math

import numpy as np

from oracle import attention as oa


def test_uniform_attention_is_harmonic_tail():
    q = np.zeros((2, 50, 8))
    k = np.random.default_rng(0).standard_normal((2, 50, 8))
    a = oa.attention_mass(q, k, 0.3)
    assert np.allclose(a[0], oa.harmonic_tail(50), rtol=0, atol=1e-12)
    assert np.allclose(a[1], oa.harmonic_tail(50), rtol=0, atol=1e-12)


def test_mass_is_conserved_and_causal():
    rng = np.random.default_rng(1)
    q, k = rng.standard_normal((3, 40, 16)), rng.standard_normal((3, 40, 16))
    a = oa.attention_mass(q, k, 0.25)
    assert np.allclose(a.sum(axis=1), 40.0, atol=1e-9)     # each query row sums to 1
    assert np.all(a >= 0)
    # the last token is only attended by itself: a[T-1] = softmax of the last row at T-1
    s = 0.25 * q[:, -1] @ np.swapaxes(k, 1, 2)
    s = np.array([s[h, h] for h in range(3)])
    p_last = np.exp(s - s.max(axis=1, keepdims=True))
    p_last /= p_last.sum(axis=1, keepdims=True)
    assert np.allclose(a[:, -1], p_last[:, -1], atol=1e-12)


def test_three_token_hand_case():
    # one head, d = 1, scale 1: q = [0, 1, 2], k = [0, 1, 0]
    q = np.array([[[0.0], [1.0], [2.0]]])
    k = np.array([[[0.0], [1.0], [0.0]]])
    a = oa.attention_mass(q, k, 1.0)
    # row 0: [1]; row 1: softmax([0, 1]); row 2: softmax([0, 2, 0])
    r1 = [1 / (1 + math.e), math.e / (1 + math.e)]
    z2 = 2 + math.e ** 2
    r2 = [1 / z2, math.e ** 2 / z2, 1 / z2]
    exp = [1 + r1[0] + r2[0], r1[1] + r2[1], r2[2]]
    assert np.allclose(a[0], exp, atol=1e-12)
