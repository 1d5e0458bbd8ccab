"""Pins for oracle/prefetch.py (Eqs. 6-8 look-ahead; SPEC S:248-274 examples)."""
import math

import numpy as np

from oracle import prefetch as pf


def _logits_for_sets(sets, M):
    """Logits whose top-2 is exactly each given pair (larger value on the first listed)."""
    L = np.zeros((len(sets), M), np.float32)
    for i, (a, b) in enumerate(sets):
        L[i, a], L[i, b] = 2.0, 1.0
    return L


def test_prefill_spec_example():
    # 3 tokens predicting {e1,e2}, {e1,e3}, {e1,e2}; t=2 -> [e1 (c=3), e2 (c=2)]
    L = _logits_for_sets([(1, 2), (1, 3), (1, 2)], 4)
    ex, pr, counts = pf.prefill_prefetch(L, 2, 2)
    assert ex == [1, 2] and pr == [3, 2]
    assert counts.tolist() == [0, 3, 2, 1]
    # t = M: every expert with c_e > 0, ordered; the zero-count expert is never requested
    ex, pr, _ = pf.prefill_prefetch(L, 2, 4)
    assert ex == [1, 2, 3] and pr == [3, 2, 1]


def test_prefill_matches_histogram_and_is_permutation_equivariant():
    rng = np.random.default_rng(0)
    L = rng.standard_normal((500, 16)).astype(np.float32)
    ex, pr, counts = pf.prefill_prefetch(L, 3, 5)
    top3 = np.argsort(-L, axis=1, kind="stable")[:, :3]
    hist = np.bincount(top3.ravel(), minlength=16)
    assert counts.tolist() == hist.tolist()
    brute = sorted(range(16), key=lambda j: (-hist[j], j))[:5]
    assert ex == brute and pr == [int(hist[j]) for j in brute]
    perm = rng.permutation(500)
    assert pf.prefill_prefetch(L[perm], 3, 5)[0] == ex


def test_decode_spec_examples():
    # g_hat = [0.5, 0.3, 0.2], t = 2 -> [e0, e1]; t = 1 -> the argmax; uniform -> index order
    L = np.log(np.array([[0.5, 0.3, 0.2]], np.float32))
    assert pf.decode_prefetch(L, 2)[0] == [0, 1]
    assert pf.decode_prefetch(L, 1)[0] == [0]
    assert pf.decode_prefetch(np.zeros((1, 3), np.float32), 2)[0] == [0, 1]
    # batch: ranks by the summed softmax
    L2 = np.array([[5, 0, 0, 0], [0, 0, 5, 0], [0, 0, 5, 0]], np.float32)
    assert pf.decode_prefetch(L2, 2)[0] == [2, 0]


def test_gate_logits_is_the_exact_product():
    # Eq. 6 fixes the product, not an order: the oracle's value is the exact one.
    # integers: exact integer dot products
    rng = np.random.default_rng(1)
    h = rng.integers(-8, 8, (5, 64)).astype(np.float32)
    w = rng.integers(-8, 8, (3, 64)).astype(np.float32)
    got = pf.gate_logits(h, w)
    assert got.dtype == np.float64
    assert np.array_equal(got, (h.astype(np.int64) @ w.T.astype(np.int64)).astype(np.float64))
    # hand case: cancellation an fp32 left-to-right sum gets wrong (2^24 + 1 - 2^24 = 0 in fp32)
    hc = np.array([[2.0 ** 12, 1.0, -(2.0 ** 12)]], np.float32)
    wc = np.array([[2.0 ** 12, 1.0, 2.0 ** 12]], np.float32)
    assert pf.gate_logits(hc, wc).tolist() == [[1.0]]
    # bf16-valued reals: equal to math.fsum (correctly rounded sum of the exact fp64 products) up
    # to the fp64 summation bound Hd * 2^-53 * sum|h w|
    def bf16(a):
        return (np.asarray(a, np.float32).view(np.uint32) & 0xffff0000).view(np.float32)
    h = bf16(rng.standard_normal((7, 512)) * np.exp2(rng.integers(-20, 20, (7, 512))))
    w = bf16(rng.standard_normal((4, 512)) / 20)
    got = pf.gate_logits(h, w)
    for t in range(7):
        for e in range(4):
            prods = [float(h[t, k]) * float(w[e, k]) for k in range(512)]
            exact = math.fsum(prods)
            assert abs(got[t, e] - exact) <= 512 * 2.0 ** -53 * math.fsum(abs(p) for p in prods)


def test_predict_next_reduces_to_route_of_the_next_gate():
    rng = np.random.default_rng(2)
    h = rng.integers(-4, 4, (40, 32)).astype(np.float32)
    w = rng.integers(-4, 4, (8, 32)).astype(np.float32)
    r = pf.predict_next("prefill", h, w, 2, 3)
    logits = (h.astype(np.int64) @ w.T.astype(np.int64)).astype(np.float64)
    assert np.array_equal(r["logits"], logits)
    assert r["experts"] == pf.prefill_prefetch(logits, 2, 3)[0]
