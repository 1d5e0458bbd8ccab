"""Pins for oracle.route (top-k gating)."""
import numpy as np
import pytest

from oracle import route
import synthetic


def test_hand_example():
    idx, w, p = route.route(np.array([[1.0, 3.0, 2.0, 3.0]], np.float32), 2)
    assert idx.tolist() == [[1, 3]]                 # tie 3.0/3.0 -> lower index first
    assert np.allclose(w, 0.5, rtol=0, atol=1e-15)
    e = np.exp([1.0, 3.0, 2.0, 3.0])
    assert np.allclose(p[0], e / e.sum(), rtol=1e-14)


def test_all_equal_and_signed_zero():
    idx, w, _ = route.route(np.zeros((3, 8), np.float32), 3)
    assert (idx == [0, 1, 2]).all()
    row = np.array([[-0.0, 0.0, -0.0, 0.0]], np.float32)
    idx, _, _ = route.route(row, 2)
    assert idx.tolist() == [[0, 1]]                 # -0.0 == +0.0 numerically


@pytest.mark.parametrize("ties", [False, True])
def test_brute_force_lexsort(ties):
    lg = synthetic.random_logits(300, 16, seed=3, ties=ties).numpy()
    idx, w, p = route.route(lg, 4)
    for t in range(lg.shape[0]):
        # independent ordering: numpy lexsort on (index, -logit) with -0.0 canonicalised
        key = -(lg[t].astype(np.float64) + 0.0)
        order = np.lexsort((np.arange(16), key))
        assert idx[t].tolist() == order[:4].tolist()
    assert np.allclose(w.sum(1), 1.0, atol=1e-12)
    # softmax over the top-k == full softmax renormalised over the top-k
    sel = np.take_along_axis(p, idx.astype(np.int64), 1)
    assert np.allclose(w, sel / sel.sum(1, keepdims=True), rtol=1e-12)
    assert np.allclose(p.sum(1), 1.0, atol=1e-12)


def test_weights_monotone_in_rank():
    lg = synthetic.random_logits(100, 8, seed=5).numpy()
    _, w, _ = route.route(lg, 3)
    assert (np.diff(w, axis=1) <= 1e-15).all()


def test_invalid_k():
    with pytest.raises(ValueError, match="k"):
        route.route(np.zeros((1, 4), np.float32), 5)
