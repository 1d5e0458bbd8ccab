"""Pins for oracle.importance (Eq. 1-3)."""
import numpy as np
import pytest

from oracle import importance as imp, route
from golden_util import load_golden
import synthetic


G = load_golden("spec_examples.json")


@pytest.mark.parametrize("case", G["heavy_hitters"])
def test_spec_heavy_hitters(case):
    got = imp.heavy_hitters(np.array(case["s"], np.float32), case["k"])
    assert sorted(got.tolist()) == case["expect"]


@pytest.mark.parametrize("case", G["prefill_counts"])
def test_spec_prefill_counts(case):
    got = imp.prefill_importance(case["heavy"], np.array(case["topk"]), case["M"])
    assert got.tolist() == case["expect"]


def test_token_scores_sequential_fp32():
    # integer-valued masses: every partial sum is exact in fp32, so S == the exact sum
    rng = np.random.default_rng(0)
    a = rng.integers(0, 1000, size=(32, 500)).astype(np.float32)
    assert np.array_equal(imp.token_scores(a), a.astype(np.int64).sum(0).astype(np.float32))
    # order matters in fp32: head order h = 0..H-1, one rounding per add
    a = np.array([[1.0], [2.0 ** -24], [2.0 ** -24]], np.float32)
    assert imp.token_scores(a)[0] == np.float32(1.0)     # (1 + e) + e rounds twice to 1
    a2 = a[[1, 2, 0]]
    assert imp.token_scores(a2)[0] > np.float32(1.0)     # (e + e) + 1 = 1 + 2**-23


def test_heavy_set_matches_eq1_mean():
    # Eq. 1 divides by H; the top-k set is unchanged by that positive constant
    cfg = synthetic.CONFIGS["tiny"]
    a = synthetic.attention_mass(cfg.with_tokens(400), seed=1).numpy()
    S = imp.token_scores(a)
    s_mean = imp.mean_head_score(a)
    heavy = imp.heavy_hitters(S, 80)
    order = np.lexsort((np.arange(400), -s_mean))
    assert set(heavy.tolist()) == set(order[:80].tolist())


def test_monotone_invariance_and_k_default():
    rng = np.random.default_rng(2)
    s = rng.random(50).astype(np.float32)
    h1 = imp.heavy_hitters(s, 10)
    h2 = imp.heavy_hitters((np.exp(s * 3) + 2).astype(np.float32), 10)
    assert h1.tolist() == h2.tolist()
    assert imp.default_k_tokens(2048) == 410 and imp.default_k_tokens(16) == 4
    assert imp.default_k_tokens(5) == 1 and imp.default_k_tokens(0) == 0
    with pytest.raises(ValueError, match="k_tokens"):
        imp.heavy_hitters(s, 51)


def test_counts_brute_force_and_mass():
    cfg = synthetic.CONFIGS["tiny"].with_tokens(200)
    x, lg, a = synthetic.layer_inputs(cfg, seed=4)
    idx, _, _ = route.route(lg.numpy(), cfg.k)
    I, heavy, _ = imp.score_prefill(a.numpy(), idx, cfg.M, 40)
    assert len(heavy) == 40
    assert I.sum() == 40 * cfg.k
    onehot = np.zeros((200, cfg.M), np.int64)
    for t in range(200):
        onehot[t, idx[t]] = 1
    assert np.array_equal(I, onehot[heavy].sum(0))               # S:130 double loop
    # equivariance under expert relabelling
    perm = np.random.default_rng(1).permutation(cfg.M)
    I2 = imp.prefill_importance(heavy, perm[idx], cfg.M)
    assert np.array_equal(I2[perm], I)


def test_decode_importance():
    lg = np.array([[0.3, 2.0, -1.0, 2.0]], np.float32)
    _, _, p = route.route(lg, 2)
    I = imp.decode_importance(lg, p)
    assert I.tolist() == [float(v) for v in lg[0]]                # B = 1: logit row
    assert int(np.argmax(I)) == int(np.argmax(p[0]))
    lg2 = synthetic.random_logits(5, 8, seed=9).numpy()
    _, _, p2 = route.route(lg2, 2)
    assert np.allclose(imp.decode_importance(lg2, p2), p2.sum(0), rtol=1e-14)
    u = np.zeros((3, 8), np.float32)
    _, _, pu = route.route(u, 2)
    assert np.allclose(imp.decode_importance(u, pu), 3 / 8)      # S:138 uniform
