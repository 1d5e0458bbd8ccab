"""Pins for oracle.moe: permutation, SwiGLU FFN, combine, layer forward, EP simulation."""
import numpy as np
import pytest
import torch

from oracle import moe, route, schedule as sc, quant
from oracle.bf16 import round_bf16
import synthetic


def _np_experts(cfg, seed):
    return [{n: e[n].float().numpy() for n in ("w1", "w3", "w2")}
            for e in synthetic.expert_weights(cfg, seed)]


def test_permute_stable_brute_force():
    rng = np.random.default_rng(0)
    T, k, M = 50, 3, 8
    idx = np.stack([rng.permutation(M)[:k] for _ in range(T)]).astype(np.int32)
    bits = np.array([4, 0, 2, 8, 16, 0, 4, 2], np.uint8)
    p = moe.permute(idx, bits, M)
    flat_e = idx.reshape(-1)
    keep = bits[flat_e] != 0
    pos = np.nonzero(keep)[0]
    order = pos[np.argsort(flat_e[pos], kind="stable")]           # independent: numpy stable sort
    assert p["perm_token"].tolist() == (order // k).tolist()
    assert p["perm_slot"].tolist() == (order % k).tolist()
    assert p["expert_off"].tolist() == [0] + np.cumsum(
        [int(((flat_e == e) & keep).sum()) for e in range(M)]).tolist()
    for r, (t, s) in enumerate(zip(p["perm_token"], p["perm_slot"])):
        assert p["inv_row"][t, s] == r
    assert (p["inv_row"][bits[idx] == 0] == -1).all()


def test_combine_renorm_and_all_skipped():
    y_perm = np.array([[1.0, 2.0], [10.0, 20.0]])
    inv = np.array([[0, -1], [-1, -1], [1, 0]])
    w = np.array([[0.75, 0.25], [0.6, 0.4], [0.5, 0.5]])
    y = moe.combine(y_perm, inv, w, renorm=True)
    assert y[0].tolist() == [1.0, 2.0]                     # 0.75/0.75
    assert y[1].tolist() == [0.0, 0.0]                     # all skipped -> 0
    assert y[2].tolist() == [5.5, 11.0]
    y = moe.combine(y_perm, inv, w, renorm=False)
    assert y[0].tolist() == [0.75, 1.5]


def _torch_swiglu(x, W1, W3, W2, round_h):
    A = x @ W1.T
    B = x @ W3.T
    h = torch.nn.functional.silu(A) * B
    if round_h:
        h = h.to(torch.float32).to(torch.bfloat16).to(torch.float64)
    return h @ W2.T


def test_dense_mixture_reduction():
    # all-BF16 ladder with k = M: the layer is the softmax-weighted mixture of every
    # expert's SwiGLU FFN (textbook dense MoE), evaluated independently in torch fp64
    cfg = synthetic.CONFIGS["tiny"]
    experts = _np_experts(cfg, 0)
    x, lg, _ = synthetic.layer_inputs(cfg, 0)
    lad = sc.Ladder(bits=(16, 16 // 2), lambdas=(1.0,))     # lambda = 1: everything BF16
    out = moe.moe_forward(x.float().numpy(), lg.numpy(), experts, 3, 32, lad, k_route=cfg.M)
    assert (out["bits"] == 16).all()
    xt = x.double()
    p = torch.softmax(lg.double(), dim=1)
    for round_h, tol in [(False, 1e-2), (True, 1e-6)]:
        ref = torch.zeros(cfg.T, cfg.hidden, dtype=torch.float64)
        for e in range(cfg.M):
            W = [torch.from_numpy(experts[e][n]).double() for n in ("w1", "w3", "w2")]
            ref += p[:, e:e + 1] * _torch_swiglu(xt, *W, round_h)
        err = np.abs(out["y"] - ref.numpy()).max() / np.abs(ref.numpy()).max()
        assert err < tol, (round_h, err)


def test_identity_down_projection():
    # Hd == F and W2 = I: y_e = h exactly (the bf16-rounded SwiGLU intermediate)
    rng = np.random.default_rng(1)
    H = 64
    W1 = round_bf16(rng.standard_normal((H, H)) / 8)
    W3 = round_bf16(rng.standard_normal((H, H)) / 8)
    x = round_bf16(rng.standard_normal((5, H)))
    y = moe.ffn(x, W1, W3, np.eye(H))
    A, B = x @ W1.T, x @ W3.T
    assert np.array_equal(y, round_bf16(A / (1 + np.exp(-A)) * B))
    assert np.abs(moe.silu(np.array([0.0, 50.0, -50.0])) - [0.0, 50.0, 0.0]).max() < 1e-15


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_ep_simulation_equals_unsharded(P):
    cfg = synthetic.CONFIGS["tiny"]
    experts = _np_experts(cfg, 2)
    x, lg, _ = synthetic.layer_inputs(cfg, 2)
    lad = sc.Ladder(bits=(8, 4, 2), lambdas=(0.25, 0.5))
    out = moe.moe_forward(x.float().numpy(), lg.numpy(), experts, 20, 32, lad, cfg.k)
    y = moe.ep_simulate(x.float().numpy(), out["topk_idx"], out["topk_w"], out["bits"],
                        experts, cfg.M, P)
    assert np.array_equal(y, out["y"])
    rows = moe.ep_dispatch_order(out["topk_idx"], out["bits"], cfg.M, P)
    assert [r[0] for r in rows] == sorted(r[0] for r in rows)
    assert all(moe.ep_owner(e, cfg.M, P) == d for d, e, _, _ in rows)


def test_forward_prefill_mixed_and_skip():
    cfg = synthetic.CONFIGS["tiny"]
    experts = _np_experts(cfg, 3)
    x, lg, a = synthetic.layer_inputs(cfg, 3)
    lad = sc.Ladder(bits=(4, 0), lambdas=(0.0,))
    out = moe.moe_forward(x.float().numpy(), lg.numpy(), experts, 31, 32, lad, cfg.k,
                          phase="prefill", attn_mass=a.numpy())
    assert out["importance"].sum() == len(out["heavy"]) * cfg.k
    assert (out["bits"] == 4).sum() == 2                       # t = max(ceil(0), k) = 2
    # executed experts only: tokens whose experts were all skipped give 0
    dead = (out["inv_row"] < 0).all(1)
    assert (out["y"][dead] == 0).all()
    # an Int4 expert's rows equal the FFN on its dequantized weights (quantized here)
    e = int(np.nonzero(out["bits"] == 4)[0][0])
    lo, hi = out["expert_off"][e], out["expert_off"][e + 1]
    W = [quant.dequant(*quant.quantize(experts[e][n], 4), 4, experts[e][n].shape[1]) for n in ("w1", "w3", "w2")]
    xr = x.float().numpy()[out["perm_token"][lo:hi]].astype(np.float64)
    assert np.array_equal(out["y_perm"][lo:hi], moe.ffn(xr, *W))


def test_route_in_forward_matches_router():
    cfg = synthetic.CONFIGS["tiny"]
    x, lg, _ = synthetic.layer_inputs(cfg, 5)
    idx, w, _ = route.route(lg.numpy(), cfg.k)
    experts = _np_experts(cfg, 5)
    out = moe.moe_forward(x.float().numpy(), lg.numpy(), experts, 0, 32, sc.paper_ladder(2), cfg.k)
    assert np.array_equal(out["topk_idx"], idx) and np.array_equal(out["topk_w"], w)
