"""Pins for oracle.stack (the C5 layer stack on the bf16 residual stream)."""
import numpy as np
import torch

from oracle import stack, schedule as sc
from oracle.bf16 import round_bf16
import synthetic

CFG = synthetic.MoEConfig("stack_tiny", M=4, k=2, hidden=128, ffn=256, T=6, heads=4, layers=4)


def _np_experts(cfg, seed):
    return [{n: e[n].float().numpy() for n in ("w1", "w3", "w2")}
            for e in synthetic.expert_weights(cfg, seed)]


def _gates(cfg, L):
    out = []
    for l in range(L):
        wg, beta = synthetic.stack_gate(cfg, l, 0)
        out.append((wg.float().numpy(), beta.numpy()))
    return out


def test_router_is_the_exact_affine_map():
    rng = np.random.default_rng(0)
    x = round_bf16(rng.standard_normal((3, 64))).astype(np.float32)
    w = round_bf16(rng.standard_normal((5, 64)) / 8).astype(np.float32)
    b = np.array([0.5, -1.25, 0.0, 3.0, -0.0], np.float32)
    base = stack.router_logits(x, w, None)
    assert base.dtype == np.float64
    assert np.array_equal(stack.router_logits(x, w, np.zeros(5, np.float32)), base)
    # independent: torch fp64 x @ w^T + b (bf16 products exact in fp64, 64 terms: exact sums at
    # these magnitudes up to 64 * 2^-53 relative)
    ref = (torch.from_numpy(x).double() @ torch.from_numpy(w).double().T
           + torch.from_numpy(b).double()).numpy()
    assert np.allclose(stack.router_logits(x, w, b), ref, rtol=0, atol=1e-13)
    # hand case: one nonzero product per entry, plus the bias
    xh = np.zeros((1, 64), np.float32)
    xh[0, 3] = 2.0
    wh = np.zeros((2, 64), np.float32)
    wh[0, 3], wh[1, 3] = 0.75, -1.5
    assert stack.router_logits(xh, wh, np.array([1.0, 0.25], np.float32)).tolist() == [[2.5, -2.75]]


def test_rmsnorm_closed_forms():
    # constant row c: u = RNE(c / sqrt(c^2 + eps)); with eps = 0 exactly +-1
    x = np.array([[3.0] * 8, [-0.5] * 8])
    assert stack.rmsnorm(x, eps=0.0).tolist() == [[1.0] * 8, [-1.0] * 8]
    assert np.array_equal(stack.rmsnorm(x), round_bf16(x / np.sqrt(x * x + stack.EPS)))
    # power-of-two scaling is exact: rmsnorm(4x) == rmsnorm(x) at eps = 0
    rng = np.random.default_rng(3)
    y = round_bf16(rng.standard_normal((5, 128)))
    assert np.array_equal(stack.rmsnorm(4 * y, eps=0.0), stack.rmsnorm(y, eps=0.0))
    # unit mean square up to the bf16 rounding of each element
    u = stack.rmsnorm(y, eps=0.0)
    assert np.abs((u * u).mean(axis=1) - 1.0).max() < 2 * 2.0 ** -8
    # hand case: [3, 4] -> mean square 12.5, u = [3, 4] / sqrt(12.5) rounded to bf16
    assert stack.rmsnorm(np.array([[3.0, 4.0]]), eps=0.0).tolist() == [[0.84765625, 1.1328125]]


def test_residual_rounds_once():
    x = np.array([1.0, 1.0, 256.0, -3.0])
    y = np.array([2.0 ** -9, 3 * 2.0 ** -9, 1.0, 0.0])   # tie -> even; above tie; ulp 2 at 256
    assert stack.residual(x, y).tolist() == [1.0, 1.0078125, 256.0, -3.0]


def test_zero_expert_outputs_leave_stream_unchanged():
    # W2 = 0 in every expert: every y_l = 0, so x_L = x_0 exactly through all layers
    L = 4
    ex = []
    for l in range(L):
        e = _np_experts(CFG, 10 + l)
        for d in e:
            d["w2"] = np.zeros_like(d["w2"])
        ex.append(e)
    x0 = synthetic.hidden_states(CFG, 1).float().numpy()
    lad = sc.Ladder(bits=(8, 4, 2), lambdas=(0.25, 0.5))
    xL, trace = stack.stack_forward(x0, _gates(CFG, L), ex, lad, CFG.k)
    assert np.array_equal(xL, x0.astype(np.float64))
    assert len(trace) == L and all(len(b) == CFG.M for _, _, b in trace)


def _torch_swiglu(x, W1, W3, W2):
    a, b = x @ W1.T, x @ W3.T
    h = torch.from_numpy(round_bf16((a * torch.sigmoid(a) * b).numpy()))
    return h @ W2.T


def test_dense_bf16_stack_equals_torch_chain():
    # lambda = 1 (all BF16) and k = M: every layer is the softmax-weighted dense mixture of all
    # SwiGLU experts; chain three layers independently in torch fp64 with the same router and the
    # same residual rounding, and compare the final stream
    L = 3
    cfg = CFG
    ex = [_np_experts(cfg, 20 + l) for l in range(L)]
    gates = _gates(cfg, L)
    x0 = synthetic.hidden_states(cfg, 2).float().numpy()
    lad = sc.Ladder(bits=(16, 8), lambdas=(1.0,))
    xL, trace = stack.stack_forward(x0, gates, ex, lad, k_route=cfg.M)
    assert all((b == 16).all() for _, _, b in trace)
    xt = torch.from_numpy(x0.astype(np.float64))
    for l in range(L):
        ut = torch.from_numpy(round_bf16((xt / torch.sqrt((xt * xt).mean(dim=1, keepdim=True)
                                                           + 1e-5)).numpy()))
        lg = ut @ torch.from_numpy(gates[l][0]).double().T + torch.from_numpy(gates[l][1]).double()
        p = torch.softmax(lg, dim=1)
        y = torch.zeros_like(xt)
        for e in range(cfg.M):
            W = [torch.from_numpy(ex[l][e][n]).double() for n in ("w1", "w3", "w2")]
            y += p[:, e:e + 1] * _torch_swiglu(ut, *W)
        xt = torch.from_numpy(round_bf16((xt + y).numpy()))
    # router logits and mixtures differ from the oracle's only by fp64 summation order ->
    # identical bf16 streams but for rare rounding ties
    diff = np.abs(xL - xt.numpy())
    ulp = np.abs(xt.numpy()) * 2.0 ** -7 + 1e-30
    assert (diff <= ulp).all() and (diff > 0).mean() < 0.01
