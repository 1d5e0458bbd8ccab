"""GPU parity for dymoe_predict_next (Eqs. 6-8 look-ahead) against oracle/prefetch.py, which
evaluates the gate product exactly (reading P1): the GPU's fp32 logits within the kernel's fp32
error bound of the exact values (tests/validity.py); requests and prefill counts equal the
oracle's wherever no token's top-k is ambiguous under that bound, and a valid selection
otherwise; decode priorities within the bound's effect on the gate sums."""
import numpy as np
import pytest
import torch

import synthetic
from oracle import prefetch as o_pf, route as o_route
from validity import check_logits, check_topk, gate_logit_bound

pytestmark = pytest.mark.gpu


def D():
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    return d


def _bf16(t):
    return t.to(torch.bfloat16)


@pytest.mark.parametrize("phase,T,Hd,M,k,t", [
    ("prefill", 300, 256, 8, 2, 4), ("prefill", 2048, 4096, 8, 2, 3), ("prefill", 97, 2048, 64, 6, 16),
    ("decode", 1, 4096, 8, 2, 2), ("decode", 8, 4096, 8, 2, 4), ("decode", 5, 1024, 64, 6, 6),
    ("prefill", 7, 64, 256, 8, 256)])
def test_predict_next(phase, T, Hd, M, k, t):
    d = D()
    g = torch.Generator().manual_seed(T * 7 + M)
    h = _bf16(torch.randn(T, Hd, generator=g))
    # next layer's gate: N(0, 1/Hd) plus a per-expert skew so the predicted demand is Zipf-like
    w = _bf16(torch.randn(M, Hd, generator=g) / Hd ** 0.5 + torch.linspace(0.02, 0, M)[:, None])
    ph = d.DYMOE_PREFILL if phase == "prefill" else d.DYMOE_DECODE
    ex, pr, lg = d.dymoe_predict_next(ph, h.cuda(), w.cuda(), k, t)
    torch.cuda.synchronize()
    hn, wn = h.float().numpy(), w.float().numpy()
    ref = o_pf.predict_next(phase, hn, wn, k, t)
    bound = gate_logit_bound(hn, wn)
    check_logits(lg.cpu().numpy(), ref["logits"], bound)
    ex, pr = ex.cpu().numpy().tolist(), pr.cpu().numpy()
    if phase == "prefill":
        # counts: each token's exact top-k is unambiguous except on the `near` tokens, each of
        # which can move one unit of count between experts
        idx, _, _ = o_route.route(ref["logits"], k)
        near = check_topk(idx, ref["logits"], bound)      # the oracle's own selection is valid
        n_near = int(near.sum())
        assert n_near <= max(2, T // 100)
        _, _, c_ref = o_pf.prefill_prefetch(ref["logits"], k, t)
        if n_near == 0:
            assert ex == ref["experts"] and pr.tolist() == ref["priority"]
        else:
            for e, c in zip(ex, pr):
                assert abs(c - c_ref[e]) <= n_near
            rest = [e for e in range(M) if e not in ex]
            if rest and len(ex) == t:
                assert min(c_ref[e] for e in ex) + n_near >= max(c_ref[e] for e in rest) - n_near
    else:
        # decode demand: B = 1 the logit row (error = the logit bound); B > 1 sum_b softmax:
        # a logit error <= b moves each probability by <= p (e^{2b} - 1), plus fp32 rounding
        demand = np.asarray(o_pf.decode_prefetch(ref["logits"], t)[2])
        if T == 1:
            tol = bound[0]
        else:
            p = np.exp(ref["logits"] - ref["logits"].max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            tol = (p * np.expm1(2 * bound.max(axis=1, keepdims=True))).sum(axis=0) + 2e-6 * T
        assert np.all(np.abs(pr - demand[ex]) <= tol[ex])
        rest = [e for e in range(M) if e not in ex]
        if rest:
            assert min(demand[e] + tol[e] for e in ex) >= max(demand[e] - tol[e] for e in rest)
        clear = len(rest) == 0 or min(demand[e] - tol[e] for e in ref["experts"]) > max(
            demand[e] + tol[e] for e in range(M) if e not in ref["experts"])
        if clear:
            assert sorted(ex) == sorted(ref["experts"])


def test_predict_next_validation():
    d = D()
    h = torch.zeros(4, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(d.DymoeError, match="t: must satisfy"):
        d.dymoe_predict_next(d.DYMOE_DECODE, h, w, 2, 9)
    # all-zero gate: every logit 0 -> index order; prefill counts = the first k experts
    ex, pr, _ = d.dymoe_predict_next(d.DYMOE_PREFILL, h, w, 2, 8)
    assert ex.cpu().tolist() == [0, 1] and pr.cpu().tolist() == [4.0, 4.0]
