"""GPU parity for dymoe_predict_next (Eqs. 6-8 look-ahead) against oracle/prefetch.py:
logits bit-exact (same fp32 op order, P1), requested experts and prefill priorities exact,
decode priorities within fp32 summation tolerance."""
import numpy as np
import pytest
import torch

import synthetic
from oracle import prefetch as o_pf

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
    ref = o_pf.predict_next(phase, h.float().numpy(), w.float().numpy(), k, t)
    assert np.array_equal(lg.cpu().numpy().view(np.uint32), ref["logits"].view(np.uint32))
    assert ex.cpu().numpy().tolist() == ref["experts"]
    if phase == "prefill":
        assert pr.cpu().numpy().tolist() == ref["priority"]
    else:
        assert np.allclose(pr.cpu().numpy(), ref["priority"], rtol=1e-6, atol=1e-6 * T)


def test_predict_next_validation():
    d = D()
    h = torch.zeros(4, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(d.DymoeError, match="t: must satisfy"):
        d.dymoe_predict_next(d.DYMOE_DECODE, h, w, 2, 9)
    # all-zero gate: every logit 0 -> index order; prefill counts = the first k experts
    ex, pr, _ = d.dymoe_predict_next(d.DYMOE_PREFILL, h, w, 2, 8)
    assert ex.cpu().tolist() == [0, 1] and pr.cpu().tolist() == [4.0, 4.0]
