"""GPU parity for dymoe_attention_mass (f3) against oracle/attention.py: within fp32 accumulation
tolerance, conservation (each query row distributes one unit), the heavy-hitter set it induces
equals the oracle's, and the closed form for uniform attention."""
import numpy as np
import pytest
import torch

from oracle import attention as oa, importance as o_imp

pytestmark = pytest.mark.gpu


def D():
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    return d


@pytest.mark.parametrize("H,T", [(2, 64), (3, 200), (1, 1), (4, 517), (2, 2048), (5, 1300)])
def test_attention_mass_matches_oracle(H, T):
    d = D()
    g = torch.Generator().manual_seed(H * 1000 + T)
    q = torch.randn(H, T, 128, generator=g).to(torch.bfloat16)
    k = torch.randn(H, T, 128, generator=g).to(torch.bfloat16)
    # a few "sink" tokens with large keys make the mass heavy-tailed
    k[:, : min(T, 3)] *= 4
    a = d.dymoe_attention_mass(q.cuda(), k.cuda()).cpu().numpy()
    ref = oa.attention_mass(q.float().numpy(), k.float().numpy(), 128 ** -0.5)
    assert np.abs(a - ref).max() <= 1e-5 * max(1.0, np.abs(ref).max()), np.abs(a - ref).max()
    assert np.allclose(a.sum(axis=1), T, rtol=1e-5)


def test_uniform_attention_closed_form_and_heavy_set():
    d = D()
    T, H = 300, 2
    q = torch.zeros(H, T, 128, dtype=torch.bfloat16)
    k = torch.randn(H, T, 128).to(torch.bfloat16)
    a = d.dymoe_attention_mass(q.cuda(), k.cuda()).cpu().numpy()
    assert np.allclose(a, np.stack([oa.harmonic_tail(T)] * H), rtol=1e-5)
    # realistic mass -> heavy-hitter set (Eq. 1) identical to the oracle's from its own mass
    q = torch.randn(4, 256, 128).to(torch.bfloat16)
    k = torch.randn(4, 256, 128).to(torch.bfloat16)
    k[:, [0, 17, 90]] *= 3
    a = d.dymoe_attention_mass(q.cuda(), k.cuda()).cpu().numpy()
    ref = oa.attention_mass(q.float().numpy(), k.float().numpy(), 128 ** -0.5)
    hh = o_imp.heavy_hitters(o_imp.token_scores(a.astype(np.float32)), 50)
    hr = o_imp.heavy_hitters(o_imp.token_scores(ref.astype(np.float32)), 50)
    assert set(hh.tolist()) == set(hr.tolist())
