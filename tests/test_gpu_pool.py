"""The pooled expert store (paper_2603_19172_b200.pool: dymoe_pool policy + runtime quantization
into one device arena + dymoe_layer_set_expert rebinding) over a 4-layer stack whose packed
formats do not all fit: every step's output equals the oracle layer run with the served widths,
served widths never fall below the assigned ones (Conservative Reuse), the arena budget holds,
and hits, misses and evictions all occur."""
import numpy as np
import pytest
import torch

import synthetic
from oracle import moe as o_moe, schedule as o_sched

pytestmark = pytest.mark.gpu

FFN_TOL = 2e-3


@pytest.mark.parametrize("phase,T", [("decode", 4), ("prefill", 40)])
def test_pooled_stack_matches_oracle(phase, T):
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200.pool import ExpertStore
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    L = 4
    masters = [[{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 40 + l)]
               for l in range(L)]
    probe = ExpertStore(masters[:1], cfg.k, cfg.hidden, cfg.ffn, 1 << 20)
    full = L * cfg.M * sum(probe.entry_bytes(b) for b in (8, 4, 2))
    del probe
    store = ExpertStore(masters, cfg.k, cfg.hidden, cfg.ffn, int(full * 0.3))
    lad_bits, lad_l = (8, 4, 2), (0.25, 0.5)
    lad = d.make_ladder(lad_bits, lad_l)
    o_lad = o_sched.Ladder(lad_bits, lad_l)
    np_masters = [[{n: t.float().cpu().numpy() for n, t in e.items()} for e in ml] for ml in masters]
    ph = d.DYMOE_PREFILL if phase == "prefill" else d.DYMOE_DECODE
    rng = np.random.default_rng(3)
    for step in range(16):
        l = int(rng.integers(0, L))
        x, lg, a = synthetic.layer_inputs(cfg, 900 + step)
        y, served, want, forced = store.forward(l, x.cuda(), lg.cuda(), lad, L, phase=ph,
                                        attn_mass=a.cuda() if ph == d.DYMOE_PREFILL else None)
        torch.cuda.synchronize()
        for e in range(cfg.M):
            if want[e]:
                assert served[e] >= want[e] or want[e] == 16, (step, e, served, want)
                assert (served[e] == 0) == (want[e] == 0)
        assert store.pool.used() <= store.pool.capacity
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), np_masters[l], l, L, o_lad, cfg.k,
                                forced_bits=np.array(forced, np.uint8))
        err = np.abs(y.cpu().numpy() - ref["y"]).max() / max(np.abs(ref["y"]).max(), 1e-30)
        assert err <= FFN_TOL, (step, err)
    s = store.stats
    assert s["hits"] > 0 and s["misses"] > 0 and s["evictions"] > 0, s


def test_host_offload_stack_matches_oracle():
    """Masters in pinned host memory: every format, BF16 included, is a pool entry
    filled by a host->device copy (+ quantization); steps equal the oracle with served widths."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200.pool import ExpertStore
    cfg = synthetic.CONFIGS["tiny"].with_tokens(6)
    L = 3
    masters = [[{n: t.pin_memory() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 60 + l)]
               for l in range(L)]
    probe = ExpertStore([[{n: t.cuda() for n, t in e.items()} for e in masters[0]]], cfg.k,
                        cfg.hidden, cfg.ffn, 1 << 20)
    per_layer = cfg.M * (probe.entry_bytes(16) + probe.entry_bytes(8))
    del probe
    store = ExpertStore(masters, cfg.k, cfg.hidden, cfg.ffn, int(per_layer * 1.2))
    assert store.host
    lad_bits, lad_l = (16, 8, 4, 2), (0.2, 0.5, 0.8)
    lad = d.make_ladder(lad_bits, lad_l)
    o_lad = o_sched.Ladder(lad_bits, lad_l)
    np_masters = [[{n: t.float().numpy() for n, t in e.items()} for e in ml] for ml in masters]
    for step in range(10):
        l = step % L
        x, lg, _ = synthetic.layer_inputs(cfg, 700 + step)
        y, served, want, forced = store.forward(l, x.cuda(), lg.cuda(), lad, 32)
        torch.cuda.synchronize()
        for e in range(cfg.M):
            if want[e]:
                assert served[e] >= want[e]
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), np_masters[l], l, 32, o_lad, cfg.k,
                                forced_bits=np.array(forced, np.uint8))
        err = np.abs(y.cpu().numpy() - ref["y"]).max() / max(np.abs(ref["y"]).max(), 1e-30)
        assert err <= FFN_TOL, (step, err)
    assert store.stats["h2d_bytes"] > 0 and store.stats["evictions"] > 0, store.stats
