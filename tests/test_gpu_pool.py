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


@pytest.mark.parametrize("phase,T", [("decode", 8), ("prefill", 64)])
def test_prefetching_stack_matches_oracle(phase, T):
    """f1 (Eqs. 6-8): a 4-layer stack over a pooled arena at 40 % of its packed formats,
    the next layer's predicted critical experts quantized on a side stream while the current
    layer runs.  Teacher-forced layer by layer: every layer equals the oracle stack layer run with
    the widths the step served; prefetches happen and some of them serve the next step."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200.pool import ExpertStore, PrefetchingStack
    from oracle import stack as o_stack
    from validity import check_logits, check_topk, gate_logit_bound
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    L = 4
    masters = [[{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 80 + l)]
               for l in range(L)]
    gates = [synthetic.stack_gate(cfg, l, 3) for l in range(L)]
    probe = ExpertStore(masters[:1], cfg.k, cfg.hidden, cfg.ffn, 1 << 20)
    full = L * cfg.M * sum(probe.entry_bytes(b) for b in (8, 4, 2))
    del probe
    np_masters = [[{n: t.float().cpu().numpy() for n, t in e.items()} for e in ml] for ml in masters]
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    o_lad = o_sched.Ladder((8, 4, 2), (0.25, 0.5))
    ph = d.DYMOE_PREFILL if phase == "prefill" else d.DYMOE_DECODE
    for prefetch in (True, False):
        store = ExpertStore(masters, cfg.k, cfg.hidden, cfg.ffn, int(full * 0.4))
        st = PrefetchingStack(store, [(w.cuda(), b.cuda()) for w, b in gates])
        attn = [synthetic.attention_mass(cfg, 300 + l).cuda() for l in range(L)] if ph == d.DYMOE_PREFILL else None
        for rep in range(3):
            x0 = synthetic.hidden_states(cfg, 50 + rep).cuda()
            xL, tr = st.forward(x0, lad, phase=ph, attn_masses=attn, prefetch=prefetch, trace=True)
            torch.cuda.synchronize()
            for l in range(L):
                x_in = tr[l][0].float().cpu().numpy().astype(np.float64)
                u = tr[l][1].float().cpu().numpy().astype(np.float64)
                wg, beta = gates[l]
                lg_ref = o_stack.router_logits(u, wg.float().numpy(), beta.numpy())
                bound = gate_logit_bound(u, wg.float().numpy(), lg_ref)
                check_logits(tr[l][2].cpu().numpy(), lg_ref, bound)
                from oracle import route as o_route
                assert not check_topk(o_route.route(tr[l][2].cpu().numpy(), cfg.k)[0], lg_ref, bound).any()
                ref = o_moe.moe_forward(u.astype(np.float32), lg_ref, np_masters[l], l, L, o_lad, cfg.k,
                                        phase=phase, attn_mass=attn[l].cpu().numpy() if attn else None,
                                        forced_bits=np.array(tr[l][3], np.uint8))["y"]
                full_ref = o_stack.residual(x_in, ref)
                x_out = (tr[l + 1][0] if l + 1 < L else xL).float().cpu().numpy().astype(np.float64)
                bound = FFN_TOL * np.abs(ref).max() + np.abs(full_ref) * 2.0 ** -7
                assert (np.abs(x_out - full_ref) <= bound).all(), (prefetch, rep, l)
        s = store.stats
        assert store.pool.used() <= store.pool.capacity
        if prefetch:
            assert s["prefetched"] > 0 and s["prefetch_hits"] > 0, s
        else:
            assert s["prefetched"] == 0, s
