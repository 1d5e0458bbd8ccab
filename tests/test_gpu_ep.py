"""Expert-parallel layer on the CUDA path with P ranks simulated by P threads on one GPU
(ThreadComm): real kernels for every step, compared with the unsharded oracle."""
import threading

import numpy as np
import pytest
import torch

import synthetic
from oracle import moe as o_moe, route as o_route, importance as o_imp, schedule as o_sched

pytestmark = pytest.mark.gpu


def _run(P, phase, bits_t, lams, layer_idx, T, cfg, ffn_mode=None):
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200 import ep
    ex_all = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    d.quantize_experts(ex_all, (8, 4, 2))
    comm = ep.ThreadComm(P)
    ops = ep.CudaOps()
    results, errors = {}, []

    def worker(r):
        try:
            comm.bind(r)
            first, last = ep.owned_range(r, cfg.M, P)
            shard = ep.EPMoELayer(comm, ops, ex_all[first:last], cfg.M, cfg.k, cfg.hidden, cfg.ffn,
                                  make_local_layer=lambda ex: d.MoELayer(ex, 1, cfg.hidden, cfg.ffn))
            x, lg, a = synthetic.layer_inputs(cfg, 500 + r)
            y, info = shard.forward(x.cuda(), lg.cuda(), d.make_ladder(bits_t, lams), layer_idx, 32,
                                    phase, attn_mass=a.cuda(), ffn_mode=ffn_mode)
            torch.cuda.synchronize()
            results[r] = (y.cpu().numpy(), info["bits"].cpu().numpy())
        except Exception as e:   # pragma: no cover
            errors.append(e)
            comm.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    return results


@pytest.mark.parametrize("P,phase,bits_t,lams,layer_idx,T", [
    (2, 0, (8, 4, 2), (0.25, 0.5), 20, 40), (4, 0, (4, 0), (0.5,), 31, 24),
    (2, 1, (8, 4, 2), (0.25, 0.5), 25, 8), (8, 0, (8, 4, 2), (0.25, 0.5), 10, 300)])
def test_ep_threads_match_unsharded(P, phase, bits_t, lams, layer_idx, T):
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    res = _run(P, phase, bits_t, lams, layer_idx, T, cfg)
    experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    I = np.zeros(cfg.M)
    ins = []
    for r in range(P):
        x, lg, a = synthetic.layer_inputs(cfg, 500 + r)
        idx, w, p = o_route.route(lg.numpy(), cfg.k)
        I = I + (o_imp.score_prefill(a.numpy(), idx, cfg.M)[0] if phase == 0
                 else o_imp.decode_importance(lg.numpy(), p))
        ins.append((x, lg))
    bits, _ = o_sched.assign_bits(I, layer_idx, 32, o_sched.Ladder(bits_t, lams), cfg.k)
    for r in range(P):
        y, gbits = res[r]
        assert np.array_equal(gbits, bits)
        x, lg = ins[r]
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), experts, layer_idx, 32,
                                o_sched.Ladder(bits_t, lams), cfg.k, forced_bits=bits)
        err = np.abs(y - ref["y"]).max() / np.abs(ref["y"]).max()
        assert err <= 2e-3, (r, err)


@pytest.mark.parametrize("P,bits_t,lams,layer_idx,T", [
    (2, (8, 4, 2), (0.25, 0.5), 25, 8), (4, (8, 4, 2), (0.25, 0.5), 3, 8), (8, (4, 0), (0.5,), 31, 5)])
def test_ep_replicated_decode_threads(P, bits_t, lams, layer_idx, T):
    """Decode, batch replicated on P ranks (threads on one GPU): local experts + all-reduce(sum)
    equals the unsharded single-GPU layer and the oracle."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200 import ep
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    ex_all = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    d.quantize_experts(ex_all, (8, 4, 2))
    x, lg, _ = synthetic.layer_inputs(cfg, 77)
    lad = d.make_ladder(bits_t, lams)
    full = d.MoELayer(ex_all, cfg.k, cfg.hidden, cfg.ffn)
    y_one, _ = full.forward(x.cuda(), lg.cuda(), lad, layer_idx, 32, phase=d.DYMOE_DECODE)
    torch.cuda.synchronize()
    comm = ep.ThreadComm(P)
    ops = ep.CudaOps()
    results, errors = {}, []

    def worker(r):
        try:
            comm.bind(r)
            first, last = ep.owned_range(r, cfg.M, P)
            shard = ep.EPMoELayer(comm, ops, ex_all[first:last], cfg.M, cfg.k, cfg.hidden, cfg.ffn,
                                  make_local_layer=lambda ex: d.MoELayer(ex, 1, cfg.hidden, cfg.ffn))
            y, info = shard.forward_replicated(x.cuda(), lg.cuda(), lad, layer_idx, 32)
            torch.cuda.synchronize()
            results[r] = y.cpu().numpy()
        except Exception as e:   # pragma: no cover
            errors.append(e)
            comm.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), experts, layer_idx, 32,
                            o_sched.Ladder(bits_t, lams), cfg.k)
    y1 = y_one.cpu().numpy()
    for r in range(P):
        assert np.abs(results[r] - y1).max() <= 1e-6 * np.abs(y1).max(), r
        err = np.abs(results[r] - ref["y"]).max() / np.abs(ref["y"]).max()
        assert err <= 2e-3, (r, err)
