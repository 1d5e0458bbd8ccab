"""The expert-parallel layer through the C ABI (dymoe_ep_create / dymoe_moe_forward_ep,
include/dymoe.h) on one GPU: P ranks simulated by P threads (each with its own CUDA stream,
windows connected by pointer, device flag barriers) for the peer-memory transport, P = 1 for the
library-owned NCCL communicator, and two processes over CUDA IPC.  Every rank's output is checked
against the unsharded oracle layer with the GLOBAL importance (sum over the ranks)."""
import threading

import numpy as np
import pytest
import torch

import synthetic
from oracle import moe as o_moe, route as o_route, importance as o_imp, schedule as o_sched
from validity import check_bits, decode_importance_tol

pytestmark = pytest.mark.gpu
FFN_TOL = 2e-3


def D():
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    return d


def _experts(cfg, widths=(8, 4, 2)):
    d = D()
    ex = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    d.quantize_experts(ex, widths)
    return ex


def _np_experts(cfg):
    return [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]


def _inputs(cfg, r, s):
    return synthetic.layer_inputs(cfg, 500 + 10 * s + r)


def _make_layers(P, cfg, ex_all, transports, max_tokens, nccl_uid=None):
    from paper_2603_19172_b200 import ep
    layers = []
    for r in range(P):
        first, last = ep.owned_range(r, cfg.M, P)
        layers.append(ep.EPLayer(r, P, cfg.M, cfg.k, cfg.hidden, cfg.ffn, max_tokens,
                                 ex_all[first:last], transports=transports, nccl_uid=nccl_uid))
    if P > 1:
        ep.connect_threads(layers)
    return layers


def _run_threads(P, cfg, phase, lad, layer_idx, steps=3, placement=0, transport=None,
                 same_batch=False, **kw):
    """Each simulated rank runs `steps` layer steps on its own stream."""
    d = D()
    transport = d.DYMOE_EP_PEER if transport is None else transport
    ex_all = _experts(cfg)
    layers = _make_layers(P, cfg, ex_all, d.DYMOE_EP_PEER, cfg.T)
    results, errors = {}, []
    # every allocation and host->device copy before the ranks start: a cudaMalloc / pageable copy
    # in one thread while another rank's flag barrier spins can wait for the device to idle
    ins = {(r, s): tuple(t.cuda() for t in _inputs(cfg, 0 if same_batch else r, s))
           for r in range(P) for s in range(steps)}
    wss = [l.workspace(cfg.T, placement=placement) for l in layers]
    outs = [torch.empty(cfg.T, cfg.hidden, device="cuda") for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    torch.cuda.synchronize()

    def worker(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                out = []
                for s in range(steps):
                    x, lg, a = ins[(r, s)]
                    y, ws = layers[r].forward(x, lg, lad, (layer_idx + s) % 32, 32, phase,
                                              transport=transport, placement=placement,
                                              attn_mass=a, ws=wss[r], out=outs[r], **kw)
                    v = layers[r].views(x.shape[0], ws, placement=placement)
                    rc, word = layers[r].check_status(x.shape[0], ws, placement=placement)
                    out.append((y.float().cpu().numpy(), v["bits"].cpu().numpy(),
                                v["importance"].cpu().numpy(), word))
                results[r] = out
        except Exception as e:   # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for l in layers:
        l.close()
    assert not errors, errors
    return results


def _oracle_global(cfg, P, phase, s, same_batch=False):
    """Global importance of step s (sum over the ranks' local importances, oracle)."""
    I = np.zeros(cfg.M)
    for r in range(P):
        x, lg, a = _inputs(cfg, 0 if same_batch else r, s)
        idx, w, p = o_route.route(lg.numpy(), cfg.k)
        if phase == 0:
            I = I + o_imp.score_prefill(a.numpy(), idx, cfg.M)[0].astype(np.float64)
        else:
            I = I + (p[0] if (x.shape[0] == 1 and P > 1) else o_imp.decode_importance(lg.numpy(), p))
    return I


def _oracle_y(x, lg, experts, bits, k, cache, renorm=True):
    """oracle.moe_forward's FFN + combine with the given widths, each (expert, width)'s
    dequantized weights computed once per test (the same oracle functions, in moe_forward's
    order)."""
    idx, w, _ = o_route.route(lg, k)
    perm = o_moe.permute(idx, bits, len(experts))
    off = perm["expert_off"]
    y_perm = np.zeros((max(int(off[-1]), 1), x.shape[1]))
    for e in range(len(experts)):
        lo, hi = int(off[e]), int(off[e + 1])
        if hi > lo:
            key = (e, int(bits[e]))
            if key not in cache:
                cache[key] = o_moe.expert_weights(experts[e], int(bits[e]))
            y_perm[lo:hi] = o_moe.ffn(x[perm["perm_token"][lo:hi]].astype(np.float64), *cache[key])
    return o_moe.combine(y_perm, perm["inv_row"], w, renorm)


def _check_a2a(res, cfg, P, phase, bits_t, lams, layer_idx, renorm=True):
    experts = _np_experts(cfg)
    cache = {}
    lad_o = o_sched.Ladder(bits_t, lams, renorm_on_skip=renorm)
    for s in range(len(res[0])):
        I = _oracle_global(cfg, P, phase, s)
        l = (layer_idx + s) % 32
        bits, _ = o_sched.assign_bits(I, l, 32, lad_o, cfg.k)
        tol = 0 if phase == 0 else decode_importance_tol(cfg.T * P)
        for r in range(P):
            y, gbits, gI, status = res[r][s]
            assert status == 0, (r, s, status)
            assert np.array_equal(gbits, res[0][s][1])           # identical widths on every rank
            if phase == 0:
                assert np.array_equal(gI, I.astype(np.float32))  # exact global counts
            else:
                assert np.allclose(gI, I, rtol=0, atol=decode_importance_tol(cfg.T * P) / 2)
            check_bits(gbits, bits, I, tol)
            x, lg, a = _inputs(cfg, r, s)
            ref = _oracle_y(x.float().numpy(), lg.numpy(), experts, gbits, cfg.k, cache, renorm)
            err = np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30)
            assert err <= FFN_TOL, (r, s, err)


@pytest.mark.parametrize("P,phase,bits_t,lams,layer_idx,T,cfg_name", [
    (2, 0, (8, 4, 2), (0.25, 0.5), 20, 40, "tiny"), (4, 0, (4, 0), (0.5,), 29, 24, "tiny"),
    (2, 1, (8, 4, 2), (0.25, 0.5), 25, 8, "tiny"), (8, 0, (8, 4, 2), (0.25, 0.5), 10, 300, "tiny"),
    (8, 1, (4, 0), (0.5,), 30, 3, "tiny"), (4, 1, (8, 4, 2), (0.25, 0.5), 7, 1, "tiny"),
    (4, 0, (16, 8, 4, 2), (0.2, 0.5, 0.8), 12, 64, "ep_small")])
def test_ep_peer_threads_match_unsharded(P, phase, bits_t, lams, layer_idx, T, cfg_name):
    """Peer-memory transport, every rank its own tokens, 3 consecutive steps (window parity and
    barrier epochs advance); prefill at T = 300 runs the tcgen05 GEMM on received rows."""
    d = D()
    cfg = synthetic.CONFIGS[cfg_name].with_tokens(T)
    res = _run_threads(P, cfg, phase, d.make_ladder(bits_t, lams), layer_idx)
    _check_a2a(res, cfg, P, phase, bits_t, lams, layer_idx)


@pytest.mark.parametrize("phase,T", [(0, 256), (1, 8)])
def test_ep_peer_finegrained_p8(phase, T):
    """BASELINE.json configs[3]'s layer (64 experts, top-6, hidden 2048, ffn 1408) over 8 ranks
    (threads, 8 experts each)."""
    d = D()
    cfg = synthetic.CONFIGS["finegrained"].with_tokens(T)
    res = _run_threads(8, cfg, phase, d.make_ladder((8, 4, 2), (0.25, 0.5)), 17, steps=2)
    _check_a2a(res, cfg, 8, phase, (8, 4, 2), (0.25, 0.5), 17)


def test_ep_peer_bf16_output_and_residual():
    """out_dtype bf16 with a residual: y = bf16(residual + sum) per element."""
    d = D()
    cfg = synthetic.CONFIGS["tiny"].with_tokens(16)
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    P = 2
    ex_all = _experts(cfg)
    layers = _make_layers(P, cfg, ex_all, d.DYMOE_EP_PEER, cfg.T)
    outs, errors = {}, []
    ins = [tuple(t.cuda() for t in _inputs(cfg, r, 0)) for r in range(P)]
    wss = [l.workspace(cfg.T) for l in layers]
    o32 = [torch.empty(cfg.T, cfg.hidden, device="cuda") for _ in range(P)]
    o16 = [torch.empty(cfg.T, cfg.hidden, device="cuda", dtype=torch.bfloat16) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    torch.cuda.synchronize()

    def worker(r):
        try:
            with torch.cuda.stream(streams[r]):
                xc, lg, a = ins[r]
                y32, _ = layers[r].forward(xc, lg, lad, 3, 32, 0, attn_mass=a, ws=wss[r], out=o32[r])
                yb, _ = layers[r].forward(xc, lg, lad, 3, 32, 0, attn_mass=a, ws=wss[r], out=o16[r],
                                          out_dtype=d.DYMOE_OUT_BF16, residual=xc)
                torch.cuda.current_stream().synchronize()
                outs[r] = (y32, yb, xc)
        except Exception as e:   # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join() for t in th]
    [l.close() for l in layers]
    assert not errors, errors
    for r in range(P):
        y32, yb, xc = outs[r]
        assert torch.equal(yb, (xc.float() + y32).to(torch.bfloat16))


@pytest.mark.parametrize("P,bits_t,lams,layer_idx,T", [
    (2, (8, 4, 2), (0.25, 0.5), 25, 8), (4, (8, 4, 2), (0.25, 0.5), 3, 8), (8, (4, 0), (0.5,), 31, 5),
    (2, (4, 2), (0.5,), 6, 1)])
def test_ep_replicated_decode_peer_threads(P, bits_t, lams, layer_idx, T):
    """Decode with the batch replicated on P ranks: local experts + the sum of the partial outputs
    over the windows equals the unsharded single-GPU layer (<= 1e-6: top-2 gives at most two
    nonzero terms per element, exact in any order) and the oracle."""
    d = D()
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    lad = d.make_ladder(bits_t, lams)
    res = _run_threads(P, cfg, 1, lad, layer_idx, steps=2, placement=d.DYMOE_EP_REPLICATED,
                       same_batch=True)
    ex_all = _experts(cfg)
    full = d.MoELayer(ex_all, cfg.k, cfg.hidden, cfg.ffn)
    experts = _np_experts(cfg)
    for s in range(2):
        x, lg, _ = _inputs(cfg, 0, s)
        l = (layer_idx + s) % 32
        y_one, _ = full.forward(x.cuda(), lg.cuda(), lad, l, 32, phase=d.DYMOE_DECODE)
        y1 = y_one.cpu().numpy()
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), experts, l, 32,
                                o_sched.Ladder(bits_t, lams), cfg.k)
        for r in range(P):
            y, gbits, _, status = res[r][s]
            assert status == 0
            assert np.abs(y - y1).max() <= 1e-6 * np.abs(y1).max(), (r, s)
            check_bits(gbits, ref["bits"], ref["importance"], 0 if T == 1 else decode_importance_tol(T))
            err = np.abs(y - ref["y"]).max() / np.abs(ref["y"]).max()
            assert err <= FFN_TOL, (r, err)


@pytest.mark.parametrize("phase,placement,T", [(0, 0, 40), (1, 0, 8), (1, 1, 8), (0, 0, 300)])
def test_ep_nccl_single_rank(phase, placement, T):
    """The library-owned NCCL communicator (one rank: every collective and send/recv runs, to
    itself) gives the peer-memory transport's output bit for bit, and the oracle's."""
    d = D()
    from paper_2603_19172_b200 import ep
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    ex_all = _experts(cfg)
    both = ep.EPLayer(0, 1, cfg.M, cfg.k, cfg.hidden, cfg.ffn, T, ex_all,
                      transports=d.DYMOE_EP_NCCL | d.DYMOE_EP_PEER, nccl_uid=ep.unique_id())
    experts = _np_experts(cfg)
    for s in range(2):
        x, lg, a = _inputs(cfg, 0, s)
        args = (x.cuda(), lg.cuda(), lad, 9 + s, 32, phase)
        y_n, ws = both.forward(*args, transport=d.DYMOE_EP_NCCL, placement=placement, attn_mass=a.cuda())
        assert both.check_status(T, ws, placement=placement) == (0, 0)
        bits = both.views(T, ws, placement=placement)["bits"].cpu().numpy()
        y_p, _ = both.forward(*args, transport=d.DYMOE_EP_PEER, placement=placement, attn_mass=a.cuda())
        torch.cuda.synchronize()
        assert torch.equal(y_n, y_p)
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), experts, 9 + s, 32,
                                o_sched.Ladder((8, 4, 2), (0.25, 0.5)), cfg.k,
                                phase="prefill" if phase == 0 else "decode", attn_mass=a.numpy(),
                                forced_bits=bits)
        err = np.abs(y_n.cpu().numpy() - ref["y"]).max() / np.abs(ref["y"]).max()
        assert err <= FFN_TOL
    both.close()


def test_ep_validation_names_the_field():
    d = D()
    from paper_2603_19172_b200 import ep
    cfg = synthetic.CONFIGS["tiny"]
    ex_all = _experts(cfg)
    with pytest.raises(d.DymoeError, match="nccl_uid"):
        ep.EPLayer(0, 1, cfg.M, cfg.k, cfg.hidden, cfg.ffn, 16, ex_all, transports=d.DYMOE_EP_NCCL)
    L = ep.EPLayer(0, 1, cfg.M, cfg.k, cfg.hidden, cfg.ffn, 16, ex_all)
    x, lg, a = _inputs(cfg, 0, 0)
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    with pytest.raises(d.DymoeError, match="transport: not enabled"):
        L.forward(x.cuda(), lg.cuda(), lad, 1, 32, 1, transport=d.DYMOE_EP_NCCL)
    x2, lg2, _ = synthetic.layer_inputs(cfg.with_tokens(17), 1)
    with pytest.raises(d.DymoeError, match="T: must satisfy"):
        L.forward(x2.cuda(), lg2.cuda(), lad, 1, 32, 1)
    with pytest.raises(d.DymoeError, match="opts.phase: DYMOE_EP_REPLICATED"):
        L.forward(x.cuda(), lg.cuda(), lad, 1, 32, 0, placement=d.DYMOE_EP_REPLICATED,
                  attn_mass=a.cuda())
    L.close()


def test_ep_peer_ipc_processes(tmp_path):
    """Two processes on one GPU: windows exchanged as CUDA IPC handles over a gloo group and
    opened in the other process; device barriers across the processes; each rank's output
    against the unsharded oracle with the global importance (3 steps, prefill and decode)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "res")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29631",
           os.path.join(root, "tests", "ep_p2p_ipc_worker.py"), out]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    for rank in range(2):
        res = json.load(open("%s.%d" % (out, rank)))
        assert res["ok"] and res["status"] == 0, res
