"""Expert-parallel layer on the CUDA path with P ranks simulated by P threads on one GPU
(ThreadComm): real kernels for every step, compared with the unsharded oracle."""
import threading

import numpy as np
import pytest
import torch

import synthetic
from oracle import moe as o_moe, route as o_route, importance as o_imp, schedule as o_sched
from validity import check_bits, decode_importance_tol

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
    tol = 0 if phase == 0 else decode_importance_tol(T * P)
    for r in range(P):
        y, gbits = res[r]
        assert np.array_equal(gbits, res[0][1])          # every rank assigns the same widths
        check_bits(gbits, bits, I, tol)                  # = the oracle's, or valid on a near-tie
        x, lg = ins[r]
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), experts, layer_idx, 32,
                                o_sched.Ladder(bits_t, lams), cfg.k, forced_bits=gbits)
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


def _run_p2p(P, phase, bits_t, lams, layer_idx, cfg, steps=3, barrier="device", ffn_mode=None):
    """Each simulated rank runs `steps` layer steps through forward_p2p (peer windows, device flag
    barriers, one CUDA stream per rank) and through forward (all-to-all through ThreadComm)."""
    import paper_2603_19172_b200.dymoe as d
    from paper_2603_19172_b200 import ep
    ex_all = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    d.quantize_experts(ex_all, (8, 4, 2))
    comm = ep.ThreadComm(P)
    ops = ep.CudaOps()
    results, errors = {}, []
    lad = d.make_ladder(bits_t, lams)

    def worker(r):
        try:
            comm.bind(r)
            with torch.cuda.stream(torch.cuda.Stream()):
                first, last = ep.owned_range(r, cfg.M, P)
                shard = ep.EPMoELayer(comm, ops, ex_all[first:last], cfg.M, cfg.k, cfg.hidden,
                                      cfg.ffn, make_local_layer=lambda ex: d.MoELayer(ex, 1, cfg.hidden, cfg.ffn))
                win = ep.PeerWindows(comm, cfg.M, cfg.hidden, cfg.T * cfg.k * P, barrier=barrier)
                out = []
                for s in range(steps):
                    x, lg, a = synthetic.layer_inputs(cfg, 500 + 10 * s + r)
                    y2, i2 = shard.forward_p2p(win, x.cuda(), lg.cuda(), lad, (layer_idx + s) % 32, 32,
                                               phase, attn_mass=a.cuda(), ffn_mode=ffn_mode)
                    y1, i1 = shard.forward(x.cuda(), lg.cuda(), lad, (layer_idx + s) % 32, 32, phase,
                                           attn_mass=a.cuda(), ffn_mode=ffn_mode)
                    torch.cuda.current_stream().synchronize()
                    out.append((y1.cpu().numpy(), y2.cpu().numpy(), i2["recv"], sum(i1["recv"]),
                                int(win.status.item())))
                results[r] = out
                comm._exchange(None)
                win.close()
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
    (2, 0, (8, 4, 2), (0.25, 0.5), 20, 40), (4, 0, (4, 0), (0.5,), 29, 24),
    (2, 1, (8, 4, 2), (0.25, 0.5), 25, 8), (8, 0, (8, 4, 2), (0.25, 0.5), 10, 300),
    (8, 1, (4, 0), (0.5,), 30, 3)])
def test_ep_p2p_equals_all_to_all(P, phase, bits_t, lams, layer_idx, T):
    """Peer-memory dispatch/combine (fused kernels, device flag barriers) gives the all-to-all
    path's output bit for bit, step after step (window parity and barrier epochs advance)."""
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    res = _run_p2p(P, phase, bits_t, lams, layer_idx, cfg)
    for r in range(P):
        for s, (y1, y2, n2, n1, status) in enumerate(res[r]):
            assert status == 0, (r, s, status)
            assert n1 == n2, (r, s)
            assert np.array_equal(y1, y2), (r, s, np.abs(y1 - y2).max())


def test_ep_p2p_host_barrier_threads():
    cfg = synthetic.CONFIGS["tiny"].with_tokens(16)
    res = _run_p2p(4, 0, (8, 4, 2), (0.25, 0.5), 12, cfg, steps=2, barrier="host")
    for r in range(4):
        for y1, y2, n2, n1, status in res[r]:
            assert status == 0 and n1 == n2 and np.array_equal(y1, y2)


def test_ep_p2p_prefill_mode_matches_oracle():
    """Large enough that every owner runs the tcgen05 prefill kernel on received rows; against the
    unsharded oracle at the FFN bar."""
    P, T, layer_idx = 2, 200, 7
    bits_t, lams = (8, 4, 2), (0.25, 0.5)
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    res = _run_p2p(P, 0, bits_t, lams, layer_idx, cfg, steps=1)
    experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    I = np.zeros(cfg.M)
    ins = []
    for r in range(P):
        x, lg, a = synthetic.layer_inputs(cfg, 500 + r)
        idx, w, p = o_route.route(lg.numpy(), cfg.k)
        I = I + o_imp.score_prefill(a.numpy(), idx, cfg.M)[0]
        ins.append((x, lg))
    bits, _ = o_sched.assign_bits(I, layer_idx, 32, o_sched.Ladder(bits_t, lams), cfg.k)
    for r in range(P):
        x, lg = ins[r]
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), experts, layer_idx, 32,
                                o_sched.Ladder(bits_t, lams), cfg.k, forced_bits=bits)
        y = res[r][0][1]
        assert res[r][0][2] > 64
        err = np.abs(y - ref["y"]).max() / np.abs(ref["y"]).max()
        assert err <= 2e-3, (r, err)


def test_ep_p2p_ipc_processes(tmp_path):
    """Two processes on one GPU: windows exchanged as CUDA IPC handles and opened in the other
    process; forward_p2p equals the all-to-all forward bit for bit."""
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


@pytest.mark.parametrize("phase,T", [(0, 256), (1, 8)])
def test_ep_p2p_finegrained_p8(phase, T):
    """BASELINE.json configs[3]'s layer (64 experts, top-6, hidden 2048, ffn 1408) over 8 ranks
    (threads, 8 experts each): peer-memory dispatch/combine equals the all-to-all path."""
    cfg = synthetic.CONFIGS["finegrained"].with_tokens(T)
    res = _run_p2p(8, phase, (8, 4, 2), (0.25, 0.5), 17, cfg, steps=2)
    for r in range(8):
        for y1, y2, n2, n1, status in res[r]:
            assert status == 0 and n1 == n2 and n2 > 0
            assert np.array_equal(y1, y2), (r, np.abs(y1 - y2).max())
