"""The expert-parallel exchange plan on CPU (no GPU): the library's host-side plan
(dymoe_ep_plan_host -- exactly the messages the NCCL transport of dymoe_moe_forward_ep sends and
receives) driven over a world_size-2 gloo group, with every step of the layer's math done by the
oracle.  Each rank owns half of the experts and brings its own tokens; the importance is summed
over the ranks; the rows travel as one message per (source, expert) chunk into the
expert-major receive rows the plan gives, the owners run their experts on exactly those rows, the
outputs come back along the same chunks into each source's permuted order, and the combine must
give the unsharded oracle layer's output with the global bits."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic
from oracle import moe as o_moe, route as o_route, importance as o_imp, schedule as o_sched


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_inputs(cfg, rank):
    x, lg, a = synthetic.layer_inputs(cfg, 500 + rank)
    return x.float(), lg, a


def _owned(rank, M, P):
    return -(-rank * M // P), -(-(rank + 1) * M // P)


def _worker(rank, world, port, phase, bits_t, lams, layer_idx, T, cfg_name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2603_19172_b200.dymoe as d
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                            world_size=world)
    try:
        cfg = synthetic.CONFIGS[cfg_name].with_tokens(T)
        M, k = cfg.M, cfg.k
        experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
        x, lg, a = _rank_inputs(cfg, rank)
        x = x.numpy()
        idx, w, p = o_route.route(lg.numpy(), k)
        if phase == 0:
            I = o_imp.score_prefill(a.numpy(), idx, M)[0].astype(np.float64)
        else:
            I = p[0] if T == 1 else o_imp.decode_importance(lg.numpy(), p)
        It = torch.from_numpy(np.asarray(I, np.float64).copy())
        dist.all_reduce(It)                                   # global importance
        lad = o_sched.Ladder(bits_t, lams)
        bits, _ = o_sched.assign_bits(It.numpy(), layer_idx, 32, lad, k)
        perm = o_moe.permute(idx, bits, M)
        cnt = torch.from_numpy(np.diff(perm["expert_off"]).astype(np.int32))
        allc = [torch.zeros(M, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allc, cnt)
        C = torch.stack(allc)                                 # [P][M]
        send_off, recv_base, recv_off = d.dymoe_ep_plan_host(world, M, rank, C)
        send_off, recv_base, recv_off = send_off.numpy(), recv_base.numpy(), recv_off.numpy()
        assert send_off[-1] == len(perm["perm_token"])
        first, last = _owned(rank, M, world)
        x_send = x[perm["perm_token"]].astype(np.float32)
        recv_x = np.zeros((max(int(recv_off[-1]), 1), cfg.hidden), np.float32)
        # dispatch, in the plan's message order (one message per non-empty chunk)
        reqs, bufs = [], []
        for dst in range(world):
            f, l = _owned(dst, M, world)
            for e in range(f, l):
                lo, hi = int(send_off[e]), int(send_off[e + 1])
                if hi > lo and dst != rank:
                    reqs.append(dist.isend(torch.from_numpy(x_send[lo:hi].copy()), dst))
        for src in range(world):
            for el in range(last - first):
                c = int(C[src, first + el])
                if c > 0:
                    at = int(recv_base[el, src])
                    if src == rank:          # own chunk: gloo has no self pair, copy it
                        lo = int(send_off[first + el])
                        recv_x[at:at + c] = x_send[lo:lo + c]
                        continue
                    b = torch.zeros(c, cfg.hidden)
                    bufs.append((at, b))
                    reqs.append(dist.irecv(b, src))
        for r in reqs:
            r.wait()
        for at, b in bufs:
            recv_x[at:at + b.shape[0]] = b.numpy()
        # the owner's experts on their expert-major receive rows
        y_out = np.zeros((recv_x.shape[0], cfg.hidden))
        for el in range(last - first):
            lo, hi = int(recv_off[el]), int(recv_off[el + 1])
            if hi > lo:
                W1, W3, W2 = o_moe.expert_weights(experts[first + el], int(bits[first + el]))
                y_out[lo:hi] = o_moe.ffn(recv_x[lo:hi].astype(np.float64), W1, W3, W2)
        # the outputs back along the same chunks, into this rank's permuted order
        y_back = np.zeros((max(int(send_off[-1]), 1), cfg.hidden))
        reqs, bufs = [], []
        for src in range(world):
            for el in range(last - first):
                c = int(C[src, first + el])
                if c > 0:
                    at = int(recv_base[el, src])
                    if src == rank:
                        lo = int(send_off[first + el])
                        y_back[lo:lo + c] = y_out[at:at + c]
                        continue
                    reqs.append(dist.isend(torch.from_numpy(y_out[at:at + c].copy()), src))
        for dst in range(world):
            f, l = _owned(dst, M, world)
            for e in range(f, l):
                lo, hi = int(send_off[e]), int(send_off[e + 1])
                if hi > lo and dst != rank:
                    b = torch.zeros(hi - lo, cfg.hidden, dtype=torch.float64)
                    bufs.append((lo, b))
                    reqs.append(dist.irecv(b, dst))
        for r in reqs:
            r.wait()
        for at, b in bufs:
            y_back[at:at + b.shape[0]] = b.numpy()
        y = o_moe.combine(y_back, perm["inv_row"], w, lad.renorm_on_skip)
        q.put((rank, y, bits, int(recv_off[-1]), int(send_off[-1])))
    except Exception as e:  # surface worker failures instead of hanging the parent
        q.put((rank, "error: %r" % e, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


CASES = [("tiny", 0, (8, 4, 2), (0.25, 0.5), 20, 16), ("tiny", 0, (4, 0), (0.5,), 31, 24),
         ("tiny", 1, (8, 4, 2), (0.25, 0.5), 25, 4), ("tiny", 1, (4, 2), (0.5,), 5, 1),
         ("ep_small", 0, (8, 4, 2), (0.25, 0.5), 12, 40)]


@pytest.mark.parametrize("case", CASES)
def test_ep_two_ranks_equals_unsharded(case):
    cfg_name, phase, bits_t, lams, layer, T = case
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, phase, bits_t, lams, layer, T,
                                               cfg_name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, y, bits, n_recv, n_sent = q.get(timeout=300)
        assert not isinstance(y, str), y
        out[r] = (y, bits, n_recv, n_sent)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded reference with the global importance
    cfg = synthetic.CONFIGS[cfg_name].with_tokens(T)
    experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    lad = o_sched.Ladder(bits_t, lams)
    I = np.zeros(cfg.M)
    per_rank = []
    for r in range(world):
        x, lg, a = _rank_inputs(cfg, r)
        idx, w, p = o_route.route(lg.numpy(), cfg.k)
        if phase == 0:
            Ir = o_imp.score_prefill(a.numpy(), idx, cfg.M)[0].astype(np.float64)
        else:
            Ir = p[0] if T == 1 else o_imp.decode_importance(lg.numpy(), p)
        I = I + Ir
        per_rank.append((x, lg))
    bits, _ = o_sched.assign_bits(I, layer, 32, lad, cfg.k)
    for r in range(world):
        y, gbits, _, _ = out[r]
        assert np.array_equal(gbits, bits)
        x, lg = per_rank[r]
        ref = o_moe.moe_forward(x.numpy(), lg.numpy(), experts, layer, 32, lad, cfg.k, forced_bits=bits)
        assert np.allclose(y, ref["y"], rtol=0, atol=1e-12 * np.abs(ref["y"]).max()), \
            np.abs(y - ref["y"]).max()
    # conservation: every routed row is received exactly once
    assert out[0][2] + out[1][2] == out[0][3] + out[1][3]


def test_plan_host_hand_example():
    """P = 2, M = 4 (rank 0 owns experts 0-1, rank 1 owns 2-3); counts[src][e] by hand."""
    import paper_2603_19172_b200.dymoe as d
    C = [[2, 0, 1, 3],    # rank 0 routes 2 rows to e0, 1 to e2, 3 to e3
         [1, 4, 0, 2]]    # rank 1
    so, rb, ro = d.dymoe_ep_plan_host(2, 4, 1, C)
    assert so.tolist() == [0, 1, 5, 5, 7]             # rank 1's permuted rows by expert
    # rank 1 receives expert 2: (src0: 1 row, src1: 0), expert 3: (src0: 3, src1: 2)
    assert rb.tolist() == [[0, 1], [1, 4]]
    assert ro.tolist() == [0, 1, 6]
    so, rb, ro = d.dymoe_ep_plan_host(2, 4, 0, C)
    assert so.tolist() == [0, 2, 2, 3, 6]
    assert rb.tolist() == [[0, 2], [3, 3]] and ro.tolist() == [0, 3, 7]
    with pytest.raises(d.DymoeError, match="counts\\[1\\]"):
        d.dymoe_ep_plan_host(2, 4, 0, [[0, -1, 0, 0], [0, 0, 0, 0]])
    with pytest.raises(d.DymoeError, match="P:"):
        d.dymoe_ep_plan_host(5, 4, 0, [[0] * 4] * 5)
