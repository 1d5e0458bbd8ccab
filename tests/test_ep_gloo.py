"""Expert-parallel orchestration (paper_2603_19172_b200.ep) on CPU: world_size 2 over gloo,
oracle-backed primitives.  Each rank owns half of the experts and its own tokens; the result
must equal the unsharded oracle layer run on that rank's tokens with the bits assigned from the
GLOBAL (all-rank) importance."""
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


def _worker(rank, world, port, phase, bits_t, lams, layer_idx, T, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from ep_oracle_ops import OracleOps, SimpleLadder
    from paper_2603_19172_b200 import ep
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                            world_size=world)
    try:
        cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
        experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
        first, last = ep.owned_range(rank, cfg.M, world)
        shard = ep.EPMoELayer(ep.TorchComm(), OracleOps(), experts[first:last], cfg.M, cfg.k,
                              cfg.hidden, cfg.ffn, make_local_layer=lambda ex: ex)
        x, lg, a = _rank_inputs(cfg, rank)
        y, info = shard.forward(x, lg, SimpleLadder(bits_t, lams), layer_idx, 32, phase, attn_mass=a)
        q.put((rank, y.numpy(), info["bits"].numpy(), info["send"], info["recv"]))
    except Exception as e:  # surface worker failures instead of hanging the parent
        q.put((rank, "error: %r" % e, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


CASES = [(0, (8, 4, 2), (0.25, 0.5), 20, 16), (0, (4, 0), (0.5,), 31, 24),
         (1, (8, 4, 2), (0.25, 0.5), 25, 4), (1, (4, 2), (0.5,), 5, 1)]


@pytest.mark.parametrize("case", CASES)
def test_ep_two_ranks_equals_unsharded(case):
    phase, bits_t, lams, layer, T = case
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, phase, bits_t, lams, layer, T, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, y, bits, send, recv = q.get(timeout=300)
        assert not isinstance(y, str), y
        out[r] = (y, bits, send, recv)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded reference with the global importance
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
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
        y, gbits, send, recv = out[r]
        assert np.array_equal(gbits, bits)
        x, lg = per_rank[r]
        ref = o_moe.moe_forward(x.numpy(), lg.numpy(), experts, layer, 32, lad, cfg.k, forced_bits=bits)
        assert np.array_equal(y, ref["y"]), np.abs(y - ref["y"]).max()
    # conservation: what rank a sends to b is what b receives from a
    assert out[0][2][1] == out[1][3][0] and out[1][2][0] == out[0][3][1]


def _worker_replicated(rank, world, port, bits_t, lams, layer_idx, T, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from ep_oracle_ops import OracleOps, SimpleLadder
    from paper_2603_19172_b200 import ep
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                            world_size=world)
    try:
        cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
        experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
        first, last = ep.owned_range(rank, cfg.M, world)
        shard = ep.EPMoELayer(ep.TorchComm(), OracleOps(), experts[first:last], cfg.M, cfg.k,
                              cfg.hidden, cfg.ffn, make_local_layer=lambda ex: ex)
        x, lg, _ = _rank_inputs(cfg, 0)          # the SAME batch on every rank
        y, info = shard.forward_replicated(x, lg, SimpleLadder(bits_t, lams), layer_idx, 32)
        q.put((rank, y.numpy(), info["bits"].numpy(), info["rows"]))
    except Exception as e:  # surface worker failures instead of hanging the parent
        q.put((rank, "error: %r" % e, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [((8, 4, 2), (0.25, 0.5), 25, 8), ((4, 0), (0.5,), 31, 6),
                                  ((4, 2), (0.5,), 5, 1)])
def test_ep_replicated_decode_two_ranks(case):
    """Decode with the batch replicated on both ranks: local experts + all-reduce(sum) equals the
    unsharded oracle layer exactly (top-2: at most two nonzero terms per element)."""
    bits_t, lams, layer, T = case
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_replicated, args=(r, world, port, bits_t, lams, layer, T, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, y, bits, rows = q.get(timeout=300)
        assert not isinstance(y, str), y
        out[r] = (y, bits, rows)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synthetic.CONFIGS["tiny"].with_tokens(T)
    experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    x, lg, _ = _rank_inputs(cfg, 0)
    ref = o_moe.moe_forward(x.numpy(), lg.numpy(), experts, layer, 32, o_sched.Ladder(bits_t, lams), cfg.k)
    assert out[0][2] + out[1][2] == len(ref["perm_token"])     # every routed pair ran exactly once
    for r in range(world):
        y, bits, _ = out[r]
        assert np.array_equal(bits, ref["bits"])
        assert np.array_equal(y, ref["y"]), np.abs(y - ref["y"]).max()
