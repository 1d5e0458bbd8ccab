"""Worker of tests/test_gpu_ep.py::test_ep_peer_ipc_processes (launched by torchrun, two processes
on one GPU): each process creates its dymoe_ep handle (peer-memory transport), the windows are
exchanged as CUDA IPC handles over a gloo group and opened, and three layer steps run through
dymoe_moe_forward_ep with device flag barriers across the processes.  Each rank checks its output
against the unsharded oracle layer with the global importance (oracle = test infrastructure)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import synthetic  # noqa: E402
import paper_2603_19172_b200.dymoe as d  # noqa: E402
from paper_2603_19172_b200 import ep  # noqa: E402
from oracle import moe as o_moe, route as o_route, importance as o_imp, schedule as o_sched  # noqa: E402
from validity import check_bits, decode_importance_tol  # noqa: E402


def main():
    out_path = sys.argv[1]
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    cfg = synthetic.CONFIGS["tiny"].with_tokens(48)
    ex_all = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    d.quantize_experts(ex_all, (8, 4, 2))
    first, last = ep.owned_range(rank, cfg.M, P)
    layer = ep.EPLayer(rank, P, cfg.M, cfg.k, cfg.hidden, cfg.ffn, cfg.T, ex_all[first:last],
                       transports=d.DYMOE_EP_PEER)
    opened = ep.connect_processes(layer)
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    lad_o = o_sched.Ladder((8, 4, 2), (0.25, 0.5))
    experts = [{n: t.float().numpy() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    ok, worst, status = True, 0.0, 0
    for s in range(3):
        phase = s % 2
        x, lg, a = synthetic.layer_inputs(cfg, 700 + 10 * s + rank)
        y, ws = layer.forward(x.cuda(), lg.cuda(), lad, 9 + s, 32, phase, attn_mass=a.cuda())
        bits = layer.views(cfg.T, ws)["bits"].cpu().numpy()
        rc, word = layer.check_status(cfg.T, ws)
        status |= word
        I = np.zeros(cfg.M)
        for r in range(P):
            xr, lgr, ar = synthetic.layer_inputs(cfg, 700 + 10 * s + r)
            idx, _, p = o_route.route(lgr.numpy(), cfg.k)
            I = I + (o_imp.score_prefill(ar.numpy(), idx, cfg.M)[0] if phase == 0
                     else o_imp.decode_importance(lgr.numpy(), p))
        ref_bits, _ = o_sched.assign_bits(I, 9 + s, 32, lad_o, cfg.k)
        check_bits(bits, ref_bits, I, 0 if phase == 0 else decode_importance_tol(cfg.T * P))
        ref = o_moe.moe_forward(x.float().numpy(), lg.numpy(), experts, 9 + s, 32, lad_o, cfg.k,
                                forced_bits=bits)["y"]
        err = float(np.abs(y.cpu().numpy() - ref).max() / np.abs(ref).max())
        worst = max(worst, err)
        ok = ok and err <= 2e-3
    torch.cuda.synchronize()
    dist.barrier()
    ep.disconnect(opened)
    layer.close()
    with open("%s.%d" % (out_path, rank), "w") as f:
        json.dump({"ok": ok, "worst": worst, "status": status}, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
