"""Worker of tests/test_gpu_ep.py::test_ep_p2p_ipc_processes (launched by torchrun, several
processes on one GPU): peer windows opened through CUDA IPC, host barriers (processes time-share
one GPU), forward_p2p compared bit for bit with the all-to-all forward over gloo."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
import paper_2603_19172_b200.dymoe as d  # noqa: E402
from paper_2603_19172_b200 import ep  # noqa: E402


def main():
    out_path = sys.argv[1]
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    cfg = synthetic.CONFIGS["tiny"].with_tokens(48)
    ex_all = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 9)]
    d.quantize_experts(ex_all, (8, 4, 2))
    comm = ep.TorchComm(stage_cpu=True)
    first, last = ep.owned_range(rank, cfg.M, P)
    shard = ep.EPMoELayer(comm, ep.CudaOps(), ex_all[first:last], cfg.M, cfg.k, cfg.hidden, cfg.ffn,
                          make_local_layer=lambda ex: d.MoELayer(ex, 1, cfg.hidden, cfg.ffn))
    win = ep.PeerWindows(comm, cfg.M, cfg.hidden, cfg.T * cfg.k * P, barrier="host")
    lad = d.make_ladder((8, 4, 2), (0.25, 0.5))
    ok, worst = True, 0.0
    for s in range(3):
        x, lg, a = synthetic.layer_inputs(cfg, 700 + 10 * s + rank)
        phase = s % 2
        y2, _ = shard.forward_p2p(win, x.cuda(), lg.cuda(), lad, 9 + s, 32, phase, attn_mass=a.cuda())
        y1, _ = shard.forward(x.cuda(), lg.cuda(), lad, 9 + s, 32, phase, attn_mass=a.cuda())
        torch.cuda.synchronize()
        y1, y2 = y1.cpu().numpy(), y2.cpu().numpy()
        ok = ok and bool(np.array_equal(y1, y2))
        worst = max(worst, float(np.abs(y1 - y2).max()))
    status = int(win.status.item())
    dist.barrier()
    win.close()
    with open("%s.%d" % (out_path, rank), "w") as f:
        json.dump({"ok": ok, "worst": worst, "status": status}, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
