"""Device bandwidth of the peer-memory EP kernels on ONE GPU (window of P = 1: every "peer" row is
local HBM), at the Mixtral prefill shape (T = 2048, top-2, Hd = 4096) and the fine-grained one
(T = 2048, top-6, Hd = 2048).  dymoe_ep_dispatch moves rows*Hd*2 bytes in and out;
dymoe_ep_combine reads rows*Hd*4 and writes T*Hd*4.  Across GPUs the same kernels run over
NVLink; this bounds their local efficiency only.  usage: python tools/ep_kernels_bench.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthetic  # noqa: E402
import paper_2603_19172_b200.dymoe as d  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    out = []
    for name in ("mixtral_prefill", "finegrained"):
        cfg = synthetic.CONFIGS[name]
        x, lg, _ = synthetic.layer_inputs(cfg, 3, dev)
        idx, w, _ = d.dymoe_route(lg.contiguous(), cfg.k)
        bits = torch.full((cfg.M,), 4, dtype=torch.uint8, device=dev)
        off, pt, ps, inv = d.dymoe_permute(idx, cfg.M, bits)
        rows = int(off[-1].item())
        base, _ = d.dymoe_ep_window_alloc(d.dymoe_ep_window_bytes(1, cfg.M, cfg.hidden, rows))
        peers = torch.tensor([base], dtype=torch.int64, device=dev)
        win = d.EpWindow(1, 0, cfg.M, cfg.hidden, rows, 0, peers.data_ptr())
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        recv_off = torch.empty(cfg.M + 1, dtype=torch.int32, device=dev)
        d.dymoe_ep_publish_counts(win, off)
        d.dymoe_ep_barrier(win, 1, status)

        def timed(fn, reps=50):
            for _ in range(5):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps * 1e3   # us

        t_disp = timed(lambda: d.dymoe_ep_dispatch(win, x, off, pt, recv_off, status))
        t_comb = timed(lambda: d.dymoe_ep_combine(win, inv, w, off, status=status))
        b_disp = rows * cfg.hidden * 2 * 2
        b_comb = rows * cfg.hidden * 4 + cfg.T * cfg.hidden * 4
        out.append({"config": name, "rows": rows, "dispatch_us": round(t_disp, 2),
                    "dispatch_GBs": round(b_disp / t_disp / 1e3, 1), "combine_us": round(t_comb, 2),
                    "combine_GBs": round(b_comb / t_comb / 1e3, 1), "status": int(status.item())})
        torch.cuda.synchronize()
        d.dymoe_ep_window_free(base)
    print(json.dumps({"ep_kernels_one_gpu": out, "hbm_peak": peak.get("hbm_gbs")}))


if __name__ == "__main__":
    main()
