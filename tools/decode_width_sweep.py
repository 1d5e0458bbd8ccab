"""Decode FFN kernel rates per width: every expert forced to one width (BF16 / Int8 / Int4 / Int2),
the bench's decode workload (B tokens, Mixtral layer shape), W13 and W2 kernels timed with CUDA
events around many steps.  Prints one JSON line per width: GB/s of algorithmic bytes per kernel.
Used to calibrate the decode kernels' per-width cost model (ffn_decode_common.cuh wcost)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--widths", default="16,8,4,2")
    ap.add_argument("--phase", default="decode", choices=["decode", "prefill"])
    args = ap.parse_args()
    import paper_2603_19172_b200.dymoe as d
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synthetic.CONFIGS["mixtral_decode"].with_tokens(args.batch)
    PH = d.DYMOE_PREFILL if args.phase == "prefill" else d.DYMOE_DECODE
    layers = bench.build_layer_copies(d, cfg, 2, dev)
    inputs = bench.step_inputs(cfg, 4, dev)
    lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
    ws = [L.workspace(cfg.T, dev) for L, _ in layers]
    stream = torch.cuda.current_stream()
    for wb in [int(w) for w in args.widths.split(",")]:
        forced = torch.full((cfg.M,), wb, dtype=torch.uint8, device=dev)
        b13 = b2 = 0.0
        for c in range(len(layers)):
            x, lg, a = inputs[c]
            L = layers[c][0]
            L.forward(x, lg, lad, 0, bench.NUM_LAYERS, phase=PH, attn_mass=a, ws=ws[c],
                      forced_bits=forced)
        torch.cuda.synchronize()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        for row in ev:
            for e_ in row:
                e_.record(stream)
        torch.cuda.synchronize()
        for i in range(args.steps):
            c = i % len(layers)
            x, lg, a = inputs[i % len(inputs)]
            L = layers[c][0]
            L.forward(x, lg, lad, 0, bench.NUM_LAYERS, phase=PH, attn_mass=a,
                      ws=ws[c], forced_bits=forced, prof_events=ev[i])
        torch.cuda.synchronize()
        t13 = np.mean([ev[i][0].elapsed_time(ev[i][1]) for i in range(args.steps)]) * 1e-3
        t2 = np.mean([ev[i][1].elapsed_time(ev[i][2]) for i in range(args.steps)]) * 1e-3
        # bytes: the steps alternate over inputs, use input 0's routing for the census (all
        # experts are normally active at B = 8 with k = 2; report the active count)
        tot13 = tot2 = 0.0
        for i in range(len(layers)):
            x, lg, a = inputs[i]
            L = layers[i][0]
            L.forward(x, lg, lad, 0, bench.NUM_LAYERS, phase=PH, attn_mass=a, ws=ws[i],
                      forced_bits=forced)
            vv = L.views(cfg.T, ws[i])
            off = vv["expert_off"].cpu().numpy()
            bits = np.full(cfg.M, wb)
            a13, a2 = bench.algorithmic_bytes(cfg, bits, off)
            tot13 += a13
            tot2 += a2
        b13, b2 = tot13 / len(layers), tot2 / len(layers)
        fl = sum(bench.algorithmic_flops(cfg, layers[i][0].views(cfg.T, ws[i])["expert_off"].cpu().numpy(),
                                         np.full(cfg.M, wb)) for i in range(len(layers))) / len(layers)
        print(json.dumps({"bits": wb, "w13_us": round(t13 * 1e6, 1), "w2_us": round(t2 * 1e6, 1),
                          "w13_TFLOPs": round(fl * 2 / 3 / t13 / 1e12), "w2_TFLOPs": round(fl / 3 / t2 / 1e12),
                          "w13_GBps": round(b13 / t13 / 1e9), "w2_GBps": round(b2 / t2 / 1e9),
                          "bytes_w13": b13, "bytes_w2": b2,
                          "active": int((np.diff(off) > 0).sum())}), flush=True)


if __name__ == "__main__":
    main()
