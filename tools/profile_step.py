"""Run one DyMoE layer step of the bench workload for ncu: W warm-up steps (not profiled when
ncu is given -s <skip>), then exactly one step at (layer l, input j), and print that step's
algorithmic bytes / flops per FFN kernel as JSON (stdout) so that the ncu dram traffic of the
same launch can be compared with them (profiles/traffic.json)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="decode",
                    choices=["decode", "prefill", "finegrained", "finegrained_decode"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--layer", type=int, default=20)
    ap.add_argument("--input", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import paper_2603_19172_b200.dymoe as d
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg, is_decode, _ = bench.workload_cfg(args)
    phase = d.DYMOE_DECODE if is_decode else d.DYMOE_PREFILL
    (layer, _), = bench.build_layer_copies(d, cfg, 1, dev)
    inputs = bench.step_inputs(cfg, args.input + 1, dev)
    x, lg, a = inputs[args.input]
    ws = layer.workspace(cfg.T, dev)
    lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
    for _ in range(args.warmup + 1):
        y, _ = layer.forward(x, lg, lad, args.layer, bench.NUM_LAYERS, phase=phase, attn_mass=a, ws=ws,
                             ffn_mode=-1)
    torch.cuda.synchronize()
    v = layer.views(cfg.T, ws)
    bits = v["bits"].cpu().numpy()
    off = v["expert_off"].cpu().numpy()
    b13, b2 = bench.algorithmic_bytes(cfg, bits, off)
    fl = bench.algorithmic_flops(cfg, off, bits)
    print(json.dumps({"workload": args.workload, "layer": args.layer, "input": args.input,
                      "bits": bits.tolist(), "rows": (off[1:] - off[:-1]).tolist(),
                      "algorithmic_bytes_w13": b13, "algorithmic_bytes_w2": b2,
                      "algorithmic_flops_w13": fl * 2 / 3, "algorithmic_flops_w2": fl / 3}))


if __name__ == "__main__":
    main()
