"""Kineto timeline of Mixtral decode steps (one layer, warm, 1 weight copy = 5.4 GB > L2):
per-kernel mean duration, gaps, per-step span.  usage: python tools/decode_timeline.py [B] [layer]"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

import bench  # noqa: E402
import synthetic  # noqa: E402
import paper_2603_19172_b200.dymoe as d  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    layer_idx = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    dev = torch.device("cuda", 0)
    cfg = synthetic.CONFIGS["mixtral_decode"].with_tokens(B)
    (layer, _), = bench.build_layer_copies(d, cfg, 1, dev)
    inputs = bench.step_inputs(cfg, 4, dev)
    ws = layer.workspace(B, dev)
    lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
    out = torch.empty(B, cfg.hidden, device=dev)
    for i in range(10):
        x, lg, a = inputs[i % 4]
        layer.forward(x, lg, lad, layer_idx, 32, ws=ws, out=out)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for i in range(20):
            x, lg, a = inputs[i % 4]
            layer.forward(x, lg, lad, layer_idx, 32, ws=ws, out=out)
        torch.cuda.synchronize()
    evs = sorted([e for e in p.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    dur = collections.defaultdict(list)
    for e in evs:
        dur[e.name[:48]].append(e.time_range.end - e.time_range.start)
    print("B = %d, layer %d" % (B, layer_idx))
    for k, v in dur.items():
        print("  %-48s n=%d mean %.1f us" % (k, len(v), sum(v) / len(v)))
    gaps = [evs[i + 1].time_range.start - evs[i].time_range.end for i in range(len(evs) - 1)]
    print("  mean gap %.2f us, max %.2f; per step %.1f us" % (
        sum(gaps) / len(gaps), max(gaps), (evs[-1].time_range.end - evs[0].time_range.start) / 20))


if __name__ == "__main__":
    main()
