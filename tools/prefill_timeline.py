"""Kineto timeline of Mixtral-shaped prefill steps (one layer, 2048 tokens, warm): per-kernel mean
duration.  usage: python tools/prefill_timeline.py [config] [tokens]"""
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
    cname = sys.argv[1] if len(sys.argv) > 1 else "mixtral_prefill"
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    dev = torch.device("cuda", 0)
    cfg = synthetic.CONFIGS[cname].with_tokens(T)
    (layer, _), = bench.build_layer_copies(d, cfg, 1, dev)
    inputs = bench.step_inputs(cfg, 4, dev)
    ws = layer.workspace(T, dev)
    lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
    out = torch.empty(T, cfg.hidden, device=dev)
    for i in range(4):
        x, lg, a = inputs[i % 4]
        layer.forward(x, lg, lad, 20, 32, phase=d.DYMOE_PREFILL, attn_mass=a, ws=ws, out=out)
    torch.cuda.synchronize()
    n = 8
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for i in range(n):
            x, lg, a = inputs[i % 4]
            layer.forward(x, lg, lad, 20, 32, phase=d.DYMOE_PREFILL, attn_mass=a, ws=ws, out=out)
        torch.cuda.synchronize()
    evs = sorted([e for e in p.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    dur = collections.defaultdict(list)
    for e in evs:
        dur[e.name[:48]].append(e.time_range.end - e.time_range.start)
    tot = sum(sum(v) for v in dur.values()) / n
    print(cname, "T", T, "kernel time per step %.1f us" % tot)
    for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
        print("  %-48s n=%d mean %.1f us  %.1f%%" % (k, len(v), sum(v) / len(v), 100 * sum(v) / n / tot))


if __name__ == "__main__":
    main()
