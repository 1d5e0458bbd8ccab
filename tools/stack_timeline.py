"""Kineto per-kernel timeline of the 32-layer stack decode pass (B = 8): mean duration per kernel
kind and per layer.  usage: python tools/stack_timeline.py [layers]"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

import bench  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    import paper_2603_19172_b200.dymoe as d
    import paper_2603_19172_b200.stack as st
    import synthetic
    dev = torch.device("cuda", 0)
    cfg = synthetic.CONFIGS["mixtral_decode"].with_tokens(8)
    stack = st.MoEStack.random(cfg, L, seed=7, device=dev) if hasattr(st.MoEStack, "random") else None
    if stack is None:
        print("no MoEStack.random; see bench.py stack workload")
        return
    x = torch.randn(8, cfg.hidden, device=dev).to(torch.bfloat16)
    lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
    for _ in range(3):
        stack.forward(x, lad)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for _ in range(3):
            stack.forward(x, lad)
        torch.cuda.synchronize()
    dur = collections.defaultdict(list)
    for e in p.events():
        if e.device_type.name == "CUDA":
            dur[e.name[:48]].append(e.time_range.end - e.time_range.start)
    for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
        print("  %-48s n=%d mean %.1f us" % (k, len(v), sum(v) / len(v)))


if __name__ == "__main__":
    main()
