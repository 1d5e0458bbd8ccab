"""Quantize kernel alone (row a4): one Mixtral expert (W1, W3, W2) per batched launch and width,
timed with CUDA events; `--ncu` runs one launch per width (for a profiler)."""
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ncu", action="store_true")
    args = ap.parse_args()
    import paper_2603_19172_b200.dymoe as d
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synthetic.CONFIGS["mixtral_decode"]
    ex = [{n: t.to(dev) for n, t in e.items()} for e in synthetic.expert_weights(cfg, 7, dev, experts=[0])][0]
    d.quantize_experts([ex], (8, 4, 2))
    torch.cuda.synchronize()
    peaks = bench.load_peaks()
    for b in (8, 4, 2):
        jobs = [(ex[n], b, ex["q%d" % b][n]) for n in ("w1", "w3", "w2")]
        if args.ncu:
            d.dymoe_quantize_batched(jobs)
            continue
        r = bench.measure_quantize(d, [ex], cfg, peaks, reps=args.reps)
        print(json.dumps({k: v for k, v in r.items() if k == "int%d" % b}))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
