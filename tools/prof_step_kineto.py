import sys, os
sys.path.insert(0, "/root/repo")
import torch, bench, synthetic
import paper_2603_19172_b200.dymoe as d
from torch.profiler import profile, ProfilerActivity
dev = torch.device("cuda", 0)
cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mixtral_decode"].with_tokens(8)
(layer, _), = bench.build_layer_copies(d, cfg, 1, dev)
inputs = bench.step_inputs(cfg, 4, dev)
ws = layer.workspace(8, dev)
lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
out = torch.empty(8, cfg.hidden, device=dev)
for i in range(10):
    x, lg, a = inputs[i % 4]
    layer.forward(x, lg, lad, 20, 32, ws=ws, out=out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for i in range(20):
        x, lg, a = inputs[i % 4]
        layer.forward(x, lg, lad, 20, 32, ws=ws, out=out)
    torch.cuda.synchronize()
evs = [e for e in p.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
import collections
dur = collections.defaultdict(list)
for e in evs:
    dur[e.name[:40]].append(e.time_range.end - e.time_range.start)
for k, v in dur.items():
    print("%-40s n=%d mean %.1f us" % (k, len(v), sum(v) / len(v)))
# gaps between consecutive kernels
gaps = [evs[i + 1].time_range.start - evs[i].time_range.end for i in range(len(evs) - 1)]
print("mean gap %.2f us, max %.2f" % (sum(gaps) / len(gaps), max(gaps)))
span = (evs[-1].time_range.end - evs[0].time_range.start) / 20
print("per step %.1f us" % span)

# the front's phases as standalone kernels (same bodies), warm, for attribution
x, lg, a = inputs[0]
for i in range(5):
    idx, w, pr = d.dymoe_route(lg, cfg.k)
    imp, _ = d.dymoe_score(d.DYMOE_DECODE, cfg.M, logits=lg)
    bits, _ = d.dymoe_assign_bits(imp, 20, 32, lad, cfg.k)
    d.dymoe_permute(idx, cfg.M, bits)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p2:
    for i in range(20):
        idx, w, pr = d.dymoe_route(lg, cfg.k)
        imp, _ = d.dymoe_score(d.DYMOE_DECODE, cfg.M, logits=lg)
        bits, _ = d.dymoe_assign_bits(imp, 20, 32, lad, cfg.k)
        d.dymoe_permute(idx, cfg.M, bits)
    torch.cuda.synchronize()
dur = collections.defaultdict(list)
for e in p2.events():
    if e.device_type.name == "CUDA":
        dur[e.name[:40]].append(e.time_range.end - e.time_range.start)
for k, v in dur.items():
    print("%-40s n=%d mean %.1f us" % (k, len(v), sum(v) / len(v)))
