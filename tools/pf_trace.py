"""Timeline of CTA 0 of the prefill grouped GEMMs (measurement tool, not product code).

  python tools/pf_trace.py --build            # here: libdymoe with -DDYMOE_PF_TRACE -> tools/trace/
  python tools/pf_trace.py [prefill|finegrained]   # on the GPU: one layer step, timeline summary

Roles of CTA 0 (csrc/kernels/ffn_prefill.cu PF_TR): 0 = MMA issuer (1 / 5 = before the next
k-block's (tile's) waits, 2 = before its full wait, 3 = after it), 1 = producer warp 2 lane 0
(11 / 12 around the raw-codes wait, 13 / 14 around the stage-empty wait, 15 after the arrive),
2 = the A-tile TMA thread (21 / 22 around the stage-empty wait).
"""
import ctypes
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tools", "trace")
LIB = os.path.join(OUT, "libdymoe_pftrace.so")


def build():
    from paper_2603_19172_b200 import build as b
    b.build()
    os.makedirs(OUT, exist_ok=True)
    obj = os.path.join(OUT, "ffn_prefill_trace.o")
    src = os.path.join(b.CSRC, "kernels", "ffn_prefill.cu")
    subprocess.check_call([b.NVCC] + b.ARCH + b.FLAGS + ["-DDYMOE_PF_TRACE", "-c", src, "-o", obj])
    objs = [o for o in glob.glob(os.path.join(b.OBJ, "*.o")) if "ffn_prefill" not in o] + [obj]
    subprocess.check_call([b.NVCC] + b.ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static"])
    print("built", LIB)


def main():
    if "--build" in sys.argv:
        build()
        return
    import torch
    import paper_2603_19172_b200.dymoe as d
    d.LIB_PATH = LIB
    import synthetic
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    work = sys.argv[1] if len(sys.argv) > 1 else "prefill"
    cfg = synthetic.CONFIGS["finegrained" if work == "finegrained" else "mixtral_prefill"]
    experts = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 0, "cuda")]
    d.quantize_experts(experts, (8, 4, 2))
    layer = d.MoELayer(experts, cfg.k, cfg.hidden, cfg.ffn)
    ladder = d.make_ladder((8, 4, 2), (0.25, 0.5))
    x, logits, attn = synthetic.layer_inputs(cfg, 4, "cuda")
    L = d.lib()
    buf = (ctypes.c_ulonglong * (2 * 3 * 8192))()
    cnt = (ctypes.c_int * 6)()
    for _ in range(2):
        layer.forward(x, logits, ladder, layer=20, num_layers=32, phase=d.DYMOE_PREFILL, attn_mass=attn)
    torch.cuda.synchronize()
    L.dymoe_pf_trace_read(buf, cnt)
    layer.forward(x, logits, ladder, layer=20, num_layers=32, phase=d.DYMOE_PREFILL, attn_mass=attn)
    torch.cuda.synchronize()
    L.dymoe_pf_trace_read(buf, cnt)
    out = {"work": work, "counts": list(cnt)}
    for g, gname in enumerate(("w13", "w2")):
        for r in range(3):
            n = min(cnt[g * 3 + r], 4096)
            base = (g * 3 + r) * 8192
            evs = [(buf[base + 2 * i], buf[base + 2 * i + 1]) for i in range(n)]
            gaps = {}
            for (e0, c0), (e1, c1) in zip(evs, evs[1:]):
                gaps.setdefault("%d->%d" % (e0, e1), []).append(c1 - c0)
            out["%s_role%d" % (gname, r)] = {k: {"n": len(v), "mean": round(sum(v) / len(v), 1),
                                                 "sum": sum(v)} for k, v in sorted(gaps.items())}
            out["%s_role%d_span" % (gname, r)] = (evs[-1][1] - evs[0][1]) if evs else 0
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
