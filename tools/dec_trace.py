"""Per-CTA timeline of the decode GEMV kernels (measurement tool, not product code).

  python tools/dec_trace.py --build             # here: libdymoe with -DDYMOE_DEC_TRACE -> tools/trace/
  python tools/dec_trace.py [mixed|16|8|4|2] [B] [config]  # on the GPU: one layer step, timeline summary

Events per CTA (csrc/kernels/ffn_decode.cu DEC_TR, globaltimer ns): 0 start, 1 allocation done,
2 x slice staged (per virtual CTA), 3 its tiles done, 4 end; 5 first items issued (before
the staging), 6 thread 0's share of the staging loop done (before the barrier).  Prints, per kernel (W13, W2): the
span from the first CTA start to the last CTA end, the ramp (start -> first staged x), the time
in run_tiles, and the spread of the CTA end times (the tail).
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
LIB = os.path.join(OUT, "libdymoe_dectrace.so")
NEV = 32


def build():
    from paper_2603_19172_b200 import build as b
    b.build()
    os.makedirs(OUT, exist_ok=True)
    obj = os.path.join(OUT, "ffn_decode_trace.o")
    src = os.path.join(b.CSRC, "kernels", "ffn_decode.cu")
    subprocess.check_call([b.NVCC] + b.ARCH + b.FLAGS + ["-DDYMOE_DEC_TRACE", "-c", src, "-o", obj])
    objs = [o for o in glob.glob(os.path.join(b.OBJ, "*.o")) if "ffn_decode" not in o] + [obj]
    subprocess.check_call([b.NVCC] + b.ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static"])
    print("built", LIB)


def summarise(buf, cnt, g, ncta):
    per = []
    for c in range(ncta):
        n = cnt[g * 256 + c]
        base = (g * 256 + c) * 2 * NEV
        per.append([(buf[base + 2 * i], buf[base + 2 * i + 1]) for i in range(n)])
    per = [p for p in per if p]
    t0 = min(p[0][1] for p in per)
    t_end = max(p[-1][1] for p in per)
    ramp, run, alloc, ends, stage = [], [], [], [], []
    prime, stg, bar = [], [], []
    sub0, sub1, sub2 = [], [], []
    units = []
    by_width = {}
    unit_first, run_all = [], []
    for p in per:
        ev = {}
        for e, t in p:
            if (e & 0xff) == 2:   # payload: the unit's width and list position
                units.append(((e >> 8) & 0xff, e >> 16))
            ev.setdefault(e & 0xff, []).append(t)
        alloc.append((ev[1][0] - ev[0][0]) / 1e3 if 1 in ev else 0)
        if 2 in ev:
            ramp.append((ev[2][0] - ev[0][0]) / 1e3)
            stage.append(sum(b - a for a, b in zip(ev[1][:1] + ev[3][:-1], ev[2])) / 1e3)
            run.append(sum(b - a for a, b in zip(ev[2], ev[3])) / 1e3)
            if len(ev[2]) == 1:
                by_width.setdefault(units[-1][0], []).append(run[-1])
            unit_first.append(units[-len(ev[2])] if units else None)
            run_all.append(run[-1])
        ends.append((p[-1][1] - t0) / 1e3)
        sb = (2 * 256 * 2 * NEV) + (g * 256 + per.index(p)) * 8
        if 5 in ev and buf[sb + 2] and buf[sb + 3]:
            sub0.append((buf[sb + 2] - ev[1][0]) / 1e3)     # allocation done -> unit decoded
            sub1.append((buf[sb + 3] - buf[sb + 2]) / 1e3)  # -> past the pass-start barrier
            sub2.append((buf[sb + 1] - buf[sb + 3]) / 1e3)  # -> first items issued (prime return)
        if 5 in ev and 6 in ev:
            prime.append((ev[5][0] - ev[1][0]) / 1e3)
            stg.append((ev[6][0] - ev[5][0]) / 1e3)
            bar.append((ev[2][0] - ev[6][0]) / 1e3)
    span = (t_end - t0) / 1e3
    starts = [(p[0][1] - t0) / 1e3 for p in per]

    def st(v):
        v = sorted(v)
        return {"min": round(v[0], 2), "med": round(v[len(v) // 2], 2), "max": round(v[-1], 2),
                "mean": round(sum(v) / len(v), 2)} if v else None
    raw = [[c, u[0] if u else -1, round(r, 2)] for c, (u, r) in enumerate(zip(unit_first, run_all))]
    return {"raw": raw, "ctas": len(per), "span_us": round(span, 2), "start_us": st(starts), "alloc_us": st(alloc),
            "ramp_to_first_x_us": st(ramp), "staging_us_total": st(stage), "run_tiles_us": st(run),
            "end_us": st(ends), "run_by_width": {str(b): st(v) for b, v in sorted(by_width.items())}, "prime_us": st(prime), "stage_loop_us": st(stg), "stage_barrier_us": st(bar), "unit_decode_us": st(sub0), "to_barrier_us": st(sub1), "to_first_issue_us": st(sub2), "busy_frac": round(sum(run) / (len(per) * span), 3)}


def main():
    if "--build" in sys.argv:
        build()
        return
    import torch
    import paper_2603_19172_b200.dymoe as d
    d.LIB_PATH = LIB
    import bench
    import synthetic
    mode = sys.argv[1] if len(sys.argv) > 1 else "mixed"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cname = sys.argv[3] if len(sys.argv) > 3 else "mixtral_decode"
    dev = torch.device("cuda", 0)
    cfg = synthetic.CONFIGS[cname].with_tokens(B)
    (layer, _), = bench.build_layer_copies(d, cfg, 1, dev)
    inputs = bench.step_inputs(cfg, 4, dev)
    ws = layer.workspace(B, dev)
    lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
    forced = None if mode == "mixed" else torch.full((cfg.M,), int(mode), dtype=torch.uint8, device=dev)
    L = d.lib()
    buf = (ctypes.c_ulonglong * (2 * 256 * 2 * NEV + 2 * 256 * 8))()
    cnt = (ctypes.c_int * (2 * 256))()
    x, lg, a = inputs[0]
    for _ in range(3):
        layer.forward(x, lg, lad, 20, 32, attn_mass=a, ws=ws, forced_bits=forced)
    torch.cuda.synchronize()
    L.dymoe_dec_trace_read(buf, cnt)
    layer.forward(x, lg, lad, 20, 32, attn_mass=a, ws=ws, forced_bits=forced)
    torch.cuda.synchronize()
    L.dymoe_dec_trace_read(buf, cnt)
    ncta = torch.cuda.get_device_properties(0).multi_processor_count
    out = {"mode": mode, "B": B, "config": cname, "w13": summarise(buf, cnt, 0, ncta), "w2": summarise(buf, cnt, 1, ncta)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
