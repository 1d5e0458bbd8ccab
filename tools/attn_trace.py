"""Timeline of one CTA of the f3 attention-mass kernels (measurement tool, not product code).

  python tools/attn_trace.py --build        # here: libdymoe with -DDYMOE_ATTN_TRACE -> tools/trace/
  python tools/attn_trace.py --build NAME -DX=1 ...   # a variant library (tools/attn_probe.py: ATTN_LIB)
  python tools/attn_trace.py [T]            # on the GPU: run H = 32, T, print the timeline summary

Roles of CTA 0 (csrc/kernels/attn_mass.cu DYMOE_TR): 0 = MMA issuer (1 before the TMEM-empty
wait, 2 before the B-full wait, 3 after it, 4 after the commit), 1 / 2 = epilogue warps 2 and 17
(11 before the TMEM-full wait, 12 after it, 13 after tcgen05.wait::ld, 14 item done, 15 after the
item's combine barrier); 100 / 101 = start of pass 1 / pass 2.
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
LIB = os.path.join(OUT, "libdymoe_trace.so")


def build(name="trace", defines=("-DDYMOE_ATTN_TRACE",)):
    """libdymoe with attn_mass.cu compiled with extra defines -> tools/trace/libdymoe_<name>.so"""
    from paper_2603_19172_b200 import build as b
    b.build()
    os.makedirs(OUT, exist_ok=True)
    obj = os.path.join(OUT, "attn_mass_%s.o" % name)
    lib = os.path.join(OUT, "libdymoe_%s.so" % name)
    src = os.path.join(b.CSRC, "kernels", "attn_mass.cu")
    subprocess.check_call([b.NVCC] + b.ARCH + b.FLAGS + list(defines) + ["-c", src, "-o", obj])
    objs = [o for o in glob.glob(os.path.join(b.OBJ, "*.o")) if "attn_mass" not in o] + [obj]
    subprocess.check_call([b.NVCC] + b.ARCH + ["-shared", "-o", lib] + objs + ["-cudart", "static"])
    print("built", lib)


def main():
    if "--build" in sys.argv:   # --build [name -DX=1 ...]
        rest = sys.argv[sys.argv.index("--build") + 1:]
        if rest:
            build(rest[0], rest[1:])
        else:
            build()
        return
    import torch
    import paper_2603_19172_b200.dymoe as d
    d.LIB_PATH = os.environ.get("ATTN_LIB") or LIB
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    H = 32
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn(H, T, 128, generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn(H, T, 128, generator=g, device="cuda").to(torch.bfloat16)
    L = d.lib()
    buf = (ctypes.c_ulonglong * (6 * 4096))()
    cnt = (ctypes.c_int * 6)()
    for _ in range(3):
        d.dymoe_attention_mass(q, k)
    torch.cuda.synchronize()
    L.dymoe_attn_trace_read(buf, cnt)   # clears the counters
    d.dymoe_attention_mass(q, k)
    torch.cuda.synchronize()
    L.dymoe_attn_trace_read(buf, cnt)
    cta = (ctypes.c_ulonglong * (2 * 160 * 3))()
    L.dymoe_attn_trace_cta(cta)
    grid = min(148, H * ((T + 127) // 128))
    for ps in (0, 1):   # COLS = 0: pass 1, 1: pass 2
        rows = [[cta[(ps * 160 + c) * 3 + k] for k in range(3)] for c in range(grid)]
        e0 = min(r[0] for r in rows)
        print("pass %d: entry spread %.2f us, setup (mean) %.2f us, end: min %.2f max %.2f us after "
              "first entry" % (ps + 1, (max(r[0] for r in rows) - e0) / 1e3,
                               sum(r[1] - r[0] for r in rows) / grid / 1e3,
                               (min(r[2] for r in rows) - e0) / 1e3, (max(r[2] for r in rows) - e0) / 1e3))
    roles = []
    for r in range(6):
        n = min(cnt[r], 2048)
        roles.append([(buf[r * 4096 + 2 * i], buf[r * 4096 + 2 * i + 1]) for i in range(n)])
    t0 = min(ev[0][1] for ev in roles if ev)
    summary = {"T": T, "counts": list(cnt)}
    for r, evs in enumerate(roles):
        gaps = {}
        for (e0, c0), (e1, c1) in zip(evs, evs[1:]):
            key = "%d->%d" % (e0, e1)
            gaps.setdefault(key, []).append(c1 - c0)
        summary["role%d" % r] = {k: {"n": len(v), "sum": sum(v), "mean": round(sum(v) / len(v), 1)}
                                  for k, v in sorted(gaps.items())}
        summary["role%d_span" % r] = (evs[-1][1] - evs[0][1]) if evs else 0
        summary["role%d_first" % r] = [(e, c - t0) for e, c in evs[:40]]
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
