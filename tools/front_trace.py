"""Phase timeline of the decode front kernel (measurement tool, not product code).

  python tools/front_trace.py --build      # here: libdymoe with -DDYMOE_FRONT_TRACE -> tools/trace/
  python tools/front_trace.py [B] [config] # on the GPU: one layer step, thread-0 stamps per phase

Stamps (csrc/kernels/route_score.cu FRONT_TR): 0 start, 1 route done, 2 importance done,
3 bits assigned, 4 probs copied, 5 permute done, 6 end (outputs written)."""
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tools", "trace")
LIB = os.path.join(OUT, "libdymoe_fronttrace.so")


def build():
    from paper_2603_19172_b200 import build as b
    b.build()
    os.makedirs(OUT, exist_ok=True)
    obj = os.path.join(OUT, "route_score_trace.o")
    src = os.path.join(b.CSRC, "kernels", "route_score.cu")
    subprocess.check_call([b.NVCC] + b.ARCH + b.FLAGS + ["-DDYMOE_FRONT_TRACE", "-c", src, "-o", obj])
    objs = [o for o in glob.glob(os.path.join(b.OBJ, "*.o")) if "route_score" not in o] + [obj]
    subprocess.check_call([b.NVCC] + b.ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static"])
    print("built", LIB)


def main():
    if "--build" in sys.argv:
        build()
        return
    import torch
    import paper_2603_19172_b200.dymoe as d
    d.LIB_PATH = LIB
    import bench
    import synthetic
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    cname = sys.argv[2] if len(sys.argv) > 2 else "mixtral_decode"
    dev = torch.device("cuda", 0)
    cfg = synthetic.CONFIGS[cname].with_tokens(B)
    (layer, _), = bench.build_layer_copies(d, cfg, 1, dev)
    inputs = bench.step_inputs(cfg, 4, dev)
    ws = layer.workspace(B, dev)
    lad = d.make_ladder(bench.LADDER_BITS, bench.LADDER_LAMBDAS)
    buf = (ctypes.c_ulonglong * 16)()
    tot = [0.0] * 6
    n = 20
    for i in range(n + 3):
        x, lg, a = inputs[i % 4]
        layer.forward(x, lg, lad, 20, 32, attn_mass=a, ws=ws)
        torch.cuda.synchronize()
        d.lib().dymoe_front_trace_read(buf)
        if i >= 3:
            for q in range(6):
                tot[q] += (buf[q + 1] - buf[q]) / 1e3
    names = ["route", "importance", "assign", "probs copy", "permute", "outputs"]
    print(cname, "B", B, " ".join("%s %.2f" % (nm, t / n) for nm, t in zip(names, tot)),
          "total %.2f us" % (sum(tot) / n))


if __name__ == "__main__":
    main()
