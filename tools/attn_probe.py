"""Times dymoe_attention_mass (f3) alone at Mixtral-shaped attention sizes (H = 32, d = 128);
usage: python tools/attn_probe.py [T ...]  -> one line per size (us, TFLOP/s, fraction of the
measured bf16 burst peak)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_19172_b200.dymoe as d  # noqa: E402

if os.environ.get("ATTN_LIB"):   # a variant library built by tools/attn_trace.py --build NAME ...
    d.LIB_PATH = os.environ["ATTN_LIB"]


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1642.7}
    g = torch.Generator(device="cuda").manual_seed(1)
    sizes = [int(a) for a in sys.argv[1:]] or [2048, 4096]
    for T in sizes:
        H = 32
        q = torch.randn(H, T, 128, generator=g, device="cuda").to(torch.bfloat16)
        k = torch.randn(H, T, 128, generator=g, device="cuda").to(torch.bfloat16)
        for _ in range(3):
            d.dymoe_attention_mass(q, k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            d.dymoe_attention_mass(q, k)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        fl = 2 * 2 * T * T * 128 * H / 2
        tf = fl / us / 1e6
        print(json.dumps({"H": H, "T": T, "us": round(us, 1), "TFLOP/s": round(tf, 1),
                          "frac_bf16_burst": round(tf / peaks["bf16_tflops"], 3)}))


if __name__ == "__main__":
    main()
