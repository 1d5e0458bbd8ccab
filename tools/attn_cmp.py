"""Accuracy of dymoe_attention_mass (or of a variant library, ATTN_LIB) against an fp64 torch
evaluation of the definition on two heads: python tools/attn_cmp.py [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_19172_b200.dymoe as d  # noqa: E402

if os.environ.get("ATTN_LIB"):
    d.LIB_PATH = os.environ["ATTN_LIB"]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
H = 32
g = torch.Generator(device="cuda").manual_seed(3)
q = torch.randn(H, T, 128, generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn(H, T, 128, generator=g, device="cuda").to(torch.bfloat16)
out = d.dymoe_attention_mass(q, k)
torch.cuda.synchronize()
s = torch.einsum("htd,hsd->hts", q[:2].double(), k[:2].double()) / 128 ** 0.5
s = s.masked_fill(torch.triu(torch.ones(T, T, dtype=torch.bool, device="cuda"), 1), float("-inf"))
a64 = torch.softmax(s, -1).sum(1)
print(os.path.basename(d.LIB_PATH), "T", T, "max |a - a64| / max a64 = %.3g" %
      float((out[:2].double() - a64).abs().max() / a64.abs().max()))
