"""Process-pool worker of tests/test_gpu_fullsize.py (test infrastructure only): the oracle's
output rows of ONE expert at ONE width for the given token rows, at full Mixtral / fine-grained
size.  The worker regenerates the expert's bf16 master from its seed on the CPU (the test builds
the GPU layer from the same CPU-generated masters), quantizes it with the oracle, checks the
GPU's packed codes / scales / zeros against the oracle's by digest, dequantizes (D17) and
evaluates the SwiGLU FFN in fp64 (O6).  Running experts in parallel processes keeps the
full-size parity tests within minutes."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(a.tobytes())
    return h.hexdigest()


def expert_rows(cfg, seed, e, b, x_rows, gpu_digests):
    """-> (y [n][Hd] fp64, {matrix: codes/scales/zeros equal}).  cfg: synthetic.MoEConfig."""
    import numpy as np
    import torch
    import synthetic
    torch.set_num_threads(max(1, (os.cpu_count() or 8) // 8))
    from oracle import moe as o_moe, quant as o_quant
    ex = synthetic.expert_weights(cfg, seed, experts=[e])[0]
    exp = {n: ex[n].float().numpy() for n in ("w1", "w3", "w2")}
    same = {}
    if b != 16:
        q = {}
        for n in ("w1", "w3", "w2"):
            codes, sc, z = o_quant.quantize(exp[n], b)
            same[n] = digest(codes.view(np.uint32), sc.view(np.uint32), z) == gpu_digests[n]
            q[n] = (codes, sc, z)
        exp["q%d" % b] = q
    W1, W3, W2 = o_moe.expert_weights(exp, b)
    return o_moe.ffn(np.asarray(x_rows, np.float64), W1, W3, W2), same
