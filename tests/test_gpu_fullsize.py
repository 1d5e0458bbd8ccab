"""GPU parity at the benchmark's full sizes, in the launch configuration bench.py times.

The whole layer runs on the GPU exactly as bench.py runs it (BASELINE.json configs[1]: Mixtral
decode, B = 8; configs[2]: Mixtral prefill, T = 2048; configs[3]: the fine-grained C4 layer).
The oracle checks, on the same seeded inputs:
  * everything cheap at full size, exactly: routing indices, per-expert importance (prefill:
    exact integer counts), bit assignment, the expert-sorted permutation;
  * sampled outputs one by one: for a few tokens the oracle quantizes the token's experts itself
    (codes / scales / zeros compared bit-exactly with the GPU's), dequantizes (D17), evaluates the
    SwiGLU FFN in fp64 and combines (D12); y[t] must match within the FFN tolerance.
"""
import numpy as np
import pytest
import torch

import synthetic
from oracle import importance as o_imp, moe as o_moe, quant as o_quant, route as o_route
from oracle import schedule as o_sched

pytestmark = pytest.mark.gpu

FFN_TOL = 2e-3
LADDER = ((8, 4, 2), (0.25, 0.5))   # bench.py's ladder
NUM_LAYERS = 32


def D():
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    return d


def rel_err(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max()
    return float(np.abs(y - ref).max() / (den if den > 0 else 1.0))


def oracle_token(x_row, t, idx, w, bits, ex_cpu, gpu_ex, renorm=True):
    """y[t] by the oracle for one token, quantizing (and cross-checking) its experts."""
    k = idx.shape[1]
    rows = np.zeros((k, x_row.shape[0]), np.float64)
    inv = np.full((1, k), -1, np.int32)
    for s in range(k):
        e = int(idx[t, s])
        b = int(bits[e])
        if b == 0:
            continue
        exp = {n: ex_cpu[e][n] for n in ("w1", "w3", "w2")}
        if b != 16:
            q = {}
            for n in ("w1", "w3", "w2"):
                codes, sc, z = o_quant.quantize(exp[n], b)
                gc, gs, gz = (a.cpu().numpy() for a in gpu_ex[e]["q%d" % b][n])
                assert np.array_equal(codes.view(np.uint32), gc.view(np.uint32)), (e, b, n)
                assert np.array_equal(sc.view(np.uint32), gs.view(np.uint32)), (e, b, n)
                assert np.array_equal(z, gz), (e, b, n)
                q[n] = (codes, sc, z)
            exp["q%d" % b] = q
        W1, W3, W2 = o_moe.expert_weights(exp, b)
        rows[s] = o_moe.ffn(x_row[None].astype(np.float64), W1, W3, W2)[0]
        inv[0, s] = s
    return o_moe.combine(rows, inv, w[t:t + 1], renorm)[0]


def run_case(cfg_name, T, phase, layer, tokens, experts_seed=11, input_seed=4):
    d = D()
    cfg = synthetic.CONFIGS[cfg_name].with_tokens(T)
    dev = torch.device("cuda")
    gpu_ex = [{n: t.to(dev) for n, t in e.items()} for e in synthetic.expert_weights(cfg, experts_seed, dev)]
    d.quantize_experts(gpu_ex, (8, 4, 2))
    L = d.MoELayer(gpu_ex, cfg.k, cfg.hidden, cfg.ffn)
    x, lg, a = synthetic.layer_inputs(cfg, input_seed, dev)
    ph = d.DYMOE_PREFILL if phase == "prefill" else d.DYMOE_DECODE
    lad = d.make_ladder(*LADDER)
    y, ws = L.forward(x, lg, lad, layer, NUM_LAYERS, phase=ph, attn_mass=a if ph == d.DYMOE_PREFILL else None)
    torch.cuda.synchronize()
    assert L.check_status(T, ws)[0] == 0
    v = L.views(T, ws)
    # exact parts at full size
    lg_np, a_np = lg.cpu().numpy(), a.cpu().numpy()
    idx, w, p = o_route.route(lg_np, cfg.k)
    if phase == "prefill":
        I, _, _ = o_imp.score_prefill(a_np, idx, cfg.M, None)
    else:
        I = o_imp.decode_importance(lg_np, p)
    active = np.zeros(cfg.M, bool)
    active[np.unique(idx)] = True
    bits, _ = o_sched.assign_bits(I, layer, NUM_LAYERS, o_sched.Ladder(bits=LADDER[0], lambdas=LADDER[1]),
                                  cfg.k, active)
    perm = o_moe.permute(idx, bits, cfg.M)
    assert np.array_equal(v["topk_idx"].cpu().numpy(), idx)
    if phase == "prefill":
        assert np.array_equal(v["importance"].cpu().numpy(), I.astype(np.float32))
    assert np.array_equal(v["bits"].cpu().numpy(), bits)
    assert np.array_equal(v["expert_off"].cpu().numpy(), perm["expert_off"])
    assert np.array_equal(v["inv_row"].cpu().numpy(), perm["inv_row"])
    # sampled outputs
    ex_cpu = {}
    for t in tokens:
        for e in idx[t]:
            e = int(e)
            if e not in ex_cpu:
                ex_cpu[e] = {n: gpu_ex[e][n].float().cpu().numpy() for n in ("w1", "w3", "w2")}
    x_np = x.float().cpu().numpy()
    y_np = y.cpu().numpy()
    for t in tokens:
        ref = oracle_token(x_np[t], t, idx, w, bits, ex_cpu, gpu_ex)
        assert rel_err(y_np[t], ref) <= FFN_TOL, (t, rel_err(y_np[t], ref))
    return bits, perm


def test_mixtral_decode_full():
    """configs[1]: Mixtral-8x7B layer, decode B = 8 (bench.py's default workload), layer 20."""
    run_case("mixtral_decode", 8, "decode", 20, tokens=[0])


def test_mixtral_prefill_full():
    """configs[2]: Mixtral-8x7B layer, prefill T = 2048 (bench --workload prefill), layer 3 (all
    three ladder tiers present); sampled tokens from both ends of the sequence."""
    run_case("mixtral_prefill", 2048, "prefill", 3, tokens=[5, 2047])


@pytest.mark.parametrize("phase,T", [("decode", 16), ("prefill", 384)])
def test_finegrained_layer(phase, T):
    """configs[3] shape (64 experts, top-6, hidden 2048, ffn 1408) on one GPU."""
    run_case("finegrained", T, phase, 9, tokens=[0, T - 1])
