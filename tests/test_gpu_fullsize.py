"""GPU parity at the benchmark's full sizes, in the launch configuration bench.py times.

The whole layer runs on the GPU exactly as bench.py runs it (BASELINE.json configs[1]: Mixtral
decode at B = 1, 2, 4, 8; configs[2]: Mixtral prefill, T = 2048; configs[3]: the fine-grained
64-expert top-6 layer; configs[4]: a Mixtral-shaped stack).  The oracle checks, on the same seeded
inputs:
  * everything cheap at full size, exactly: routing indices, importance (prefill: exact integer
    counts), bit assignment (decode B > 1: a valid assignment on near-tied gate sums,
    tests/validity.py), the expert-sorted permutation;
  * outputs: decode -- EVERY token through EVERY active expert; prefill -- for every 256-row
    pair tile of every expert its first, middle and last row (so every tile the grouped GEMM
    schedules, the experts' tails and both K halves of the split W2 GEMM are covered); the
    fine-grained layer -- every token at T = 384, a sample at T = 2048.  For each (expert, width)
    a worker process regenerates the expert's master, quantizes it with the oracle (codes /
    scales / zeros compared with the GPU's by digest), dequantizes (D17) and runs the SwiGLU FFN
    in fp64; y[t] must be within the FFN tolerance (north_star: 2e-3 of max|y_ref|).
"""
import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import synthetic
from fullsize_worker import digest, expert_rows
from oracle import importance as o_imp, moe as o_moe, route as o_route, schedule as o_sched
from oracle import stack as o_stack
from validity import check_bits, check_logits, check_topk, decode_importance_tol, gate_logit_bound

pytestmark = pytest.mark.gpu

FFN_TOL = 2e-3
LADDER = ((8, 4, 2), (0.25, 0.5))   # bench.py's ladder
NUM_LAYERS = 32
SEED = 11
_POOL = None


def D():
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    return d


def pool():
    global _POOL
    if _POOL is None:
        n = max(1, min(8, (os.cpu_count() or 2) // 2))
        _POOL = cf.ProcessPoolExecutor(n, mp_context=mp.get_context("spawn"))
    return _POOL


def rel_err(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max()
    return float(np.abs(y - ref).max() / (den if den > 0 else 1.0))


_LAYERS = {}


def gpu_layer(cfg, seed=SEED, widths=(8, 4, 2)):
    """The layer on the GPU from CPU-generated bf16 masters (the workers regenerate the same)."""
    key = (cfg.M, cfg.hidden, cfg.ffn, seed)      # the weights depend on the shape and seed only
    if key not in _LAYERS:
        _LAYERS.clear()
        torch.cuda.empty_cache()
        d = D()
        ex = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, seed)]
        d.quantize_experts(ex, widths)
        _LAYERS[key] = (d.MoELayer(ex, cfg.k, cfg.hidden, cfg.ffn), ex)
    return _LAYERS[key]


def gpu_digests(ex, e, b):
    if b == 16:
        return None
    return {n: digest(*(a.cpu().numpy() for a in ex[e]["q%d" % b][n])) for n in ("w1", "w3", "w2")}


def oracle_outputs(cfg, seed, ex_gpu, x_np, idx, w, bits, tokens):
    """y_ref[t] for the given tokens: one worker task per (expert, width) with the rows of the
    tokens routed to it; the combine (D12) over the token's live slots."""
    tokens = sorted(set(int(t) for t in tokens))
    jobs = {}
    for t in tokens:
        for s in range(idx.shape[1]):
            e = int(idx[t, s])
            if bits[e]:
                jobs.setdefault(e, []).append(t)
    futs = {e: pool().submit(expert_rows, cfg, seed, e, int(bits[e]), x_np[ts].astype(np.float32),
                             gpu_digests(ex_gpu, e, int(bits[e])))
            for e, ts in jobs.items()}
    rows = {}
    for e, f in futs.items():
        y_e, same = f.result()
        assert all(same.values()), ("packed codes / scales / zeros differ", e, int(bits[e]), same)
        for t, r in zip(jobs[e], y_e):
            rows[(t, e)] = r
    out = {}
    for t in tokens:
        k = idx.shape[1]
        y_rows = np.zeros((k, x_np.shape[1]))
        inv = np.full((1, k), -1, np.int32)
        for s in range(k):
            e = int(idx[t, s])
            if bits[e]:
                y_rows[s] = rows[(t, e)]
                inv[0, s] = s
        out[t] = o_moe.combine(y_rows, inv, w[t:t + 1], True)[0]
    return out


def run_case(cfg_name, T, phase, layer, pick, seed=SEED, input_seed=4):
    d = D()
    cfg = synthetic.CONFIGS[cfg_name].with_tokens(T)
    L, ex = gpu_layer(synthetic.CONFIGS[cfg_name], seed)
    x, lg, a = synthetic.layer_inputs(cfg, input_seed)
    ph = d.DYMOE_PREFILL if phase == "prefill" else d.DYMOE_DECODE
    lad = d.make_ladder(*LADDER)
    y, ws = L.forward(x.cuda(), lg.cuda(), lad, layer, NUM_LAYERS, phase=ph,
                      attn_mass=a.cuda() if ph == d.DYMOE_PREFILL else None)
    torch.cuda.synchronize()
    assert L.check_status(T, ws)[0] == 0
    v = L.views(T, ws)
    # exact parts at full size
    lg_np, a_np = lg.numpy(), a.numpy()
    idx, w, p = o_route.route(lg_np, cfg.k)
    if phase == "prefill":
        I, _, _ = o_imp.score_prefill(a_np, idx, cfg.M, None)
    else:
        I = o_imp.decode_importance(lg_np, p)
    active = np.zeros(cfg.M, bool)
    active[np.unique(idx)] = True
    bits, _ = o_sched.assign_bits(I, layer, NUM_LAYERS, o_sched.Ladder(bits=LADDER[0], lambdas=LADDER[1]),
                                  cfg.k, active)
    assert np.array_equal(v["topk_idx"].cpu().numpy(), idx)
    if phase == "prefill":
        assert np.array_equal(v["importance"].cpu().numpy(), I.astype(np.float32))
    gbits = v["bits"].cpu().numpy()
    check_bits(gbits, bits, I, 0 if (phase == "prefill" or T == 1) else decode_importance_tol(T))
    bits = gbits                    # equal, or a valid assignment on a near-tie
    perm = o_moe.permute(idx, bits, cfg.M)
    assert np.array_equal(v["expert_off"].cpu().numpy(), perm["expert_off"])
    assert np.array_equal(v["inv_row"].cpu().numpy(), perm["inv_row"])
    tokens = pick(perm, T)
    x_np = x.float().numpy()
    ref = oracle_outputs(cfg, seed, ex, x_np, idx, w, bits, tokens)
    y_np = y.cpu().numpy()
    for t, r in ref.items():
        assert rel_err(y_np[t], r) <= FFN_TOL, (t, rel_err(y_np[t], r))
    return bits, perm, len(ref)


def every_token(perm, T):
    return range(T)


def tile_rows(perm, T, tile=256):
    """first, middle and last row of every 256-row pair tile of every expert -> their tokens"""
    off, pt = perm["expert_off"], perm["perm_token"]
    rows = set()
    for e in range(len(off) - 1):
        lo, hi = int(off[e]), int(off[e + 1])
        for t0 in range(lo, hi, tile):
            t1 = min(hi, t0 + tile)
            rows.update({t0, (t0 + t1 - 1) // 2, t1 - 1})
    return sorted(int(pt[r]) for r in rows)


@pytest.mark.parametrize("B", [1, 2, 4, 8])
def test_mixtral_decode_full(B):
    """configs[1]: Mixtral-8x7B layer, decode B tokens (bench.py's default B = 8 and its B = 1
    sub-line), layer 20: every token through every active expert."""
    bits, perm, n = run_case("mixtral_decode", B, "decode", 20, every_token, input_seed=4 + B)
    assert n == B


def test_mixtral_prefill_full():
    """configs[2]: Mixtral-8x7B layer, prefill T = 2048 (bench's prefill line), layer 24 (Eq. 4-5:
    3 x Int8, 2 x Int4, 3 x Int2): every pair tile of every expert sampled at its first / middle /
    last row (multi-tile experts, ragged tails, the split-K W2 GEMM)."""
    bits, perm, n = run_case("mixtral_prefill", 2048, "prefill", 24, tile_rows)
    rows = np.diff(perm["expert_off"])
    assert (rows > 256).any() and len(set(int(b) for b in bits[rows > 0])) >= 2


@pytest.mark.parametrize("phase,T,pick", [("decode", 16, every_token), ("prefill", 384, every_token),
                                          ("prefill", 2048, tile_rows)])
def test_finegrained_layer(phase, T, pick):
    """configs[3] shape (64 experts, top-6, hidden 2048, ffn 1408) on one GPU; at T = 2048 the
    small-expert GEMV split and the grouped GEMM both run."""
    run_case("finegrained", T, phase, 9, pick)


def test_mixtral_stack_two_layers_teacher_forced():
    """configs[4]'s structure at full Mixtral shape: a 2-layer stack (RMSNorm -> router -> MoE ->
    residual, depth schedule over L = 2: layer 0 all Int8, layer 1 at r = lambda), decode B = 8,
    teacher-forced layer by layer against oracle.stack (as tests/test_gpu_stack.py at Hd = 256)."""
    d = D()
    from paper_2603_19172_b200.stack import MoEStack
    cfg = synthetic.CONFIGS["stack"].with_tokens(8)
    L = 2
    layers, exs, gates = [], [], []
    for l in range(L):
        ex = [{n: t.cuda() for n, t in e.items()} for e in synthetic.expert_weights(cfg, 300 + l)]
        d.quantize_experts(ex, (8, 4, 2))
        layers.append(ex)
        gates.append(synthetic.stack_gate(cfg, l, 5))
    st = MoEStack(layers, [(w.cuda(), b.cuda()) for w, b in gates], cfg.k, cfg.hidden, cfg.ffn)
    x0 = synthetic.hidden_states(cfg, 6).cuda()
    lad = d.make_ladder(*LADDER)
    xL, trace = st.forward(x0, lad, phase=d.DYMOE_DECODE, trace=True)
    torch.cuda.synchronize()
    seen = set()
    for l in range(L):
        x_in = trace[l][0].float().cpu().numpy().astype(np.float64)
        u_gpu = trace[l][1].float().cpu().numpy().astype(np.float64)
        u_ref = o_stack.rmsnorm(x_in)
        ulp = np.where(u_ref != 0, 2.0 ** (np.floor(np.log2(np.abs(np.where(u_ref != 0, u_ref, 1)))) - 7), 0)
        assert (np.abs(u_gpu - u_ref) <= ulp).all(), "rmsnorm, layer %d" % l
        wg, beta = gates[l]
        lg_ref = o_stack.router_logits(u_gpu, wg.float().numpy(), beta.numpy())
        check_logits(trace[l][2].cpu().numpy(), lg_ref, gate_logit_bound(u_gpu, wg.float().numpy(), lg_ref))
        idx_gpu = trace[l][4].cpu().numpy()
        near = check_topk(idx_gpu, lg_ref, gate_logit_bound(u_gpu, wg.float().numpy(), lg_ref))
        assert not near.any()          # no ambiguous routing on these seeded inputs
        idx, w, p = o_route.route(lg_ref, cfg.k)
        assert np.array_equal(idx_gpu, idx)
        I = o_imp.decode_importance(lg_ref, p)
        bits_ref, _ = o_sched.assign_bits(I, l, L, o_sched.Ladder(*LADDER), cfg.k)
        bits = trace[l][3].cpu().numpy()
        check_bits(bits, bits_ref, I, decode_importance_tol(8))
        seen.update(int(b) for b in bits)
        ref = oracle_outputs(cfg, 300 + l, layers[l], u_gpu, idx, w, bits, range(8))
        x_out = (trace[l + 1][0] if l + 1 < L else xL).float().cpu().numpy().astype(np.float64)
        for t in range(8):
            y_ref = ref[t]
            full = o_stack.residual(x_in[t], y_ref)
            bound = FFN_TOL * np.abs(y_ref).max() + np.abs(full) * 2.0 ** -7
            assert (np.abs(x_out[t] - full) <= bound).all(), ("stream", l, t)
    assert {8, 4, 2} <= seen
