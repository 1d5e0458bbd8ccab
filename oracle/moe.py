"""Permutation, SwiGLU expert FFN, combine and the whole MoE layer, SURVEY §8c O5-O8.

Test infrastructure only (see oracle/__init__.py).

Paper: the MoE layer replaces the dense FFN by M experts and a gate that selects a
few experts per token; the executor runs every expert "on a unified
mixed-precision weight set" (P:203 step 4) whose widths come from the scheduler
(P:250-259).  A "0-bit" (skipped) expert costs no compute.

Readings:
  D18 expert FFN = SwiGLU with Mixtral naming: y = W2 (silu(W1 x) * (W3 x)).
  D17 weights enter the FFN dequantized (quant.dequant); BF16-tier experts use
      the bf16 masters directly.
  O6  h = RNE_bf16(silu(A) * B) -- the one activation rounding point (the input of
      the second bf16 matmul); everything else in float64.
  D12 when a routed expert is skipped, the remaining routing weights of that token
      are renormalised over the executed experts (default; flag); a token whose
      routed experts are all skipped outputs 0.
  O8  permutation = stable order of (token, slot) pairs by expert id; pairs routed
      to a skipped expert are dropped.  Expert parallel: by (destination rank,
      expert, token, slot) with expert e on rank floor(e * P / M).
"""

import numpy as np

from .bf16 import round_bf16
from . import quant as _q
from . import route as _route
from . import importance as _imp
from . import schedule as _sched


def silu(a):
    """silu(a) = a / (1 + exp(-a)) in float64."""
    a = np.asarray(a, dtype=np.float64)
    return a / (1.0 + np.exp(-a))


def permute(topk_idx, bits, M):
    """O8.  Returns dict(expert_off int32[M+1], perm_token, perm_slot int32[R], inv_row int32[T,k])."""
    topk_idx = np.asarray(topk_idx)
    T, k = topk_idx.shape
    rows = []
    for e in range(M):
        if int(bits[e]) == 0:
            continue
        for t in range(T):
            for s in range(k):
                if int(topk_idx[t, s]) == e:
                    rows.append((e, t, s))
    off = np.zeros(M + 1, dtype=np.int32)
    for e, _, _ in rows:
        off[e + 1] += 1
    off = np.cumsum(off).astype(np.int32)
    perm_token = np.asarray([t for _, t, _ in rows], dtype=np.int32)
    perm_slot = np.asarray([s for _, _, s in rows], dtype=np.int32)
    inv_row = np.full((T, k), -1, dtype=np.int32)
    for r, (_, t, s) in enumerate(rows):
        inv_row[t, s] = r
    return dict(expert_off=off, perm_token=perm_token, perm_slot=perm_slot, inv_row=inv_row)


def expert_weights(expert, bits, group=128):
    """Dequantized (W1, W3, W2) in float64 for the given width.

    expert: dict with bf16 masters 'w1','w3' [F,Hd], 'w2' [Hd,F] (float32 holding bf16
    values) and, per quantized width b, 'q{b}' = dict(w1=(codes,s,z), w3=..., w2=...).
    If 'q{b}' is absent the masters are quantized here with quant.quantize.
    """
    if bits == 16:
        return tuple(np.asarray(expert[n], dtype=np.float64) for n in ("w1", "w3", "w2"))
    key = "q%d" % bits
    out = []
    for n in ("w1", "w3", "w2"):
        K = expert[n].shape[1]
        if key in expert:
            codes, s, z = expert[key][n]
        else:
            codes, s, z = _q.quantize(expert[n], bits, group)
        out.append(_q.dequant(codes, s, z, bits, K, group))
    return tuple(out)


def ffn(x_rows, W1, W3, W2):
    """O6 for one expert: x_rows float64 [R, Hd] -> y float64 [R, Hd]."""
    A = x_rows @ W1.T
    Bm = x_rows @ W3.T
    h = round_bf16(silu(A) * Bm)
    return h @ W2.T


def combine(y_perm, inv_row, topk_w, renorm=True):
    """O7: y[t] = sum_slot w'[t,slot] * y_perm[inv_row[t,slot]] in slot order (float64)."""
    inv_row = np.asarray(inv_row)
    T, k = inv_row.shape
    Hd = y_perm.shape[1] if y_perm.ndim == 2 and y_perm.shape[0] else None
    if Hd is None:
        raise ValueError("y_perm: need the hidden size")
    y = np.zeros((T, Hd), dtype=np.float64)
    for t in range(T):
        live = [s for s in range(k) if inv_row[t, s] >= 0]
        if not live:
            continue
        denom = sum(float(topk_w[t, s]) for s in live) if renorm else 1.0
        for s in live:
            y[t] += (float(topk_w[t, s]) / denom) * y_perm[inv_row[t, s]]
    return y


def moe_forward(x, logits, experts, l, L, ladder, k_route, phase="decode",
                attn_mass=None, k_tokens=None, group=128, forced_bits=None):
    """The whole layer (SURVEY §3 CS3/CS4 order): route -> score -> assign -> permute
    -> FFN per expert on its assigned width -> combine.

    x: float32 [T, Hd] (bf16 values); logits float32 [T, M]; experts: list of expert
    dicts (see expert_weights).  forced_bits overrides the schedule (uniform sweeps).
    Returns dict with y (float64 [T,Hd]) and every intermediate.
    """
    x = np.asarray(x, dtype=np.float32)
    T, Hd = x.shape
    M = len(experts)
    idx, w, p = _route.route(logits, k_route)
    heavy = None
    if phase == "prefill":
        I, heavy, _ = _imp.score_prefill(attn_mass, idx, M, k_tokens)
    else:
        I = _imp.decode_importance(logits, p)
    active = np.zeros(M, dtype=bool)
    active[np.unique(idx)] = True
    if forced_bits is not None:
        bits = np.asarray(forced_bits, dtype=np.uint8)
        counts = None
    else:
        bits, counts = _sched.assign_bits(I, l, L, ladder, k_route, active)
    perm = permute(idx, bits, M)
    R = len(perm["perm_token"])
    y_perm = np.zeros((max(R, 1), Hd), dtype=np.float64)
    off = perm["expert_off"]
    for e in range(M):
        lo, hi = int(off[e]), int(off[e + 1])
        if hi == lo:
            continue
        W1, W3, W2 = expert_weights(experts[e], int(bits[e]), group)
        xr = x[perm["perm_token"][lo:hi]].astype(np.float64)
        y_perm[lo:hi] = ffn(xr, W1, W3, W2)
    y = combine(y_perm, perm["inv_row"], w, ladder.renorm_on_skip)
    return dict(y=y, topk_idx=idx, topk_w=w, probs=p, importance=I, heavy=heavy,
                bits=bits, counts=counts, y_perm=y_perm[:R], **perm)


def ep_owner(e, M, P):
    """Expert e lives on rank floor(e * P / M) (contiguous blocks)."""
    return (e * P) // M


def ep_dispatch_order(topk_idx, bits, M, P):
    """O8 for expert parallelism: list of (dest_rank, expert, token, slot), sorted."""
    topk_idx = np.asarray(topk_idx)
    T, k = topk_idx.shape
    rows = [(ep_owner(int(topk_idx[t, s]), M, P), int(topk_idx[t, s]), t, s)
            for t in range(T) for s in range(k) if int(bits[int(topk_idx[t, s])]) != 0]
    return sorted(rows)


def ep_simulate(x, topk_idx, topk_w, bits, experts, M, P, group=128, renorm=True):
    """Expert-parallel layer simulated on one host: every rank computes only its
    experts' rows (dispatched in ep_dispatch_order), results return to the source
    and are combined as in `combine`.  Must equal the unsharded layer.
    """
    x = np.asarray(x, dtype=np.float32)
    T, Hd = x.shape
    k = topk_idx.shape[1]
    rows = ep_dispatch_order(topk_idx, bits, M, P)
    inv_row = np.full((T, k), -1, dtype=np.int32)
    y_rows = np.zeros((max(len(rows), 1), Hd), dtype=np.float64)
    for rank in range(P):
        mine = [(r, e, t, s) for r, (dst, e, t, s) in enumerate(rows) if dst == rank]
        for e in sorted({e for _, e, _, _ in mine}):
            rs = [(r, t, s) for r, ee, t, s in mine if ee == e]
            W1, W3, W2 = expert_weights(experts[e], int(bits[e]), group)
            xr = x[[t for _, t, _ in rs]].astype(np.float64)
            ye = ffn(xr, W1, W3, W2)
            for i, (r, t, s) in enumerate(rs):
                y_rows[r] = ye[i]
                inv_row[t, s] = r
    return combine(y_rows, inv_row, topk_w, renorm)
