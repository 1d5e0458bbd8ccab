"""Validity rules for the places where several results are correct (SURVEY §8(c) parity note,
DESIGN.md §4): an fp32 evaluation of a quantity the oracle computes exactly (the Eq. 6 gate
product, the Eq. 3 decode gate sums) can only be held to an error bound, so a selection made
from it (top-k experts, tiers of Eq. 5) is exact wherever the margin exceeds that bound and
otherwise only has to be *a* valid selection under it.

Nothing here computes the method: the helpers take the oracle's exact values and the GPU's
outputs and check the GPU's outputs are consistent with the exact values within the bound.
"""
import numpy as np

U32 = 2.0 ** -24          # unit roundoff of fp32


def gamma(n):
    """Higham's gamma_n = n u / (1 - n u): |fl(sum) - sum| <= gamma_depth * sum |terms| for any
    evaluation whose every partial sum passes through at most `depth` roundings."""
    return n * U32 / (1.0 - n * U32)


def gate_logit_bound(h, w, exact_plus_bias=None):
    """Error bound of dymoe_gate_logits / dymoe_predict_next's logits (include/dymoe.h: fp32
    accumulation of depth <= Hd/32 + 5 over exact bf16 products, then one rounding of the bias
    add): gamma_depth * |h| |w|^T (+ u * (|exact + bias| + that bound) with a bias).
    h [T][Hd], w [M][Hd] (bf16 values) -> float64 [T][M]."""
    h = np.abs(np.asarray(h, np.float64))
    w = np.abs(np.asarray(w, np.float64))
    depth = h.shape[1] // 32 + 5
    b = gamma(depth) * (h @ w.T)
    if exact_plus_bias is not None:
        b = b + U32 * (np.abs(exact_plus_bias) + b)
    return b


def check_logits(gpu, exact, bound):
    gpu = np.asarray(gpu, np.float64)
    err = np.abs(gpu - exact)
    assert (err <= bound).all(), "logit error %.3e over bound %.3e" % (
        (err - bound).max(), bound.ravel()[np.argmax(err - bound)])


def check_topk(idx_gpu, exact, bound):
    """idx_gpu [T][k]: each row must be a valid top-k of the exact row under the bound (every
    selected expert within 2 bounds of every unselected one, in order within the selection up to
    the bound).  Returns the boolean mask of tokens whose exact top-k is ambiguous under the
    bound (on all other tokens validity forces the oracle's selection exactly)."""
    idx_gpu = np.asarray(idx_gpu)
    T, k = idx_gpu.shape
    M = exact.shape[1]
    near = np.zeros(T, bool)
    for t in range(T):
        sel = [int(j) for j in idx_gpu[t]]
        assert len(set(sel)) == k, (t, sel)
        rest = [j for j in range(M) if j not in sel]
        lo = min(exact[t, j] + bound[t, j] for j in sel)
        if rest:
            hi = max(exact[t, j] - bound[t, j] for j in rest)
            assert lo >= hi, ("invalid top-k", t, sel)
        for a, b in zip(sel, sel[1:]):
            assert exact[t, a] + bound[t, a] >= exact[t, b] - bound[t, b], ("order", t, sel)
        order = sorted(range(M), key=lambda j: (-exact[t, j], j))
        if k < M:
            kk, nx = order[k - 1], order[k]
            near[t] = exact[t, kk] - bound[t, kk] <= exact[t, nx] + bound[t, nx]
    return near


def check_bits(bits_gpu, bits_ref, importance, tol, active=None):
    """Eq. 5 tiers on importances the GPU evaluates to within `tol` (decode B > 1: fp32 sums of
    the gate probabilities).  The tier sizes come from the host's fp64 Eq. 4-5 arithmetic, so the
    multiset of widths must equal the oracle's; within the active set a higher width may never
    go to an expert whose exact importance is more than `tol` below a lower-width one's.  With
    tol = 0 (exact importances: counts, the B = 1 logit row) the assignment must equal the
    oracle's.  Returns True when it equals the oracle's assignment."""
    bits_gpu = np.asarray(bits_gpu).astype(np.int64)
    bits_ref = np.asarray(bits_ref).astype(np.int64)
    if tol == 0:
        assert np.array_equal(bits_gpu, bits_ref), (bits_gpu, bits_ref)
        return True
    assert sorted(bits_gpu.tolist()) == sorted(bits_ref.tolist()), (bits_gpu, bits_ref)
    I = np.asarray(importance, np.float64)
    M = len(I)
    act = np.ones(M, bool) if active is None else np.asarray(active, bool)
    if active is not None:
        assert np.array_equal(bits_gpu[~act], bits_ref[~act])
    for j in range(M):
        for jj in range(M):
            if act[j] and act[jj] and bits_gpu[j] > bits_gpu[jj]:
                assert I[j] >= I[jj] - tol, ("rank-inconsistent", j, jj, I[j], I[jj])
    return bool(np.array_equal(bits_gpu, bits_ref))


def decode_importance_tol(B):
    """|I_gpu - I_exact| for the decode gate sums (fp32 softmax rows summed over B tokens):
    the parity bar of the decode scorer (<= 1e-6 B, test_gpu_parity::test_score_decode), doubled
    for a pair of experts."""
    return 2e-6 * max(B, 1)
