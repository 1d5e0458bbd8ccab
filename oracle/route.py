"""Top-k gating (router), SURVEY §8c O1.

Test infrastructure only (see oracle/__init__.py).

Paper: "the router selects a small subset of experts per token"; the gate
is ``Softmax(h W_g)`` (Eq. 6) and ``g_j`` is "the routing weight assigned to
expert E_j" (Eq. 3).  The gate GEMM is outside the path (reading R19): the
caller supplies fp32 logits.

Readings: experts are ordered by (logit descending, index
ascending) -- lower index wins ties (R11), and -0.0 equals +0.0 because the
comparison is numeric; the k routing weights are the softmax over the k selected
logits (identical to the full softmax renormalised over the top-k); ``p`` is the
softmax over all M experts (used by decode importance, Eq. 3).
"""

import math

import numpy as np


def topk_order(row, k):
    """First ``k`` expert indices of ``sorted(range(M), key=(-logit, index))``."""
    M = len(row)
    order = sorted(range(M), key=lambda j: (-float(row[j]), j))
    return order[:k]


def route(logits, k):
    """Route every token.

    logits: float32 [T, M] (float64 is taken as is: the exact router logits of a gate product,
    reading P1).  Returns (topk_idx int32 [T,k], topk_w float64 [T,k],
    probs float64 [T,M]).  Softmaxes are evaluated in float64 with the max
    subtracted (mathematically identical to the plain definition).
    """
    logits = np.asarray(logits)
    if logits.dtype != np.float64:
        logits = logits.astype(np.float32)
    T, M = logits.shape
    if not (1 <= k <= M):
        raise ValueError("k: must satisfy 1 <= k <= M")
    idx = np.zeros((T, k), dtype=np.int32)
    w = np.zeros((T, k), dtype=np.float64)
    p = np.zeros((T, M), dtype=np.float64)
    for t in range(T):
        row = [float(v) for v in logits[t]]
        sel = topk_order(row, k)
        idx[t] = sel
        lmax = max(row)
        e_all = [math.exp(v - lmax) for v in row]
        z_all = sum(e_all)
        p[t] = [e / z_all for e in e_all]
        e_sel = [math.exp(row[j] - lmax) for j in sel]
        z_sel = sum(e_sel)
        w[t] = [e / z_sel for e in e_sel]
    return idx, w, p
