"""Phase-adaptive expert importance, SURVEY §8c O2.

Test infrastructure only (see oracle/__init__.py).

Prefill, token-guided (§4.2.1):
  Eq. 1  s_i = (1/H) * sum_h a_i^(h)
  P:223              T_imp = the top-k tokens by s_i
  Eq. 2  I_prefill(E_j) = |{ t_i in Tokens_j : t_i in T_imp }|
Decode, gate-guided (§4.2.2):
  Eq. 3  I_decode(E_j) = g_j

Readings:
  R1  a[h][i] is the attention mass *received* by token i in head h (column sum
      of the head's attention matrix); the caller supplies it as fp32 [H][T].
  R1b The 1/H factor is a positive constant and cannot change the top-k set, so
      the ranking key is S_i = sum_h a[h][i], accumulated in fp32 in head order
      h = 0..H-1 (one rounding per add, never a pairwise/tree sum).
  R3  k_tokens defaults to ceil(0.2 * T).
  R11 ties broken by lower token index.
  R10 decode: B = 1 ranks experts by the token's logit row (order-equivalent to
      g = softmax(logits) and exact); B > 1 sums g over the batch.
"""

import math

import numpy as np


def default_k_tokens(T):
    """R3: ceil(0.2 * T) (integer arithmetic: ceil(T/5))."""
    return (T + 4) // 5


def token_scores(attn_mass):
    """S_i = a[0][i] + a[1][i] + ... + a[H-1][i] in fp32, head order (Eq. 1 up to 1/H)."""
    a = np.asarray(attn_mass, dtype=np.float32)
    H, T = a.shape
    S = a[0].copy()
    for h in range(1, H):
        S = (S + a[h]).astype(np.float32)   # elementwise fp32 add, one rounding each
    return S


def heavy_hitters(S, k_tokens):
    """T_imp: first k_tokens of sorted(range(T), key=(-S_i, i)) (R11)."""
    T = len(S)
    if not (0 <= k_tokens <= T):
        raise ValueError("k_tokens: must satisfy 0 <= k_tokens <= T")
    order = sorted(range(T), key=lambda i: (-float(S[i]), i))
    return np.asarray(order[:k_tokens], dtype=np.int32)


def prefill_importance(heavy, topk_idx, M):
    """Eq. 2: I[j] = number of heavy tokens whose routed set contains expert j."""
    I = np.zeros(M, dtype=np.int64)
    topk_idx = np.asarray(topk_idx)
    for i in heavy:
        for j in topk_idx[i]:
            I[int(j)] += 1
    return I


def decode_importance(logits, probs):
    """Eq. 3.  B == 1: the logit row itself (R10: same order as g, exact).

    B > 1: I[j] = sum_b g[b][j] with g the full softmax (float64 here).
    """
    logits = np.asarray(logits)
    if logits.dtype != np.float64:        # float64 = exact gate-product logits (reading P1)
        logits = logits.astype(np.float32)
    B = logits.shape[0]
    if B == 1:
        return logits[0].astype(np.float64)
    I = np.zeros(logits.shape[1], dtype=np.float64)
    for b in range(B):
        I = I + np.asarray(probs[b], dtype=np.float64)
    return I


def score_prefill(attn_mass, topk_idx, M, k_tokens=None):
    """Full prefill scorer: returns (I int64[M], heavy int32[k_tokens], S fp32[T])."""
    S = token_scores(attn_mass)
    if k_tokens is None or k_tokens == 0:
        k_tokens = default_k_tokens(len(S))
    heavy = heavy_hitters(S, k_tokens)
    return prefill_importance(heavy, topk_idx, M), heavy, S


def mean_head_score(attn_mass):
    """Eq. 1 literally, in float64: (1/H) sum_h a_i^(h).  Used only by pins."""
    a = np.asarray(attn_mass, dtype=np.float64)
    return a.sum(axis=0) / a.shape[0]


__all__ = [
    "default_k_tokens", "token_scores", "heavy_hitters", "prefill_importance",
    "decode_importance", "score_prefill", "mean_head_score", "math",
]
