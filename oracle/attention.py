"""Heavy-hitter attention mass (Eq. 1 input; reading R1): the
mass token j receives from the causal softmax attention of head h,

    a[h][j] = sum_{i >= j} softmax_j'( s[h][i][j'] )[j],   s[h][i][j] = scale * q[h][i] . k[h][j],
    the softmax over j' <= i (causal),

evaluated in float64 straight from the definition (row max subtracted).  Test infrastructure only
(see oracle/__init__.py).
"""
import numpy as np


def attention_mass(q, k, scale):
    """q, k float [H, T, d] -> a float64 [H, T]."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    H, T, _ = q.shape
    a = np.zeros((H, T), dtype=np.float64)
    for h in range(H):
        s = scale * (q[h] @ k[h].T)                  # [T queries, T keys]
        for i in range(T):
            row = s[i, :i + 1]
            p = np.exp(row - row.max())
            a[h, :i + 1] += p / p.sum()
    return a


def harmonic_tail(T):
    """Closed form for q = 0 (uniform causal attention): a[j] = sum_{i=j}^{T-1} 1/(i+1)."""
    inv = 1.0 / np.arange(1, T + 1, dtype=np.float64)
    return np.cumsum(inv[::-1])[::-1]
