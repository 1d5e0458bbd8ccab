"""Look-ahead prediction of the next layer's experts (PAPER.md §"Phase-Adaptive
Prefetcher", Eqs. 6-8).

Test infrastructure only (see oracle/__init__.py).

Eq. 6: g_hat_i^(l+1) = Softmax(h_i^(l) W_g^(l+1)) -- the next layer's gate applied to the current
hidden state.  s_i = TopK_k(g_hat_i) are the experts token i is likely to activate.
Eq. 7 (prefill): c_e = sum_i 1[e in s_i]; prefetch the top-t experts by c_e.
Eq. 8 (decode):  prefetch TopK_t(g_hat) of the current token.

Readings:
  P1  Eq. 6 states the product, not an evaluation order: the oracle evaluates it exactly (fp64
      on bf16 operands; see gate_logits).  TopK over g_hat equals TopK over the logits (softmax
      is monotonic), ties to the lower index (R11) -- the routing oracle (route.route) is reused
      as is, on the exact logits.  A device evaluates the product in some fp32 order; the tests
      accept its logits within the fp32 error bound of the exact value and its selections
      wherever they are a valid top-k under that bound (several results are correct there).
  P2  Eq. 7's membership test uses k_route (SPEC S:263 open question; "likely-to-be-activated").
      Experts with c_e = 0 are never requested; requests are ordered by (c_e desc, index asc),
      priority = c_e.
  P3  Eq. 8 is stated for one token.  For a decode batch of B tokens the predicted demand is the
      decode importance of the predicted gate (Eq. 3 reading R10: B = 1 ranks by the logit row,
      B > 1 by sum_b g_hat[b]); requests are its top-t, priority = that value.
"""

import numpy as np

from . import importance as _imp
from . import route as _route


def gate_logits(h, w_gate):
    """Eq. 6's gate product h W_g^(l+1)T, evaluated exactly (reading P1).

    Eq. 6 fixes no summation order and no precision, so the oracle computes the value itself:
    every product of two bf16 values is exact in fp64 (8-bit x 8-bit significands) and the fp64
    sum of Hd <= 2^16 of them is within Hd * 2^-53 * sum|h w| of the exact sum -- 2^-29 of the unit
    fp32 bound the tests apply to the GPU's fp32 evaluation, i.e. exact for every comparison here.

    h float32 [T, Hd] (bf16 values), w_gate float32 [M, Hd] (bf16 values) -> float64 [T, M].
    """
    h = np.asarray(h, dtype=np.float64)
    w = np.asarray(w_gate, dtype=np.float64)
    return h @ w.T


def _top_t(values, t, drop_zero):
    order = sorted(range(len(values)), key=lambda j: (-float(values[j]), j))
    out = [j for j in order if not (drop_zero and values[j] <= 0)][:t]
    return out


def prefill_prefetch(logits_next, k_route, t):
    """Eq. 7 with P2.  Returns (experts list, priorities list, counts int64 [M])."""
    idx, _, _ = _route.route(logits_next, k_route)
    M = np.asarray(logits_next).shape[1]
    counts = np.zeros(M, dtype=np.int64)
    for row in idx:
        for e in row:
            counts[int(e)] += 1
    ex = _top_t(counts, t, drop_zero=True)
    return ex, [int(counts[e]) for e in ex], counts


def decode_prefetch(logits_next, t):
    """Eq. 8 with P3.  Returns (experts list, priorities list, predicted demand [M])."""
    logits_next = np.asarray(logits_next, dtype=np.float32)
    _, _, p = _route.route(logits_next, 1)
    demand = _imp.decode_importance(logits_next, p)
    ex = _top_t(demand, t, drop_zero=False)
    return ex, [float(demand[e]) for e in ex], demand


def predict_next(phase, h, w_gate_next, k_route, t):
    """The whole look-ahead step: Eq. 6 then Eq. 7 (phase 'prefill') or Eq. 8 ('decode')."""
    logits = gate_logits(h, w_gate_next)
    if phase == "prefill":
        ex, pr, _ = prefill_prefetch(logits, k_route, t)
    else:
        ex, pr, _ = decode_prefetch(logits, t)
    return dict(logits=logits, experts=ex, priority=pr)
