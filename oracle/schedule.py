"""Depth-aware precision scheduling, SURVEY §8c O3.

Test infrastructure only (see oracle/__init__.py).

PAPER.md §4.3:
  Eq. 4  r(l) = (1 - lambda) * (cos(pi * l / (L - 1)) + 1) / 2 + lambda
  Eq. 5  t_l = ceil(r(l) * M)
  P:312              configs "4/2" (critical Int4, sub-critical Int2) and "4/0"
                     (sub-critical experts bypassed)
The t_l experts with the highest importance are critical.

Readings:
  D5  M_eff = M (TOTAL, default) or the number of experts with >= 1 routed token
      in this step (ACTIVE).
  D7  t = ceil(r * M_eff - 1e-9), evaluated in float64 (absorbs cos() noise such
      as r*M = 2.000000000000001).
  D8  optional clamp t_1 >= min(k_route, M_eff) (default on; the SPEC's choice).
  D9  ladder of n tiers b_1 > ... > b_n (b_n may be 0 = skip) with thresholds
      lambda_1 <= ... <= lambda_{n-1}; t_k = ceil(r(l; lambda_k) * M_eff); ranks
      [0, t_1) get b_1, [t_1, t_2) get b_2, ..., the rest b_n.  n = 2 is exactly the
      paper's High/Low scheme.
  D11 experts ranked by (importance descending, index ascending).
  L = 1 => r = 1.
"""

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

VALID_BITS = (16, 8, 4, 2, 0)


@dataclass(frozen=True)
class Ladder:
    """Tier ladder: bits per tier (high to low) and the n-1 lambda thresholds."""
    bits: Sequence[int]
    lambdas: Sequence[float]
    clamp_to_k: bool = True
    m_active: bool = False       # D5: False = TOTAL, True = ACTIVE
    renorm_on_skip: bool = True  # D12 (used by the combine step)

    def validate(self):
        if len(self.bits) < 1 or len(self.lambdas) != len(self.bits) - 1:
            raise ValueError("ladder.lambdas: need len(bits)-1 thresholds")
        for b in self.bits:
            if b not in VALID_BITS:
                raise ValueError("ladder.bits: each width must be one of 16, 8, 4, 2, 0")
        for a, b in zip(self.bits, self.bits[1:]):
            if not a > b:
                raise ValueError("ladder.bits: widths must be strictly decreasing")
        for lam in self.lambdas:
            if not (0.0 <= lam <= 1.0):
                raise ValueError("ladder.lambdas: each lambda must lie in [0, 1]")
        for a, b in zip(self.lambdas, self.lambdas[1:]):
            if a > b:
                raise ValueError("ladder.lambdas: must be non-decreasing")


def paper_ladder(low_bits=2, lam=0.5):
    """The paper's "4/2" (low_bits=2) or "4/0" (low_bits=0) configuration."""
    return Ladder(bits=(4, low_bits), lambdas=(lam,))


def retention_ratio(l, L, lam):
    """Eq. 4 in float64 with math.cos; L = 1 gives 1."""
    if L < 1 or not (0 <= l < L):
        raise ValueError("layer: must satisfy 0 <= layer < num_layers")
    if L == 1:
        return 1.0
    return (1.0 - lam) * (math.cos(math.pi * l / (L - 1)) + 1.0) / 2.0 + lam


def critical_count(l, L, lam, M):
    """Eq. 5 with reading D7: ceil(r(l) * M - 1e-9)."""
    return int(math.ceil(retention_ratio(l, L, lam) * M - 1e-9))


def tier_counts(l, L, ladder, M_eff, k_route):
    """Cumulative tier boundaries t_1 <= ... <= t_{n-1} (each <= M_eff)."""
    ladder.validate()
    t = []
    for i, lam in enumerate(ladder.lambdas):
        c = critical_count(l, L, lam, M_eff)
        if i == 0 and ladder.clamp_to_k:
            c = max(c, min(k_route, M_eff))
        if t:
            c = max(c, t[-1])
        t.append(min(c, M_eff))
    return t


def rank_experts(importance, candidates=None):
    """Experts sorted by (importance desc, index asc) -- D11."""
    M = len(importance)
    cand = range(M) if candidates is None else candidates
    return sorted(cand, key=lambda j: (-float(importance[j]), j))


def assign_bits(importance, l, L, ladder, k_route, active=None):
    """Bit width per expert for layer l.  Returns (bits uint8[M], counts list).

    importance: length-M vector (int counts for prefill, floats for decode).
    active: bool[M] (needed only when ladder.m_active) -- experts with a routed token.
    """
    M = len(importance)
    if ladder.m_active:
        if active is None:
            raise ValueError("active_mask: required in ACTIVE mode")
        cand = [j for j in range(M) if active[j]]
    else:
        cand = list(range(M))
    M_eff = len(cand)
    counts = tier_counts(l, L, ladder, M_eff, k_route)
    bits = np.full(M, ladder.bits[-1], dtype=np.uint8)
    for rank, j in enumerate(rank_experts(importance, cand)):
        tier = len(counts)
        for i, c in enumerate(counts):
            if rank < c:
                tier = i
                break
        bits[j] = ladder.bits[tier]
    return bits, counts


__all__ = ["Ladder", "paper_ladder", "retention_ratio", "critical_count", "tier_counts",
           "rank_experts", "assign_bits", "VALID_BITS", "field"]
