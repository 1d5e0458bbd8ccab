"""Pins for oracle.schedule (Eq. 4-5; tiers P:312)."""
import itertools
import math

import numpy as np
import pytest

from oracle import schedule as sc
from golden_util import load_golden

SPEC = load_golden("spec_examples.json")
TAB = load_golden("schedule_tables.json")


@pytest.mark.parametrize("L", [2, 5, 8, 32, 33])
@pytest.mark.parametrize("lam", [0.0, 0.25, 0.5, 0.8, 1.0])
def test_closed_forms(L, lam):
    assert sc.retention_ratio(0, L, lam) == pytest.approx(1.0, abs=1e-15)
    assert sc.retention_ratio(L - 1, L, lam) == pytest.approx(lam, abs=1e-12)
    if (L - 1) % 2 == 0:
        assert sc.retention_ratio((L - 1) // 2, L, lam) == pytest.approx((1 + lam) / 2, abs=1e-12)
    r = [sc.retention_ratio(l, L, lam) for l in range(L)]
    # terms l and L-1-l cancel the cosine: the layer mean is exactly (1+lam)/2 (reading D6)
    assert sum(r) / L == pytest.approx((1 + lam) / 2, abs=1e-12)
    assert all(a >= b - 1e-15 for a, b in zip(r, r[1:]))           # S:210 non-increasing
    # S:514 acceptance: schedule exact to 1e-12 against the formula typed from P:252
    for l in range(L):
        want = (1 - lam) * (math.cos(math.pi * l / (L - 1)) + 1) / 2 + lam
        assert abs(r[l] - want) < 1e-12


@pytest.mark.parametrize("case", SPEC["retention"])
def test_spec_retention(case):
    assert sc.retention_ratio(case["l"], case["L"], case["lambda"]) == pytest.approx(case["r"], abs=1e-12)


def test_spec_counts_and_single_layer():
    assert math.ceil(0.75 * 8 - 1e-9) == 6                            # S:196 arithmetic
    assert sc.critical_count(0, 32, 0.5, 8) == 8
    assert sc.retention_ratio(0, 1, 0.3) == 1.0                       # S:185 L = 1
    with pytest.raises(ValueError, match="layer"):
        sc.retention_ratio(3, 3, 0.5)


def _expand(tab):
    if "values" in tab:
        return tab["values"]
    return [v for v, n in tab["runs"] for _ in range(n)]


@pytest.mark.parametrize("tab", TAB["tables"])
def test_survey_tables(tab):
    got = [sc.critical_count(l, TAB["L"], tab["lambda"], tab["M"]) for l in range(TAB["L"])]
    assert got == _expand(tab)


def test_fp_noise_case():
    c = TAB["fp_noise_case"]
    assert sc.retention_ratio(c["l"], c["L"], c["lambda"]) * c["M"] > 2.0   # the noise exists
    assert sc.critical_count(c["l"], c["L"], c["lambda"], c["M"]) == c["t"]


def test_ladder_example():
    ex = TAB["ladder_example"]
    lad = sc.Ladder(bits=tuple(ex["bits"]), lambdas=tuple(ex["lambdas"]))
    for l, sizes in ex["per_layer_tier_sizes"].items():
        t = sc.tier_counts(int(l), 32, lad, ex["M"], ex["k_route"])
        got = [t[0], t[1] - t[0], ex["M"] - t[1]]
        assert got == sizes


@pytest.mark.parametrize("case", SPEC["assign"])
def test_spec_assign(case):
    scores = np.array(case["scores"], np.float64)
    M = len(scores)
    # a 2-tier ladder whose t equals case["t"] at l = 0 of L = 1 needs lambda only via M:
    order = sc.rank_experts(scores)
    high = sorted(order[: case["t"]])
    assert high == case["high"]


def test_lambda_one_is_all_high():
    # Table 2 at r = 1.0 equals Table 1's Int4 column (P:367 vs P:421): lambda = 1 => every expert High
    lad = sc.paper_ladder(low_bits=0, lam=1.0)
    rng = np.random.default_rng(0)
    for l in range(32):
        bits, _ = sc.assign_bits(rng.random(8), l, 32, lad, 2)
        assert (bits == 4).all()


def test_clamp_and_paper_literal():
    lad = sc.paper_ladder(low_bits=0, lam=0.0)
    bits, t = sc.assign_bits(np.arange(8, dtype=float), 31, 32, lad, 2)
    assert t == [2] and (bits == 4).sum() == 2                      # clamp to k_route (D8)
    lit = sc.Ladder(bits=(4, 0), lambdas=(0.0,), clamp_to_k=False)
    bits, t = sc.assign_bits(np.arange(8, dtype=float), 31, 32, lit, 2)
    assert t == [0] and (bits == 0).all()                           # paper-literal t = ceil(0) = 0


def _brute_force(importance, sizes, bits_of_tier):
    """Enumerate all bit vectors with the given tier sizes; keep the rank-consistent ones."""
    M = len(importance)
    found = []
    for assign in set(itertools.permutations([i for i, n in enumerate(sizes) for _ in range(n)])):
        ok = True
        for a in range(M):
            for b in range(M):
                # a ranks before b  <=>  (I_a > I_b) or (I_a == I_b and a < b)
                before = importance[a] > importance[b] or (importance[a] == importance[b] and a < b)
                if before and assign[a] > assign[b]:
                    ok = False
        if ok:
            found.append([bits_of_tier[i] for i in assign])
    return found


@pytest.mark.parametrize("seed", range(120))
def test_brute_force_tiny_layers(seed):
    rng = np.random.default_rng(seed)
    M = int(rng.integers(2, 7))
    imp = rng.integers(0, 4, size=M).astype(float)          # many ties on purpose
    lad = sc.Ladder(bits=(8, 4, 2), lambdas=(float(rng.random() * 0.5), 0.5 + float(rng.random() * 0.5)))
    l, L = int(rng.integers(0, 8)), 8
    bits, t = sc.assign_bits(imp, l, L, lad, k_route=1)
    sizes = [t[0], t[1] - t[0], M - t[1]]
    sols = _brute_force(imp, sizes, lad.bits)
    assert len(sols) == 1 and sols[0] == bits.tolist()
    # higher importance never receives fewer bits (BASELINE.json invariant)
    for a in range(M):
        for b in range(M):
            if imp[a] > imp[b]:
                assert bits[a] >= bits[b]


def test_active_mode_and_monotone_in_lambda():
    imp = np.array([5.0, 0, 3, 0, 1, 0, 0, 2])
    active = imp > 0
    lad = sc.Ladder(bits=(4, 2), lambdas=(0.5,), m_active=True)
    bits, t = sc.assign_bits(imp, 31, 32, lad, 2, active)
    assert t == [2]                                           # M_eff = 4 active: ceil(0.5 * 4 - 1e-9) = 2
    assert bits.tolist() == [4, 2, 4, 2, 2, 2, 2, 2]
    bits_total, t_total = sc.assign_bits(imp, 31, 32, sc.paper_ladder(2, 0.5), 2)
    assert t_total == [4] and bits_total.tolist() == [4, 2, 4, 2, 4, 2, 2, 4]
    # S:521-style: the number of High experts never decreases as lambda grows
    prev = -1
    for lam in np.linspace(0, 1, 41):
        n = (sc.assign_bits(imp, 20, 32, sc.paper_ladder(2, float(lam)), 2)[0] == 4).sum()
        assert n >= prev
        prev = n


def test_ladder_validation():
    with pytest.raises(ValueError, match="lambdas"):
        sc.Ladder(bits=(8, 4, 2), lambdas=(0.6, 0.5)).validate()
    with pytest.raises(ValueError, match="bits"):
        sc.Ladder(bits=(4, 3), lambdas=(0.5,)).validate()
    with pytest.raises(ValueError, match="lambdas"):
        sc.Ladder(bits=(4, 2), lambdas=(1.5,)).validate()
