"""The C pool (dymoe_pool_*, host-side policy in libdymoe) against oracle/pool.py on the SPEC
examples and on random operation sequences: outcomes, served widths, offsets, eviction lists,
errors and snapshots must agree exactly (integer work).  Runs on CPU: the pool never touches the
device."""
import numpy as np
import pytest

from oracle import pool as op


def D():
    import paper_2603_19172_b200.dymoe as d
    d.lib()
    return d


def test_spec_examples_through_the_abi():
    d = D()
    p = d.Pool(100)
    assert p.lookup(0, 0, 4)[0] == d.POOL_MISS
    p.insert(0, 1, 4, 40)
    p.insert(0, 2, 4, 40)
    off, ev = p.insert(0, 3, 4, 40)
    assert ev == [(0, 1)] and off == 0
    assert p.lookup(0, 2, 8)[0] == d.POOL_PROMOTE
    off, ev = p.insert(0, 2, 8, 60)
    assert ev == [] and off == 40 and p.used() == 100
    assert p.lookup(0, 2, 4)[:2] == (d.POOL_HIT, 8)             # conservative reuse
    p.pin(0, 2)
    with pytest.raises(d.DymoeError) as ei:
        p.insert(5, 5, 16, 70)
    assert ei.value.args[0].startswith("dymoe error 7")          # capacity; nothing changed
    assert [k for k, _ in p.snapshot()] == [(0, 3), (0, 2)]
    with pytest.raises(d.DymoeError, match="pinned, cannot replace"):
        p.insert(0, 2, 16, 10)
    p.unpin(0, 2)
    with pytest.raises(d.DymoeError, match="not pinned"):
        p.unpin(0, 2)
    with pytest.raises(d.DymoeError, match="bits: must be"):
        p.lookup(0, 0, 3)


@pytest.mark.parametrize("seed,cap", [(0, 200), (1, 97), (2, 1000)])
def test_random_sequences_match_the_oracle(seed, cap):
    d = D()
    rng = np.random.default_rng(seed)
    sizes = {16: 64, 8: 33, 4: 17, 2: 9}
    ref = op.Pool(cap)
    p = d.Pool(cap)
    for _ in range(4000):
        key = (int(rng.integers(0, 3)), int(rng.integers(0, 6)))
        b = int(rng.choice([2, 4, 8, 16]))
        r = rng.random()
        if r < 0.55:
            o_ref = ref.lookup(key, b)
            o_got = p.lookup(key[0], key[1], b)
            assert o_got == o_ref
            if o_ref[0] != op.HIT:
                try:
                    exp = ref.insert(key, b, sizes[b])
                except op.CapacityError:
                    exp = "capacity"
                except op.PoolError:
                    exp = "invalid"
                try:
                    got = p.insert(key[0], key[1], b, sizes[b])
                except d.DymoeError as e:
                    got = "capacity" if e.args[0].startswith("dymoe error 7") else "invalid"
                assert got == exp if isinstance(exp, str) else got == (exp[0], list(exp[1]))
        elif r < 0.75 and ref.entries:
            k = list(ref.entries)[int(rng.integers(0, len(ref.entries)))]
            ref.pin(k)
            p.pin(*k)
        else:
            pinned = [k for k, e in ref.entries.items() if e["pins"] > 0]
            if pinned:
                k = pinned[int(rng.integers(0, len(pinned)))]
                ref.unpin(k)
                p.unpin(*k)
        assert p.used() == ref.used()
    snap = p.snapshot()
    rs = ref.snapshot()
    assert [k for k, _ in snap] == [k for k, _ in rs]
    for (_, a), (_, b) in zip(snap, rs):
        assert (a["bits"], a["nbytes"], a["offset"], a["pins"]) == (b["bits"], b["nbytes"], b["offset"], b["pins"])
