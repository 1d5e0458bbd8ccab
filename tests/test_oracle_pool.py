"""Pins for oracle/pool.py: the SPEC's worked examples, the paper's three rules
(P:305-308), textbook-LRU equivalence and invariants on random operation sequences."""
import collections

import numpy as np
import pytest

from oracle import pool as op


def test_spec_lookup_table():
    p = op.Pool(1000)
    assert p.lookup((0, 0), 4)[0] == op.MISS                      # cold miss
    p.insert((3, 1), 4, 100)
    assert p.lookup((3, 1), 8)[0] == op.PROMOTE                   # Precision Promotion
    p.insert((3, 2), 8, 100)
    out, served, _ = p.lookup((3, 2), 4)
    assert out == op.HIT and served == 8                          # Conservative Reuse
    assert p.lookup((3, 1), 4)[:2] == (op.HIT, 4)


def test_spec_insert_examples():
    p = op.Pool(100)
    p.insert("A", 4, 40)
    p.insert("B", 4, 40)
    off, ev = p.insert("C", 4, 40)
    assert ev == ["A"] and off == 0                               # LRU victim, first fit
    # replacing a key's format frees its old range first (No Duplication)
    off2, ev2 = p.insert("B", 8, 60)
    assert ev2 == [] and p.entries["B"]["bits"] == 8 and off2 == 40 and p.used() == 100
    # a pinned entry blocks eviction
    q = op.Pool(100)
    q.insert("A", 8, 60)
    q.pin("A")
    with pytest.raises(op.CapacityError):
        q.insert("C", 4, 50)
    assert set(q.entries) == {"A"}                                # nothing changed
    q.unpin("A")
    assert q.insert("C", 4, 50)[1] == ["A"]


def test_pin_counts():
    p = op.Pool(100)
    p.insert("A", 4, 60)
    p.pin("A")
    p.pin("A")
    p.unpin("A")
    with pytest.raises(op.CapacityError):
        p.insert("B", 4, 50)                                      # still pinned once
    p.unpin("A")
    assert p.insert("B", 4, 50)[1] == ["A"]
    with pytest.raises(op.PoolError):
        p.unpin("B")
    with pytest.raises(op.PoolError):
        p.pin("zz")


def test_textbook_lru_equivalence():
    """Equal-size single-precision entries: identical to an N-slot LRU (OrderedDict)."""
    rng = np.random.default_rng(0)
    p = op.Pool(5 * 10)
    ref = collections.OrderedDict()
    for _ in range(2000):
        k = int(rng.integers(0, 12))
        hit = p.lookup(k, 4)[0] == op.HIT
        assert hit == (k in ref)
        if hit:
            ref.move_to_end(k)
        else:
            _, ev = p.insert(k, 4, 10)
            exp = []
            if len(ref) == 5:
                exp = [ref.popitem(last=False)[0]]
            ref[k] = True
            assert ev == exp
    assert [k for k, _ in p.snapshot()] == list(ref)


def test_random_sequences_keep_invariants():
    rng = np.random.default_rng(1)
    sizes = {16: 64, 8: 33, 4: 17, 2: 9}
    p = op.Pool(200)
    for _ in range(3000):
        key = (int(rng.integers(0, 3)), int(rng.integers(0, 6)))
        b = int(rng.choice([2, 4, 8, 16]))
        r = rng.random()
        if r < 0.6:
            out, served, _ = p.lookup(key, b)
            if out == op.HIT:
                assert served >= b
            else:
                if key in p.entries:
                    assert p.entries[key]["bits"] < b and out == op.PROMOTE
                try:
                    p.insert(key, b, sizes[b])
                except (op.CapacityError, op.PoolError):
                    pass
        elif r < 0.8 and p.entries:
            k = list(p.entries)[int(rng.integers(0, len(p.entries)))]
            p.pin(k)
        elif p.entries:
            pinned = [k for k, e in p.entries.items() if e["pins"] > 0]
            if pinned:
                p.unpin(pinned[int(rng.integers(0, len(pinned)))])
        # invariants: budget, disjoint in-range placements, free list = complement
        assert p.used() <= p.capacity
        spans = sorted((e["offset"], e["nbytes"]) for e in p.entries.values()) + list(p.free)
        spans.sort()
        pos = 0
        for o, s in spans:
            assert o == pos and s > 0
            pos = o + s
        assert pos == p.capacity
