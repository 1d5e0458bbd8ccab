"""Byte-budgeted mixed-precision expert pool (PAPER.md §"Mixed-Precision Cache
Management"; "cache" module), as a plain reference model.

Test infrastructure only (see oracle/__init__.py).

Paper rules, restated for bit widths (reading P4: "High" / "Low" generalise to the
order 16 > 8 > 4 > 2 of the resident formats):
  * No Duplication: an expert is stored in one format only;
  * Precision Promotion: a request for b with a narrower format cached is a miss -- load b and
    evict the narrower one;
  * Conservative Reuse: a request for b with a wider (or equal) format cached is served by it.
An LRU policy chooses victims ("extend the standard LRU cache").

SPEC decision table and behaviour, with the readings of DESIGN.md §3:
  lookup(key, b): absent -> MISS; cached b' >= b -> HIT (served b', recency refreshed);
                  cached b' < b -> PROMOTE (a miss; no recency change).
  insert(key, b, nbytes): an existing entry of the key is replaced (its space freed first;
      replacing a pinned entry is an error -- P5); then least-recently-used unpinned entries are
      evicted until a contiguous free range of nbytes exists; placement is first fit (lowest
      offset) in a free list with coalescing (P6: the pool is an arena of device memory, so the
      model includes addresses).  If the entry cannot fit even with every unpinned entry evicted,
      nothing changes and CapacityError is raised.
  pin / unpin: counted; eviction skips pinned entries; pin of an absent key and
      unpin below zero are errors.
  snapshot: entries from least to most recently used.
Skip-tier experts (b = 0) never enter the pool.
"""


class CapacityError(Exception):
    pass


class PoolError(Exception):
    pass


HIT, MISS, PROMOTE = 0, 1, 2


class Pool:
    def __init__(self, capacity):
        if capacity <= 0:
            raise PoolError("capacity: must be > 0")
        self.capacity = int(capacity)
        self.entries = {}            # key -> dict(bits, nbytes, offset, last_use, pins)
        self.free = [(0, self.capacity)]   # sorted, coalesced (offset, size)
        self.clock = 0

    # ---------------------------------------------------------------- free list
    @staticmethod
    def _release(free, off, size):
        free = sorted(free + [(off, size)])
        merged = []
        for o, s in free:
            if merged and merged[-1][0] + merged[-1][1] == o:
                merged[-1] = (merged[-1][0], merged[-1][1] + s)
            else:
                merged.append((o, s))
        return merged

    @staticmethod
    def _first_fit(free, size):
        for o, s in free:
            if s >= size:
                return o
        return None

    @staticmethod
    def _take(free, off, size):
        out = []
        for o, s in free:
            if o <= off < o + s:
                if off > o:
                    out.append((o, off - o))
                if off + size < o + s:
                    out.append((off + size, o + s - off - size))
            else:
                out.append((o, s))
        return out

    # ---------------------------------------------------------------- operations
    def lookup(self, key, bits):
        if bits not in (2, 4, 8, 16):
            raise PoolError("bits: must be 2, 4, 8 or 16")
        e = self.entries.get(key)
        if e is None:
            return MISS, bits, None
        if e["bits"] >= bits:
            self.clock += 1
            e["last_use"] = self.clock
            return HIT, e["bits"], e["offset"]
        return PROMOTE, bits, None

    def insert(self, key, bits, nbytes):
        """Returns (offset, evicted keys in eviction order)."""
        if bits not in (2, 4, 8, 16):
            raise PoolError("bits: must be 2, 4, 8 or 16")
        if nbytes <= 0:
            raise PoolError("nbytes: must be > 0")
        old = self.entries.get(key)
        if old is not None and old["pins"] > 0:
            raise PoolError("key is pinned: cannot replace")
        # plan on copies; commit only if the entry fits
        free = list(self.free)
        live = dict(self.entries)
        evicted = []
        if old is not None:
            free = self._release(free, old["offset"], old["nbytes"])
            del live[key]
        off = self._first_fit(free, nbytes)
        victims = sorted((e["last_use"], k) for k, e in live.items() if e["pins"] == 0)
        vi = 0
        while off is None:
            if vi == len(victims):
                raise CapacityError("cannot fit %d bytes" % nbytes)
            _, k = victims[vi]
            vi += 1
            free = self._release(free, live[k]["offset"], live[k]["nbytes"])
            del live[k]
            evicted.append(k)
            off = self._first_fit(free, nbytes)
        free = self._take(free, off, nbytes)
        self.clock += 1
        live[key] = dict(bits=bits, nbytes=nbytes, offset=off, last_use=self.clock, pins=0)
        self.entries, self.free = live, free
        return off, evicted

    def pin(self, key):
        if key not in self.entries:
            raise PoolError("key not cached")
        self.entries[key]["pins"] += 1

    def unpin(self, key):
        if key not in self.entries:
            raise PoolError("key not cached")
        if self.entries[key]["pins"] == 0:
            raise PoolError("key not pinned")
        self.entries[key]["pins"] -= 1

    def snapshot(self):
        return [(k, dict(e)) for k, e in sorted(self.entries.items(), key=lambda kv: kv[1]["last_use"])]

    def used(self):
        return sum(e["nbytes"] for e in self.entries.values())
