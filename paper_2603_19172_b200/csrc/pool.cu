// Mixed-precision expert pool: host-side policy over a caller-owned arena.
// PAPER.md P:303-309 (No Duplication, Precision Promotion, Conservative Reuse, LRU), SPEC
// S:299-383; readings P4-P6.  Mirrors oracle/pool.py operation for operation
// (tests/test_pool_abi.py compares outcomes, offsets, evictions and snapshots on random
// sequences); the two share no code.
#include <algorithm>
#include <map>
#include <new>
#include <utility>
#include <vector>

#include "dymoe_internal.cuh"

struct dymoe_pool {
  struct Entry {
    int bits;
    size_t bytes, offset;
    unsigned long long last_use;
    int pins;
  };
  using Key = std::pair<int, int>;   // (layer, expert)
  size_t capacity = 0;
  std::map<Key, Entry> entries;
  std::vector<std::pair<size_t, size_t>> free_list;   // sorted, coalesced (offset, size)
  unsigned long long clock = 0;
};

namespace {

using FreeList = std::vector<std::pair<size_t, size_t>>;

FreeList release(FreeList f, size_t off, size_t size) {
  f.emplace_back(off, size);
  std::sort(f.begin(), f.end());
  FreeList m;
  for (const auto& r : f) {
    if (!m.empty() && m.back().first + m.back().second == r.first) m.back().second += r.second;
    else m.push_back(r);
  }
  return m;
}
bool first_fit(const FreeList& f, size_t size, size_t* off) {
  for (const auto& r : f)
    if (r.second >= size) {
      *off = r.first;
      return true;
    }
  return false;
}
FreeList take(const FreeList& f, size_t off, size_t size) {
  FreeList out;
  for (const auto& r : f) {
    if (r.first <= off && off < r.first + r.second) {
      if (off > r.first) out.emplace_back(r.first, off - r.first);
      if (off + size < r.first + r.second) out.emplace_back(off + size, r.first + r.second - off - size);
    } else {
      out.push_back(r);
    }
  }
  return out;
}
bool valid_bits(int b) { return b == 2 || b == 4 || b == 8 || b == 16; }

}  // namespace

using dymoe::set_error;

extern "C" {

int dymoe_pool_create(size_t capacity, dymoe_pool** out) {
  if (!out) return set_error(DYMOE_ERR_INVALID, "out: must not be NULL");
  *out = nullptr;
  if (capacity == 0) return set_error(DYMOE_ERR_INVALID, "capacity: must be > 0");
  dymoe_pool* p = new (std::nothrow) dymoe_pool();
  if (!p) return set_error(DYMOE_ERR_INVALID, "out of host memory");
  p->capacity = capacity;
  p->free_list.emplace_back(0, capacity);
  *out = p;
  dymoe::clear_error();
  return DYMOE_OK;
}

int dymoe_pool_destroy(dymoe_pool* pool) {
  delete pool;
  dymoe::clear_error();
  return DYMOE_OK;
}

int dymoe_pool_lookup(dymoe_pool* pool, int layer, int expert, int bits, int* outcome,
                      int* served_bits, size_t* offset) {
  if (!pool) return set_error(DYMOE_ERR_INVALID, "pool: must not be NULL");
  if (!outcome || !served_bits) return set_error(DYMOE_ERR_INVALID, "outcome/served_bits: must not be NULL");
  if (!valid_bits(bits)) return set_error(DYMOE_ERR_INVALID, "bits: must be 2, 4, 8 or 16");
  auto it = pool->entries.find({layer, expert});
  if (it == pool->entries.end()) {
    *outcome = DYMOE_POOL_MISS;
    *served_bits = bits;
  } else if (it->second.bits >= bits) {
    it->second.last_use = ++pool->clock;
    *outcome = DYMOE_POOL_HIT;
    *served_bits = it->second.bits;
    if (offset) *offset = it->second.offset;
  } else {
    *outcome = DYMOE_POOL_PROMOTE;
    *served_bits = bits;
  }
  dymoe::clear_error();
  return DYMOE_OK;
}

int dymoe_pool_insert(dymoe_pool* pool, int layer, int expert, int bits, size_t bytes,
                      size_t* offset, int32_t* evicted, int max_evicted, int* n_evicted) {
  if (!pool) return set_error(DYMOE_ERR_INVALID, "pool: must not be NULL");
  if (!offset || !n_evicted) return set_error(DYMOE_ERR_INVALID, "offset/n_evicted: must not be NULL");
  if (!valid_bits(bits)) return set_error(DYMOE_ERR_INVALID, "bits: must be 2, 4, 8 or 16");
  if (bytes == 0) return set_error(DYMOE_ERR_INVALID, "bytes: must be > 0");
  const dymoe_pool::Key key{layer, expert};
  auto old = pool->entries.find(key);
  if (old != pool->entries.end() && old->second.pins > 0)
    return set_error(DYMOE_ERR_INVALID, "(layer %d, expert %d): pinned, cannot replace", layer, expert);
  // plan on copies, commit only if the entry fits
  FreeList f = pool->free_list;
  std::map<dymoe_pool::Key, dymoe_pool::Entry> live = pool->entries;
  if (old != pool->entries.end()) {
    f = release(f, old->second.offset, old->second.bytes);
    live.erase(key);
  }
  std::vector<std::pair<unsigned long long, dymoe_pool::Key>> victims;
  for (const auto& kv : live)
    if (kv.second.pins == 0) victims.emplace_back(kv.second.last_use, kv.first);
  std::sort(victims.begin(), victims.end());
  std::vector<dymoe_pool::Key> ev;
  size_t off = 0;
  size_t vi = 0;
  while (!first_fit(f, bytes, &off)) {
    if (vi == victims.size())
      return set_error(DYMOE_ERR_CAPACITY, "bytes: %zu cannot fit (capacity %zu, pinned entries stay)",
                       bytes, pool->capacity);
    const auto k = victims[vi++].second;
    f = release(f, live[k].offset, live[k].bytes);
    live.erase(k);
    ev.push_back(k);
  }
  f = take(f, off, bytes);
  live[key] = dymoe_pool::Entry{bits, bytes, off, ++pool->clock, 0};
  pool->entries.swap(live);
  pool->free_list.swap(f);
  *offset = off;
  *n_evicted = (int)ev.size();
  if (evicted)
    for (int i = 0; i < (int)ev.size() && i < max_evicted; ++i) {
      evicted[2 * i] = ev[i].first;
      evicted[2 * i + 1] = ev[i].second;
    }
  dymoe::clear_error();
  return DYMOE_OK;
}

int dymoe_pool_pin(dymoe_pool* pool, int layer, int expert) {
  if (!pool) return set_error(DYMOE_ERR_INVALID, "pool: must not be NULL");
  auto it = pool->entries.find({layer, expert});
  if (it == pool->entries.end())
    return set_error(DYMOE_ERR_INVALID, "(layer %d, expert %d): not cached", layer, expert);
  ++it->second.pins;
  dymoe::clear_error();
  return DYMOE_OK;
}

int dymoe_pool_unpin(dymoe_pool* pool, int layer, int expert) {
  if (!pool) return set_error(DYMOE_ERR_INVALID, "pool: must not be NULL");
  auto it = pool->entries.find({layer, expert});
  if (it == pool->entries.end())
    return set_error(DYMOE_ERR_INVALID, "(layer %d, expert %d): not cached", layer, expert);
  if (it->second.pins == 0)
    return set_error(DYMOE_ERR_INVALID, "(layer %d, expert %d): not pinned", layer, expert);
  --it->second.pins;
  dymoe::clear_error();
  return DYMOE_OK;
}

int dymoe_pool_snapshot(const dymoe_pool* pool, dymoe_pool_entry* out, int max, int* n) {
  if (!pool) return set_error(DYMOE_ERR_INVALID, "pool: must not be NULL");
  if (!n) return set_error(DYMOE_ERR_INVALID, "n: must not be NULL");
  std::vector<std::pair<unsigned long long, dymoe_pool::Key>> order;
  for (const auto& kv : pool->entries) order.emplace_back(kv.second.last_use, kv.first);
  std::sort(order.begin(), order.end());
  *n = (int)order.size();
  for (int i = 0; out && i < (int)order.size() && i < max; ++i) {
    const auto& e = pool->entries.at(order[i].second);
    out[i] = dymoe_pool_entry{order[i].second.first, order[i].second.second, e.bits, e.pins,
                              e.bytes, e.offset, e.last_use};
  }
  dymoe::clear_error();
  return DYMOE_OK;
}

size_t dymoe_pool_used(const dymoe_pool* pool) {
  if (!pool) return 0;
  size_t u = 0;
  for (const auto& kv : pool->entries) u += kv.second.bytes;
  return u;
}

}  // extern "C"
