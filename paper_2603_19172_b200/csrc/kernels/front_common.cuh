// Block-level bodies of the latency-bound front of the layer -- route (a1), decode score (a2),
// assign (a3), permute (a5) -- shared by their standalone kernels (route_score.cu,
// permute_combine.cu) and by the fused decode front k_front_decode (route_score.cu), so that the
// fused kernel computes bit-for-bit what the four launches compute.
//
// Shared memory is passed in by the caller (the fused kernel overlays the phases' buffers).
// Pointers a phase reads after an earlier phase of the SAME kernel wrote them are plain (no
// __restrict__ const): they must not be read through the non-coherent load path.
#pragma once
#include <cfloat>
#include <math.h>

#include "../dymoe_internal.cuh"

namespace dymoe {
namespace front {

__device__ __forceinline__ bool better(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

// Route one token (Eq. 6, readings D10/D11) with one warp: top-k by (logit desc,
// index asc) as k rounds of a warp arg-max (plain float compares: -0.0 == +0.0); w = softmax over
// the selected logits (max = the first selected, fp32, slot order); probs (nullable) = softmax
// over all M (lane partial sums in i order, then an xor butterfly).
__device__ __forceinline__ void route_token(const float* row, int M, int k, int lane,
                                            int32_t* topk_idx, float* topk_w, float* probs) {
  float v[8];
  uint32_t taken = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < M ? row[j] : -FLT_MAX;
  }
  // k rounds of a warp arg-max on an order-preserving unsigned key of the logit (monotonic in
  // the float order, -0.0 and +0.0 mapped to one key, 0 = not a candidate): each lane scans its
  // 8 candidates in index order (strict > keeps the lower index on ties), then two warp
  // reductions (REDUX: max of the keys, min of the indices holding it) -- the same (value desc,
  // index asc) order as `better` with two reduction instructions per round instead of five
  // dependent shuffle-compare steps.
  unsigned key[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = lane + 32 * i;
    const unsigned u = v[i] == 0.f ? 0u : __float_as_uint(v[i]);
    key[i] = j < M ? ((u & 0x80000000u) ? ~u : (u | 0x80000000u)) : 0u;
  }
  float sel_v[8];
  int sel_i[8];
  for (int r = 0; r < k; ++r) {
    unsigned bk = 0u;
    int bj = 0x7fffffff;
    float bv = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const unsigned kk = (taken >> i & 1u) ? 0u : key[i];
      if (kk > bk) {
        bk = kk;
        bj = lane + 32 * i;
        bv = v[i];
      }
    }
    const unsigned kmax = __reduce_max_sync(0xffffffffu, bk);
    const int bi = (int)__reduce_min_sync(0xffffffffu, bk == kmax ? (unsigned)bj : 0x7fffffffu);
    sel_v[r] = __shfl_sync(0xffffffffu, bv, bi & 31);
    sel_i[r] = bi;
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
  }

  const float vmax = sel_v[0];
  float e[8];
  float z = 0.f;
  for (int r = 0; r < k; ++r) {
    e[r] = expf(sel_v[r] - vmax);
    z += e[r];
  }
  if (lane < k) {
    float my_e = 0.f;
    int my_i = 0;
    for (int r = 0; r < k; ++r)
      if (r == lane) { my_e = e[r]; my_i = sel_i[r]; }
    topk_idx[lane] = my_i;
    topk_w[lane] = my_e / z;
  }
  if (probs != nullptr) {
    float ev[8];
    float zs = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = lane + 32 * i;
      ev[i] = j < M ? expf(v[i] - vmax) : 0.f;
      zs += ev[i];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) zs += __shfl_xor_sync(0xffffffffu, zs, off);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = lane + 32 * i;
      if (j < M) probs[j] = ev[i] / zs;
    }
  }
}

// Full softmax of one logit row by one warp into p[0..M): exactly route_token's probs (the row
// max is the first top-1 pick, the same value however it is found).
__device__ __forceinline__ void softmax_row(const float* row, int M, int lane, float* p) {
  float v[8];
  float m = -FLT_MAX;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < M ? row[j] : -FLT_MAX;
    m = fmaxf(m, v[i]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  float ev[8];
  float zs = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = lane + 32 * i;
    ev[i] = j < M ? expf(v[i] - m) : 0.f;
    zs += ev[i];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) zs += __shfl_xor_sync(0xffffffffu, zs, off);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int j = lane + 32 * i;
    if (j < M) p[j] = ev[i] / zs;
  }
}

// Decode importance (Eq. 3, reading D10), whole block: B == 1 -> the logit row; B > 1 ->
// I_j = sum_b softmax(l_b)_j in fp32, b ascending.  sp: shared [nwarps][M] floats.  Ends with a
// __syncthreads (importance may be re-read by the block).
__device__ __forceinline__ void decode_importance(const float* logits, int B, int M, float* sp,
                                                  float* importance) {
  const int j = threadIdx.x, lane = j & 31, w = j >> 5, nw = blockDim.x >> 5;
  if (B == 1) {
    if (j < M) importance[j] = logits[j];
    __syncthreads();
    return;
  }
  float acc = 0.f;
  for (int b0 = 0; b0 < B; b0 += nw) {
    if (b0 + w < B) softmax_row(logits + (size_t)(b0 + w) * M, M, lane, sp + w * M);
    __syncthreads();
    const int nb = B - b0 < nw ? B - b0 : nw;
    if (j < M)
      for (int q = 0; q < nb; ++q) acc = __fadd_rn(acc, sp[q * M + j]);
    __syncthreads();
  }
  if (j < M) importance[j] = acc;
  __syncthreads();
}

// Assign bits (Eq. 5 + tiers; readings D5, D7-D9, D11), whole block (blockDim >= M): thread j =
// expert j; rank_j = #{i active : I_i > I_j or (I_i == I_j and i < j)}; t_k = ceil(r_k*M_eff -
// 1e-9) in fp64 (explicit _rn, no contraction) from the host-evaluated r_k.  Shared: I [M]
// floats, act [M] ints, n_act.  Ends with a __syncthreads.
__device__ __forceinline__ void assign_bits(const float* importance, const uint8_t* active_mask,
                                            const int32_t* topk_idx, int T, const AssignParams& p,
                                            uint8_t* bits, uint8_t* active_out, float* I, int* act,
                                            int* n_act) {
  const int j = threadIdx.x;
  if (j < p.M) {
    I[j] = importance[j];
    act[j] = p.m_active ? (active_mask != nullptr ? (active_mask[j] != 0) : 0) : 1;
  }
  __syncthreads();
  if (p.m_active && active_mask == nullptr) {
    for (int q = j; q < T * p.k_route; q += blockDim.x) act[topk_idx[q]] = 1;  // benign race
    __syncthreads();
  }
  const int M_eff = __syncthreads_count(j < p.M && act[j]);   // the active count (a barrier)
  if (j == 0) *n_act = M_eff;
  if (j < p.M) {
    if (active_out != nullptr) active_out[j] = (uint8_t)act[j];
    if (!act[j]) {
      bits[j] = (uint8_t)p.bits[p.n_tiers - 1];
    } else {
      const float Ij = I[j];
      int rank = 0;   // independent terms (no loop-carried branch): unrolled broadcast reads
#pragma unroll 8
      for (int i = 0; i < p.M; ++i)
        rank += (act[i] != 0) & ((I[i] > Ij) | ((I[i] == Ij) & (i < j)));
      int tier = p.n_tiers - 1;
      int prev = 0;
      for (int q = 0; q < p.n_tiers - 1; ++q) {
        const double x = __dsub_rn(__dmul_rn(p.r[q], (double)M_eff), 1e-9);
        int t = (int)ceil(x);
        if (q == 0 && p.clamp_to_k) t = max(t, min(p.k_route, M_eff));
        t = max(t, prev);
        t = min(t, M_eff);
        prev = t;
        if (rank < t && tier == p.n_tiers - 1) tier = q;
      }
      bits[j] = (uint8_t)p.bits[tier];
    }
  }
  __syncthreads();
}

// Permute (P:203 step 3): stable counting sort of the T*k (token, slot) pairs by expert id,
// pairs of skipped experts (bits == 0) dropped; a block of NT threads.  Token-major chunks of NT
// pairs: a pair's stable rank = running offset + same-expert pairs of earlier warps (per-warp
// histogram) + same-expert lanes before it (__match_any_sync).  Shared: running [M] ints,
// warp_cnt [NT/32][kMaxE] ints, keep [M] bytes.  Integer-only, bit-exact by construction (the
// result does not depend on NT).
constexpr int kPermThreads = 1024;
constexpr int kPermWarps = kPermThreads / 32;

template <int NT = kPermThreads>
__device__ __forceinline__ void permute(const int32_t* topk_idx, int T, int k, int M,
                                        const uint8_t* bits, int32_t* expert_off,
                                        int32_t* perm_token, int32_t* perm_slot, int32_t* inv_row,
                                        int32_t* active_list, int* running, int* warp_cnt,
                                        uint8_t* keep) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int P = T * k;
  for (int e = tid; e < M; e += NT) {
    running[e] = 0;
    keep[e] = bits[e] != 0;
  }
  __syncthreads();
  for (int p = tid; p < P; p += NT) {   // counts per expert
    const int e = topk_idx[p];
    if (keep[e]) atomicAdd(&running[e], 1);
  }
  __syncthreads();
  if (tid < 32) {   // exclusive scan of the counts (M <= 256) and the active list, one warp
    const int per = (M + 31) / 32;
    const int e0 = lane * per, e1 = min(M, e0 + per);
    int sum = 0, nz = 0;
    for (int e = e0; e < e1; ++e) {
      sum += running[e];
      nz += running[e] > 0;
    }
    int is = sum, in = nz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int vs = __shfl_up_sync(0xffffffffu, is, o), vn = __shfl_up_sync(0xffffffffu, in, o);
      if (lane >= o) { is += vs; in += vn; }
    }
    int acc = is - sum, na = in - nz;
    for (int e = e0; e < e1; ++e) {
      const int c = running[e];
      expert_off[e] = acc;
      running[e] = acc;
      if (c > 0) active_list[1 + na++] = e;
      acc += c;
    }
    if (lane == 31) {
      expert_off[M] = acc;
      active_list[0] = na;
    }
  }
  __syncthreads();
  for (int c0 = 0; c0 < P; c0 += NT) {   // stable placement, chunk by chunk
    for (int q = tid; q < (NT / 32) * M; q += NT)
      warp_cnt[(q / M) * DYMOE_MAX_EXPERTS + (q % M)] = 0;
    __syncthreads();
    const int p = c0 + tid;
    int e = -1;
    if (p < P) {
      e = topk_idx[p];
      if (!keep[e]) {
        inv_row[p] = -1;
        e = -1;
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank_in_warp = __popc(peers & ((1u << lane) - 1u));
    if (e >= 0 && rank_in_warp == 0) warp_cnt[w * DYMOE_MAX_EXPERTS + e] = __popc(peers);
    __syncthreads();
    if (e >= 0) {
      int r = running[e] + rank_in_warp;
      for (int q = 0; q < w; ++q) r += warp_cnt[q * DYMOE_MAX_EXPERTS + e];
      perm_token[r] = p / k;
      perm_slot[r] = p - (p / k) * k;
      inv_row[p] = r;
    }
    __syncthreads();
    for (int e2 = tid; e2 < M; e2 += NT) {
      int add = 0;
      for (int q = 0; q < (NT / 32); ++q) add += warp_cnt[q * DYMOE_MAX_EXPERTS + e2];
      running[e2] += add;
    }
    __syncthreads();
  }
}

// The same permutation by ONE warp for P = T*k <= 256 pairs (the decode front: 8 tokens x top-2
// .. top-8): pairs are taken 32 at a time in token-major order (round r: pair 32 r + lane); per
// round one __match_any_sync gives every pair its expert's count and its rank among the round's
// earlier pairs, and the single leader of each expert group adds the count -- a pair's stable
// position is its expert's offset + the same-expert pairs of earlier rounds + its in-round rank,
// the stable counting sort of permute, with __syncwarp instead of permute's block barriers
// (seven per chunk).  Bit-identical outputs: the stable counting sort is unique.
// Shared: running [M] ints.  RMAX = the largest round count the instance handles (1: P <= 32).
template <int RMAX>
__device__ __forceinline__ void permute_small(const int32_t* topk_idx, int T, int k, int M,
                                              const uint8_t* bits, int32_t* expert_off,
                                              int32_t* perm_token, int32_t* perm_slot,
                                              int32_t* inv_row, int32_t* active_list,
                                              int* running) {
  const int lane = threadIdx.x & 31;
  const int P = T * k;
  const int R = (P + 31) / 32;   // <= RMAX
  for (int e = lane; e < M; e += 32) running[e] = 0;
  __syncwarp();
  int ex[RMAX];
  unsigned peers[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    if (r >= R) break;
    const int p = 32 * r + lane;
    int e = -1;
    if (p < P) {
      e = topk_idx[p];
      if (bits[e] == 0) {
        inv_row[p] = -1;
        e = -1;
      }
    }
    ex[r] = e;
    peers[r] = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && (peers[r] & ((1u << lane) - 1u)) == 0) running[e] += __popc(peers[r]);
    __syncwarp();
  }
  {   // exclusive scan of the counts and the active list (permute's warp scan)
    const int per = (M + 31) / 32;
    const int e0 = lane * per, e1 = min(M, e0 + per);
    int sum = 0, nz = 0;
    for (int q = e0; q < e1; ++q) {
      sum += running[q];
      nz += running[q] > 0;
    }
    int is = sum, in = nz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int vs = __shfl_up_sync(0xffffffffu, is, o), vn = __shfl_up_sync(0xffffffffu, in, o);
      if (lane >= o) { is += vs; in += vn; }
    }
    int acc = is - sum, na = in - nz;
    for (int q = e0; q < e1; ++q) {
      const int c = running[q];
      expert_off[q] = acc;
      running[q] = acc;
      if (c > 0) active_list[1 + na++] = q;
      acc += c;
    }
    if (lane == 31) {
      expert_off[M] = acc;
      active_list[0] = na;
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    if (r >= R) break;
    const int e = ex[r];
    const unsigned lower = peers[r] & ((1u << lane) - 1u);
    int base = 0;
    if (e >= 0) base = running[e];
    __syncwarp();   // every lane has read its expert's running offset before the leaders advance it
    if (e >= 0) {
      const int p = 32 * r + lane;
      const int pos = base + __popc(lower);
      perm_token[pos] = p / k;
      perm_slot[pos] = p - (p / k) * k;
      inv_row[p] = pos;
      if (lower == 0) running[e] = base + __popc(peers[r]);
    }
    __syncwarp();
  }
}

}  // namespace front
}  // namespace dymoe
