// Router (row a1), importance scoring (a2) and bit assignment (a3) kernels for sm_100a.
//
// Paper: PAPER.md P:111 (router), Eq. 6 P:278 (softmax gate), Eq. 1-2 P:216-227 (prefill
// token-guided importance), Eq. 3 P:236-241 (decode gate-guided importance), Eq. 4-5
// P:250-259 (depth-aware schedule), P:312 (tiers).  Readings R1b, R3, D5, D7-D11.
//
// All three are latency-bound (a few KB of input per layer); they are written for one launch
// each with no host round trip so that a decode step can be captured in a CUDA graph.
#include "front_common.cuh"

namespace dymoe {

// ===========================================================================================
// Route: one warp per token (front::route_token: top-k by (logit desc, index asc), softmax over
// the k, full softmax).
// ===========================================================================================
__global__ void __launch_bounds__(256) k_route(const float* __restrict__ logits, int T, int M,
                                               int k, int32_t* __restrict__ topk_idx,
                                               float* __restrict__ topk_w,
                                               float* __restrict__ probs) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= T) return;
  front::route_token(logits + (size_t)warp * M, M, k, threadIdx.x & 31, topk_idx + (size_t)warp * k,
                     topk_w + (size_t)warp * k, probs != nullptr ? probs + (size_t)warp * M : nullptr);
}

cudaError_t launch_route(const float* logits, int T, int M, int k, int32_t* topk_idx,
                         float* topk_w, float* probs, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int warps_per_block = 8;
  dim3 grid((T + warps_per_block - 1) / warps_per_block);
  k_route<<<grid, 32 * warps_per_block, 0, s>>>(logits, T, M, k, topk_idx, topk_w, probs);
  return cudaGetLastError();
}

// ===========================================================================================
// Prefill score: one CTA of 1024 threads.
//   1. S_i = sum_h a[h][i], fp32, heads in order (Eq. 1 without the 1/H factor, R1b).
//   2. T_imp = top-k_tokens by (S desc, i asc): 4-pass 8-bit radix select on an order-preserving
//      u32 key (with -0.0 folded onto +0.0), then the lowest-index ties at the threshold.
//   3. importance[j] = #{i in T_imp : j in topk_idx[i]} (Eq. 2), exact integer counts.
// ===========================================================================================
__device__ __forceinline__ uint32_t order_key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;                  // -0.0 == +0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, int* sh_warp, int& total) {
  // returns exclusive prefix of v over threads in index order; total = sum
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) sh_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < NT / 32 ? sh_warp[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, off);
      if (lane >= off) t += y;
    }
    if (lane < NT / 32) sh_warp[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  int base = w > 0 ? sh_warp[w - 1] : 0;
  total = sh_warp[NT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

constexpr int kScoreThreads = 1024;

__global__ void __launch_bounds__(kScoreThreads)
k_score_prefill(const float* __restrict__ attn, int H, const int32_t* __restrict__ topk_idx,
                int T, int M, int k, int k_tokens, float* __restrict__ importance,
                int32_t* __restrict__ heavy, float* __restrict__ S) {
  __shared__ int hist[256];
  __shared__ int cnt[DYMOE_MAX_EXPERTS];
  __shared__ int sh_warp[32];
  __shared__ uint32_t sh_prefix;
  __shared__ int sh_krem;
  const int tid = threadIdx.x;

  // 1. token scores, sequential over heads (coalesced over tokens).  One CTA pulls the whole
  // [H][T] mass (256 KB at H = 32, T = 2048), so the loads are 16 bytes wide (4 tokens) with 8
  // heads in flight; each token's sum keeps the head order.
  const int T4 = (T % 4 == 0 && ((reinterpret_cast<uintptr_t>(attn) | reinterpret_cast<uintptr_t>(S)) & 15) == 0)
                     ? T / 4 : 0;
  for (int i4 = tid; i4 < T4; i4 += kScoreThreads) {
    const float4* a4 = reinterpret_cast<const float4*>(attn);
    float4 acc = a4[i4];
    int h = 1;
    for (; h + 8 <= H; h += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a4[(size_t)(h + u) * T4 + i4];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x = __fadd_rn(acc.x, v[u].x);
        acc.y = __fadd_rn(acc.y, v[u].y);
        acc.z = __fadd_rn(acc.z, v[u].z);
        acc.w = __fadd_rn(acc.w, v[u].w);
      }
    }
    for (; h < H; ++h) {
      const float4 v = a4[(size_t)h * T4 + i4];
      acc.x = __fadd_rn(acc.x, v.x);
      acc.y = __fadd_rn(acc.y, v.y);
      acc.z = __fadd_rn(acc.z, v.z);
      acc.w = __fadd_rn(acc.w, v.w);
    }
    reinterpret_cast<float4*>(S)[i4] = acc;
  }
  for (int i = 4 * T4 + tid; i < T; i += kScoreThreads) {
    float acc = attn[i];
    int h = 1;
    for (; h + 8 <= H; h += 8) {   // 8 loads in flight, then the adds in head order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = attn[(size_t)(h + u) * T + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
    }
    for (; h < H; ++h) acc = __fadd_rn(acc, attn[(size_t)h * T + i]);
    S[i] = acc;
  }
  for (int j = tid; j < M; j += kScoreThreads) cnt[j] = 0;
  if (tid == 0) {
    sh_prefix = 0u;
    sh_krem = k_tokens;
  }
  __syncthreads();
  if (k_tokens <= 0) {
    for (int j = tid; j < M; j += kScoreThreads) importance[j] = 0.f;
    return;
  }

  // 2. radix select of the k_tokens-th largest key (MSB first, 8 bits per pass)
  uint32_t prefix_mask = 0u;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int b = tid; b < 256; b += kScoreThreads) hist[b] = 0;
    __syncthreads();
    const uint32_t prefix = sh_prefix;
    for (int i = tid; i < T; i += kScoreThreads) {
      uint32_t key = order_key(S[i]);
      if ((key & prefix_mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
    }
    __syncthreads();
    if (tid < 32) {
      // find digit d (from 255 down) where the cumulative count reaches k_rem
      const int krem = sh_krem;
      // each lane owns 8 consecutive digits from the top: lane 0 -> 255..248
      int local[8];
      int lsum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        local[q] = hist[255 - (tid * 8 + q)];
        lsum += local[q];
      }
      int incl = lsum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (tid >= off) incl += y;
      }
      int excl = incl - lsum;
      bool mine = excl < krem && incl >= krem;
      if (mine) {
        int run = excl;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (run < krem && run + local[q] >= krem) {
            const uint32_t d = 255u - (uint32_t)(tid * 8 + q);
            sh_prefix = prefix | (d << shift);
            sh_krem = krem - run;
          }
          run += local[q];
        }
      }
    }
    prefix_mask |= 255u << shift;
    __syncthreads();
  }
  const uint32_t thresh = sh_prefix;
  const int need_eq = sh_krem;  // how many tokens with key == thresh belong to T_imp

  // 3. membership in token order; count routed experts of heavy tokens; compact `heavy`
  int eq_base = 0, out_base = 0;
  for (int c0 = 0; c0 < T; c0 += kScoreThreads) {
    const int i = c0 + tid;
    uint32_t key = i < T ? order_key(S[i]) : 0u;
    const int is_eq = (i < T && key == thresh) ? 1 : 0;
    int eq_total;
    const int eq_rank = eq_base + block_exclusive_scan<kScoreThreads>(is_eq, sh_warp, eq_total);
    const int is_heavy = (i < T && (key > thresh || (is_eq && eq_rank < need_eq))) ? 1 : 0;
    int h_total;
    const int h_pos = out_base + block_exclusive_scan<kScoreThreads>(is_heavy, sh_warp, h_total);
    if (is_heavy) {
      if (heavy != nullptr) heavy[h_pos] = i;
      for (int r = 0; r < k; ++r) atomicAdd(&cnt[topk_idx[(size_t)i * k + r]], 1);
    }
    eq_base += eq_total;
    out_base += h_total;
  }
  __syncthreads();
  for (int j = tid; j < M; j += kScoreThreads) importance[j] = (float)cnt[j];
}

cudaError_t launch_score_prefill(const float* attn, int H, const int32_t* topk_idx, int T,
                                 int M, int k, int k_tokens, float* importance, int32_t* heavy,
                                 float* S_scratch, cudaStream_t s) {
  k_score_prefill<<<1, kScoreThreads, 0, s>>>(attn, H, topk_idx, T, M, k, k_tokens, importance,
                                              heavy, S_scratch);
  return cudaGetLastError();
}

// ===========================================================================================
// Decode score (Eq. 3, reading D10): B == 1 -> the logit row; B > 1 -> sum_b softmax(l_b)
// (fp32, b ascending; each softmax exactly route's probs).  One CTA of 8 warps.
// ===========================================================================================
__global__ void __launch_bounds__(256) k_score_decode(const float* __restrict__ logits, int B,
                                                      int M, float* __restrict__ importance) {
  __shared__ float sp[8 * DYMOE_MAX_EXPERTS];
  front::decode_importance(logits, B, M, sp, importance);
}

cudaError_t launch_score_decode(const float* logits, int B, int M, float* importance,
                                cudaStream_t s) {
  k_score_decode<<<1, 256, 0, s>>>(logits, B, M, importance);
  return cudaGetLastError();
}

// ===========================================================================================
// Assign bits (Eq. 5 + tiers, readings D5, D7-D9, D11): one CTA, thread j = expert j
// (front::assign_bits).
// ===========================================================================================
__global__ void __launch_bounds__(256) k_assign(const float* __restrict__ importance,
                                                const uint8_t* __restrict__ active_mask,
                                                const int32_t* __restrict__ topk_idx, int T,
                                                AssignParams p, uint8_t* __restrict__ bits,
                                                uint8_t* __restrict__ active_out) {
  __shared__ float I[DYMOE_MAX_EXPERTS];
  __shared__ int act[DYMOE_MAX_EXPERTS];
  __shared__ int n_act;
  front::assign_bits(importance, active_mask, topk_idx, T, p, bits, active_out, I, act, &n_act);
}

cudaError_t launch_assign(const float* importance, const uint8_t* active_mask,
                          const int32_t* topk_idx, int T, const AssignParams& p, uint8_t* bits,
                          uint8_t* active_out, cudaStream_t s) {
  k_assign<<<1, 256, 0, s>>>(importance, active_mask, topk_idx, T, p, bits, active_out);
  return cudaGetLastError();
}

// ===========================================================================================
// Fused decode front: route -> score -> assign -> permute in ONE single-CTA launch of 256 threads
// for a decode batch, with exactly the arithmetic of the four standalone kernels (the same front::
// bodies; none of their results depends on the block size).  The intermediates the later phases
// read back (top-k indices, importance, bits) stay in shared memory and are copied out at the
// end.  A decode step's front is latency-bound (a few KB), so three launches and their gaps were
// ~10 % of the step.  forced_bits != nullptr skips score/assign.
// ===========================================================================================
constexpr int kFrontThreads = 256;

// Optional phase timeline of the decode front (a build with -DDYMOE_FRONT_TRACE, tools/front_trace.py;
// the product build has no trace code): globaltimer stamps of thread 0 after each phase.
#ifdef DYMOE_FRONT_TRACE
__device__ unsigned long long g_front_tr[16];
#define FRONT_TR(i)                                                         \
  do {                                                                      \
    if (threadIdx.x == 0) {                                                 \
      unsigned long long t_;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                \
      g_front_tr[i] = t_;                                                   \
    }                                                                       \
  } while (0)
extern "C" int dymoe_front_trace_read(unsigned long long* host) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(host, g_front_tr, sizeof(g_front_tr));
}
#else
#define FRONT_TR(i) do {} while (0)
#endif

__global__ void __launch_bounds__(kFrontThreads)
k_front_decode(const float* logits, int T, int M, int k, AssignParams p,
               const uint8_t* forced_bits, int32_t* topk_idx, float* topk_w, float* probs,
               float* importance, uint8_t* bits, uint8_t* active, int32_t* expert_off,
               int32_t* perm_token, int32_t* perm_slot, int32_t* inv_row, int32_t* active_list) {
  constexpr int NW = kFrontThreads / 32;
  // phase buffers: the score's per-warp softmax rows and the permute's per-warp histograms are
  // never live at the same time (block barriers between the phases)
  __shared__ __align__(16) int big[NW * DYMOE_MAX_EXPERTS];
  __shared__ int running[DYMOE_MAX_EXPERTS];
  __shared__ float I[DYMOE_MAX_EXPERTS];
  __shared__ int act[DYMOE_MAX_EXPERTS];
  __shared__ uint8_t keep[DYMOE_MAX_EXPERTS];
  __shared__ int n_act;
  __shared__ int32_t s_idx[kFrontDecodeMaxT * 8];
  __shared__ float s_imp[DYMOE_MAX_EXPERTS];
  __shared__ uint8_t s_bits[DYMOE_MAX_EXPERTS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  FRONT_TR(0);
  // T <= NW (one token per warp): route's full-softmax rows go to shared memory, where the score
  // phase sums them -- they are exactly the rows decode_importance would recompute
  // (front::softmax_row), so the importance is unchanged; copied to `probs` below
  const bool rows_in_smem = T <= NW && T > 1;
  float* sp = reinterpret_cast<float*>(big);
  for (int t = w; t < T; t += NW)
    front::route_token(logits + (size_t)t * M, M, k, lane, s_idx + (size_t)t * k,
                       topk_w + (size_t)t * k,
                       rows_in_smem ? sp + t * M : (probs != nullptr ? probs + (size_t)t * M : nullptr));
  __syncthreads();
  FRONT_TR(1);
  const uint8_t* b = forced_bits;
  if (b == nullptr) {
    if (rows_in_smem) {
      if ((int)threadIdx.x < M) {   // Eq. 3, b ascending (decode_importance's sum)
        float acc = 0.f;
        for (int q = 0; q < T; ++q) acc = __fadd_rn(acc, sp[q * M + threadIdx.x]);
        s_imp[threadIdx.x] = acc;
      }
      __syncthreads();
    } else {
      front::decode_importance(logits, T, M, sp, s_imp);
    }
    FRONT_TR(2);
    front::assign_bits(s_imp, nullptr, s_idx, T, p, s_bits, active, I, act, &n_act);
    b = s_bits;
  }
  FRONT_TR(3);
  if (rows_in_smem && probs != nullptr)
    for (int i = threadIdx.x; i < T * M; i += kFrontThreads) probs[i] = sp[i];
  __syncthreads();   // sp (= big) is reused by the permute's histograms
  FRONT_TR(4);
  if (T * k <= 256) {   // one warp, no block barriers (front::permute_small)
    if (threadIdx.x < 32) {
      if (T * k <= 32)
        front::permute_small<1>(s_idx, T, k, M, b, expert_off, perm_token, perm_slot, inv_row,
                                active_list, running);
      else
        front::permute_small<8>(s_idx, T, k, M, b, expert_off, perm_token, perm_slot, inv_row,
                                active_list, running);
    }
  } else {
    front::permute<kFrontThreads>(s_idx, T, k, M, b, expert_off, perm_token, perm_slot, inv_row,
                                  active_list, running, big, keep);
  }
  FRONT_TR(5);
  for (int i = threadIdx.x; i < T * k; i += kFrontThreads) topk_idx[i] = s_idx[i];
  if (forced_bits == nullptr)
    for (int j = threadIdx.x; j < M; j += kFrontThreads) {
      importance[j] = s_imp[j];
      bits[j] = s_bits[j];
    }
  FRONT_TR(6);
}

cudaError_t launch_front_decode(const float* logits, int T, int M, int k, const AssignParams& p,
                                const uint8_t* forced_bits, int32_t* topk_idx, float* topk_w,
                                float* probs, float* importance, uint8_t* bits, uint8_t* active,
                                int32_t* expert_off, int32_t* perm_token, int32_t* perm_slot,
                                int32_t* inv_row, int32_t* active_list, cudaStream_t s) {
  k_front_decode<<<1, kFrontThreads, 0, s>>>(logits, T, M, k, p, forced_bits, topk_idx, topk_w,
                                                   probs, importance, bits, active, expert_off,
                                                   perm_token, perm_slot, inv_row, active_list);
  return cudaGetLastError();
}

cudaError_t preload_route_score() {
  return preload_kernels(k_route, k_score_prefill, k_score_decode, k_assign, k_front_decode);
}

}  // namespace dymoe
