// Token permutation (row a5) and weighted combine (row a8) for sm_100a.
//
// Permute (P:203 step 3; BASELINE.json "(c)"): stable counting sort of the T*k (token, slot)
// pairs by expert id; pairs routed to a skipped expert (bits == 0, "4/0") are dropped.
// One CTA of 1024 threads walks the pairs in token-major chunks of 1024; inside a chunk the
// stable rank of a pair among same-expert pairs is (running offset) + (same-expert pairs in
// earlier warps, from a per-warp histogram in shared memory) + (same-expert lanes before it,
// from __match_any_sync).  Integer-only, bit-exact by construction.
//
// Combine (reading D12): y[t] = sum_slot w'[t,slot] * y_perm[inv_row[t,slot]], slot order, fp32.
#include "front_common.cuh"

namespace dymoe {

using front::kPermThreads;
using front::kPermWarps;

__global__ void __launch_bounds__(kPermThreads)
k_permute(const int32_t* __restrict__ topk_idx, int T, int k, int M,
          const uint8_t* __restrict__ bits, int32_t* __restrict__ expert_off,
          int32_t* __restrict__ perm_token, int32_t* __restrict__ perm_slot,
          int32_t* __restrict__ inv_row, int32_t* __restrict__ active_list) {
  __shared__ int running[DYMOE_MAX_EXPERTS];
  __shared__ int warp_cnt[kPermWarps * DYMOE_MAX_EXPERTS];
  __shared__ uint8_t keep[DYMOE_MAX_EXPERTS];
  front::permute(topk_idx, T, k, M, bits, expert_off, perm_token, perm_slot, inv_row, active_list,
                 running, warp_cnt, keep);
}

// Multi-CTA permute for long pair lists: the single-CTA kernel walks its token-major chunks of
// kPermThreads pairs one after another; here chunk c is CTA c.  k_perm_count: per-chunk expert
// counts; k_perm_scan: per expert, the exclusive prefix over chunks plus the expert offset (one
// CTA; the expert scan and active list exactly as front::permute); k_perm_place: the body of one
// iteration of front::permute's chunk loop with running[] = that prefix.  Same placement order
// (chunk, warp, lane), so the same arrays bit for bit.
__global__ void __launch_bounds__(kPermThreads)
k_perm_count(const int32_t* __restrict__ topk_idx, int P, int M, const uint8_t* __restrict__ bits,
             int32_t* __restrict__ cnt) {
  __shared__ int c_sh[DYMOE_MAX_EXPERTS];
  for (int e = threadIdx.x; e < M; e += kPermThreads) c_sh[e] = 0;
  __syncthreads();
  const int p = blockIdx.x * kPermThreads + threadIdx.x;
  if (p < P) {
    const int e = topk_idx[p];
    if (bits[e] != 0) atomicAdd(&c_sh[e], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < M; e += kPermThreads) cnt[(size_t)blockIdx.x * M + e] = c_sh[e];
}

__global__ void __launch_bounds__(256)
k_perm_scan(int G, int M, int32_t* __restrict__ cnt, int32_t* __restrict__ expert_off,
            int32_t* __restrict__ active_list) {
  __shared__ int tot[DYMOE_MAX_EXPERTS];
  for (int e = threadIdx.x; e < M; e += blockDim.x) {
    int acc = 0;
    for (int c = 0; c < G; ++c) {
      const int v = cnt[(size_t)c * M + e];
      cnt[(size_t)c * M + e] = acc;
      acc += v;
    }
    tot[e] = acc;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int per = (M + 31) / 32;
    const int e0 = lane * per, e1 = min(M, e0 + per);
    int sum = 0, nz = 0;
    for (int e = e0; e < e1; ++e) {
      sum += tot[e];
      nz += tot[e] > 0;
    }
    int is = sum, in = nz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int vs = __shfl_up_sync(0xffffffffu, is, o), vn = __shfl_up_sync(0xffffffffu, in, o);
      if (lane >= o) { is += vs; in += vn; }
    }
    int acc = is - sum, na = in - nz;
    for (int e = e0; e < e1; ++e) {
      const int c = tot[e];
      expert_off[e] = acc;
      tot[e] = acc;   // now the expert's first row
      if (c > 0) active_list[1 + na++] = e;
      acc += c;
    }
    if (lane == 31) {
      expert_off[M] = acc;
      active_list[0] = na;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < M; e += blockDim.x)
    for (int c = 0; c < G; ++c) cnt[(size_t)c * M + e] += tot[e];
}

__global__ void __launch_bounds__(kPermThreads)
k_perm_place(const int32_t* __restrict__ topk_idx, int T, int k, int M,
             const uint8_t* __restrict__ bits, const int32_t* __restrict__ base,
             int32_t* __restrict__ perm_token, int32_t* __restrict__ perm_slot,
             int32_t* __restrict__ inv_row) {
  __shared__ int warp_cnt[kPermWarps * DYMOE_MAX_EXPERTS];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int P = T * k;
  for (int q = tid; q < kPermWarps * M; q += kPermThreads)
    warp_cnt[(q / M) * DYMOE_MAX_EXPERTS + (q % M)] = 0;
  __syncthreads();
  const int p = blockIdx.x * kPermThreads + tid;
  int e = -1;
  if (p < P) {
    e = topk_idx[p];
    if (bits[e] == 0) {
      inv_row[p] = -1;
      e = -1;
    }
  }
  const unsigned peers = __match_any_sync(0xffffffffu, e);
  const int rank_in_warp = __popc(peers & ((1u << lane) - 1u));
  if (e >= 0 && rank_in_warp == 0) warp_cnt[w * DYMOE_MAX_EXPERTS + e] = __popc(peers);
  __syncthreads();
  if (e >= 0) {
    int r = base[(size_t)blockIdx.x * M + e] + rank_in_warp;
    for (int q = 0; q < w; ++q) r += warp_cnt[q * DYMOE_MAX_EXPERTS + e];
    perm_token[r] = p / k;
    perm_slot[r] = p - (p / k) * k;
    inv_row[p] = r;
  }
}

size_t permute_scratch_bytes(int T, int k, int M) {
  return (size_t)((T * k + kPermThreads - 1) / kPermThreads) * M * sizeof(int32_t);
}

cudaError_t launch_permute(const int32_t* topk_idx, int T, int k, int M, const uint8_t* bits,
                           int32_t* expert_off, int32_t* perm_token, int32_t* perm_slot,
                           int32_t* inv_row, int32_t* active_list, cudaStream_t s,
                           int32_t* scratch) {
  const int G = (T * k + kPermThreads - 1) / kPermThreads;
  if (scratch != nullptr && G > kPermMultiMinChunks) {
    k_perm_count<<<G, kPermThreads, 0, s>>>(topk_idx, T * k, M, bits, scratch);
    k_perm_scan<<<1, 256, 0, s>>>(G, M, scratch, expert_off, active_list);
    k_perm_place<<<G, kPermThreads, 0, s>>>(topk_idx, T, k, M, bits, scratch, perm_token,
                                            perm_slot, inv_row);
    return cudaGetLastError();
  }
  k_permute<<<1, kPermThreads, 0, s>>>(topk_idx, T, k, M, bits, expert_off, perm_token,
                                       perm_slot, inv_row, active_list);
  return cudaGetLastError();
}

// -------------------------------------------------------------------------------------------
// Expert parallelism helpers: expert e lives on rank floor(e * P / M); because that
// owner is non-decreasing in e, the expert-sorted permutation is already sorted by destination.
__global__ void k_ep_plan(const int32_t* __restrict__ off, int M, int P,
                          int32_t* __restrict__ send_counts, int32_t* __restrict__ row_expert) {
  const int e = blockIdx.x;
  const int lo = off[e], hi = off[e + 1];
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) row_expert[i] = e;
  if (e == 0 && threadIdx.x < P) {
    int c = 0;
    for (int x = 0; x < M; ++x)
      if ((int)(((long long)x * P) / M) == (int)threadIdx.x) c += off[x + 1] - off[x];
    send_counts[threadIdx.x] = c;
  }
}

cudaError_t launch_ep_plan(const int32_t* expert_off, int M, int P, int32_t* send_counts,
                           int32_t* row_expert, cudaStream_t s) {
  k_ep_plan<<<M, 128, 0, s>>>(expert_off, M, P, send_counts, row_expert);
  return cudaGetLastError();
}

// out[i] = x[rows[i]] (bf16 rows of Hd elements, 16-byte vectors)
__global__ void k_gather_rows(const uint4* __restrict__ x, int vec_per_row,
                              const int32_t* __restrict__ rows, int n, uint4* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)n * vec_per_row;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / vec_per_row, c = i - r * vec_per_row;
    out[i] = __ldg(x + (size_t)rows[r] * vec_per_row + c);
  }
}

cudaError_t launch_gather_rows(const uint16_t* x, int Hd, const int32_t* rows, int n,
                               uint16_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int vpr = Hd / 8;
  const size_t total = (size_t)n * vpr;
  const unsigned blocks = (unsigned)((total + 255) / 256 < 8192 ? (total + 255) / 256 : 8192);
  k_gather_rows<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(x), vpr, rows, n,
                                       reinterpret_cast<uint4*>(out));
  return cudaGetLastError();
}

// -------------------------------------------------------------------------------------------
// Combine: one CTA per token, float4 over Hd.  With n_parts > 1 the expert outputs arrive as
// K-slice partials (decode W2 kernel) and are summed in slice order first.
__device__ __forceinline__ float4 load_row(const float* __restrict__ y_perm, int n_parts,
                                           size_t part_stride, int row, int Hd, int c) {
  float4 v = *reinterpret_cast<const float4*>(y_perm + (size_t)row * Hd + c);
  for (int p = 1; p < n_parts; ++p) {
    const float4 u = *reinterpret_cast<const float4*>(y_perm + p * part_stride + (size_t)row * Hd + c);
    v.x = __fadd_rn(v.x, u.x);
    v.y = __fadd_rn(v.y, u.y);
    v.z = __fadd_rn(v.z, u.z);
    v.w = __fadd_rn(v.w, u.w);
  }
  return v;
}

__global__ void __launch_bounds__(256) k_reduce_parts(const float* __restrict__ y_part, int n_parts,
                                                      int part_rows, int rows, int Hd,
                                                      float* __restrict__ y_perm,
                                                      const int32_t* __restrict__ rows_dev) {
  if (rows_dev != nullptr) rows = min(rows, *rows_dev);
  const size_t stride = (size_t)part_rows * Hd;
  const size_t total4 = (size_t)rows * Hd / 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total4;
       i += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(i * 4 / Hd), c = (int)(i * 4 - (size_t)row * Hd);
    *reinterpret_cast<float4*>(y_perm + (size_t)row * Hd + c) =
        load_row(y_part, n_parts, stride, row, Hd, c);
  }
}

cudaError_t launch_reduce_parts(const float* y_part, int n_parts, int part_rows, int rows, int Hd,
                                float* y_perm, cudaStream_t s, const int32_t* rows_dev) {
  if (rows == 0) return cudaSuccess;
  const size_t total4 = (size_t)rows * Hd / 4;
  const int blocks = (int)((total4 + 255) / 256 < 4096 ? (total4 + 255) / 256 : 4096);
  k_reduce_parts<<<blocks, 256, 0, s>>>(y_part, n_parts, part_rows, rows, Hd, y_perm, rows_dev);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_zero_rows(float4* __restrict__ y, int Hd, int cap_rows,
                                                   const int32_t* __restrict__ rows_dev) {
  const int rows = rows_dev != nullptr ? min(cap_rows, *rows_dev) : cap_rows;
  const size_t n4 = (size_t)rows * Hd / 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

cudaError_t launch_zero_rows(float* y, int Hd, int cap_rows, const int32_t* rows_dev, cudaStream_t s) {
  if (cap_rows == 0) return cudaSuccess;
  const size_t n4 = (size_t)cap_rows * Hd / 4;
  const int blocks = (int)((n4 + 255) / 256 < 2 * 148 * 4 ? (n4 + 255) / 256 : 2 * 148 * 4);
  k_zero_rows<<<blocks, 256, 0, s>>>(reinterpret_cast<float4*>(y), Hd, cap_rows, rows_dev);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_combine(const float* __restrict__ y_perm, int n_parts,
                                                 int part_rows,
                                                 const int32_t* __restrict__ inv_row,
                                                 const float* __restrict__ topk_w, int k, int Hd,
                                                 int renorm, int out_bf16,
                                                 const uint16_t* __restrict__ residual,
                                                 void* __restrict__ y) {
  const size_t part_stride = (size_t)part_rows * Hd;
  const int t = blockIdx.x;
  int rows[8];
  float wt[8];
  float denom = 0.f;
  int live = 0;
  for (int s = 0; s < k; ++s) {
    rows[s] = inv_row[(size_t)t * k + s];
    wt[s] = topk_w[(size_t)t * k + s];
    if (rows[s] >= 0) {
      denom += wt[s];
      ++live;
    }
  }
  for (int s = 0; s < k; ++s) wt[s] = renorm ? wt[s] / denom : wt[s];
  // blockIdx.y splits Hd so that a small decode batch still spreads over many SMs
  for (int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4; c < Hd; c += gridDim.y * blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n_parts == 1) {
      // every live slot's row loaded first (k loads in flight), then summed in slot order
      float4 v[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < k && rows[s] >= 0)
          v[s] = *reinterpret_cast<const float4*>(y_perm + (size_t)rows[s] * Hd + c);
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (s >= k || rows[s] < 0) continue;
        acc.x = __fadd_rn(acc.x, __fmul_rn(wt[s], v[s].x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(wt[s], v[s].y));
        acc.z = __fadd_rn(acc.z, __fmul_rn(wt[s], v[s].z));
        acc.w = __fadd_rn(acc.w, __fmul_rn(wt[s], v[s].w));
      }
    } else if (k <= 2 && n_parts <= 4) {
      // decode W2 partials (top-2, <= 4 K slices): all 8 loads in flight before the sums, which
      // keep load_row's order (slices in order per slot, then slots in order)
      float4 v[2][4];
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (s < k && rows[s] >= 0 && q < n_parts)
            v[s][q] = *reinterpret_cast<const float4*>(y_perm + q * part_stride + (size_t)rows[s] * Hd + c);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (s >= k || rows[s] < 0) continue;
        float4 u = v[s][0];
#pragma unroll
        for (int q = 1; q < 4; ++q) {
          if (q >= n_parts) break;
          u.x = __fadd_rn(u.x, v[s][q].x);
          u.y = __fadd_rn(u.y, v[s][q].y);
          u.z = __fadd_rn(u.z, v[s][q].z);
          u.w = __fadd_rn(u.w, v[s][q].w);
        }
        acc.x = __fadd_rn(acc.x, __fmul_rn(wt[s], u.x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(wt[s], u.y));
        acc.z = __fadd_rn(acc.z, __fmul_rn(wt[s], u.z));
        acc.w = __fadd_rn(acc.w, __fmul_rn(wt[s], u.w));
      }
    } else {
      for (int s = 0; s < k; ++s) {
        if (rows[s] < 0) continue;
        const float4 v = load_row(y_perm, n_parts, part_stride, rows[s], Hd, c);
        acc.x = __fadd_rn(acc.x, __fmul_rn(wt[s], v.x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(wt[s], v.y));
        acc.z = __fadd_rn(acc.z, __fmul_rn(wt[s], v.z));
        acc.w = __fadd_rn(acc.w, __fmul_rn(wt[s], v.w));
      }
    }
    if (residual != nullptr) {   // x_{l+1} = x_l + y_l (one fp32 add), rounded below if bf16
      const uint2 r = *reinterpret_cast<const uint2*>(residual + (size_t)t * Hd + c);
      acc.x = __fadd_rn(__uint_as_float(r.x << 16), acc.x);
      acc.y = __fadd_rn(__uint_as_float(r.x & 0xffff0000u), acc.y);
      acc.z = __fadd_rn(__uint_as_float(r.y << 16), acc.z);
      acc.w = __fadd_rn(__uint_as_float(r.y & 0xffff0000u), acc.w);
    }
    if (out_bf16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(y) + (size_t)t * Hd + c) = o;
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + (size_t)t * Hd + c) = acc;
    }
  }
  (void)live;
}

cudaError_t launch_combine(const float* y_perm, int n_parts, int part_rows, const int32_t* inv_row,
                           const float* topk_w, int T, int k, int Hd, int renorm, int out_dtype,
                           void* y, cudaStream_t s, const uint16_t* residual) {
  if (T == 0) return cudaSuccess;
  // ~4 CTAs of 128 threads x float4 per SM in total, at least one column chunk per token
  const int chunks = (Hd + 511) / 512;
  int gy = (4 * 148 + T - 1) / T;
  gy = gy < 1 ? 1 : (gy > chunks ? chunks : gy);
  k_combine<<<dim3(T, gy), 128, 0, s>>>(y_perm, n_parts, part_rows, inv_row, topk_w, k, Hd, renorm,
                                        out_dtype == DYMOE_OUT_BF16, residual, y);
  return cudaGetLastError();
}

// Global-live-set combine weights (D12): one thread per token, slot order, fp32 -- the same
// arithmetic k_combine applies when it renormalises.
__global__ void k_renorm_weights(const int32_t* __restrict__ topk_idx, const float* __restrict__ topk_w,
                                 const uint8_t* __restrict__ bits, int T, int k, int renorm,
                                 float* __restrict__ w_out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float w[8];
  bool live[8];
  float denom = 0.f;
  for (int s = 0; s < k; ++s) {
    w[s] = topk_w[(size_t)t * k + s];
    live[s] = bits[topk_idx[(size_t)t * k + s]] != 0;
    if (live[s]) denom += w[s];
  }
  for (int s = 0; s < k; ++s)
    w_out[(size_t)t * k + s] = live[s] ? (renorm ? w[s] / denom : w[s]) : 0.f;
}

cudaError_t launch_renorm_weights(const int32_t* topk_idx, const float* topk_w, const uint8_t* bits,
                                  int T, int k, int renorm, float* w_out, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  k_renorm_weights<<<(T + 127) / 128, 128, 0, s>>>(topk_idx, topk_w, bits, T, k, renorm, w_out);
  return cudaGetLastError();
}

cudaError_t preload_permute_combine() {
  return preload_kernels(k_permute, k_perm_count, k_perm_scan, k_perm_place, k_ep_plan, k_gather_rows, k_reduce_parts, k_zero_rows, k_combine,
                         k_renorm_weights);
}

}  // namespace dymoe
