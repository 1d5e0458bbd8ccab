// Expert-parallel dispatch and combine over peer memory (include/dymoe.h
// "Expert-parallel dispatch and combine over peer memory").  The NCCL all-to-all pair of ep.py's
// default path becomes two kernels that move the bytes themselves over NVLink / NVSwitch:
//   k_ep_dispatch  gather of the permuted token rows FUSED with the dispatch: each warp reads
//                  x[perm_token[j]] from local HBM and stores it, 16 bytes per lane, straight
//                  into the owner's receive window at its final expert-major row;
//   k_ep_combine   the reverse transfer FUSED with the weighted combine: each token's CTA loads
//                  its live slots' output rows from the owners' windows and sums them with the
//                  dymoe_combine arithmetic (reading D12, slot order, fp32).
// Barriers are flag counters in the windows (release / acquire at system scope), bounded by a
// wall-clock timeout so that a missing peer sets a status bit instead of hanging the device.
#include <cstring>

#include "dymoe_internal.cuh"

namespace dymoe {
namespace {

constexpr unsigned long long kBarrierTimeoutNs = 5ull * 1000 * 1000 * 1000;

__device__ __forceinline__ int32_t* cnt_of(const EpWin& a, int p) {
  return reinterpret_cast<int32_t*>(a.peers[p] + a.L.cnt) + (size_t)a.parity * a.P * a.M;
}
__device__ __forceinline__ float* imp_of(const EpWin& a, int p) {
  return reinterpret_cast<float*>(a.peers[p] + a.L.imp) + (size_t)a.parity * a.P * a.M;
}
__device__ __forceinline__ float* red_of(const EpWin& a, int p) {
  return reinterpret_cast<float*>(a.peers[p] + a.L.red) + (size_t)a.parity * kEpRedRows * a.Hd;
}
// rows rank s sends to expert e this step: the published count, 0 for a skipped expert
__device__ __forceinline__ int cnt_at(const EpWin& a, const int32_t* cnt, int s, int e) {
  return (a.bits != nullptr && a.bits[e] == 0) ? 0 : cnt[(size_t)s * a.M + e];
}

// Row layout of the step (computed from this rank's own, complete count matrix):
//   tot[e]  = sum_src cnt[src][e];  gex[e] = sum_{e' < e} tot[e'] (global exclusive prefix)
//   base(e) = gex[e] - gex[first expert of owner(e)]  (expert e's first row in its owner's recv_x)
//   row0[e] = base(e) + sum_{src < rank} cnt[src][e]   (this rank's first row of expert e there)
// The prefix is one warp scan over contiguous blocks of experts (owners hold contiguous expert
// blocks, so a per-owner base is a difference of the global prefix).
__device__ void ep_layout(const EpWin& a, int* s_row0, int* s_gex, int* s_tot) {
  const int32_t* cnt = cnt_of(a, a.rank);
  for (int e = threadIdx.x; e < a.M; e += blockDim.x) {
    int tot = 0, pre = 0;
    for (int s = 0; s < a.P; ++s) {
      const int c = cnt_at(a, cnt, s, e);
      tot += c;
      if (s < a.rank) pre += c;
    }
    s_tot[e] = tot;
    s_row0[e] = pre;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int per = (a.M + 31) / 32;
    const int e0 = lane * per, e1 = min(a.M, e0 + per);
    int sum = 0;
    for (int e = e0; e < e1; ++e) sum += s_tot[e];
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int acc = incl - sum;
    for (int e = e0; e < e1; ++e) {
      s_gex[e] = acc;
      acc += s_tot[e];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < a.M; e += blockDim.x)
    s_row0[e] += s_gex[e] - s_gex[ep_first_of_owner(ep_owner_of(e, a.M, a.P), a.M, a.P)];
  __syncthreads();
}

__device__ __forceinline__ int expert_of_row(const int32_t* off, int M, int j) {
  // largest e with off[e] <= j (off non-decreasing; rows of empty experts are never hit)
  int lo = 0, hi = M - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= j) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void k_ep_publish(EpWin a, const int32_t* __restrict__ off) {
  for (int i = threadIdx.x; i < a.P * a.M; i += blockDim.x) {
    const int p = i / a.M, e = i - p * a.M;
    cnt_of(a, p)[(size_t)a.rank * a.M + e] = off[e + 1] - off[e];
  }
}

// one CTA: histogram of this rank's routing (pre-skip) and its importance into every window
__global__ void __launch_bounds__(1024) k_ep_publish_pre(EpWin a, const float* __restrict__ imp,
                                                         const int32_t* __restrict__ topk_idx,
                                                         int n_pairs) {
  __shared__ int h[DYMOE_MAX_EXPERTS];
  for (int e = threadIdx.x; e < a.M; e += blockDim.x) h[e] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n_pairs; i += blockDim.x) atomicAdd(&h[topk_idx[i]], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < a.P * a.M; i += blockDim.x) {
    const int p = i / a.M, e = i - p * a.M;
    cnt_of(a, p)[(size_t)a.rank * a.M + e] = h[e];
    imp_of(a, p)[(size_t)a.rank * a.M + e] = imp[e];
  }
}

__global__ void k_ep_reduce_imp(EpWin a, float* __restrict__ imp, uint8_t* __restrict__ active) {
  const float* src = imp_of(a, a.rank);
  const int32_t* cnt = cnt_of(a, a.rank);
  for (int e = threadIdx.x; e < a.M; e += blockDim.x) {
    float v = src[e];
    int c = cnt[e];
    for (int s = 1; s < a.P; ++s) {
      v = __fadd_rn(v, src[(size_t)s * a.M + e]);
      c += cnt[(size_t)s * a.M + e];
    }
    imp[e] = v;
    if (active) active[e] = c > 0;
  }
}

__global__ void k_ep_barrier(EpWin a, uint32_t epoch, uint32_t* status) {
  const int p = threadIdx.x;
  if (p < a.P) {
    // every write this stream issued before (previous kernels included) is ordered before the flag
    __threadfence_system();
    uint32_t* f = reinterpret_cast<uint32_t*>(a.peers[p] + a.L.flags) + a.rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.peers[a.rank] + a.L.flags) + p;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int)(v - epoch) >= 0) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > kBarrierTimeoutNs) {
        if (status) atomicOr(status, (uint32_t)DYMOE_STATUS_EP_TIMEOUT);
        break;
      }
      __nanosleep(64);
    }
  }
}

__global__ void __launch_bounds__(256) k_ep_dispatch(EpWin a, const uint4* __restrict__ x,
                                                      const int32_t* __restrict__ off,
                                                      const int32_t* __restrict__ perm_token,
                                                      int32_t* __restrict__ recv_off,
                                                      uint32_t* status) {
  __shared__ int s_row0[DYMOE_MAX_EXPERTS], s_gex[DYMOE_MAX_EXPERTS], s_tot[DYMOE_MAX_EXPERTS];
  __shared__ int s_off[DYMOE_MAX_EXPERTS + 1];
  ep_layout(a, s_row0, s_gex, s_tot);
  for (int e = threadIdx.x; e <= a.M; e += blockDim.x) s_off[e] = off[e];
  if (blockIdx.x == 0) {
    // local experts' offsets in this rank's own recv_x (the receiver side of the same layout),
    // clamped to the window: rows past cap_rows are never stored, so the FFN never reads them
    const int first = ep_first_of_owner(a.rank, a.M, a.P);
    const int last = ep_first_of_owner(a.rank + 1, a.M, a.P);
    for (int i = threadIdx.x; i <= last - first; i += blockDim.x) {
      const int v = i < last - first
                        ? s_gex[first + i] - s_gex[first]
                        : (last > first ? s_gex[last - 1] + s_tot[last - 1] - s_gex[first] : 0);
      recv_off[i] = min(v, a.cap);
      if (v > a.cap && i == last - first && status)
        atomicOr(status, (uint32_t)DYMOE_STATUS_EP_OVERFLOW);
    }
  }
  __syncthreads();
  const int R = s_off[a.M];
  const int vpr = a.Hd / 8;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x / 32;
  for (int j = blockIdx.x * warps + (threadIdx.x >> 5); j < R; j += gridDim.x * warps) {
    const int e = expert_of_row(s_off, a.M, j);
    const int dest = ep_owner_of(e, a.M, a.P);
    const int row = s_row0[e] + (j - s_off[e]);
    if (row >= a.cap) {
      if (lane == 0 && status) atomicOr(status, (uint32_t)DYMOE_STATUS_EP_OVERFLOW);
      continue;
    }
    const uint4* src = x + (size_t)perm_token[j] * vpr;
    uint4* dst = reinterpret_cast<uint4*>(a.peers[dest] + a.L.recv_x) + (size_t)row * vpr;
    for (int c = lane; c < vpr; c += 32) dst[c] = __ldg(src + c);
  }
}

__device__ __forceinline__ void store_out(void* y, int out_bf16, size_t at, float4 acc) {
  if (out_bf16) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&lo);
    o.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(y) + at) = o;
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + at) = acc;
  }
}

__device__ __forceinline__ float4 add_residual(float4 acc, const uint16_t* residual, size_t at) {
  if (residual == nullptr) return acc;
  const uint2 r = *reinterpret_cast<const uint2*>(residual + at);
  acc.x = __fadd_rn(__uint_as_float(r.x << 16), acc.x);
  acc.y = __fadd_rn(__uint_as_float(r.x & 0xffff0000u), acc.y);
  acc.z = __fadd_rn(__uint_as_float(r.y << 16), acc.z);
  acc.w = __fadd_rn(__uint_as_float(r.y & 0xffff0000u), acc.w);
  return acc;
}

__global__ void __launch_bounds__(128) k_ep_combine(EpWin a, const int32_t* __restrict__ inv_row,
                                                     const float* __restrict__ topk_w, int k,
                                                     const int32_t* __restrict__ off, int renorm,
                                                     int out_bf16, void* __restrict__ y,
                                                     const uint16_t* __restrict__ residual,
                                                     uint32_t* status) {
  __shared__ int s_row0[DYMOE_MAX_EXPERTS], s_gex[DYMOE_MAX_EXPERTS], s_tot[DYMOE_MAX_EXPERTS];
  __shared__ int s_off[DYMOE_MAX_EXPERTS + 1];
  for (int e = threadIdx.x; e <= a.M; e += blockDim.x) s_off[e] = off[e];
  ep_layout(a, s_row0, s_gex, s_tot);   // ends with a barrier: s_off is visible below
  const int t = blockIdx.x;
  const float* src[8];
  float wt[8];
  float denom = 0.f;
  for (int s = 0; s < k; ++s) {
    const int j = inv_row[(size_t)t * k + s];
    wt[s] = topk_w[(size_t)t * k + s];
    src[s] = nullptr;
    if (j >= 0) {
      denom += wt[s];
      const int e = expert_of_row(s_off, a.M, j);
      const int row = s_row0[e] + (j - s_off[e]);
      if (row < a.cap) {
        src[s] = reinterpret_cast<const float*>(a.peers[ep_owner_of(e, a.M, a.P)] + a.L.y_out) +
                 (size_t)row * a.Hd;
      } else if (status && threadIdx.x == 0 && blockIdx.y == 0) {
        // the row never reached its owner (dispatch overflow): a dead slot, flagged
        atomicOr(status, (uint32_t)DYMOE_STATUS_EP_OVERFLOW);
      }
    }
  }
  for (int s = 0; s < k; ++s) wt[s] = renorm ? wt[s] / denom : wt[s];
  for (int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4; c < a.Hd; c += gridDim.y * blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < k; ++s) {
      if (src[s] == nullptr) continue;
      const float4 v = *reinterpret_cast<const float4*>(src[s] + c);
      acc.x = __fadd_rn(acc.x, __fmul_rn(wt[s], v.x));
      acc.y = __fadd_rn(acc.y, __fmul_rn(wt[s], v.y));
      acc.z = __fadd_rn(acc.z, __fmul_rn(wt[s], v.z));
      acc.w = __fadd_rn(acc.w, __fmul_rn(wt[s], v.w));
    }
    const size_t at = (size_t)t * a.Hd + c;
    store_out(y, out_bf16, at, add_residual(acc, residual, at));
  }
}

// replicated decode: y[t] = out(residual + sum_src red[parity][t] of window src), src order
__global__ void __launch_bounds__(256) k_ep_reduce_red(EpWin a, int B, int out_bf16,
                                                        void* __restrict__ y,
                                                        const uint16_t* __restrict__ residual) {
  const size_t n4 = (size_t)B * a.Hd / 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(red_of(a, 0))[i];
    for (int s = 1; s < a.P; ++s) {
      const float4 v = reinterpret_cast<const float4*>(red_of(a, s))[i];
      acc.x = __fadd_rn(acc.x, v.x);
      acc.y = __fadd_rn(acc.y, v.y);
      acc.z = __fadd_rn(acc.z, v.z);
      acc.w = __fadd_rn(acc.w, v.w);
    }
    store_out(y, out_bf16, i * 4, add_residual(acc, residual, i * 4));
  }
}

}  // namespace

cudaError_t launch_ep_publish(const EpWin& w, const int32_t* off, cudaStream_t s) {
  k_ep_publish<<<1, 256, 0, s>>>(w, off);
  return cudaGetLastError();
}
cudaError_t launch_ep_publish_pre(const EpWin& w, const float* importance, const int32_t* topk_idx,
                                  int T, int k, cudaStream_t s) {
  k_ep_publish_pre<<<1, 1024, 0, s>>>(w, importance, topk_idx, T * k);
  return cudaGetLastError();
}
cudaError_t launch_ep_reduce_imp(const EpWin& w, float* importance, uint8_t* active, cudaStream_t s) {
  k_ep_reduce_imp<<<1, 256, 0, s>>>(w, importance, active);
  return cudaGetLastError();
}
cudaError_t launch_ep_barrier(const EpWin& w, uint32_t epoch, uint32_t* status, cudaStream_t s) {
  k_ep_barrier<<<1, kEpMaxP, 0, s>>>(w, epoch, status);
  return cudaGetLastError();
}
cudaError_t launch_ep_dispatch(const EpWin& w, const uint16_t* x, const int32_t* off,
                               const int32_t* perm_token, int32_t* recv_off, uint32_t* status,
                               cudaStream_t s) {
  // a fixed grid (the row count lives on the device): two CTAs of 8 warps per SM
  k_ep_dispatch<<<2 * 148, 256, 0, s>>>(w, reinterpret_cast<const uint4*>(x), off, perm_token,
                                        recv_off, status);
  return cudaGetLastError();
}
cudaError_t launch_ep_combine(const EpWin& w, const int32_t* inv_row, const float* topk_w, int T,
                              int k, const int32_t* off, int renorm, int out_dtype, void* y,
                              const uint16_t* residual, uint32_t* status, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const int chunks = (w.Hd + 511) / 512;
  int gy = (4 * 148 + T - 1) / T;
  gy = gy < 1 ? 1 : (gy > chunks ? chunks : gy);
  k_ep_combine<<<dim3(T, gy), 128, 0, s>>>(w, inv_row, topk_w, k, off, renorm,
                                           out_dtype == DYMOE_OUT_BF16, y, residual, status);
  return cudaGetLastError();
}
cudaError_t launch_ep_reduce_red(const EpWin& w, int B, int out_dtype, void* y,
                                 const uint16_t* residual, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const size_t n4 = (size_t)B * w.Hd / 4;
  const int blocks = (int)((n4 + 255) / 256 < 4 * 148 ? (n4 + 255) / 256 : 4 * 148);
  k_ep_reduce_red<<<blocks, 256, 0, s>>>(w, B, out_dtype == DYMOE_OUT_BF16, y, residual);
  return cudaGetLastError();
}
cudaError_t preload_ep() {
  return preload_kernels(k_ep_publish, k_ep_publish_pre, k_ep_reduce_imp, k_ep_barrier,
                         k_ep_dispatch, k_ep_combine, k_ep_reduce_red);
}

}  // namespace dymoe

namespace {

int check_window(const dymoe_ep_window* w) {
  using dymoe::set_error;
  if (!w) return set_error(DYMOE_ERR_INVALID, "window: must not be NULL");
  if (!w->peers) return set_error(DYMOE_ERR_INVALID, "window.peers: must not be NULL");
  if (w->M < 1 || w->M > DYMOE_MAX_EXPERTS)
    return set_error(DYMOE_ERR_INVALID, "window.M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  if (w->P < 1 || w->P > w->M || w->P > dymoe::kEpMaxP)
    return set_error(DYMOE_ERR_INVALID, "window.P: must satisfy 1 <= P <= min(M, %d)", dymoe::kEpMaxP);
  if (w->rank < 0 || w->rank >= w->P)
    return set_error(DYMOE_ERR_INVALID, "window.rank: must be in [0, P)");
  if (w->Hd <= 0 || w->Hd % 8 != 0)
    return set_error(DYMOE_ERR_INVALID, "window.Hd: must be a positive multiple of 8");
  if (w->cap_rows < 0) return set_error(DYMOE_ERR_INVALID, "window.cap_rows: must be >= 0");
  if (w->parity != 0 && w->parity != 1)
    return set_error(DYMOE_ERR_INVALID, "window.parity: must be 0 or 1");
  return DYMOE_OK;
}

dymoe::EpWin args_of(const dymoe_ep_window* w) {
  dymoe::EpWin a;
  a.P = w->P;
  a.rank = w->rank;
  a.M = w->M;
  a.Hd = w->Hd;
  a.cap = w->cap_rows;
  a.parity = w->parity;
  a.peers = reinterpret_cast<char* const*>(w->peers);
  a.bits = nullptr;
  a.L = dymoe::ep_win_layout(w->P, w->M, w->Hd, w->cap_rows);
  return a;
}

int cuda_err(cudaError_t e, const char* where) {
  return dymoe::set_error(DYMOE_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

int done(cudaError_t e, const char* where) {
  if (e != cudaSuccess) return cuda_err(e, where);
  dymoe::clear_error();
  return DYMOE_OK;
}

}  // namespace

extern "C" {

int dymoe_preload(void) {
  using namespace dymoe;
  cudaError_t e = preload_ep();
  cudaError_t (*const fns[])() = {preload_route_score, preload_permute_combine, preload_ffn_decode,
                                  preload_ffn_prefill,  preload_quantize,        preload_attn_mass,
                                  preload_predict,      preload_norm,            preload_api,
                                  preload_ep_layer};
  for (auto f : fns)
    if (e == cudaSuccess) e = f();
  return done(e, "dymoe_preload");
}

size_t dymoe_ep_window_bytes(int P, int M, int Hd, int cap_rows) {
  if (P < 1 || M < 1 || Hd < 1 || cap_rows < 0) return 0;
  return dymoe::ep_win_layout(P, M, Hd, cap_rows).total;
}

int dymoe_ep_window_alloc(size_t bytes, void** base, void* ipc_handle) {
  if (!base) return dymoe::set_error(DYMOE_ERR_INVALID, "base: must not be NULL");
  if (bytes == 0) return dymoe::set_error(DYMOE_ERR_INVALID, "bytes: must be > 0");
  *base = nullptr;
  // every kernel loaded before any peer can spin in a barrier (see dymoe_preload)
  int rc = dymoe_preload();
  if (rc) return rc;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return cuda_err(e, "dymoe_ep_window_alloc");
  e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess && ipc_handle) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, p);
    if (e == cudaSuccess) std::memcpy(ipc_handle, &h, sizeof(h));
  }
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_err(e, "dymoe_ep_window_alloc");
  }
  *base = p;
  return done(cudaSuccess, "");
}

int dymoe_ep_window_open(const void* ipc_handle, void** base) {
  if (!ipc_handle || !base) return dymoe::set_error(DYMOE_ERR_INVALID, "ipc_handle/base: must not be NULL");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  *base = nullptr;
  return done(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess), "dymoe_ep_window_open");
}

int dymoe_ep_window_close(void* base) {
  if (!base) return dymoe::set_error(DYMOE_ERR_INVALID, "base: must not be NULL");
  return done(cudaIpcCloseMemHandle(base), "dymoe_ep_window_close");
}

int dymoe_ep_window_free(void* base) {
  if (!base) return dymoe::set_error(DYMOE_ERR_INVALID, "base: must not be NULL");
  return done(cudaFree(base), "dymoe_ep_window_free");
}

int dymoe_ep_publish_counts(const dymoe_ep_window* w, const int32_t* expert_off,
                            dymoe_stream_t stream) {
  int rc = check_window(w);
  if (rc) return rc;
  if (!expert_off) return dymoe::set_error(DYMOE_ERR_INVALID, "expert_off: must not be NULL");
  return done(dymoe::launch_ep_publish(args_of(w), expert_off, (cudaStream_t)stream),
              "dymoe_ep_publish_counts");
}

int dymoe_ep_barrier(const dymoe_ep_window* w, uint32_t epoch, uint32_t* status,
                     dymoe_stream_t stream) {
  int rc = check_window(w);
  if (rc) return rc;
  return done(dymoe::launch_ep_barrier(args_of(w), epoch, status, (cudaStream_t)stream),
              "dymoe_ep_barrier");
}

int dymoe_ep_dispatch(const dymoe_ep_window* w, const uint16_t* x, int T,
                      const int32_t* expert_off, const int32_t* perm_token, int32_t* recv_off,
                      uint32_t* status, dymoe_stream_t stream) {
  int rc = check_window(w);
  if (rc) return rc;
  if (T < 0) return dymoe::set_error(DYMOE_ERR_INVALID, "T: must be >= 0");
  if (!expert_off || !recv_off || (T > 0 && (!x || !perm_token)))
    return dymoe::set_error(DYMOE_ERR_INVALID, "x/expert_off/perm_token/recv_off: must not be NULL");
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0)
    return dymoe::set_error(DYMOE_ERR_INVALID, "x: must be 16-byte aligned");
  return done(dymoe::launch_ep_dispatch(args_of(w), x, expert_off, perm_token, recv_off, status,
                                        (cudaStream_t)stream),
              "dymoe_ep_dispatch");
}

int dymoe_ep_combine(const dymoe_ep_window* w, const int32_t* inv_row, const float* topk_w,
                     int T, int k, const int32_t* expert_off, int renorm, int out_dtype, void* y,
                     uint32_t* status, dymoe_stream_t stream) {
  int rc = check_window(w);
  if (rc) return rc;
  if (T < 0) return dymoe::set_error(DYMOE_ERR_INVALID, "T: must be >= 0");
  if (k < 1 || k > 8) return dymoe::set_error(DYMOE_ERR_INVALID, "k: must be in [1, 8]");
  if (out_dtype != DYMOE_OUT_F32 && out_dtype != DYMOE_OUT_BF16)
    return dymoe::set_error(DYMOE_ERR_INVALID, "out_dtype: must be DYMOE_OUT_F32 or DYMOE_OUT_BF16");
  if (T == 0) return done(cudaSuccess, "");
  if (!inv_row || !topk_w || !expert_off || !y)
    return dymoe::set_error(DYMOE_ERR_INVALID, "inv_row/topk_w/expert_off/y: must not be NULL");
  return done(dymoe::launch_ep_combine(args_of(w), inv_row, topk_w, T, k, expert_off, renorm,
                                       out_dtype, y, nullptr, status, (cudaStream_t)stream),
              "dymoe_ep_combine");
}

}  // extern "C"
