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

namespace {

constexpr int kMaxP = 64;
constexpr unsigned long long kBarrierTimeoutNs = 5ull * 1000 * 1000 * 1000;

struct WinLayout {
  size_t flags, cnt, recv_x, y_out, total;
};

__host__ __device__ inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

__host__ __device__ inline WinLayout win_layout(int P, int M, int Hd, int cap) {
  WinLayout L;
  L.flags = 0;
  L.cnt = align256((size_t)P * 4);
  L.recv_x = L.cnt + align256((size_t)2 * P * M * 4);
  L.y_out = L.recv_x + align256((size_t)cap * Hd * 2);
  L.total = L.y_out + align256((size_t)cap * Hd * 4);
  return L;
}

struct WinArgs {
  int P, rank, M, Hd, cap, parity;
  char* const* peers;
  WinLayout L;
};

__device__ __forceinline__ int owner_of(int e, int M, int P) {
  return (int)(((long long)e * P) / M);
}

__device__ __forceinline__ int32_t* cnt_of(const WinArgs& a, int p) {
  return reinterpret_cast<int32_t*>(a.peers[p] + a.L.cnt) + (size_t)a.parity * a.P * a.M;
}

// Row layout of the step (computed from this rank's own, complete count matrix):
//   tot[e]  = sum_src cnt[src][e];  gex[e] = sum_{e' < e} tot[e'] (global exclusive prefix)
//   base(e) = gex[e] - gex[first expert of owner(e)]  (expert e's first row in its owner's recv_x)
//   row0[e] = base(e) + sum_{src < rank} cnt[src][e]   (this rank's first row of expert e there)
// The prefix is one warp scan over contiguous blocks of experts (owners hold contiguous expert
// blocks, so a per-owner base is a difference of the global prefix).
__device__ __forceinline__ int first_of_owner(int o, int M, int P) {
  return (int)(((long long)o * M + P - 1) / P);
}

__device__ void ep_layout(const WinArgs& a, int* s_row0, int* s_gex, int* s_tot) {
  const int32_t* cnt = cnt_of(a, a.rank);
  for (int e = threadIdx.x; e < a.M; e += blockDim.x) {
    int tot = 0, pre = 0;
    for (int s = 0; s < a.P; ++s) {
      const int c = cnt[(size_t)s * a.M + e];
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
    s_row0[e] += s_gex[e] - s_gex[first_of_owner(owner_of(e, a.M, a.P), a.M, a.P)];
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

__global__ void k_ep_publish(WinArgs a, const int32_t* __restrict__ off) {
  for (int i = threadIdx.x; i < a.P * a.M; i += blockDim.x) {
    const int p = i / a.M, e = i - p * a.M;
    cnt_of(a, p)[(size_t)a.rank * a.M + e] = off[e + 1] - off[e];
  }
}

__global__ void k_ep_barrier(WinArgs a, uint32_t epoch, uint32_t* status) {
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

__global__ void __launch_bounds__(256) k_ep_dispatch(WinArgs a, const uint4* __restrict__ x,
                                                      const int32_t* __restrict__ off,
                                                      const int32_t* __restrict__ perm_token,
                                                      int32_t* __restrict__ recv_off,
                                                      uint32_t* status) {
  __shared__ int s_row0[DYMOE_MAX_EXPERTS], s_gex[DYMOE_MAX_EXPERTS], s_tot[DYMOE_MAX_EXPERTS];
  __shared__ int s_off[DYMOE_MAX_EXPERTS + 1];
  ep_layout(a, s_row0, s_gex, s_tot);
  for (int e = threadIdx.x; e <= a.M; e += blockDim.x) s_off[e] = off[e];
  if (blockIdx.x == 0) {
    // local experts' offsets in this rank's own recv_x (the receiver side of the same layout)
    const int first = first_of_owner(a.rank, a.M, a.P);
    const int last = first_of_owner(a.rank + 1, a.M, a.P);
    for (int i = threadIdx.x; i <= last - first; i += blockDim.x)
      recv_off[i] = i < last - first ? s_gex[first + i] - s_gex[first]
                                     : (last > first ? s_gex[last - 1] + s_tot[last - 1] - s_gex[first] : 0);
  }
  __syncthreads();
  const int R = s_off[a.M];
  const int vpr = a.Hd / 8;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x / 32;
  for (int j = blockIdx.x * warps + (threadIdx.x >> 5); j < R; j += gridDim.x * warps) {
    const int e = expert_of_row(s_off, a.M, j);
    const int dest = owner_of(e, a.M, a.P);
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

__global__ void __launch_bounds__(128) k_ep_combine(WinArgs a, const int32_t* __restrict__ inv_row,
                                                     const float* __restrict__ topk_w, int k,
                                                     const int32_t* __restrict__ off, int renorm,
                                                     int out_bf16, void* __restrict__ y) {
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
      src[s] = reinterpret_cast<const float*>(a.peers[owner_of(e, a.M, a.P)] + a.L.y_out) +
               (size_t)row * a.Hd;
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
    if (out_bf16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(y) + (size_t)t * a.Hd + c) = o;
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + (size_t)t * a.Hd + c) = acc;
    }
  }
}

int check_window(const dymoe_ep_window* w) {
  using dymoe::set_error;
  if (!w) return set_error(DYMOE_ERR_INVALID, "window: must not be NULL");
  if (!w->peers) return set_error(DYMOE_ERR_INVALID, "window.peers: must not be NULL");
  if (w->M < 1 || w->M > DYMOE_MAX_EXPERTS)
    return set_error(DYMOE_ERR_INVALID, "window.M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  if (w->P < 1 || w->P > w->M || w->P > kMaxP)
    return set_error(DYMOE_ERR_INVALID, "window.P: must satisfy 1 <= P <= min(M, %d)", kMaxP);
  if (w->rank < 0 || w->rank >= w->P)
    return set_error(DYMOE_ERR_INVALID, "window.rank: must be in [0, P)");
  if (w->Hd <= 0 || w->Hd % 8 != 0)
    return set_error(DYMOE_ERR_INVALID, "window.Hd: must be a positive multiple of 8");
  if (w->cap_rows < 0) return set_error(DYMOE_ERR_INVALID, "window.cap_rows: must be >= 0");
  if (w->parity != 0 && w->parity != 1)
    return set_error(DYMOE_ERR_INVALID, "window.parity: must be 0 or 1");
  return DYMOE_OK;
}

WinArgs args_of(const dymoe_ep_window* w) {
  WinArgs a;
  a.P = w->P;
  a.rank = w->rank;
  a.M = w->M;
  a.Hd = w->Hd;
  a.cap = w->cap_rows;
  a.parity = w->parity;
  a.peers = reinterpret_cast<char* const*>(w->peers);
  a.L = win_layout(w->P, w->M, w->Hd, w->cap_rows);
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
  cudaError_t e = preload_kernels(k_ep_publish, k_ep_barrier, k_ep_dispatch, k_ep_combine);
  cudaError_t (*const fns[])() = {preload_route_score, preload_permute_combine, preload_ffn_decode,
                                  preload_ffn_prefill,  preload_quantize,        preload_attn_mass,
                                  preload_predict,      preload_norm,            preload_api};
  for (auto f : fns)
    if (e == cudaSuccess) e = f();
  return done(e, "dymoe_preload");
}

size_t dymoe_ep_window_bytes(int P, int M, int Hd, int cap_rows) {
  if (P < 1 || M < 1 || Hd < 1 || cap_rows < 0) return 0;
  return win_layout(P, M, Hd, cap_rows).total;
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
  k_ep_publish<<<1, 256, 0, (cudaStream_t)stream>>>(args_of(w), expert_off);
  return done(cudaGetLastError(), "dymoe_ep_publish_counts");
}

int dymoe_ep_barrier(const dymoe_ep_window* w, uint32_t epoch, uint32_t* status,
                     dymoe_stream_t stream) {
  int rc = check_window(w);
  if (rc) return rc;
  k_ep_barrier<<<1, kMaxP, 0, (cudaStream_t)stream>>>(args_of(w), epoch, status);
  return done(cudaGetLastError(), "dymoe_ep_barrier");
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
  // a fixed grid (the row count lives on the device): two CTAs of 8 warps per SM
  k_ep_dispatch<<<2 * 148, 256, 0, (cudaStream_t)stream>>>(
      args_of(w), reinterpret_cast<const uint4*>(x), expert_off, perm_token, recv_off, status);
  return done(cudaGetLastError(), "dymoe_ep_dispatch");
}

int dymoe_ep_combine(const dymoe_ep_window* w, const int32_t* inv_row, const float* topk_w,
                     int T, int k, const int32_t* expert_off, int renorm, int out_dtype, void* y,
                     dymoe_stream_t stream) {
  int rc = check_window(w);
  if (rc) return rc;
  if (T < 0) return dymoe::set_error(DYMOE_ERR_INVALID, "T: must be >= 0");
  if (k < 1 || k > 8) return dymoe::set_error(DYMOE_ERR_INVALID, "k: must be in [1, 8]");
  if (out_dtype != DYMOE_OUT_F32 && out_dtype != DYMOE_OUT_BF16)
    return dymoe::set_error(DYMOE_ERR_INVALID, "out_dtype: must be DYMOE_OUT_F32 or DYMOE_OUT_BF16");
  if (T == 0) return done(cudaSuccess, "");
  if (!inv_row || !topk_w || !expert_off || !y)
    return dymoe::set_error(DYMOE_ERR_INVALID, "inv_row/topk_w/expert_off/y: must not be NULL");
  const int chunks = (w->Hd + 511) / 512;
  int gy = (4 * 148 + T - 1) / T;
  gy = gy < 1 ? 1 : (gy > chunks ? chunks : gy);
  k_ep_combine<<<dim3(T, gy), 128, 0, (cudaStream_t)stream>>>(
      args_of(w), inv_row, topk_w, k, expert_off, renorm, out_dtype == DYMOE_OUT_BF16, y);
  return done(cudaGetLastError(), "dymoe_ep_combine");
}

}  // extern "C"
