// Look-ahead prediction of the next layer's experts (Eqs. 6-8,
// P:275-298), for sm_100a.  Readings P1-P3:
//   Eq. 6  logits = h^(l) · W_g^(l+1)^T in fp32, accumulation depth <= Hd/32 + 5 (the accuracy
//          contract of include/dymoe.h, reading P1); g_hat = softmax (routing kernel);
//   Eq. 7  prefill: c_e = #{tokens whose top-k_route predicted experts contain e} (exact ints);
//   Eq. 8  decode:  predicted demand = decode importance of the predicted gate (B = 1: the
//          logit row; B > 1: sum_b g_hat[b], fp32 in b order -- the decode scoring kernel);
//   requests = top-t by (value desc, index asc); prefill drops c_e = 0.
// Roofline: HBM (h [T][Hd] read once, W_g^(l+1) [M][Hd] from L2); microseconds per layer.
#include "../dymoe_internal.cuh"

namespace dymoe {

// one warp per (token, expert): lane l accumulates the 8-element chunks l, l + 32, l + 64, ...
// of the dot product in order (16-byte loads, fp32 FMA: Hd/32 roundings per lane), then an xor
// butterfly over the lanes (5 more): the depth the header's error bound states
__global__ void __launch_bounds__(256) k_gate_logits(const uint4* __restrict__ h,
                                                     const uint4* __restrict__ w, int T, int Hd,
                                                     int M, const float* __restrict__ bias,
                                                     float* __restrict__ logits) {
  const long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= (long long)T * M) return;
  const int t = (int)(i / M), e = (int)(i - (long long)t * M);
  const uint4* hp = h + (size_t)t * (Hd / 8);
  const uint4* wp = w + (size_t)e * (Hd / 8);
  float acc = 0.f;
  for (int c = lane; c < Hd / 8; c += 32) {
    const uint4 a = __ldg(hp + c), b = __ldg(wp + c);
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc = __fmaf_rn(__uint_as_float(aw[q] << 16), __uint_as_float(bw[q] << 16), acc);
      acc = __fmaf_rn(__uint_as_float(aw[q] & 0xffff0000u), __uint_as_float(bw[q] & 0xffff0000u), acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if (lane == 0) logits[i] = bias != nullptr ? __fadd_rn(acc, bias[e]) : acc;
}

cudaError_t launch_gate_logits(const uint16_t* h, const uint16_t* wg, const float* bias, int T,
                               int Hd, int M, float* logits, cudaStream_t s) {
  const long long n = (long long)T * M * 32;   // one warp per (token, expert)
  if (n == 0) return cudaSuccess;
  k_gate_logits<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(reinterpret_cast<const uint4*>(h),
                                                           reinterpret_cast<const uint4*>(wg), T,
                                                           Hd, M, bias, logits);
  return cudaGetLastError();
}

__global__ void k_predict_counts(const int32_t* __restrict__ topk_idx, int n, int M,
                                 float* __restrict__ counts) {
  __shared__ int c[DYMOE_MAX_EXPERTS];
  for (int e = threadIdx.x; e < M; e += blockDim.x) c[e] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&c[topk_idx[i]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < M; e += blockDim.x) counts[e] = (float)c[e];   // exact (< 2^24)
}

// thread e: rank = #{j : v_j > v_e or (v_j == v_e and j < e)}
__global__ void k_select_top(const float* __restrict__ v, int M, int t, int drop_zero,
                             int32_t* __restrict__ experts, float* __restrict__ priority,
                             int32_t* __restrict__ n_out) {
  __shared__ float s[DYMOE_MAX_EXPERTS];
  __shared__ int n_valid;
  const int e = threadIdx.x;
  if (e == 0) n_valid = 0;
  if (e < M) s[e] = v[e];
  __syncthreads();
  if (e < M) {
    const float ve = s[e];
    int rank = 0;
    for (int j = 0; j < M; ++j) rank += (s[j] > ve) || (s[j] == ve && j < e);
    const bool ok = !drop_zero || ve > 0.f;
    if (ok) atomicAdd(&n_valid, 1);
    if (ok && rank < t) {
      experts[rank] = e;
      priority[rank] = ve;
    }
  }
  __syncthreads();
  if (e == 0) *n_out = min(t, n_valid);
}

cudaError_t launch_predict_next(int phase, const uint16_t* h, const uint16_t* wg, int T, int Hd,
                                int M, int k, int t, float* logits, int32_t* topk_idx,
                                float* topk_w, float* probs, float* value, int32_t* experts,
                                float* priority, int32_t* n_out, cudaStream_t s) {
  cudaError_t e = launch_gate_logits(h, wg, nullptr, T, Hd, M, logits, s);
  if (e != cudaSuccess) return e;
  if (phase == DYMOE_PREFILL) {
    e = launch_route(logits, T, M, k, topk_idx, topk_w, probs, s);
    if (e != cudaSuccess) return e;
    k_predict_counts<<<1, 1024, 0, s>>>(topk_idx, T * k, M, value);
  } else {
    e = launch_score_decode(logits, T, M, value, s);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_select_top<<<1, 256, 0, s>>>(value, M, t, phase == DYMOE_PREFILL, experts, priority, n_out);
  return cudaGetLastError();
}

cudaError_t preload_predict() {
  return preload_kernels(k_gate_logits, k_predict_counts, k_select_top);
}

}  // namespace dymoe
