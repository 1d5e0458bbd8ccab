// RMSNorm of the residual stream for the layer stack (Mixtral applies it before
// every MoE block, and the synthetic recipe's x ~ N(0, 1) is "as after an RMSNorm"):
//   u[t] = RNE_bf16(x[t] / sqrt(mean_i x[t][i]^2 + eps)),  unit weight (random-init stack).
// One CTA of 128 threads per token row; each thread sums the squares of its 16-byte granules in
// order (fp32 FMA), then a warp butterfly and the 4 warp sums in order; one rsqrt.
// Roofline: HBM (T x Hd bf16 read once, written once; a few microseconds per layer).
#include "../dymoe_internal.cuh"

namespace dymoe {

__global__ void __launch_bounds__(128) k_rmsnorm(const uint4* __restrict__ x, int vpr, float inv_hd,
                                                 float eps, uint4* __restrict__ u) {
  __shared__ float wsum[4];
  const int t = blockIdx.x;
  const uint4* xr = x + (size_t)t * vpr;
  uint4* ur = u + (size_t)t * vpr;
  float ss = 0.f;
  for (int c = threadIdx.x; c < vpr; c += blockDim.x) {
    const uint4 v = xr[c];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float lo = __uint_as_float(w[q] << 16), hi = __uint_as_float(w[q] & 0xffff0000u);
      ss = __fmaf_rn(lo, lo, ss);
      ss = __fmaf_rn(hi, hi, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = ss;
  __syncthreads();
  const float tot = __fadd_rn(__fadd_rn(__fadd_rn(wsum[0], wsum[1]), wsum[2]), wsum[3]);
  const float r = rsqrtf(__fadd_rn(__fmul_rn(tot, inv_hd), eps));
  for (int c = threadIdx.x; c < vpr; c += blockDim.x) {
    const uint4 v = xr[c];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 p = __floats2bfloat162_rn(__fmul_rn(__uint_as_float(w[q] << 16), r),
                                               __fmul_rn(__uint_as_float(w[q] & 0xffff0000u), r));
      o[q] = *reinterpret_cast<uint32_t*>(&p);
    }
    ur[c] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

cudaError_t launch_rmsnorm(const uint16_t* x, int T, int Hd, float eps, uint16_t* u, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  k_rmsnorm<<<T, 128, 0, s>>>(reinterpret_cast<const uint4*>(x), Hd / 8, 1.f / (float)Hd, eps,
                              reinterpret_cast<uint4*>(u));
  return cudaGetLastError();
}

cudaError_t preload_norm() { return preload_kernels(k_rmsnorm); }

}  // namespace dymoe
