// Group-wise runtime quantization + bit packing (row a4) for sm_100a.
//
// Paper: experts quantized with GPTQ at 4/2 bits; readings D14-D16: round-to-
// nearest on GPTQ's asymmetric min-max grid, G = 128 along K, fp32 scale, u8 zero, reciprocal
// form.  Per group, in fp32 with one rounding per operation (explicit _rn intrinsics, so nvcc
// cannot contract anything into an FMA):
//   mn = min(0, min w), mx = max(0, max w), s = (mx - mn) / maxq;
//   s < 2^-126 -> (mn, mx) = (-1, +1), s recomputed (D14b);
//   inv = 1/s; z = rint(-mn * inv); q = clamp(rint(w * inv) + z, 0, maxq)
//
// HBM-bound: per weight it reads 2 B and writes b/8 B (+5 B per group).  Mapping: a half-warp
// (16 lanes x 16 B = 128 bf16) owns one group; lanes min/max-reduce with 4 xor-shuffles inside
// the half-warp, quantize their 8 weights and write their packed bits contiguously, so a warp
// reads 512 contiguous bytes and writes 64 (int2) .. 256 (int8) contiguous bytes per group
// pair.  Each thread keeps UNROLL groups of loads in flight.  Grid: a multiple of the SM
// count (grid-stride over group pairs), so one launch covers any number of matrices.
#include "../dymoe_internal.cuh"

namespace dymoe {

struct QJob {
  const uint16_t* W;
  uint32_t* codes;
  float* scales;
  uint8_t* zeros;
  long long first_pair;  // global index of this job's first group pair
  int N, K, bits;
};

constexpr int kMaxJobs = 64;
struct QJobs {
  QJob j[kMaxJobs];
  int n;
  long long total_pairs;
};

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

template <int BITS>
__device__ __forceinline__ void quant_group(const uint4 raw, int lane16, long long grp_in_job,
                                            const QJob& J, bool valid) {
  // grp_in_job: index of this half-warp's group within the job (row-major over [N][K/128])
  float w[8] = {bf16lo(raw.x), bf16hi(raw.x), bf16lo(raw.y), bf16hi(raw.y),
                bf16lo(raw.z), bf16hi(raw.z), bf16lo(raw.w), bf16hi(raw.w)};
  float mn = 0.f, mx = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mn = fminf(mn, w[i]);
    mx = fmaxf(mx, w[i]);
  }
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) {  // xor within the 16-lane half
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  }
  constexpr float maxq = (float)((1 << BITS) - 1);
  float s = __fdiv_rn(__fsub_rn(mx, mn), maxq);
  if (!(s >= 1.17549435e-38f)) {  // s < 2^-126 (D14b)
    mn = -1.f;
    mx = 1.f;
    s = __fdiv_rn(__fsub_rn(mx, mn), maxq);
  }
  const float inv = __frcp_rn(s);
  const float z = rintf(__fmul_rn(-mn, inv));
  uint32_t q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float v = __fadd_rn(rintf(__fmul_rn(w[i], inv)), z);
    v = fminf(fmaxf(v, 0.f), maxq);
    q[i] = (uint32_t)v;
  }
  const int K = J.K;
  const long long gpr = K / DYMOE_GROUP;           // groups per row
  const long long row = grp_in_job / gpr;
  const long long g = grp_in_job - row * gpr;
  // packed words of this lane: lane16 covers k = g*128 + lane16*8 .. +8
  uint32_t* rowp = J.codes + row * ((long long)K * BITS / 32);
  if (BITS == 8) {
    uint2 o;
    o.x = q[0] | q[1] << 8 | q[2] << 16 | q[3] << 24;
    o.y = q[4] | q[5] << 8 | q[6] << 16 | q[7] << 24;
    if (valid) reinterpret_cast<uint2*>(rowp)[(g * 128 + lane16 * 8) / 8] = o;
  } else if (BITS == 4) {
    uint32_t o = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) o |= q[i] << (4 * i);
    if (valid) rowp[(g * 128 + lane16 * 8) / 8] = o;
  } else {  // BITS == 2: 16 bits per lane, pair lanes (even | odd << 16)
    uint32_t o = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) o |= q[i] << (2 * i);
    uint32_t other = __shfl_xor_sync(0xffffffffu, o, 1);
    if (valid && (lane16 & 1) == 0) rowp[(g * 128 + lane16 * 8) / 16] = o | (other << 16);
  }
  if (valid && lane16 == 0) {
    J.scales[grp_in_job] = s;
    J.zeros[grp_in_job] = (uint8_t)z;
  }
}

constexpr int kQuantUnroll = 4;

__global__ void __launch_bounds__(256) k_quantize(const __grid_constant__ QJobs jobs) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4, lane16 = lane & 15;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  // each warp handles kQuantUnroll consecutive pairs per iteration
  for (long long base = warp * kQuantUnroll; base < jobs.total_pairs;
       base += nwarps * kQuantUnroll) {
    uint4 raw[kQuantUnroll];
    int jid[kQuantUnroll];
    long long gij[kQuantUnroll];
    bool ok[kQuantUnroll];
#pragma unroll
    for (int u = 0; u < kQuantUnroll; ++u) {
      const long long pair = base + u;
      ok[u] = pair < jobs.total_pairs;
      int jj = 0;
      if (ok[u]) {
        while (jj + 1 < jobs.n && jobs.j[jj + 1].first_pair <= pair) ++jj;
      }
      jid[u] = jj;
      const QJob& J = jobs.j[jj];
      const long long ngroups = (long long)J.N * (J.K / DYMOE_GROUP);
      gij[u] = (pair - J.first_pair) * 2 + half;
      ok[u] = ok[u] && gij[u] < ngroups;
      raw[u] = make_uint4(0, 0, 0, 0);
      if (ok[u]) {
        const long long gpr = J.K / DYMOE_GROUP;
        const long long row = gij[u] / gpr, g = gij[u] - row * gpr;
        const uint4* src = reinterpret_cast<const uint4*>(J.W + row * J.K + g * DYMOE_GROUP);
        raw[u] = __ldcs(src + lane16);  // streamed once: evict-first
      }
    }
#pragma unroll
    for (int u = 0; u < kQuantUnroll; ++u) {
      const QJob& J = jobs.j[jid[u]];
      // the half-warp shuffles need all 32 lanes: compute even when !ok, store only if ok
      switch (J.bits) {
        case 2: quant_group<2>(raw[u], lane16, gij[u], J, ok[u]); break;
        case 4: quant_group<4>(raw[u], lane16, gij[u], J, ok[u]); break;
        default: quant_group<8>(raw[u], lane16, gij[u], J, ok[u]); break;
      }
    }
  }
}

// Derived dequant metadata: meta[i] = bf16bits(RNE_bf16(scales[i])) << 16 | zeros[i].
__global__ void __launch_bounds__(256) k_build_meta(const float* __restrict__ scales,
                                                    const uint8_t* __restrict__ zeros, size_t n,
                                                    uint32_t* __restrict__ meta) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const __nv_bfloat16 sb = __float2bfloat16_rn(scales[i]);
    meta[i] = ((uint32_t)*reinterpret_cast<const uint16_t*>(&sb) << 16) | (uint32_t)zeros[i];
  }
}

cudaError_t launch_build_meta(const float* scales, const uint8_t* zeros, size_t n, uint32_t* meta,
                              cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const size_t blocks = (n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192;
  k_build_meta<<<(unsigned)blocks, 256, 0, s>>>(scales, zeros, n, meta);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const dymoe_quant_job* jobs_host, int n_jobs, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int start = 0; start < n_jobs; start += kMaxJobs) {
    QJobs J{};
    J.n = 0;
    long long pairs = 0;
    for (int i = start; i < n_jobs && J.n < kMaxJobs; ++i) {
      const dymoe_quant_job& h = jobs_host[i];
      const long long ng = (long long)h.N * (h.K / DYMOE_GROUP);
      if (ng == 0) continue;
      QJob& q = J.j[J.n++];
      q.W = h.W; q.codes = h.codes; q.scales = h.scales; q.zeros = h.zeros;
      q.N = h.N; q.K = h.K; q.bits = h.bits;
      q.first_pair = pairs;
      pairs += (ng + 1) / 2;
    }
    J.total_pairs = pairs;
    if (pairs == 0) continue;
    const long long warps_needed = (pairs + kQuantUnroll - 1) / kQuantUnroll;
    long long blocks = (warps_needed + 7) / 8;
    const long long cap = (long long)sms * 8;   // 8 CTAs of 256 threads per SM resident
    if (blocks > cap) blocks = cap;
    k_quantize<<<(unsigned)blocks, 256, 0, s>>>(J);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace dymoe
