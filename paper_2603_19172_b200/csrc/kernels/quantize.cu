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
// HBM-bound in bytes (2 B read + b/8 B written per weight) but, at HBM rate, tight in ALU issue
// slots (~2.6 T weights/s).  So one LANE owns one whole 128-weight group: the per-group scalar
// work (two IEEE divisions, z) is amortised over 128 weights instead of 8, the min/max runs on
// packed bf16 pairs (HMNMX2, exact), and rint(w*inv) uses the 1.5*2^23 magic add (exact
// round-half-even for |x| < 2^22) whose bit pattern is the integer, so one IADD also adds z.
// A warp owns 32 consecutive groups = 8 KB of contiguous input, which it stages through its own
// shared-memory buffer with coalesced 16-byte cp.async (each instruction covers 512 contiguous
// bytes; rows padded to 272 B so that the per-lane 16-byte reads are bank-conflict free), double
// buffered: the next 8 KB is in flight while the lanes quantize the current one.  Each lane
// writes its group's packed codes back into its own staging row (it has read the row into
// registers), and the warp then stores the 32 groups' codes -- one contiguous 1-4 KB range --
// with 16-byte stores of 512 contiguous bytes per instruction (a lane storing its own 128-byte
// group directly made every store instruction touch 32 separate lines).  Jobs are padded to whole
// warps, so a warp never straddles two matrices; groups past a job's end are zero-filled and not
// stored.
#include "../dymoe_internal.cuh"

namespace dymoe {

struct QJob {
  const uint16_t* W;
  uint32_t* codes;
  float* scales;
  uint8_t* zeros;
  long long first_warp;  // global warp index of this job's first 32 groups
  long long n_groups;
  int K, bits;
};

constexpr int kMaxJobs = 64;
struct QJobs {
  QJob j[kMaxJobs];
  int n;
  long long total_warps;
};

__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmin2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

// one code: clamp(rint(w * inv) + z, 0, maxq) with w the bf16 in the high (hi=1) / low half of u
template <int BITS>
__device__ __forceinline__ uint32_t qcode(uint32_t u, bool hi, float inv, int zbias) {
  const float w = __uint_as_float(hi ? (u & 0xffff0000u) : (u << 16));
  // |w * inv| <= maxq + 1 < 2^22, so adding 1.5 * 2^23 rounds to an integer (half to even) and
  // the low mantissa bits hold it in two's-complement offset by 0x4B400000
  const float t = __fadd_rn(__fmul_rn(w, inv), 12582912.0f);
  int q = (int)__float_as_uint(t) - zbias;   // zbias = 0x4B400000 - z
  q = max(q, 0);
  q = min(q, (1 << BITS) - 1);
  return (uint32_t)q;
}

constexpr int kQWarps = 4;               // warps per CTA
constexpr int kRow = 272;                // padded bytes per staged group (256 + 16)
constexpr int kBuf = 32 * kRow;          // one warp's 32 groups

// stage the 32 groups of warp-item w (global warp index) of job J into smem buffer `buf`
__device__ __forceinline__ void stage_groups(const QJob& J, long long w, long long first_warp,
                                             uint32_t buf, int lane) {
  const long long g0 = (w - first_warp) * 32;
  const char* base = reinterpret_cast<const char*>(J.W) + g0 * 256;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int gl = 2 * j + (lane >> 4);                 // group within the warp's 32
    const uint32_t dst = buf + gl * kRow + (lane & 15) * 16;
    const bool ok = g0 + gl < J.n_groups;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                 "l"(base + j * 512 + lane * 16), "r"(ok ? 16 : 0) : "memory");
  }
}

template <int BITS>
__device__ __forceinline__ void quant_lane_group(const QJob& J, long long g, uint32_t row) {
  constexpr float maxq = (float)((1 << BITS) - 1);
  uint4 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i)
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w) : "r"(row + i * 16));
  // packed min / max over the 64 bf16 pairs (exact), then the two halves, then 0 (GPTQ grid)
  uint32_t mn2 = v[0].x, mx2 = v[0].x;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t a[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mn2 = hmin2(mn2, a[j]);
      mx2 = hmax2(mx2, a[j]);
    }
  }
  float mn = fminf(__uint_as_float(mn2 << 16), __uint_as_float(mn2 & 0xffff0000u));
  float mx = fmaxf(__uint_as_float(mx2 << 16), __uint_as_float(mx2 & 0xffff0000u));
  mn = fminf(mn, 0.f);
  mx = fmaxf(mx, 0.f);
  float s = __fdiv_rn(__fsub_rn(mx, mn), maxq);
  if (!(s >= 1.17549435e-38f)) {  // s < 2^-126 (D14b)
    mn = -1.f;
    s = __fdiv_rn(2.f, maxq);
  }
  const float inv = __frcp_rn(s);
  const float zf = rintf(__fmul_rn(-mn, inv));
  const int z = (int)zf;
  const int zbias = 0x4B400000 - z;
  J.scales[g] = s;
  J.zeros[g] = (uint8_t)z;
  // codes: group g's 128*BITS/8 bytes go to the start of this lane's staging row (already read
  // into v); the warp stores them to global memory afterwards (store_codes)
  auto sts = [&](int i, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(row + i * 16), "r"(a), "r"(b), "r"(c),
                 "r"(d) : "memory");
  };
  if constexpr (BITS == 8) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {   // 16 codes per 16-byte store
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 a = v[i + h];
        o[2 * h] = qcode<8>(a.x, false, inv, zbias) | qcode<8>(a.x, true, inv, zbias) << 8 |
                   qcode<8>(a.y, false, inv, zbias) << 16 | qcode<8>(a.y, true, inv, zbias) << 24;
        o[2 * h + 1] = qcode<8>(a.z, false, inv, zbias) | qcode<8>(a.z, true, inv, zbias) << 8 |
                       qcode<8>(a.w, false, inv, zbias) << 16 | qcode<8>(a.w, true, inv, zbias) << 24;
      }
      sts(i / 2, o[0], o[1], o[2], o[3]);
    }
  } else if constexpr (BITS == 4) {
#pragma unroll
    for (int i = 0; i < 16; i += 4) {   // 32 codes per 16-byte store
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const uint4 a = v[i + h];
        const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          word |= (qcode<4>(w4[j], false, inv, zbias) | qcode<4>(w4[j], true, inv, zbias) << 4) << (8 * j);
        o[h] = word;
      }
      sts(i / 4, o[0], o[1], o[2], o[3]);
    }
  } else {   // 2
#pragma unroll
    for (int i = 0; i < 16; i += 8) {   // 64 codes per 16-byte store
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        uint32_t word = 0;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint4 a = v[i + 2 * h + hh];
          const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            word |= (qcode<2>(w4[j], false, inv, zbias) | qcode<2>(w4[j], true, inv, zbias) << 2)
                    << (16 * hh + 4 * j);
        }
        o[h] = word;
      }
      sts(i / 8, o[0], o[1], o[2], o[3]);
    }
  }
}

// The warp's 32 staged groups (BITS 16-byte chunks each, at the start of each staging row) ->
// contiguous global codes, 32 consecutive chunks per store instruction.
__device__ __forceinline__ void store_codes(const QJob& J, long long g0, uint32_t buf, int lane) {
  const long long left = J.n_groups - g0;
  const int ng = left < 32 ? (int)left : 32;
  const int nch = ng * J.bits;                    // 16-byte chunks (BITS per group)
  uint4* dst = reinterpret_cast<uint4*>(J.codes) + g0 * J.bits;
  for (int c = lane; c < nch; c += 32) {
    const int gl = c / J.bits, off = c - gl * J.bits;
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(buf + gl * kRow + off * 16));
    dst[c] = v;
  }
}

__global__ void __launch_bounds__(kQWarps * 32) k_quantize(const __grid_constant__ QJobs jobs) {
  extern __shared__ __align__(16) uint8_t qsm[];
  const int lane = threadIdx.x & 31;
  const uint32_t buf0 = (uint32_t)__cvta_generic_to_shared(qsm) + (threadIdx.x >> 5) * (2 * kBuf);
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  auto job_of = [&](long long ww) {
    int jj = 0;
    while (jj + 1 < jobs.n && jobs.j[jj + 1].first_warp <= ww) ++jj;
    return jj;
  };
  if (w >= jobs.total_warps) return;
  int jj = job_of(w);
  stage_groups(jobs.j[jj], w, jobs.j[jj].first_warp, buf0, lane);
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int it = 0; w < jobs.total_warps; w += nwarps, ++it) {
    const uint32_t cur = buf0 + (it & 1) * kBuf;
    // prefetch the next item into the other buffer, then wait for the current one
    const long long wn = w + nwarps;
    int jn = jj;
    if (wn < jobs.total_warps) {
      jn = job_of(wn);
      stage_groups(jobs.j[jn], wn, jobs.j[jn].first_warp, buf0 + ((it + 1) & 1) * kBuf, lane);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const QJob& J = jobs.j[jj];
    const long long g = (w - J.first_warp) * 32 + lane;
    if (g < J.n_groups) {
      const uint32_t row = cur + lane * kRow;
      switch (J.bits) {
        case 2: quant_lane_group<2>(J, g, row); break;
        case 4: quant_lane_group<4>(J, g, row); break;
        default: quant_lane_group<8>(J, g, row); break;
      }
    }
    __syncwarp();   // every lane's codes are staged
    store_codes(J, (w - J.first_warp) * 32, cur, lane);
    __syncwarp();   // every lane has read `cur` before it is refilled (two items later)
    jj = jn;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Derived dequant metadata, group-major: meta[g * N + n] = bf16bits(RNE_bf16(scales[n * gpr + g]))
// << 16 | zeros[n * gpr + g].  One thread per output word (coalesced writes).
__global__ void __launch_bounds__(256) k_build_meta(const float* __restrict__ scales,
                                                    const uint8_t* __restrict__ zeros, int N,
                                                    int gpr, uint32_t* __restrict__ meta) {
  const size_t n_all = (size_t)N * gpr;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_all;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t g = i / N, n = i - g * N;
    const size_t src = n * gpr + g;
    const __nv_bfloat16 sb = __float2bfloat16_rn(scales[src]);
    meta[i] = ((uint32_t)*reinterpret_cast<const uint16_t*>(&sb) << 16) | (uint32_t)zeros[src];
  }
}

cudaError_t launch_build_meta(const float* scales, const uint8_t* zeros, int N, int gpr,
                              uint32_t* meta, cudaStream_t s) {
  const size_t n = (size_t)N * gpr;
  if (n == 0) return cudaSuccess;
  const size_t blocks = (n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192;
  k_build_meta<<<(unsigned)blocks, 256, 0, s>>>(scales, zeros, N, gpr, meta);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const dymoe_quant_job* jobs_host, int n_jobs, cudaStream_t s) {
  static const int sms = [] {   // one-time setup, thread-safe (magic static)
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_quantize, cudaFuncAttributeMaxDynamicSharedMemorySize, kQWarps * 2 * kBuf);
    return n;
  }();
  for (int start = 0; start < n_jobs; start += kMaxJobs) {
    QJobs J{};
    J.n = 0;
    long long warps = 0;
    for (int i = start; i < n_jobs && i < start + kMaxJobs; ++i) {
      const dymoe_quant_job& h = jobs_host[i];
      const long long ng = (long long)h.N * (h.K / DYMOE_GROUP);
      if (ng == 0) continue;
      QJob& q = J.j[J.n++];
      q.W = h.W; q.codes = h.codes; q.scales = h.scales; q.zeros = h.zeros;
      q.K = h.K; q.bits = h.bits;
      q.n_groups = ng;
      q.first_warp = warps;
      warps += (ng + 31) / 32;
    }
    J.total_warps = warps;
    if (warps == 0) continue;
    long long blocks = (warps + kQWarps - 1) / kQWarps;
    const long long cap = (long long)sms * 3;   // 3 CTAs of 4 warps (2 x 8.5 KB each) per SM
    if (blocks > cap) blocks = cap;
    k_quantize<<<(unsigned)blocks, kQWarps * 32, kQWarps * 2 * kBuf, s>>>(J);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t preload_quantize() { return preload_kernels(k_build_meta, k_quantize); }

}  // namespace dymoe
