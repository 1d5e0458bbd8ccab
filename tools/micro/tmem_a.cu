// Probe for a tcgen05 decode GEMV with the dequantized weights as the A operand in TMEM:
//  (1) layout check: A [128][64] bf16 written to TMEM by 4 warps (tcgen05.st.32x32b, lane = row,
//      column c = k pair (2c, 2c+1)), B = x [N][64] bf16 in shared memory (K-major, 128B
//      swizzle), tcgen05.mma.kind::f16 M=128 N=16 K=16 x4, D read back and compared on the host;
//      also with SBO = 0 (8 real B rows aliased as rows 8..15).
//  (2) throughput: W writer warps dequantize Int4-style codes into A stages (64 k each), one
//      thread issues 4 MMAs per stage; weights per cycle per SM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
#define ST32(taddr, r)                                                                              \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), \
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),         \
               "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),       \
               "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory")

__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ----------------------------------------------------------------------------- (1) layout check
__global__ void k_check(const uint16_t* A, const uint16_t* B, int nb_rows, uint32_t sbo, float* D) {
  __shared__ __align__(1024) uint8_t xs[2048];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B rows into the 128B-swizzled K-major tile: row r at (r/8)*1024 + (r%8)*128, chunk j ^ (r%8)
  for (int i = threadIdx.x; i < nb_rows * 8; i += blockDim.x) {
    const int r = i / 8, j = i % 8;
    *reinterpret_cast<uint4*>(xs + (r / 8) * 1024 + (r % 8) * 128 + ((j ^ (r % 8)) << 4)) =
        *reinterpret_cast<const uint4*>(B + r * 64 + j * 8);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  const uint32_t a_col = 32, d_col = 0;
  if (warp < 4) {
    const int row = warp * 32 + lane;
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = (uint32_t)A[row * 64 + 2 * c] | ((uint32_t)A[row * 64 + 2 * c + 1] << 16);
    ST32(tm + ((uint32_t)(warp * 32) << 16) + a_col, r);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 128) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int kk = 0; kk < 4; ++kk)
      mma_ts(tm + d_col, tm + a_col + kk * 8, sw_desc(smem_u32(xs) + kk * 32, sbo), make_idesc(128, 16), kk > 0);
    commit(smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    float v[16];
    ld16(tm + ((uint32_t)(warp * 32) << 16) + d_col, v);
    const int row = warp * 32 + lane;
    for (int n = 0; n < 16; ++n) D[row * 16 + n] = v[n];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}

// ----------------------------------------------------------------------------- (2) throughput
template <int NW, int S, bool NOMMA = false, int NN = 16>
__global__ void k_tput(int steps, uint32_t seed, float* out, long long* cyc) {
  __shared__ __align__(1024) uint8_t xs[NN >= 64 ? ((NN + 7) / 8) * 1024 : 1024 * 4];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t full[S], empty[S], done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (int)sizeof(xs) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(xs)[i] = 0x3f803f80u;
  if (warp == NW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(&full[s]), 4);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(&done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  long long t0 = clock64();
  if (warp < NW) {
    const int q = warp & 3, grp = warp >> 2, ngrp = NW / 4;
    uint32_t w = seed * (threadIdx.x + 1);
    const uint32_t zz = 0x43044304u, ss = 0x3c003c00u;
    for (int i = grp; i < steps; i += ngrp) {
      const int s = i % S;
      mbar_wait(smem_u32(&empty[s]), ((i / S) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {   // 8 words of 8 Int4 codes -> 32 bf16 pairs
        const uint32_t x = w + c * 0x11111111u;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          uint32_t v;
          asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(v) : "r"(x >> (4 * t)), "r"(0x000F000Fu), "r"(0x43004300u));
          __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v);
          b = __hmul2(__hsub2(b, *reinterpret_cast<const __nv_bfloat162*>(&zz)), *reinterpret_cast<const __nv_bfloat162*>(&ss));
          r[c * 4 + t] = *reinterpret_cast<uint32_t*>(&b);
        }
      }
      w = w * 1664525u + 1013904223u;
      ST32(tm + ((uint32_t)(q * 32) << 16) + (NN >= 64 ? NN : 64) + s * 32, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&full[s]));
    }
  } else if (warp == NW && lane == 0) {
    // each stage is written by the 4 warps of one group; full[s] counts NW arrivals per phase, so
    // with 2 groups a phase spans 2 stages' worth -- use group-major stage ownership instead
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      mbar_wait(smem_u32(&full[s]), (i / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (NOMMA) {
        mbar_arrive(smem_u32(&empty[s]));
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(NN >= 64 ? tm : tm + (i & 1) * 16, tm + (NN >= 64 ? NN : 64) + s * 32 + kk * 8,
                 sw_desc(smem_u32(xs) + kk * 32, NN >= 64 ? 1024 : 0), make_idesc(128, NN), kk > 0);
        commit(smem_u32(&empty[s]));
      }
    }
    commit(smem_u32(&done));
  }
  if (warp == NW && lane == 0) mbar_wait(smem_u32(&done), 0);
  __syncthreads();
  long long t1 = clock64();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    float v[16];
    ld16(tm + ((uint32_t)(warp * 32) << 16), v);
    float s = 0;
    for (int n = 0; n < 16; ++n) s += v[n];
    out[blockIdx.x * 128 + warp * 32 + lane] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == NW) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}


// ----------------------------------------------------------------------------- (3) MMA issue rate
template <int M, int N, bool TS, int ROT = 1>
__global__ void k_mma_rate(int n, long long* cyc, float* out) {
  __shared__ __align__(1024) uint8_t sm[32768];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_base;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          mma_ts(tm + (kk % ROT) * 64, tm + 256 + kk * 8, sw_desc(smem_u32(sm) + kk * 32, 1024), make_idesc(M, N), 1);
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tm), "l"(sw_desc(smem_u32(sm) + 16384 + kk * 32, 1024)), "l"(sw_desc(smem_u32(sm) + kk * 32, 1024)),
                       "r"(make_idesc(M, N)), "r"(1) : "memory");
      }
    }
    commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

static float bf(uint16_t h) { uint32_t u = (uint32_t)h << 16; float f; memcpy(&f, &u, 4); return f; }
static uint16_t tobf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }

int main() {
  // (1)
  const int K = 64;
  uint16_t hA[128 * K], hB[16 * K];
  srand(1);
  for (int i = 0; i < 128 * K; ++i) hA[i] = tobf((float)((rand() % 17) - 8) * 0.25f);
  for (int i = 0; i < 16 * K; ++i) hB[i] = tobf((float)((rand() % 9) - 4) * 0.5f);
  uint16_t *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, 128 * 16 * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 2; ++variant) {
    const int nb = variant == 0 ? 16 : 8;
    const uint32_t sbo = variant == 0 ? 1024 : 0;
    cudaMemset(dD, 0, 128 * 16 * 4);
    k_check<<<1, 160>>>(dA, dB, nb, sbo, dD);
    cudaError_t e = cudaDeviceSynchronize();
    float hD[128 * 16];
    cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 16; ++n) {
        double ref = 0;
        const int bn = variant == 0 ? n : n % 8;
        for (int k = 0; k < K; ++k) ref += (double)bf(hA[m * K + k]) * bf(hB[bn * K + k]);
        maxerr = fmax(maxerr, fabs(ref - hD[m * 16 + n]));
      }
    printf("layout check variant %d (B rows %d, SBO %u): %s, max |err| = %g  (D[0][0..3] = %g %g %g %g)\n",
           variant, nb, sbo, cudaGetErrorString(e), maxerr, hD[0], hD[1], hD[2], hD[3]);
  }
  // (2)
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 128 * 4);
  cudaMalloc(&cyc, 8);
  const int steps = 20000;
  auto run = [&](auto kern, int nw, const char* name) {
    kern<<<148, nw * 32 + 32>>>(steps, 3u, out, cyc);
    cudaDeviceSynchronize();
    kern<<<148, nw * 32 + 32>>>(steps, 3u, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s: %s cycles %lld, weights/cycle/SM %.1f\n", name, cudaGetErrorString(e), c, 128.0 * 64 * steps / c);
  };
  {
    auto mr = [&](auto kern, int M, int N, const char* kind) {
      const int n = 4096;
      kern<<<148, 128>>>(n, cyc, out);
      cudaDeviceSynchronize();
      kern<<<148, 128>>>(n, cyc, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("MMA %s M=%d N=%d K=16: %s %.1f cycles per MMA, A-rows*K per cycle %.1f\n", kind, M, N,
             cudaGetErrorString(e), (double)c / (4.0 * n), M * 16.0 * 4 * n / c);
    };
    mr(k_mma_rate<128, 16, true>, 128, 16, "TS");
    mr(k_mma_rate<128, 16, true, 4>, 128, 16, "TS 4 accumulators");
    mr(k_mma_rate<128, 16, false, 1>, 128, 16, "SS");
    mr(k_mma_rate<128, 32, true>, 128, 32, "TS");
    mr(k_mma_rate<128, 64, true>, 128, 64, "TS");
    mr(k_mma_rate<128, 256, true>, 128, 256, "TS");
    mr(k_mma_rate<128, 16, false>, 128, 16, "SS");
    mr(k_mma_rate<128, 64, false>, 128, 64, "SS");
    mr(k_mma_rate<128, 256, false>, 128, 256, "SS");
    mr(k_mma_rate<128, 128, false>, 128, 128, "SS");
    mr(k_mma_rate<128, 192, false>, 128, 192, "SS");
    mr(k_mma_rate<64, 8, true>, 64, 8, "TS");
    mr(k_mma_rate<64, 8, false>, 64, 8, "SS");
  }
  run(k_tput<8, 4, false, 256>, 8, "N=256: 8 writer warps, 4 stages (A in TMEM, prefill shape)");
  run(k_tput<8, 4, true, 256>, 8, "N=256 NO MMA: 8 writer warps, 4 stages");
  run(k_tput<4, 4, false, 256>, 4, "N=256: 4 writer warps, 4 stages");
  run(k_tput<8, 6, false, 128>, 8, "N=128: 8 writer warps, 6 stages");
  run(k_tput<8, 4, false, 192>, 8, "N=192: 8 writer warps, 4 stages (MMA-bound = 21.3)");
  run(k_tput<8, 4, false, 160>, 8, "N=160: 8 writer warps, 4 stages (MMA-bound = 25.6)");
  run(k_tput<4, 4, true>, 4, "NO MMA: 4 writer warps, 4 stages");
  run(k_tput<8, 4, true>, 8, "NO MMA: 8 writer warps, 4 stages");
  run(k_tput<4, 4>, 4, "4 writer warps, 4 stages");
  run(k_tput<8, 4>, 8, "8 writer warps, 4 stages");
  run(k_tput<8, 8>, 8, "8 writer warps, 8 stages");
  run(k_tput<12, 6>, 12, "12 writer warps, 6 stages");
  return 0;
}
