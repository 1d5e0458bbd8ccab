// Microbenchmark: issue throughput of the dequant instruction classes on sm_100a (warp
// instructions per cycle per SM), 8 independent chains per thread, 16 warps per SM.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

template <int OP>
__global__ void k(uint32_t* out, int iters, uint32_t seed, long long* cyc) {
  uint32_t r[8];
  float4 acc[2] = {make_float4(0, 0, 0, 0), make_float4(0, 0, 0, 0)};
  for (int i = 0; i < 8; ++i) r[i] = seed * (threadIdx.x + 1) + i * 0x01010101u;
  const uint32_t c1 = seed | 0x3f803f80u, c2 = seed ^ 0x3c003c00u;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {  // bf16x2 mul
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&r[i]);
        __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&c1);
        a = __hmul2(a, b);
        r[i] = *reinterpret_cast<uint32_t*>(&a);
      } else if (OP == 1) {  // fp16x2 mul
        __half2 a = *reinterpret_cast<__half2*>(&r[i]);
        __half2 b = *reinterpret_cast<const __half2*>(&c2);
        a = __hmul2(a, b);
        r[i] = *reinterpret_cast<uint32_t*>(&a);
      } else if (OP == 2) {  // fp32 fma
        float a = __uint_as_float(r[i]);
        a = __fmaf_rn(a, __uint_as_float(c1), __uint_as_float(c2));
        r[i] = __float_as_uint(a);
      } else if (OP == 3) {  // lop3
        uint32_t x;
        asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(r[i]), "r"(c1), "r"(c2));
        r[i] = x;
      } else if (OP == 4) {  // prmt
        uint32_t x;
        asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(x) : "r"(c1), "r"(c2), "r"(r[i]));
        r[i] = x;
      } else if (OP == 5) {  // imad
        r[i] = r[i] * c1 + c2;
      } else if (OP == 6) {  // bf16x2 fma
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&r[i]);
        __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&c1);
        __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(&c2);
        a = __hfma2(a, b, c);
        r[i] = *reinterpret_cast<uint32_t*>(&a);
      } else if (OP == 7) {  // bf16x2 sub
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&r[i]);
        __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&c1);
        a = __hsub2(a, b);
        r[i] = *reinterpret_cast<uint32_t*>(&a);
      } else if (OP == 8) {  // mixed: lop3 + bf16 sub + bf16 mul (the Int4 dequant)
        uint32_t x;
        asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(r[i]), "r"(0x000f000fu), "r"(0x43004300u));
        __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&x);
        __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&c1);
        a = __hmul2(__hsub2(a, b), b);
        r[i] ^= *reinterpret_cast<uint32_t*>(&a);
      } else if (OP == 20) {  // MUFU.EX2 (ex2.approx.ftz.f32)
        float y;   // a pure chain: 2^x of the previous result (the value does not matter)
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint_as_float(r[i])));
        r[i] = __float_as_uint(y);
      } else if (OP == 21) {  // FFMA2 (fma.rn.f32x2)
        uint64_t a, y;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(r[i]), "r"(r[(i + 1) & 7]));
        const uint64_t b = ((uint64_t)c1 << 32) | c1, c = ((uint64_t)c2 << 32) | c2;
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(y) : "l"(a), "l"(b), "l"(c));
        r[i] = (uint32_t)y ^ (uint32_t)(y >> 32);
      } else if (OP == 10) {  // mma.sync m16n8k16 bf16, 2 independent accumulators per chain pair
        if (i < 2) {
          float* d = &acc[i].x;
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                       : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                       : "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]));
        }
      } else if (OP == 11) {  // Int4 dequant of 4 A regs + 1 mma per 2 chains (realistic inner step)
        if ((i & 1) == 0) {
          uint32_t a[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t x;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(r[i] >> (4 * q)), "r"(0x000f000fu), "r"(0x43004300u));
            __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&x);
            __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&c1);
            v = __hmul2(__hsub2(v, b), b);
            a[q] = *reinterpret_cast<uint32_t*>(&v);
          }
          float* d = &acc[(i >> 1) & 1].x;
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                       : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                       : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(c1), "r"(c2));
          r[i] = r[i] * 0x9E3779B9u;
        }
      } else if (OP >= 12 && OP <= 15) {  // 1 mma + 8 ops of one class per 2 chains
        if ((i & 1) == 0) {
          uint32_t a[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t x = r[i] + q;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (OP == 12) {
                __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&x);
                __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&c1);
                v = __hmul2(v, b);
                x = *reinterpret_cast<uint32_t*>(&v);
              } else if (OP == 13) {
                x = __float_as_uint(__fmul_rn(__uint_as_float(x), __uint_as_float(c1)));
              } else if (OP == 14) {
                asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(x) : "r"(x), "r"(c1), "r"(c2));
              } else {
                x = x * c1 + c2;
              }
            }
            a[q] = x;
          }
          float* d = &acc[(i >> 1) & 1].x;
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                       : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                       : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(c1), "r"(c2));
          r[i] = r[i] * 0x9E3779B9u;
        }
      } else if (OP == 9) {  // fp32 sub (FADD)
        r[i] = __float_as_uint(__fsub_rn(__uint_as_float(r[i]), __uint_as_float(c1)));
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s ^= r[i];
  s ^= __float_as_uint(acc[0].x + acc[1].y + acc[0].z + acc[1].w);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* out, long long* cyc, int threads = 512) {
  const int iters = 4096;
  k<OP><<<148, threads>>>(out, iters, 7u, cyc);
  cudaDeviceSynchronize();
  k<OP><<<148, threads>>>(out, iters, 7u, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // warp instructions per SM: 16 warps x iters x 8 (op 8: x4 instr incl. the xor)
  double wi = threads / 32.0 * iters * 8;
  printf("[%4d thr] %-28s cycles %lld  warp-instr/cycle/SM (ops of this kind) %.3f\n", threads, name, c, wi / c);
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  run<0>("HMUL2.BF16", out, cyc);
  run<7>("HSUB2.BF16 (HADD2)", out, cyc);
  run<6>("HFMA2.BF16", out, cyc);
  run<1>("HMUL2.F16", out, cyc);
  run<2>("FFMA", out, cyc);
  run<9>("FADD", out, cyc);
  run<3>("LOP3", out, cyc);
  run<4>("PRMT", out, cyc);
  run<5>("IMAD", out, cyc);
  run<8>("int4 dequant (lop+sub+mul+xor)", out, cyc);
  run<10>("mma m16n8k16 (x2 per 8 chains: /4)", out, cyc);
  run<11>("int4 deq4+mma (/2 -> per mma x4)", out, cyc);
  run<12>("mma + 8 HMUL2.BF16", out, cyc);
  run<13>("mma + 8 FMUL", out, cyc);
  run<14>("mma + 8 LOP3", out, cyc);
  run<15>("mma + 8 IMAD", out, cyc);
  run<20>("MUFU.EX2", out, cyc);
  run<21>("FFMA2 (+MOV +XOR)", out, cyc);
  return 0;
}
