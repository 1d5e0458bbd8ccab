// Heavy-hitter attention mass without materializing P (Eq. 1 input,
// P:216-221, reading R1): a[h][j] = sum_{i >= j} softmax_{j' <= i}(scale q_i . k_j')[j].
//
// Two passes over causal 64 x 64 blocks of S = Q K^T on the tensor cores (mma.sync m16n8k16,
// bf16 -> fp32; the score tiles stay in registers):
//   pass 1 (row statistics): per query row i, m_i = max_j s_ij and l_i = sum_j exp(s_ij - m_i)
//            (online over key blocks, as in flash attention);
//   pass 2 (column sums): each warp owns 16 keys and walks every query block at or below the
//            diagonal, computing S^T = K Q^T so that the column sums of P are row sums of its
//            accumulator tile, adds exp(s_ij - m_i) / l_i, and writes its 16 a[h][j] once.
// Sums run in a fixed order (deterministic).  Roofline: tensor (2 x T^2 d H flops, causal half).
#include "../dymoe_internal.cuh"

namespace dymoe {
namespace attn {

constexpr int D = 128;        // head dim
constexpr int BQ = 64;        // rows per block (4 warps x 16)
constexpr int RS = D / 2 + 4; // padded smem row stride in 32-bit words (conflict-free fragments)

__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                    uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// rows [r0, r0 + 64) of a [T][D] bf16 matrix into smem (words, stride RS); rows >= T zero-filled
__device__ __forceinline__ void load_block(uint32_t* dst, const uint16_t* src, int r0, int T) {
  for (int i = threadIdx.x; i < BQ * (D / 8); i += blockDim.x) {
    const int r = i / (D / 8), c = i - r * (D / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r0 + r < T) v = *reinterpret_cast<const uint4*>(src + (size_t)(r0 + r) * D + c * 8);
    *reinterpret_cast<uint4*>(dst + r * RS + c * 4) = v;
  }
}

// A fragments of 16 rows (r0 .. r0+15 of the smem block) over all D: 8 k-steps x 4 words
__device__ __forceinline__ void a_frags(const uint32_t* s, int r0, uint32_t (&a)[D / 16][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    a[ks][0] = s[(r0 + g) * RS + ks * 8 + c];
    a[ks][1] = s[(r0 + g + 8) * RS + ks * 8 + c];
    a[ks][2] = s[(r0 + g) * RS + ks * 8 + 4 + c];
    a[ks][3] = s[(r0 + g + 8) * RS + ks * 8 + 4 + c];
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

// acc[n][.] = (rows of A) x (rows n*8.. of the smem block B)^T, 8 n-tiles of 8 columns.
// B fragments by ldmatrix.x4: matrices (k 0-7, k 8-15) x (n-tiles 2p, 2p+1) of each k16 step.
__device__ __forceinline__ void tile_product(const uint32_t (&a)[D / 16][4], const uint32_t* sb,
                                             float (&acc)[8][4]) {
  const int lane = threadIdx.x & 31;
  // lane l supplies the row address of matrix l / 8: n-tile 2p + (l / 16), k half (l / 8) & 1
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sb) +
                        (uint32_t)(((lane >> 4) * 8 + (lane & 7)) * RS * 4 + ((lane >> 3) & 1) * 16);
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks)
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      uint32_t b00, b01, b10, b11;
      ldsm_x4(base + p * 16 * RS * 4 + ks * 32, b00, b01, b10, b11);
      mma(acc[2 * p], a[ks][0], a[ks][1], a[ks][2], a[ks][3], b00, b01);
      mma(acc[2 * p + 1], a[ks][0], a[ks][1], a[ks][2], a[ks][3], b10, b11);
    }
}

// Pass 1: one CTA per (head, 64-query block); warp w owns queries q0 + 16w ..
__global__ void __launch_bounds__(128) k_row_stats(const uint16_t* __restrict__ Q,
                                                   const uint16_t* __restrict__ K, int T,
                                                   float scale_log2, float* __restrict__ m_out,
                                                   float* __restrict__ l_out) {
  __shared__ __align__(16) uint32_t sq[BQ * RS], sk[BQ * RS];
  const int h = blockIdx.y, qb = blockIdx.x, q0 = qb * BQ;
  const uint16_t* Qh = Q + (size_t)h * T * D;
  const uint16_t* Kh = K + (size_t)h * T * D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  load_block(sq, Qh, q0, T);
  __syncthreads();
  uint32_t a[D / 16][4];
  a_frags(sq, warp * 16, a);
  const int i0 = q0 + warp * 16 + g, i1 = i0 + 8;   // this thread's two query rows
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  for (int kb = 0; kb <= qb; ++kb) {
    __syncthreads();
    load_block(sk, Kh, kb * BQ, T);
    __syncthreads();
    float acc[8][4];
    tile_product(a, sk, acc);
    // scores in log2 units; causal / tail mask
    float bm0 = -INFINITY, bm1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = kb * BQ + n * 8 + 2 * c + (e & 1);
        const int i = e < 2 ? i0 : i1;
        const float s = (j <= i && j < T) ? acc[n][e] * scale_log2 : -INFINITY;
        acc[n][e] = s;
        if (e < 2) bm0 = fmaxf(bm0, s);
        else bm1 = fmaxf(bm1, s);
      }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, off));
      bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, off));
    }
    const float n0 = fmaxf(m0, bm0), n1 = fmaxf(m1, bm1);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      s0 += exp2f(acc[n][0] - n0) + exp2f(acc[n][1] - n0);
      s1 += exp2f(acc[n][2] - n1) + exp2f(acc[n][3] - n1);
    }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, off);
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    }
    l0 = (m0 == -INFINITY ? 0.f : l0 * exp2f(m0 - n0)) + s0;
    l1 = (m1 == -INFINITY ? 0.f : l1 * exp2f(m1 - n1)) + s1;
    m0 = n0;
    m1 = n1;
  }
  if (c == 0) {
    if (i0 < T) { m_out[(size_t)h * T + i0] = m0; l_out[(size_t)h * T + i0] = l0; }
    if (i1 < T) { m_out[(size_t)h * T + i1] = m1; l_out[(size_t)h * T + i1] = l1; }
  }
}

// Pass 2: one CTA per (head, 64-key block); warp w owns keys k0 + 16w ..; S^T = K Q^T
__global__ void __launch_bounds__(128) k_col_sums(const uint16_t* __restrict__ Q,
                                                  const uint16_t* __restrict__ K, int T,
                                                  float scale_log2, const float* __restrict__ m_in,
                                                  const float* __restrict__ l_in,
                                                  float* __restrict__ a_out) {
  __shared__ __align__(16) uint32_t sk[BQ * RS], sq[BQ * RS];
  __shared__ float sm[BQ], sl[BQ];   // row max (log2 units) and 1 / row sum of the query block
  const int h = blockIdx.y, kb = blockIdx.x, k0 = kb * BQ;
  const uint16_t* Qh = Q + (size_t)h * T * D;
  const uint16_t* Kh = K + (size_t)h * T * D;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  load_block(sk, Kh, k0, T);
  __syncthreads();
  uint32_t a[D / 16][4];
  a_frags(sk, warp * 16, a);
  const int j0 = k0 + warp * 16 + g, j1 = j0 + 8;   // this thread's two keys
  float col0 = 0.f, col1 = 0.f;
  const int nqb = (T + BQ - 1) / BQ;
  for (int qb = kb; qb < nqb; ++qb) {
    __syncthreads();
    load_block(sq, Qh, qb * BQ, T);
    if (threadIdx.x < BQ) {
      const int i = qb * BQ + threadIdx.x;
      sm[threadIdx.x] = i < T ? m_in[(size_t)h * T + i] : 0.f;
      sl[threadIdx.x] = i < T ? 1.f / l_in[(size_t)h * T + i] : 1.f;
    }
    __syncthreads();
    float acc[8][4];
    tile_product(a, sq, acc);    // acc[n][e]: key (e < 2 ? j0 : j1), query qb*64 + 8n + 2c + (e & 1)
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = n * 8 + 2 * c + (e & 1);
        const int i = qb * BQ + qi;
        const int j = e < 2 ? j0 : j1;
        const float p = (j <= i && i < T) ? exp2f(acc[n][e] * scale_log2 - sm[qi]) * sl[qi] : 0.f;
        if (e < 2) col0 += p;
        else col1 += p;
      }
  }
#pragma unroll
  for (int off = 1; off < 4; off <<= 1) {
    col0 += __shfl_xor_sync(0xffffffffu, col0, off);
    col1 += __shfl_xor_sync(0xffffffffu, col1, off);
  }
  if (c == 0) {
    if (j0 < T) a_out[(size_t)h * T + j0] = col0;
    if (j1 < T) a_out[(size_t)h * T + j1] = col1;
  }
}

}  // namespace attn

cudaError_t launch_attention_mass(const uint16_t* Q, const uint16_t* K, int H, int T, int d,
                                  float scale, float* m_scratch, float* l_scratch, float* a_out,
                                  cudaStream_t s) {
  using namespace attn;
  if (d != D) return cudaErrorInvalidValue;
  if (T == 0 || H == 0) return cudaSuccess;
  const float sl2 = scale * 1.4426950408889634f;
  const dim3 grid((T + BQ - 1) / BQ, H);
  k_row_stats<<<grid, 128, 0, s>>>(Q, K, T, sl2, m_scratch, l_scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_col_sums<<<grid, 128, 0, s>>>(Q, K, T, sl2, m_scratch, l_scratch, a_out);
  return cudaGetLastError();
}

cudaError_t preload_attn_mass() { return preload_kernels(attn::k_row_stats, attn::k_col_sums); }

}  // namespace dymoe
