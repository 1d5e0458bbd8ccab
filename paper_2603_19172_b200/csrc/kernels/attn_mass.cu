// Heavy-hitter attention mass without materializing P (Eq. 1 input,
// P:216-221, reading R1): a[h][j] = sum_{i >= j} softmax_{j' <= i}(scale q_i . k_j')[j].
//
// Two passes over causal 128 x 128 blocks of the score matrix on the 5th-generation tensor cores
// (tcgen05.mma.cta_group::1.kind::f16, M = N = 128, K = d = 128, bf16 -> fp32 in TMEM):
//   pass 1 (row statistics): one work item = (head, 128-query block); S = Q_blk K_blk^T for every
//            key block at or below the diagonal; each epilogue thread owns one query row (one TMEM
//            lane) and keeps m_i = max_j s_ij, l_i = sum_j exp(s_ij - m_i) online; it stores
//            n_i = m_i + log2 l_i (log2 units), so that p_ij = 2^(s_ij - n_i);
//   pass 2 (column sums): one work item = (head, 128-key block); S^T = K_blk Q_blk^T for every
//            query block at or after the diagonal, so that a TMEM lane holds one KEY and its
//            row of 128 queries: each epilogue thread adds 2^(s_ij - n_i) over the
//            queries (ascending, four interleaved fp32 chains per key combined in a fixed order --
//            deterministic) and writes a[h][j].
// Per CTA (persistent, one per SM): warp 0 lane 0 streams the tiles by TMA (the work item's A
// tile once into one of two buffers, B tiles through a 3-stage ring; 128B-swizzled K-major, two 64-column boxes per
// 128 x 128 tile), warp 1 owns TMEM (two 128-column accumulators) and one lane issues the MMAs,
// warps 2-9 drain TMEM (tcgen05.ld 32x32b, two warps per lane quarter, 64 columns each) and do
// the softmax arithmetic -- the MMA of block n + 1 overlaps the exponentials of block n.  Work
// items are ordered longest first and dealt out in alternating directions.  (Taking every 4th
// exponential on the FMA pipe with a degree-6 polynomial unloaded the SFU but raised the
// instruction count 70 % and cost 20 %: the epilogue is issue-bound, not SFU-bound.)
// Roofline: tensor (2 passes x 2 T^2 d H / 2 causal flops) with the SFU's exp2 alongside.
#include "../dymoe_internal.cuh"

namespace dymoe {
namespace attn {

constexpr int D = 128;            // head dim (= MMA K)
constexpr int BT = 128;           // rows / columns per block (MMA M = N)
constexpr int NST = 3;            // B-tile ring stages
constexpr int CHUNK = BT * 128;   // one 64-column box: 128 rows x 128 bytes
constexpr int TILE = 2 * CHUNK;   // 32 KB
constexpr int kSmem = (2 + NST) * TILE + 1024;   // A double-buffered by item, B ring
constexpr int kEpi = 16;          // epilogue warps: four per TMEM lane quarter, 32 columns each
constexpr int NQ = kEpi / 4;      // column parts per block (warps sharing a lane quarter)
constexpr int HC = BT / NQ;       // columns per part
constexpr int kThreads = (2 + kEpi) * 32;   // warps 0 (TMA), 1 (TMEM + MMA), 2.. (epilogue)
constexpr uint32_t TMEM_COLS = 2 * BT;
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BT >> 3) << 17) |
                           ((uint32_t)(BT >> 4) << 24);   // kind::f16: bf16 x bf16 -> f32, K-major

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(m), "r"(x), "r"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(IDESC), "r"(acc)
      : "memory");
}
// K-major, 128-byte swizzle, 8-row atoms 1024 B apart (rows of 128 bytes)
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t (&r)[32] = reinterpret_cast<uint32_t(&)[32]>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {   // 2^x on the SFU (ex2(-inf) = +0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void epi_sync() {   // the epilogue threads only
  asm volatile("bar.sync 1, %0;" ::"n"(kEpi * 32) : "memory");
}

// Work item n (longest first) -> (head, block of the A operand, first and end B block).
// Pass 1: A = query block qb, B = key blocks 0 .. qb.  Pass 2: A = key block kb, B = query
// blocks kb .. nb - 1.
template <bool COLS>
__device__ __forceinline__ void item_at(int n, int H, int nb, int& h, int& a, int& b0, int& b1) {
  const int r = n / H;   // rank in the cost order
  h = n - r * H;
  if (COLS) { a = r; b0 = r; b1 = nb; }
  else { a = nb - 1 - r; b0 = 0; b1 = a + 1; }
}

// The work item of round j for CTA c of G: the rounds alternate direction (round 0: c, round 1:
// 2G-1-c, ...), so a CTA that took a long item in one round takes a short one in the next
// (items are ordered longest first).
__device__ __forceinline__ int snake(int j, int c, int G) { return j * G + ((j & 1) ? G - 1 - c : c); }

template <bool COLS>
__global__ void __launch_bounds__(kThreads, 1)
k_attn_mass(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            int H, int T, float scale_log2, float* __restrict__ m_io, float* __restrict__ l_io,
            float* __restrict__ a_out) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[NST], empty_bar[NST], tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t a_full[2], a_empty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ float x_m[NQ][BT], x_l[NQ][BT];                 // the column parts' partials
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sA0 = smem_u32(smem);
  auto sA = [&](int it) { return sA0 + (uint32_t)(it & 1) * TILE; };
  auto sB = [&](int s) { return sA0 + (uint32_t)(2 + s) * TILE; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = (T + BT - 1) / BT;
  const int n_items = H * nb;
  const CUtensorMap* tmA = COLS ? &tmK : &tmQ;
  const CUtensorMap* tmB = COLS ? &tmQ : &tmK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull_bar[b]), 1);
      mbar_init(smem_u32(&tempty_bar[b]), kEpi);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&a_full[b]), 1);
      mbar_init(smem_u32(&a_empty[b]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0, it = 0;
      uint32_t phase = 0;
      for (int j = 0;; ++j, ++it) {
        const int n = snake(j, blockIdx.x, gridDim.x);
        if (n >= n_items) break;
        int h, ab, b0, b1;
        item_at<COLS>(n, H, nb, h, ab, b0, b1);
        const uint32_t af = smem_u32(&a_full[it & 1]);
        mbar_wait(smem_u32(&a_empty[it & 1]), ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(af, TILE);
        tma2d(sA(it), tmA, 0, h * T + ab * BT, af);
        tma2d(sA(it) + CHUNK, tmA, 64, h * T + ab * BT, af);
        for (int bb = b0; bb < b1; ++bb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          mbar_expect_tx(smem_u32(&full_bar[stage]), TILE);
          tma2d(sB(stage), tmB, 0, h * T + bb * BT, smem_u32(&full_bar[stage]));
          tma2d(sB(stage) + CHUNK, tmB, 64, h * T + bb * BT, smem_u32(&full_bar[stage]));
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0, it = 0, blk = 0;
      uint32_t phase = 0;
      for (int j = 0;; ++j, ++it) {
        const int n = snake(j, blockIdx.x, gridDim.x);
        if (n >= n_items) break;
        int h, ab, b0, b1;
        item_at<COLS>(n, H, nb, h, ab, b0, b1);
        mbar_wait(smem_u32(&a_full[it & 1]), (it >> 1) & 1);
        tc_fence_after();
        for (int bb = b0; bb < b1; ++bb, ++blk) {
          const int b = blk & 1;
          mbar_wait(smem_u32(&tempty_bar[b]), ((blk >> 1) & 1) ^ 1);
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (uint32_t)(kk >> 2) * CHUNK + (uint32_t)(kk & 3) * 32;
            tc_mma(tmem + (uint32_t)(b * BT), sw_desc(sA(it) + off), sw_desc(sB(stage) + off), kk != 0);
          }
          tc_commit(smem_u32(&empty_bar[stage]));
          tc_commit(smem_u32(&tfull_bar[b]));
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        tc_commit(smem_u32(&a_empty[it & 1]));   // every MMA reading this A buffer has completed
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2..)
    // NQ warps per TMEM lane quarter (one per HC-column part of the block), so every SM
    // sub-partition runs NQ epilogue warps -- the epilogue is latency-bound, not issue-bound; each
    // row's reductions run as 4 interleaved chains per part, combined in a fixed order (chains,
    // then parts 0, 1, ...) at the end of the item.  Blocks strictly off the diagonal and inside
    // the sequence take a mask-free path.
    const int q = warp & 3;                    // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;          // column part 0 .. NQ-1
    const int r = q * 32 + lane;               // A row = TMEM lane owned by this thread
    int blk = 0;
    for (int j = 0;; ++j) {
      const int n = snake(j, blockIdx.x, gridDim.x);
      if (n >= n_items) break;
      int h, ab, b0, b1;
      item_at<COLS>(n, H, nb, h, ab, b0, b1);
      const int row = ab * BT + r;            // query (pass 1) / key (pass 2) of this thread
      float m = -INFINITY, l = 0.f;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int bb = b0; bb < b1; ++bb, ++blk) {
        const int b = blk & 1;
        float s[HC];
        const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BT + half * HC);
        const bool full = bb != ab && (bb + 1) * BT <= T;   // no causal / tail mask (uniform)
        const int c0 = half * HC;
        if (COLS) {
          // n_i of this part's 32 queries (pass 1): one address per load across the warp (a
          // broadcast from L1), issued before the wait for the MMA so that their latency
          // overlaps it -- no shared memory, no barrier
          const float* mq = m_io + (size_t)h * T + bb * BT + c0;
          float4 mm4[HC / 4];
          if (full && (T & 3) == 0) {           // 16-byte aligned rows of the scratch
#pragma unroll
            for (int c = 0; c < HC / 4; ++c) mm4[c] = __ldg(reinterpret_cast<const float4*>(mq) + c);
          } else {
            const int nv = min(HC, T - bb * BT - c0);   // queries of this part inside the sequence
#pragma unroll
            for (int c = 0; c < HC / 4; ++c) {
              float t0[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) t0[e] = 4 * c + e < nv ? __ldg(mq + 4 * c + e) : 0.f;
              mm4[c] = make_float4(t0[0], t0[1], t0[2], t0[3]);
            }
          }
          mbar_wait(smem_u32(&tfull_bar[b]), (blk >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < HC / 32; ++c)
            tmem_ld32(tb + c * 32, reinterpret_cast<float(&)[32]>(s[c * 32]));
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[b]));
          // queries i = bb*128 + c0 + c; valid when i >= row (causal) and i < T
          if (full) {
#pragma unroll
            for (int c = 0; c < HC; c += 4) {
              const float4 mm = mm4[c / 4];
              acc[0] += ex2(__fmaf_rn(s[c], scale_log2, -mm.x));
              acc[1] += ex2(__fmaf_rn(s[c + 1], scale_log2, -mm.y));
              acc[2] += ex2(__fmaf_rn(s[c + 2], scale_log2, -mm.z));
              acc[3] += ex2(__fmaf_rn(s[c + 3], scale_log2, -mm.w));
            }
          } else {
            const int cmin = row - bb * BT - c0;   // first valid column of this half
            const int cmax = T - bb * BT - c0;     // columns >= cmax are past the sequence
#pragma unroll
            for (int c = 0; c < HC; c += 4) {
              const float4 mm = mm4[c / 4];
              const float mv[4] = {mm.x, mm.y, mm.z, mm.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const bool ok = c + e >= cmin && c + e < cmax;
                const float p = ex2(__fmaf_rn(s[c + e], scale_log2, -mv[e]));
                acc[e] += ok ? p : 0.f;
              }
            }
          }
        } else {
          mbar_wait(smem_u32(&tfull_bar[b]), (blk >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < HC / 32; ++c)
            tmem_ld32(tb + c * 32, reinterpret_cast<float(&)[32]>(s[c * 32]));
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[b]));
          // keys j = bb*128 + c0 + c, valid when j <= row (causal) and j < T; the max is taken on
          // the raw scores (scale > 0), the exponent is fma(s, scale_log2, -max * scale_log2)
          if (!full) {
            const int cmax = min(row - bb * BT + 1, T - bb * BT) - c0;
#pragma unroll
            for (int c = 0; c < HC; ++c) s[c] = c < cmax ? s[c] : -INFINITY;
          }
          float bm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = 0; c < HC; ++c) bm[c & 3] = fmaxf(bm[c & 3], s[c]);
          const float nm = fmaxf(m, fmaxf(fmaxf(bm[0], bm[1]), fmaxf(bm[2], bm[3])));
          float sum[4] = {0.f, 0.f, 0.f, 0.f};
          if (nm != -INFINITY) {
            const float nms = -nm * scale_log2;
#pragma unroll
            for (int c = 0; c < HC; ++c) sum[c & 3] += ex2(__fmaf_rn(s[c], scale_log2, nms));
          }
          l = (m == -INFINITY ? 0.f : l * ex2((m - nm) * scale_log2)) +
              ((sum[0] + sum[1]) + (sum[2] + sum[3]));
          m = nm;
        }
      }
      // combine the column parts of each row: parts 1.. hand their partials to part 0
      x_m[half][r] = COLS ? (acc[0] + acc[1]) + (acc[2] + acc[3]) : m;
      x_l[half][r] = l;
      epi_sync();
      if (half == 0 && row < T) {
        if (COLS) {
          float a = x_m[0][r];
#pragma unroll
          for (int p = 1; p < NQ; ++p) a += x_m[p][r];
          a_out[(size_t)h * T + row] = a;
        } else {
          float mt = x_m[0][r];   // raw-score maxima; m, l in the scaled log2 domain
#pragma unroll
          for (int p = 1; p < NQ; ++p) mt = fmaxf(mt, x_m[p][r]);
          float lt = 0.f;
#pragma unroll
          for (int p = 0; p < NQ; ++p)
            lt += x_m[p][r] == -INFINITY ? 0.f : x_l[p][r] * ex2((x_m[p][r] - mt) * scale_log2);
          // p_ij = 2^(s_ij c - m_i) / l_i = 2^(s_ij c - (m_i + log2 l_i)): pass 2 needs one value
          m_io[(size_t)h * T + row] = __fadd_rn(mt * scale_log2, log2f(lt));
          l_io[(size_t)h * T + row] = lt;
        }
      }
      epi_sync();   // x_m / x_l are rewritten by the next item
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace attn

cudaError_t launch_attention_mass(const uint16_t* Q, const uint16_t* K, int H, int T, int d,
                                  float scale, float* m_scratch, float* l_scratch, float* a_out,
                                  cudaStream_t s) {
  using namespace attn;
  if (d != D) return cudaErrorInvalidValue;
  if (T == 0 || H == 0) return cudaSuccess;
  static const int sms = [] {   // one-time setup, thread-safe (magic static)
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_attn_mass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_attn_mass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    return n;
  }();
  // Q, K as 2-D [H*T][128] bf16 tensors; boxes of 64 columns x 128 rows, 128-byte swizzle (rows
  // of a block past T read the next head's rows or TMA's zero fill: masked in the epilogue)
  CUtensorMap tq, tk;
  const uint64_t rows = (uint64_t)H * T;
  if (!encode_tmap_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Q, D, rows, D * 2, 64, BT,
                      CU_TENSOR_MAP_SWIZZLE_128B) ||
      !encode_tmap_2d(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, K, D, rows, D * 2, 64, BT,
                      CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const float sl2 = scale * 1.4426950408889634f;
  const int items = H * ((T + BT - 1) / BT);
  const int grid = items < sms ? items : sms;
  k_attn_mass<false><<<grid, kThreads, kSmem, s>>>(tq, tk, H, T, sl2, m_scratch, l_scratch, a_out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_attn_mass<true><<<grid, kThreads, kSmem, s>>>(tq, tk, H, T, sl2, m_scratch, l_scratch, a_out);
  return cudaGetLastError();
}

cudaError_t preload_attn_mass() {
  return preload_kernels(attn::k_attn_mass<false>, attn::k_attn_mass<true>);
}

}  // namespace dymoe
