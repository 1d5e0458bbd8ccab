// Decode expert FFN (row a7): fused-dequant SwiGLU GEMV for few tokens per expert, sm_100a.
//
// Paper: P:203 step 4 (executor on a unified mixed-precision weight set), P:312 (Int4/Int2
// experts, skip), P:356 (decode is dominated by fetching expert weights).  Readings D13, D17,
// D18, O6: A = x·deq(W1)^T, B = x·deq(W3)^T in fp32, h = RNE_bf16(silu(A)·B),
// y = h·deq(W2)^T in fp32, deq = RNE_bf16((q - z)·RNE_bf16(s)).
//
// Roofline: HBM.  Every active expert's packed W1/W3/W2 is streamed once per 8-token chunk
// (3·Hd·F·(b/8 + 5/128) bytes per expert).
//
// Arithmetic.  At Int2 there are only ~2 ALU issue slots per weight at the HBM rate:
//  * multiply-adds on the tensor cores: mma.sync m16n8k16, 16 weight rows as A, the (<= 8)
//    tokens as the N = 8 columns of B, fp32 accumulation;
//  * dequant in registers straight into A fragments: Int2/Int4 codes are OR-ed into the mantissa
//    of bf16 128.0 (one LOP3 per 2 weights gives 128+q exactly), HSUB2 (128+z) gives q-z
//    exactly, HMUL2 by bf16(s) gives RNE((q-z)·s) — bit-identical to D17.  Int8 uses the fp32
//    magic 2^23+q, FADD, FMUL (exact) and one cvt.rn.bf16x2;
//  * the dot product is permutation-invariant in k, so A fragments take codes in the order the
//    LOP3 extracts them (code i and i+4 of a word) and the x values are permuted to match (PRMT
//    on registers loaded from shared memory).
//
// Work decomposition (one launch per matrix pair, persistent, cost-balanced):
//  * grid = 1 CTA of two 8-warp groups per SM (alternate tiles, one named barrier per group); each CTA walks "virtual CTAs".  Every CTA computes the same
//    allocation of virtual CTAs to the active experts, proportional to each expert's streamed
//    bytes (width x token chunks), so CTAs of Int8 and Int2 experts finish together.
//  * a virtual CTA = (expert, K-slice, range of 16-row tiles).  Its 8 warps split every tile's K
//    round-robin by 64-byte chunk and reduce the 16x8 partial tiles through shared memory in
//    warp order (deterministic, double-buffered, one barrier per tile).  The tokens' x slice is
//    staged once per virtual CTA in shared memory (XOR-swizzled: conflict-free LDS.128).
//  * each warp streams its weights through its own cp.async (LDGSTS, L1-bypassing) shared-memory
//    ring of 4 (W1/W3) or 5 (W2) stages of one 64-byte chunk per row plus the rows' per-group
//    dequant words, so 2-4 chunks per warp (64 KB per SM) are in flight while it computes.
//  * W1/W3 (gate/up): one K-slice (x = 8 x Hd bf16 in smem), SwiGLU applied in the reduction
//    epilogue, h written as bf16.  W2 (down): K = F is split into SK slices (x slice <= 64 KB),
//    each writes fp32 partials y_part[slice]; the combine kernel sums the slices in order.
#include "ffn_decode_common.cuh"

namespace dymoe {
namespace dec {

// partial-tile reduction buffer: [tok 8][row16 + 4 pad] floats (conflict-free fragment stores)
constexpr int kRedStride = 20;
constexpr int kRedTile = 8 * kRedStride;

// Per-warp cp.async (LDGSTS) ring.  A pipeline item is (tile, chunk): 64 contiguous bytes of each
// of the tile's rows (16 rows per matrix) plus those rows' dequant metadata words for the groups
// the chunk covers.  Copy: 4 lanes per row, 8 rows per instruction (512 contiguous smem bytes);
// compute reads it back in the mma lane mapping (lane quad c of row g reads granule c), which is
// bank-conflict free without swizzling.  The metadata copy is one 4/8-byte cp.async per row.
template <int NM>
struct Ring {
  static constexpr int ROWS = NM * 16;
  static constexpr int W_BYTES = ROWS * 64;
  static constexpr int META = ROWS * 8;        // up to 2 groups per row per chunk (Int2)
  static constexpr int STAGE = W_BYTES + META;
};
template <bool W13>
struct Pipe {
  static constexpr int STAGES = W13 ? 3 : 5;
};

template <int BYTES>
__device__ __forceinline__ void cp_async(uint32_t saddr, const void* g) {
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(saddr), "l"(g));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(saddr), "l"(g), "n"(BYTES));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
// x slice loads: the slice is constant for the whole run_tiles call, so the load is a pure function
// of its address (non-volatile: the compiler may schedule it freely)
__device__ __forceinline__ uint4 lds128_const(uint32_t a) {
  uint4 r;
  asm("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
  return r;
}

// Dequant parameters from a metadata word (bf16 scale bits << 16 | zero).
template <int BITS>
__device__ __forceinline__ DQ dq_from_meta(uint32_t w) {
  DQ d;
  d.ss = prmt(w, 0u, 0x3232u);                       // (s, s)
  if constexpr (BITS == 2) {
    const uint32_t zl2 = prmt(w, 0u, 0x4040u);       // (z, z)
    d.zz = zl2 + 0x43004300u;                        // bf16(128 + z)
    d.zz1 = zl2 * 4u + 0x42004200u;                  // bf16(32 + z)
    d.zz2 = zl2 * 16u + 0x41004100u;                 // bf16(8 + z)
  } else {
    d.zz = prmt(w, 0x43u, 0x4040u);                  // (bf16(128 + z), bf16(128 + z))
  }
  d.sf = __uint_as_float(w & 0xffff0000u);
  d.zf = __uint_as_float(prmt(w, 0x4B000000u, 0x7440u));   // 2^23 + z
  return d;
}

// Per-lane producer state: the global addresses this lane copies for the current tile at chunk
// `warp` (j = 0).  Item j of the tile is these + j * 512 bytes (codes) / + j * GADV words (meta):
// no per-item address arithmetic beyond one 64-bit add per copy.
template <int BITS, int NM>
struct Producer {
  static constexpr int RG = Ring<NM>::ROWS / 8;               // row groups of 8 rows
  static constexpr int CK = WT<BITS>::CHUNK_K;
  static constexpr int GADV = kWarps * CK / DYMOE_GROUP;      // meta words per item step
  const uint8_t* src[RG];
  const uint32_t* msrc;
  size_t tile_step;      // bytes between this lane's rows of tile t and t + 2
  int mtile_step;        // meta words between ...
  int k_lane0;           // k of this lane's granule at j = 0 (relative to the slice)
  bool meta8;            // Int2: the chunk's two metadata words are one aligned 8-byte copy

  __device__ __forceinline__ void init(const uint8_t* const (&mat)[NM],
                                       const uint32_t* const (&meta)[NM], size_t row_bytes,
                                       int gpr, int tile, int k0, int warp, int lane) {
    const int gr = lane & 3;
    const size_t kbytes = (size_t)k0 * BITS / 8 + (size_t)warp * 64 + gr * 16;
#pragma unroll
    for (int i = 0; i < RG; ++i) {
      const int r = i * 8 + (lane >> 2), m = r >> 4, rr = r & 15;
      src[i] = mat[m] + (size_t)(tile * 16 + rr) * row_bytes + kbytes;
    }
    tile_step = (size_t)32 * row_bytes;
    k_lane0 = warp * CK + gr * WT<BITS>::CODES;
    if constexpr (BITS != 16) {
      const int r = lane < Ring<NM>::ROWS ? lane : 0, m = r >> 4, rr = r & 15;
      msrc = meta[m] + (size_t)(tile * 16 + rr) * gpr + (k0 + warp * CK) / DYMOE_GROUP;
      mtile_step = 32 * gpr;
      meta8 = (((uintptr_t)msrc) & 7) == 0;   // invariant: every step is an even word count
    }
  }
  __device__ __forceinline__ void next_tile() {
#pragma unroll
    for (int i = 0; i < RG; ++i) src[i] += tile_step;
    if constexpr (BITS != 16) msrc += mtile_step;
  }
  // copy item j (chunk ci = warp + 8 j) into the stage at shared address st
  __device__ __forceinline__ void issue(uint32_t st, int j, int ci, int nck, int kl, bool ragged,
                                       int lane) const {
    if (ci >= nck) return;
    const int gr = lane & 3;
    const uint32_t dst = st + (lane >> 2) * 64 + gr * 16;
    if (!ragged || k_lane0 + j * kWarps * CK < kl) {
#pragma unroll
      for (int i = 0; i < RG; ++i) cp_async<16>(dst + i * 512, src[i] + (size_t)j * 512);
    }
    if constexpr (BITS != 16) {
      if (lane < Ring<NM>::ROWS) {
        const uint32_t* p = msrc + j * GADV;
        const uint32_t mdst = st + Ring<NM>::W_BYTES + lane * 8;
        if constexpr (BITS == 2) {
          const bool both = !ragged || ci * CK + DYMOE_GROUP < kl;
          if (both && meta8) {
            cp_async<8>(mdst, p);
          } else {
            cp_async<4>(mdst, p);
            if (both) cp_async<4>(mdst + 4, p + 1);
          }
        } else {
          cp_async<4>(mdst, p);
        }
      }
    }
  }
};

// One virtual CTA: expert e, k-slice [k0, k0 + kl), tiles [t0, t1), nt tokens whose x slice is
// staged at shared address xs (x_pos layout, row_gran granules per token).  Outputs: W13 -> bf16
// h at out[tok * ostride + n]; W2 -> fp32 partials at out[tok * ostride + n].
template <bool W13, int BITS>
__device__ __noinline__ void run_tiles(const DevExpert* __restrict__ experts, int e, int K, int k0,
                                       int kl, int t0, int t1, int nt, void* out, int ostride,
                                       uint32_t xs, int row_gran, float* red, uint32_t ring_base,
                                       int* sync) {
  using Tr = WT<BITS>;
  constexpr int NM = W13 ? 2 : 1;
  constexpr int S = Pipe<W13>::STAGES;
  constexpr int STAGE = Ring<NM>::STAGE;
  constexpr int CK = Tr::CHUNK_K;
  const int lane = threadIdx.x & 31;
  const int grp = threadIdx.x >> 8;                 // warp group: tiles t0 + grp, +2, ...
  const int warp = (threadIdx.x >> 5) & (kWarps - 1);  // warp within the group
  const int g = lane >> 2, c = lane & 3;
  const DevExpert& E = experts[e];
  const int wi = width_index(BITS);
  const uint8_t* mat[NM];
  const uint32_t* meta[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int mi = W13 ? m : 2;
    if constexpr (BITS == 16) {
      mat[m] = reinterpret_cast<const uint8_t*>(E.w[mi]);
      meta[m] = nullptr;
    } else {
      mat[m] = reinterpret_cast<const uint8_t*>(E.q[wi][mi].codes);
      meta[m] = E.q[wi][mi].meta;
    }
  }
  const int nck = (kl + CK - 1) / CK;            // chunks per tile (slice)
  const int cmax = (nck + kWarps - 1) / kWarps;  // per warp (same for all warps)
  const bool ragged = (kl % CK) != 0;
  const int my_tiles = (t1 - t0 - grp + 1) / 2;
  const int n_items = (my_tiles > 0 ? my_tiles : 0) * cmax;
  if (n_items == 0) return;
  const uint32_t ring = ring_base + (threadIdx.x >> 5) * (S * STAGE);
  red += grp * (2 * kWarps * NM * kRedTile);
  sync += grp * 4;   // [arrivals buf0, arrivals buf1, generation buf0, generation buf1]

  Producer<BITS, NM> pr;
  pr.init(mat, meta, (size_t)K * BITS / 8, K / DYMOE_GROUP, t0 + grp, k0, warp, lane);

  float acc[NM][4];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;

  // producer cursor: the next item to issue is chunk warp + 8 * j_iss of the producer's tile
  int j_iss = 0;
#pragma unroll
  for (int p = 0; p < S - 1; ++p) {
    if (p < n_items) pr.issue(ring + p * STAGE, j_iss, warp + kWarps * j_iss, nck, kl, ragged, lane);
    cp_commit();
    if (++j_iss == cmax) { j_iss = 0; pr.next_tile(); }
  }

  // this lane's x address at chunk 0: token row g, quad position c (x_pos layout)
  const uint32_t xlane = xs + (uint32_t)(g * row_gran + c) * 16;
  int tile_seq = 0;
  int tile = t0 + grp, j = 0;      // consumer cursor
  int slot = 0, slot_iss = S - 1;  // ring slots of the consumer / producer
  for (int q = 0; q < n_items; ++q) {
    // refill: item q + S - 1 goes into the slot consumed in the previous iteration
    if (q + S - 1 < n_items)
      pr.issue(ring + slot_iss * STAGE, j_iss, warp + kWarps * j_iss, nck, kl, ragged, lane);
    cp_commit();
    if (++j_iss == cmax) { j_iss = 0; pr.next_tile(); }
    if (++slot_iss == S) slot_iss = 0;
    const int ci = warp + kWarps * j;
    const bool live = ci < nck;
    // x for this chunk: beyond the slice the staged x is zero, so stale ring bytes (always
    // finite: the ring is zeroed at kernel start and only ever holds weights) contribute nothing
    const uint32_t xa = xlane + (uint32_t)ci * (2 * CK);
    cp_wait<S - 1>();
    __syncwarp();   // the stage's rows were copied by other lanes
    const uint32_t st = ring + slot * STAGE;
    if (live) {
      DQ dq[NM][2];
      if constexpr (BITS != 16) {
        const int gi = BITS == 2 ? (c >> 1) : 0;            // group within the chunk
#pragma unroll
        for (int m = 0; m < NM; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            dq[m][h] = dq_from_meta<BITS>(lds32(st + Ring<NM>::W_BYTES + (m * 16 + 8 * h + g) * 8 + gi * 4));
      }
      uint4 w[NM][2];
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) w[m][h] = lds128(st + (m * 16 + 8 * h + g) * 64 + c * 16);
      using X = XB<BITS>;
#pragma unroll
      for (int blk = 0; blk < X::NB; ++blk) {
        uint4 xb[X::GPB];
#pragma unroll
        for (int i = 0; i < X::GPB; ++i) xb[i] = lds128_const(xa + (blk * X::GPB + i) * 64);
#pragma unroll
        for (int ss = 0; ss < X::SPB; ++ss) {
          const int s = blk * X::SPB + ss;
          uint32_t b0, b1;
          b_frag<BITS>(xb, ss, b0, b1);
#pragma unroll
          for (int m = 0; m < NM; ++m) {
            uint32_t glo, ghi, g8lo, g8hi;
            a_frag<BITS>(w[m][0], dq[m][0], s, glo, ghi);
            a_frag<BITS>(w[m][1], dq[m][1], s, g8lo, g8hi);
            mma16816(acc[m], glo, g8lo, ghi, g8hi, b0, b1);
          }
        }
      }
    }
    __syncwarp();   // every lane is done with this stage before it is refilled
    if (++slot == S) slot = 0;
    if (++j == cmax) {
      // end of tile: partials -> red[buf][warp][m][tok][row16 (+pad)]; the LAST warp of the
      // group to arrive (shared-memory counter) reduces in warp order and applies the
      // epilogue -- no barrier, so warps drift up to one tile apart.  Buffer b = tile_seq & 1 is
      // reused by tile_seq + 2 only after its reduction bumped gen[b].
      j = 0;
      const int b = tile_seq & 1;
      if (lane == 0)
        while (*reinterpret_cast<volatile int*>(&sync[2 + b]) != (tile_seq >> 1)) {}
      __syncwarp();
      float* rb = red + b * (kWarps * NM * kRedTile);
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        float* pp = rb + (warp * NM + m) * kRedTile;
        pp[(2 * c) * kRedStride + g] = acc[m][0];
        pp[(2 * c + 1) * kRedStride + g] = acc[m][1];
        pp[(2 * c) * kRedStride + g + 8] = acc[m][2];
        pp[(2 * c + 1) * kRedStride + g + 8] = acc[m][3];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[m][i] = 0.f;
      }
      __threadfence_block();
      __syncwarp();
      int old = 0;
      if (lane == 0) old = atomicAdd(&sync[b], 1);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old == kWarps - 1) {
        __threadfence_block();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int o = lane + 32 * i, tok = o >> 4, r16 = o & 15;
          if (tok < nt) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
              const float* pp = rb + (w * NM) * kRedTile + tok * kRedStride + r16;
              s0 = __fadd_rn(s0, pp[0]);
              if (NM == 2) s1 = __fadd_rn(s1, pp[kRedTile]);
            }
            const int n = tile * 16 + r16;
            if (W13) {
              // silu(A) * B, fast exp / divide (well inside the FFN tolerance)
              const float silu = __fdividef(s0, 1.f + __expf(-s0));
              const __nv_bfloat16 hv = __float2bfloat16_rn(__fmul_rn(silu, s1));
              reinterpret_cast<__nv_bfloat16*>(out)[(size_t)tok * ostride + n] = hv;
            } else {
              reinterpret_cast<float*>(out)[(size_t)tok * ostride + n] = s0;
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          sync[b] = 0;
          __threadfence_block();
          *reinterpret_cast<volatile int*>(&sync[2 + b]) = (tile_seq >> 1) + 1;
        }
      }
      ++tile_seq;
      tile += 2;
    }
  }
  cp_wait<0>();
}

// x slice layout in shared memory ("x_pos"): [8 tokens][row_gran granules of 16 B].  Within each
// chunk of CK k values (4 * XU4 granules), the granule lane quad position c reads as its i-th
// (logical granule c * XU4 + i) is stored at position i * 4 + c, so a lane's XU4 loads are 64 B
// apart (immediate offsets) and the 4 lanes of a quad hit 4 consecutive bank groups; row_gran = 4
// (mod 8) puts the other token row of an LDS.128 phase on the other four.
__device__ __forceinline__ int x_logical(int pos, int xu4) {
  const int span = 4 * xu4;
  const int chunk = pos / span, w = pos - chunk * span;
  return chunk * span + (w & 3) * xu4 + (w >> 2);
}
__host__ __device__ inline int x_row_gran(int sliceK) { return (sliceK + 255) / 256 * 32 + 4; }

template <bool W13>
__global__ void __launch_bounds__(2 * kThreads, 1) k_decode_gemv(const FfnArgs a, int SK, int sliceK) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ Alloc A;
  __shared__ int tile_sync[8];   // per warp group: arrival counters + generations (run_tiles)
  constexpr int NM = W13 ? 2 : 1;
  const size_t red_bytes = 2 * 2 * kWarps * NM * kRedTile * sizeof(float);  // [group][buf]
  float* red = reinterpret_cast<float*>(smem);
  const uint32_t ring_base = (uint32_t)__cvta_generic_to_shared(smem + red_bytes);
  const size_t ring_bytes = (size_t)2 * kWarps * Pipe<W13>::STAGES * Ring<NM>::STAGE;
  uint4* xs = reinterpret_cast<uint4*>(smem + red_bytes + ring_bytes);
  const int K = W13 ? a.Hd : a.F;
  const int N = W13 ? a.F : a.Hd;
  const int NT = N / 16;
  const int row_gran = x_row_gran(sliceK);
  if (threadIdx.x == 0) compute_alloc(a, gridDim.x / SK, W13, A);
  {  // zero the weight ring once: stale stage bytes are then always finite (see run_tiles)
    uint4* rz = reinterpret_cast<uint4*>(smem + red_bytes);
    const int n16 = (int)(ring_bytes / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) rz[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  if (A.n_act == 0) return;
  const int V = A.units_total * SK;
  for (int v = blockIdx.x; v < V; v += gridDim.x) {
    const int unit = v / SK, ks = v - unit * SK;
    int i = 0;
    while (A.first_unit[i + 1] <= unit) ++i;
    const int e = A.expert[i];
    const int u_e = A.first_unit[i + 1] - A.first_unit[i];
    const int part = unit - A.first_unit[i];
    const int t0 = (int)((long long)part * NT / u_e), t1 = (int)((long long)(part + 1) * NT / u_e);
    const int k0 = ks * sliceK;
    const int kl = min(sliceK, K - k0);
    const int be = a.bits[e];
    const int r_lo = a.expert_off[e], r_hi = a.expert_off[e + 1];
    // residency check (device-side fault -> status word; outputs zeroed)
    bool resident = true;
    const DevExpert& E = a.experts[e];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const int mi = W13 ? m : 2;
      if (be == 16) resident &= E.w[mi] != nullptr;
      else resident &= width_index(be) >= 0 && E.q[width_index(be)][mi].codes != nullptr;
    }
    if (!resident) {
      if (threadIdx.x == 0 && a.status) atomicOr(a.status, (unsigned)DYMOE_STATUS_WIDTH_NOT_RESIDENT);
      for (int r = r_lo; r < r_hi; ++r)
        for (int n = t0 * 16 + threadIdx.x; n < t1 * 16; n += blockDim.x) {
          if (W13) a.h[(size_t)r * a.F + n] = 0;
          else a.y_part[((size_t)ks * a.part_rows + r) * a.Hd + n] = 0.f;
        }
      continue;
    }
    if (t1 <= t0 || kl <= 0) continue;
    int xu4;
    switch (be) {
      case 2: xu4 = WT<2>::XU4; break;
      case 4: xu4 = WT<4>::XU4; break;
      case 8: xu4 = WT<8>::XU4; break;
      default: xu4 = WT<16>::XU4; break;
    }
    const int gran = kl / 8;                        // granules of real x
    const int npos = (kl + 255) / 256 * 32;         // staged positions (zero beyond gran)
    for (int tok0 = r_lo; tok0 < r_hi; tok0 += kMaxTok) {
      const int nt = min(kMaxTok, r_hi - tok0);
      // stage the x slice of this pass's tokens (zero rows beyond nt), x_pos layout
      __syncthreads();  // the previous pass is done with xs / red / tile_sync
      if (threadIdx.x < 8) tile_sync[threadIdx.x] = 0;
      for (int idx = threadIdx.x; idx < kMaxTok * npos; idx += blockDim.x) {
        const int t = idx / npos, pos = idx - t * npos;
        const int gl = x_logical(pos, xu4);
        uint4 v4 = make_uint4(0, 0, 0, 0);
        if (t < nt && gl < gran) {
          const int r = tok0 + t;
          const uint16_t* src = W13 ? a.x + (size_t)a.perm_token[r] * a.Hd : a.h + (size_t)r * a.F;
          v4 = *reinterpret_cast<const uint4*>(src + k0 + gl * 8);
        }
        xs[t * row_gran + pos] = v4;
      }
      __syncthreads();
      void* out = W13 ? (void*)(a.h + (size_t)tok0 * a.F)
                      : (void*)(a.y_part + ((size_t)ks * a.part_rows + tok0) * a.Hd);
      const int ostride = W13 ? a.F : a.Hd;
      const uint32_t xsa = (uint32_t)__cvta_generic_to_shared(xs);
#define DYMOE_RUN(B) run_tiles<W13, B>(a.experts, e, K, k0, kl, t0, t1, nt, out, ostride, xsa, \
                                       row_gran, red, ring_base, tile_sync)
      switch (be) {
        case 2: DYMOE_RUN(2); break;
        case 4: DYMOE_RUN(4); break;
        case 8: DYMOE_RUN(8); break;
        default: DYMOE_RUN(16); break;
      }
#undef DYMOE_RUN
    }
  }
}

size_t smem_bytes(bool w13, int sliceK) {
  const int NM = w13 ? 2 : 1;
  const size_t ring = w13 ? (size_t)2 * kWarps * Pipe<true>::STAGES * Ring<2>::STAGE
                          : (size_t)2 * kWarps * Pipe<false>::STAGES * Ring<1>::STAGE;
  return 2 * 2 * kWarps * NM * kRedTile * sizeof(float) + ring +
         (size_t)kMaxTok * x_row_gran(sliceK) * 16;
}

}  // namespace dec
using namespace dec;

int decode_w2_slice_k(int F) {
  // K = F is split into slices so that each virtual CTA's x slice (<= 8 tokens of h) stays
  // L1-resident: 2048 when it divides F, else the smallest multiple of 512 giving <= 4096.
  if (F % 2048 == 0) return 2048;
  const int sk = (F + 4095) / 4096;
  const int per = (F + sk - 1) / sk;
  return (per + 511) / 512 * 512;
}
int decode_w2_slices(int F) {
  const int sl = decode_w2_slice_k(F);
  return (F + sl - 1) / sl;
}

cudaError_t launch_ffn_decode(const FfnArgs& a, cudaStream_t s, void* const* ev) {
  static int sms = 0, dyn_max13 = 0, dyn_max2 = 0;
  const int SK = decode_w2_slices(a.F), sliceK = decode_w2_slice_k(a.F);
  const size_t sm13 = smem_bytes(true, a.Hd), sm2 = smem_bytes(false, sliceK);
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // opt in to the maximum once (227 KB per block minus the static Alloc table); the
    // per-launch size is what each launch requests
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa13{}, fa2{};
    cudaFuncGetAttributes(&fa13, k_decode_gemv<true>);
    cudaFuncGetAttributes(&fa2, k_decode_gemv<false>);
    dyn_max13 = optin - (int)fa13.sharedSizeBytes;
    dyn_max2 = optin - (int)fa2.sharedSizeBytes;
    cudaFuncSetAttribute(k_decode_gemv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max13);
    cudaFuncSetAttribute(k_decode_gemv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max2);
  }
  if ((int)sm13 > dyn_max13 || (int)sm2 > dyn_max2) return cudaErrorInvalidConfiguration;
  const int grid = sms;   // one 512-thread CTA (two 8-warp groups) per SM
  record_ev(ev, 0, s);
  k_decode_gemv<true><<<grid, 2 * kThreads, sm13, s>>>(a, 1, a.Hd);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  record_ev(ev, 1, s);
  const int g2 = grid / SK * SK;
  k_decode_gemv<false><<<g2 > 0 ? g2 : SK, 2 * kThreads, sm2, s>>>(a, SK, sliceK);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  record_ev(ev, 2, s);
  return cudaSuccess;
}

}  // namespace dymoe
