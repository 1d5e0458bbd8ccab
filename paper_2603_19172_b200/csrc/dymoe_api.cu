// Host side of the C ABI declared in include/dymoe.h: argument validation (messages name the
// offending field), the fp64 depth-aware schedule (Eq. 4-5), workspace layout, the expert-table
// handle, and launch orchestration of the per-step kernels on the caller's stream.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "dymoe_internal.cuh"

using namespace dymoe;


namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int ok() {
  g_err.clear();
  return DYMOE_OK;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(DYMOE_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CHECK_ARG(cond, ...) \
  do {                       \
    if (!(cond)) return fail(DYMOE_ERR_INVALID, __VA_ARGS__); \
  } while (0)

#define CHECK_LAUNCH(expr, where)                    \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

bool valid_width(int b) { return b == 16 || b == 8 || b == 4 || b == 2 || b == 0; }

int check_ladder(const dymoe_ladder* L) {
  CHECK_ARG(L != nullptr, "ladder: must not be NULL");
  CHECK_ARG(L->n_tiers >= 1 && L->n_tiers <= DYMOE_MAX_TIERS, "ladder.n_tiers: must be in [1, %d]",
            DYMOE_MAX_TIERS);
  for (int i = 0; i < L->n_tiers; ++i)
    CHECK_ARG(valid_width(L->bits[i]), "ladder.bits[%d]: %d is not one of 16, 8, 4, 2, 0", i,
              L->bits[i]);
  for (int i = 0; i + 1 < L->n_tiers; ++i) {
    CHECK_ARG(L->bits[i] > L->bits[i + 1], "ladder.bits: widths must be strictly decreasing");
    CHECK_ARG(L->lambdas[i] >= 0.0 && L->lambdas[i] <= 1.0,
              "ladder.lambdas[%d]: must lie in [0, 1]", i);
    if (i > 0)
      CHECK_ARG(L->lambdas[i] >= L->lambdas[i - 1], "ladder.lambdas: must be non-decreasing");
  }
  CHECK_ARG(L->m_mode == DYMOE_M_TOTAL || L->m_mode == DYMOE_M_ACTIVE,
            "ladder.m_mode: must be DYMOE_M_TOTAL or DYMOE_M_ACTIVE");
  return DYMOE_OK;
}

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

constexpr int kPrefillSmallRows = 16;

struct WsLayout {
  size_t topk_idx, topk_w, probs, importance, heavy, bits, active, active_list, expert_off,
      perm_token, perm_slot, inv_row, h, y_perm, y_part, status, score_scratch, perm_scratch, total;
};

WsLayout ws_layout(int M, int k, int Hd, int F, int T) {
  WsLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + bytes);
    return at;
  };
  const size_t TK = (size_t)T * k;
  L.topk_idx = take(TK * 4);
  L.topk_w = take(TK * 4);
  L.probs = take((size_t)T * M * 4);
  L.importance = take((size_t)M * 4);
  L.heavy = take((size_t)T * 4);
  L.bits = take((size_t)M);
  L.active = take((size_t)M);
  L.active_list = take((size_t)3 * (M + 1) * 4);   // + the two lists of the prefill split
  L.expert_off = take((size_t)(M + 1) * 4);
  L.perm_token = take(TK * 4);
  L.perm_slot = take(TK * 4);
  L.inv_row = take(TK * 4);
  L.h = take(TK * F * 2);
  L.y_perm = take(TK * Hd * 4);
  L.y_part = take((size_t)decode_w2_slices(F) * TK * Hd * 4);
  L.status = take(4);
  L.score_scratch = take((size_t)T * 4);
  L.perm_scratch = take(permute_scratch_bytes(T, k, M));
  L.total = o;
  return L;
}

cudaStream_t S(dymoe_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int check_ptr_align(const void* p, size_t a, const char* name) {
  CHECK_ARG(((uintptr_t)p % a) == 0, "%s: must be %zu-byte aligned", name, a);
  return DYMOE_OK;
}

}  // namespace

extern "C" {

const char* dymoe_last_error(void) { return g_err.c_str(); }
const char* dymoe_version(void) { return "dymoe-b200 0.1 (sm_100a)"; }

// ------------------------------------------------------------------------------------------
int dymoe_route(const float* logits, int T, int M, int k, int32_t* topk_idx, float* topk_w,
                float* probs, dymoe_stream_t stream) {
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(k >= 1 && k <= M && k <= 8, "k: must satisfy 1 <= k <= min(M, 8)");
  if (T > 0) {
    CHECK_ARG(logits != nullptr, "logits: must not be NULL");
    CHECK_ARG(topk_idx != nullptr, "topk_idx: must not be NULL");
    CHECK_ARG(topk_w != nullptr, "topk_w: must not be NULL");
  }
  CHECK_LAUNCH(launch_route(logits, T, M, k, topk_idx, topk_w, probs, S(stream)), "dymoe_route");
  return ok();
}

size_t dymoe_score_scratch_bytes(int T) { return (size_t)(T > 0 ? T : 1) * 4; }

int dymoe_score(int phase, const float* attn_mass, int H, const int32_t* topk_idx,
                const float* logits, int T, int M, int k, int k_tokens, float* importance,
                int32_t* heavy, void* scratch, dymoe_stream_t stream) {
  CHECK_ARG(phase == DYMOE_PREFILL || phase == DYMOE_DECODE, "phase: must be DYMOE_PREFILL or DYMOE_DECODE");
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(importance != nullptr, "importance: must not be NULL");
  if (phase == DYMOE_PREFILL) {
    CHECK_ARG(k >= 1 && k <= M, "k: must satisfy 1 <= k <= M");
    CHECK_ARG(H >= 1, "H: must be >= 1");
    if (k_tokens == 0) k_tokens = (T + 4) / 5;
    CHECK_ARG(k_tokens >= 0 && k_tokens <= T, "k_tokens: must satisfy 0 <= k_tokens <= T");
    if (T > 0) {
      CHECK_ARG(attn_mass != nullptr, "attn_mass: must not be NULL in PREFILL");
      CHECK_ARG(topk_idx != nullptr, "topk_idx: must not be NULL in PREFILL");
      CHECK_ARG(scratch != nullptr, "scratch: must not be NULL in PREFILL");
    }
    CHECK_LAUNCH(launch_score_prefill(attn_mass, H, topk_idx, T, M, k, k_tokens, importance,
                                      heavy, reinterpret_cast<float*>(scratch), S(stream)),
                 "dymoe_score");
  } else {
    CHECK_ARG(T >= 1, "T: DECODE needs at least one token");
    CHECK_ARG(logits != nullptr, "logits: must not be NULL in DECODE");
    CHECK_LAUNCH(launch_score_decode(logits, T, M, importance, S(stream)), "dymoe_score");
  }
  return ok();
}

// ------------------------------------------------------------------------------------------
double dymoe_retention_ratio(int layer, int num_layers, double lambda) {
  if (num_layers <= 1) return 1.0;
  const double pi = 3.14159265358979323846;
  return (1.0 - lambda) * (std::cos(pi * (double)layer / (double)(num_layers - 1)) + 1.0) / 2.0 +
         lambda;
}

int dymoe_tier_counts(int layer, int num_layers, const dymoe_ladder* ladder, int M_eff,
                      int k_route, int32_t* counts) {
  int rc = check_ladder(ladder);
  if (rc) return rc;
  CHECK_ARG(num_layers >= 1, "num_layers: must be >= 1");
  CHECK_ARG(layer >= 0 && layer < num_layers, "layer: must satisfy 0 <= layer < num_layers");
  CHECK_ARG(M_eff >= 0, "M_eff: must be >= 0");
  CHECK_ARG(counts != nullptr || ladder->n_tiers == 1, "counts: must not be NULL");
  int prev = 0;
  for (int q = 0; q + 1 < ladder->n_tiers; ++q) {
    const double r = dymoe_retention_ratio(layer, num_layers, ladder->lambdas[q]);
    int t = (int)std::ceil(r * (double)M_eff - 1e-9);
    if (q == 0 && ladder->clamp_to_k) t = std::max(t, std::min(k_route, M_eff));
    t = std::max(t, prev);
    t = std::min(t, M_eff);
    prev = t;
    counts[q] = t;
  }
  return ok();
}

}  // extern "C"

int dymoe::assign_params(const dymoe_ladder* ladder, int M, int k_route, int layer,
                         int num_layers, AssignParams& p) {
  int rc = check_ladder(ladder);
  if (rc) return rc;
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(num_layers >= 1, "num_layers: must be >= 1");
  CHECK_ARG(layer >= 0 && layer < num_layers, "layer: must satisfy 0 <= layer < num_layers");
  CHECK_ARG(k_route >= 1 && k_route <= M, "k_route: must satisfy 1 <= k_route <= M");
  p.M = M;
  p.k_route = k_route;
  p.n_tiers = ladder->n_tiers;
  p.clamp_to_k = ladder->clamp_to_k;
  p.m_active = ladder->m_mode == DYMOE_M_ACTIVE;
  for (int i = 0; i < DYMOE_MAX_TIERS; ++i) p.bits[i] = i < ladder->n_tiers ? ladder->bits[i] : 0;
  for (int i = 0; i + 1 < DYMOE_MAX_TIERS; ++i)
    p.r[i] = i + 1 < ladder->n_tiers ? dymoe_retention_ratio(layer, num_layers, ladder->lambdas[i])
                                     : 0.0;
  return DYMOE_OK;
}

extern "C" {

int dymoe_assign_bits(const float* importance, int M, int layer, int num_layers,
                      const dymoe_ladder* ladder, int k_route, const uint8_t* active_mask,
                      uint8_t* bits, int32_t* tier_counts, dymoe_stream_t stream) {
  AssignParams p{};
  int rc = assign_params(ladder, M, k_route, layer, num_layers, p);
  if (rc) return rc;
  CHECK_ARG(importance != nullptr, "importance: must not be NULL");
  CHECK_ARG(bits != nullptr, "bits: must not be NULL");
  CHECK_ARG(!p.m_active || active_mask != nullptr, "active_mask: required in DYMOE_M_ACTIVE mode");
  if (tier_counts != nullptr && !p.m_active) {
    rc = dymoe_tier_counts(layer, num_layers, ladder, M, k_route, tier_counts);
    if (rc) return rc;
  }
  CHECK_LAUNCH(launch_assign(importance, active_mask, nullptr, 0, p, bits, nullptr, S(stream)),
               "dymoe_assign_bits");
  return ok();
}

// ------------------------------------------------------------------------------------------
static int check_quant_job(const dymoe_quant_job& j, int idx, int group) {
  CHECK_ARG(group == DYMOE_GROUP, "group: only %d is supported", DYMOE_GROUP);
  CHECK_ARG(j.bits == 2 || j.bits == 4 || j.bits == 8, "jobs[%d].bits: must be 2, 4 or 8", idx);
  CHECK_ARG(j.N >= 0, "jobs[%d].N: must be >= 0", idx);
  CHECK_ARG(j.K > 0 && j.K % DYMOE_GROUP == 0, "jobs[%d].K: must be a positive multiple of %d", idx,
            DYMOE_GROUP);
  if (j.N > 0) {
    CHECK_ARG(j.W != nullptr, "jobs[%d].W: must not be NULL", idx);
    CHECK_ARG(j.codes != nullptr, "jobs[%d].codes: must not be NULL", idx);
    CHECK_ARG(j.scales != nullptr, "jobs[%d].scales: must not be NULL", idx);
    CHECK_ARG(j.zeros != nullptr, "jobs[%d].zeros: must not be NULL", idx);
    int rc = check_ptr_align(j.W, 16, "W");
    if (rc) return rc;
    rc = check_ptr_align(j.codes, 16, "codes");
    if (rc) return rc;
  }
  return DYMOE_OK;
}

int dymoe_quantize(const uint16_t* W, int N, int K, int bits, int group, uint32_t* codes,
                   float* scales, uint8_t* zeros, dymoe_stream_t stream) {
  dymoe_quant_job j{W, N, K, bits, codes, scales, zeros};
  int rc = check_quant_job(j, 0, group);
  if (rc) {
    // rename "jobs[0]." to the flat argument names
    std::string m = g_err;
    const std::string pre = "jobs[0].";
    if (m.compare(0, pre.size(), pre) == 0) g_err = m.substr(pre.size());
    return rc;
  }
  CHECK_LAUNCH(launch_quantize(&j, 1, S(stream)), "dymoe_quantize");
  return ok();
}

int dymoe_quantize_batched(const dymoe_quant_job* jobs, int n_jobs, int group,
                           dymoe_stream_t stream) {
  CHECK_ARG(n_jobs >= 0, "n_jobs: must be >= 0");
  CHECK_ARG(jobs != nullptr || n_jobs == 0, "jobs: must not be NULL");
  for (int i = 0; i < n_jobs; ++i) {
    int rc = check_quant_job(jobs[i], i, group);
    if (rc) return rc;
  }
  CHECK_LAUNCH(launch_quantize(jobs, n_jobs, S(stream)), "dymoe_quantize_batched");
  return ok();
}

// ------------------------------------------------------------------------------------------
// TMA descriptors (driver entry point fetched once through the runtime: no -lcuda)
namespace {
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {   // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}
// tiled map over a row-major tensor of rank 2 or 3 (strides in bytes for dims 1.., box per dim)
bool encode(CUtensorMap* m, CUtensorMapDataType dt, const void* base, int rank, const uint64_t* dims,
            const uint64_t* strides, const uint32_t* box, CUtensorMapSwizzle swz) {
  auto fn = tmap_encoder();
  if (fn == nullptr) return false;
  cuuint64_t d[3], st[2];
  cuuint32_t b[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    if (i + 1 < rank) st[i] = strides[i];
  }
  return fn(m, dt, rank, const_cast<void*>(base), d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// codes / bf16 rows: u8 {row_bytes, N}, 128 x 16 boxes, 128-byte swizzle (decode kernel items)
bool encode_rows(CUtensorMap* m, const void* base, uint64_t row_bytes, uint64_t N) {
  const uint64_t dims[2] = {row_bytes, N}, str[1] = {row_bytes};
  const uint32_t box[2] = {128, 16};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}
// group-major meta [n_mat][gpr][N] u32: boxes {rows, gq groups, n_mat} (W1 / W3: the 16 rows of a
// decode tile of both matrices; W2: the 32 rows of a W2 tile in one box)
bool encode_meta(CUtensorMap* m, const void* base, uint64_t N, uint64_t gpr, int n_mat, uint32_t gq,
                 uint32_t rows) {
  const uint64_t dims[3] = {N, gpr, (uint64_t)n_mat}, str[2] = {N * 4, N * gpr * 4};
  const uint32_t box[3] = {rows, gq, (uint32_t)n_mat};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, base, n_mat > 1 ? 3 : 2, dims, str, box,
                CU_TENSOR_MAP_SWIZZLE_NONE);
}
constexpr int kMapsPerExpert = 42;   // 3 + 3 bf16 masters (decode, prefill boxes) + 3 widths x 3
                                     // matrices x (codes, meta) x (decode, prefill boxes)
}  // namespace

namespace {
// Expert e's slice of the layer's derived metadata: [width][W1 | W3 | W2] group-major words, W1
// and W3 adjacent (one 3-D TMA box feeds both).  Allocated for every width at create, so that a
// format bound later (dymoe_layer_set_expert) has its slot.
size_t meta_words_per_expert(int Hd, int F) { return (size_t)3 * 3 * F * (Hd / DYMOE_GROUP); }
uint32_t* meta_slot(dymoe_layer* L, int e, int wi, int m) {
  const size_t w13 = (size_t)L->F * (L->Hd / DYMOE_GROUP);   // == W2's N * gpr as well
  return L->meta_pool + (size_t)e * meta_words_per_expert(L->Hd, L->F) + ((size_t)wi * 3 + m) * w13;
}

int validate_expert(const dymoe_expert_desc& x, int e) {
  for (int wi = 0; wi < 3; ++wi)
    for (int m = 0; m < 3; ++m) {
      if (x.q[wi][m].codes != nullptr && (x.q[wi][m].scales == nullptr || x.q[wi][m].zeros == nullptr))
        return fail(DYMOE_ERR_INVALID, "desc.experts[%d].q[%d][%d]: scales/zeros must be set with codes", e, wi, m);
      if (((uintptr_t)x.q[wi][m].codes) % 16)
        return fail(DYMOE_ERR_INVALID, "desc.experts[%d].q[%d][%d].codes: must be 16-byte aligned", e, wi, m);
    }
  const uint16_t* w[3] = {x.w1, x.w3, x.w2};
  for (int m = 0; m < 3; ++m)
    if (((uintptr_t)w[m]) % 16)
      return fail(DYMOE_ERR_INVALID, "desc.experts[%d].w%d: must be 16-byte aligned", e, m == 0 ? 1 : m == 1 ? 3 : 2);
  return DYMOE_OK;
}

// (Re)bind expert e to the formats in x: table entry, derived metadata (k_build_meta on stream)
// and TMA descriptors; the device copies are stream-ordered.
int bind_expert(dymoe_layer* L, int e, const dymoe_expert_desc& x, cudaStream_t stream) {
  DevExpert& y = L->host[e];
  y.w[0] = x.w1;
  y.w[1] = x.w3;
  y.w[2] = x.w2;
  for (int wi = 0; wi < 3; ++wi)
    for (int m = 0; m < 3; ++m) {
      DevQMat& q = y.q[wi][m];
      q.codes = x.q[wi][m].codes;
      q.scales = x.q[wi][m].scales;
      q.zeros = x.q[wi][m].zeros;
      q.meta = nullptr;
      if (q.codes == nullptr) continue;
      const size_t N = m == 2 ? L->Hd : L->F, K = m == 2 ? L->F : L->Hd;
      q.meta = meta_slot(L, e, wi, m);
      cudaError_t err = launch_build_meta(q.scales, q.zeros, (int)N, (int)(K / DYMOE_GROUP),
                                          const_cast<uint32_t*>(q.meta), stream);
      if (err != cudaSuccess) return cuda_fail(err, "bind expert");
    }
  std::vector<CUtensorMap> hm(kMapsPerExpert);
  memset(hm.data(), 0, hm.size() * sizeof(CUtensorMap));
  const CUtensorMap* dm = L->tmap_pool + (size_t)e * kMapsPerExpert;
  bool maps_ok = true;
  for (int m = 0; m < 3; ++m) {
    const uint64_t N = m == 2 ? L->Hd : L->F, K = m == 2 ? L->F : L->Hd;
    y.tm_w[m] = y.tm_wp[m] = nullptr;
    if (y.w[m] != nullptr) {
      maps_ok &= encode_rows(&hm[m], y.w[m], 2 * K, N);
      y.tm_w[m] = dm + m;
      const uint64_t dims[2] = {K, N}, str[1] = {2 * K};
      const uint32_t box[2] = {64, 128};
      maps_ok &= encode(&hm[21 + m], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y.w[m], 2, dims, str, box,
                        CU_TENSOR_MAP_SWIZZLE_128B);
      y.tm_wp[m] = dm + 21 + m;
    }
    for (int wi = 0; wi < 3; ++wi) {
      DevQMat& q = y.q[wi][m];
      q.tm_codes = q.tm_meta = q.tm_raw = q.tm_rawmeta = nullptr;
      if (q.codes == nullptr) continue;
      const int b = wi == 0 ? 8 : wi == 1 ? 4 : 2;
      const uint32_t gq = (uint32_t)(2 * 512 / b / DYMOE_GROUP);   // groups per 128-byte item
      const int ic = 3 + (wi * 3 + m) * 2, im = ic + 1;
      maps_ok &= encode_rows(&hm[ic], q.codes, K * b / 8, N);
      q.tm_codes = dm + ic;
      {  // prefill producer boxes: 64 k x 128 rows of codes, one group's words of 128 rows
        const int ir = 24 + (wi * 3 + m) * 2, irm = ir + 1;
        const uint64_t rb = K * b / 8;
        const uint64_t dims[2] = {rb, N}, str[1] = {rb};
        const uint32_t box[2] = {(uint32_t)(64 * b / 8), 128};
        const CUtensorMapSwizzle swz = b == 8 ? CU_TENSOR_MAP_SWIZZLE_64B
                                     : b == 4 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
        maps_ok &= encode(&hm[ir], CU_TENSOR_MAP_DATA_TYPE_UINT8, q.codes, 2, dims, str, box, swz);
        const uint64_t mdims[2] = {N, K / DYMOE_GROUP}, mstr[1] = {N * 4};
        const uint32_t mbox[2] = {128, 1};
        maps_ok &= encode(&hm[irm], CU_TENSOR_MAP_DATA_TYPE_UINT32, q.meta, 2, mdims, mstr, mbox,
                          CU_TENSOR_MAP_SWIZZLE_NONE);
        q.tm_raw = dm + ir;
        q.tm_rawmeta = dm + irm;
      }
      // W2: 2-D meta; W1: 3-D over the adjacent W1 / W3 meta (one box feeds both matrices);
      // W3's own descriptor is not needed by the kernels
      const bool pair = m == 0 && y.q[wi][1].codes != nullptr;
      if (m == 2 || pair) {
        maps_ok &= encode_meta(&hm[im], q.meta, N, K / DYMOE_GROUP, pair ? 2 : 1, gq, m == 2 ? 32 : 16);
        q.tm_meta = dm + im;
      }
    }
  }
  if (!maps_ok) return fail(DYMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  // pageable sources: the copies are staged before cudaMemcpyAsync returns
  cudaError_t err = cudaMemcpyAsync(const_cast<CUtensorMap*>(dm), hm.data(),
                                    hm.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice, stream);
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(L->dev + e, &y, sizeof(DevExpert), cudaMemcpyHostToDevice, stream);
  if (err != cudaSuccess) return cuda_fail(err, "bind expert");
  return DYMOE_OK;
}
}  // namespace

int dymoe_layer_create(const dymoe_layer_desc* d, dymoe_layer** out) {
  CHECK_ARG(out != nullptr, "out: must not be NULL");
  *out = nullptr;
  CHECK_ARG(d != nullptr, "desc: must not be NULL");
  CHECK_ARG(d->M >= 1 && d->M <= DYMOE_MAX_EXPERTS, "desc.M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(d->k_route >= 1 && d->k_route <= d->M && d->k_route <= 8,
            "desc.k_route: must satisfy 1 <= k_route <= min(M, 8)");
  CHECK_ARG(d->hidden > 0 && d->hidden % 128 == 0, "desc.hidden: must be a positive multiple of 128");
  CHECK_ARG(d->ffn > 0 && d->ffn % 128 == 0, "desc.ffn: must be a positive multiple of 128");
  CHECK_ARG(d->experts != nullptr, "desc.experts: must not be NULL");
  for (int e = 0; e < d->M; ++e) {
    const int rc = validate_expert(d->experts[e], e);
    if (rc) return rc;
  }
  dymoe_layer* L = new (std::nothrow) dymoe_layer();
  if (!L) return fail(DYMOE_ERR_INVALID, "out of host memory");
  L->M = d->M;
  L->k = d->k_route;
  L->Hd = d->hidden;
  L->F = d->ffn;
  L->host.resize(d->M);
  cudaError_t e = cudaMalloc(&L->meta_pool, meta_words_per_expert(d->hidden, d->ffn) * d->M * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&L->dev, sizeof(DevExpert) * d->M);
  if (e == cudaSuccess) e = cudaMalloc(&L->tmap_pool, (size_t)d->M * kMapsPerExpert * sizeof(CUtensorMap));
  if (e != cudaSuccess) {
    dymoe_layer_destroy(L);
    return cuda_fail(e, "dymoe_layer_create");
  }
  for (int ex = 0; ex < d->M; ++ex) {
    const int rc = bind_expert(L, ex, d->experts[ex], nullptr);
    if (rc) {
      dymoe_layer_destroy(L);
      return rc;
    }
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    dymoe_layer_destroy(L);
    return cuda_fail(e, "dymoe_layer_create");
  }
  *out = L;
  return ok();
}

int dymoe_layer_set_expert(dymoe_layer* L, int expert, const dymoe_expert_desc* desc,
                           dymoe_stream_t stream) {
  CHECK_ARG(L != nullptr, "layer: must not be NULL");
  CHECK_ARG(desc != nullptr, "desc: must not be NULL");
  CHECK_ARG(expert >= 0 && expert < L->M, "expert: must be in [0, %d)", L->M);
  const int rc = validate_expert(*desc, expert);
  if (rc) return rc;
  const int rb = bind_expert(L, expert, *desc, S(stream));
  if (rb) return rb;
  return ok();
}

int dymoe_layer_refresh(dymoe_layer* L, dymoe_stream_t stream) {
  CHECK_ARG(L != nullptr, "layer: must not be NULL");
  for (int ex = 0; ex < L->M; ++ex)
    for (int wi = 0; wi < 3; ++wi)
      for (int m = 0; m < 3; ++m) {
        const DevQMat& q = L->host[ex].q[wi][m];
        if (q.codes == nullptr) continue;
        const size_t N = m == 2 ? L->Hd : L->F, K = m == 2 ? L->F : L->Hd;
        CHECK_LAUNCH(launch_build_meta(q.scales, q.zeros, (int)N, (int)(K / DYMOE_GROUP),
                                       const_cast<uint32_t*>(q.meta), S(stream)),
                     "dymoe_layer_refresh");
      }
  return ok();
}

int dymoe_layer_destroy(dymoe_layer* L) {
  if (!L) return ok();
  if (L->dev) cudaFree(L->dev);
  if (L->meta_pool) cudaFree(L->meta_pool);
  if (L->tmap_pool) cudaFree(L->tmap_pool);
  delete L;
  return ok();
}

// ------------------------------------------------------------------------------------------
size_t dymoe_permute_scratch_bytes(int T, int k, int M) {
  if (T < 0 || k < 1 || M < 1) return 0;
  return align_up((size_t)(M + 1) * sizeof(int32_t)) + align_up(permute_scratch_bytes(T, k, M));
}

int dymoe_permute(const int32_t* topk_idx, int T, int k, int M, const uint8_t* bits,
                  int32_t* expert_off, int32_t* perm_token, int32_t* perm_slot, int32_t* inv_row,
                  void* scratch_ws, size_t scratch_bytes, dymoe_stream_t stream) {
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(k >= 1 && k <= M, "k: must satisfy 1 <= k <= M");
  CHECK_ARG(bits != nullptr, "bits: must not be NULL");
  CHECK_ARG(expert_off != nullptr, "expert_off: must not be NULL");
  if (T > 0) {
    CHECK_ARG(topk_idx != nullptr, "topk_idx: must not be NULL");
    CHECK_ARG(perm_token && perm_slot && inv_row, "perm_token/perm_slot/inv_row: must not be NULL");
  }
  const size_t need = dymoe_permute_scratch_bytes(T, k, M);
  CHECK_ARG(scratch_ws != nullptr, "scratch: must not be NULL");
  if (scratch_bytes < need)
    return fail(DYMOE_ERR_WORKSPACE, "scratch_bytes: %zu < dymoe_permute_scratch_bytes = %zu",
                scratch_bytes, need);
  int rc = check_ptr_align(scratch_ws, 256, "scratch");
  if (rc) return rc;
  // the active list is an internal by-product (first section of the scratch)
  int32_t* active = reinterpret_cast<int32_t*>(scratch_ws);
  int32_t* scratch = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(scratch_ws) +
                                                align_up((size_t)(M + 1) * sizeof(int32_t)));
  CHECK_LAUNCH(launch_permute(topk_idx, T, k, M, bits, expert_off, perm_token, perm_slot, inv_row,
                              active, S(stream), scratch),
               "dymoe_permute");
  return ok();
}

int dymoe_ep_plan(const int32_t* expert_off, int M, int P, int32_t* send_counts,
                  int32_t* row_expert, dymoe_stream_t stream) {
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(P >= 1 && P <= M && P <= 64, "P: must satisfy 1 <= P <= min(M, 64)");
  CHECK_ARG(expert_off != nullptr, "expert_off: must not be NULL");
  CHECK_ARG(send_counts != nullptr, "send_counts: must not be NULL");
  CHECK_ARG(row_expert != nullptr, "row_expert: must not be NULL");
  CHECK_LAUNCH(launch_ep_plan(expert_off, M, P, send_counts, row_expert, S(stream)), "dymoe_ep_plan");
  return ok();
}

int dymoe_gather_rows(const uint16_t* x, int Hd, const int32_t* rows, int n, uint16_t* out,
                      dymoe_stream_t stream) {
  CHECK_ARG(Hd > 0 && Hd % 8 == 0, "Hd: must be a positive multiple of 8");
  CHECK_ARG(n >= 0, "n: must be >= 0");
  if (n > 0) {
    CHECK_ARG(x && rows && out, "x/rows/out: must not be NULL");
    int rc = check_ptr_align(x, 16, "x");
    if (rc) return rc;
    rc = check_ptr_align(out, 16, "out");
    if (rc) return rc;
  }
  CHECK_LAUNCH(launch_gather_rows(x, Hd, rows, n, out, S(stream)), "dymoe_gather_rows");
  return ok();
}

int dymoe_combine(const float* y_perm, const int32_t* inv_row, const float* topk_w, int T, int k,
                  int Hd, int renorm, int out_dtype, void* y, dymoe_stream_t stream) {
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(k >= 1 && k <= 8, "k: must be in [1, 8]");
  CHECK_ARG(Hd > 0 && Hd % 4 == 0, "Hd: must be a positive multiple of 4");
  CHECK_ARG(out_dtype == DYMOE_OUT_F32 || out_dtype == DYMOE_OUT_BF16, "out_dtype: must be DYMOE_OUT_F32 or DYMOE_OUT_BF16");
  if (T > 0) {
    CHECK_ARG(y_perm && inv_row && topk_w && y, "y_perm/inv_row/topk_w/y: must not be NULL");
    int rc = check_ptr_align(y_perm, 16, "y_perm");
    if (rc) return rc;
  }
  CHECK_LAUNCH(launch_combine(y_perm, 1, T * k, inv_row, topk_w, T, k, Hd, renorm, out_dtype, y,
                              S(stream)),
               "dymoe_combine");
  return ok();
}

int dymoe_attention_mass(const uint16_t* q, const uint16_t* k, int H, int T, int d, float scale,
                         float* scratch, float* a_out, dymoe_stream_t stream) {
  CHECK_ARG(H >= 0 && T >= 0, "H/T: must be >= 0");
  CHECK_ARG(d == 128, "d: only head dim 128 is implemented");
  CHECK_ARG(scale > 0.f, "scale: must be > 0");
  if (H == 0 || T == 0) return ok();
  CHECK_ARG(q && k && scratch && a_out, "q/k/scratch/a_out: must not be NULL");
  int rc = check_ptr_align(q, 16, "q");
  if (rc) return rc;
  rc = check_ptr_align(k, 16, "k");
  if (rc) return rc;
  CHECK_LAUNCH(launch_attention_mass(q, k, H, T, d, scale, scratch, scratch + (size_t)H * T, a_out,
                                     S(stream)),
               "dymoe_attention_mass");
  return ok();
}

size_t dymoe_predict_ws_bytes(int T, int M, int k_route) {
  if (T < 1 || M < 1 || k_route < 1) return 0;
  const size_t TM = (size_t)T * M, TK = (size_t)T * k_route;
  return align_up(TM * 4) + align_up(TK * 4) + align_up(TK * 4) + align_up(TM * 4) + align_up((size_t)M * 4);
}

int dymoe_rmsnorm(const uint16_t* x, int T, int Hd, float eps, uint16_t* u, dymoe_stream_t stream) {
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(Hd > 0 && Hd % 8 == 0, "Hd: must be a positive multiple of 8");
  CHECK_ARG(eps >= 0.f, "eps: must be >= 0");
  if (T == 0) return ok();
  CHECK_ARG(x != nullptr, "x: must not be NULL");
  CHECK_ARG(u != nullptr, "u: must not be NULL");
  CHECK_ARG(x != u, "u: must not alias x");
  int rc = check_ptr_align(x, 16, "x");
  if (rc) return rc;
  rc = check_ptr_align(u, 16, "u");
  if (rc) return rc;
  CHECK_LAUNCH(launch_rmsnorm(x, T, Hd, eps, u, S(stream)), "dymoe_rmsnorm");
  return ok();
}

int dymoe_gate_logits(const uint16_t* h, const uint16_t* w_gate, const float* bias, int T, int Hd,
                      int M, float* logits, dymoe_stream_t stream) {
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(Hd > 0 && Hd % 8 == 0, "Hd: must be a positive multiple of 8");
  if (T == 0) return ok();
  CHECK_ARG(h != nullptr, "h: must not be NULL");
  CHECK_ARG(w_gate != nullptr, "w_gate: must not be NULL");
  CHECK_ARG(logits != nullptr, "logits: must not be NULL");
  int rc = check_ptr_align(h, 16, "h");
  if (rc) return rc;
  rc = check_ptr_align(w_gate, 16, "w_gate");
  if (rc) return rc;
  CHECK_LAUNCH(launch_gate_logits(h, w_gate, bias, T, Hd, M, logits, S(stream)), "dymoe_gate_logits");
  return ok();
}

int dymoe_predict_next(int phase, const uint16_t* h, const uint16_t* w_gate_next, int T, int Hd,
                       int M, int k_route, int t, void* ws, size_t ws_bytes, int32_t* experts,
                       float* priority, int32_t* n_out, float* logits_out, dymoe_stream_t stream) {
  CHECK_ARG(phase == DYMOE_PREFILL || phase == DYMOE_DECODE, "phase: must be DYMOE_PREFILL or DYMOE_DECODE");
  CHECK_ARG(T >= 1, "T: must be >= 1");
  CHECK_ARG(Hd > 0 && Hd % 8 == 0, "Hd: must be a positive multiple of 8");
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  CHECK_ARG(k_route >= 1 && k_route <= M && k_route <= 8, "k_route: must satisfy 1 <= k_route <= min(M, 8)");
  CHECK_ARG(t >= 1 && t <= M, "t: must satisfy 1 <= t <= M");
  CHECK_ARG(h && w_gate_next && ws && experts && priority && n_out,
            "h/w_gate_next/ws/experts/priority/n_out: must not be NULL");
  int rc = check_ptr_align(h, 16, "h");
  if (rc) return rc;
  rc = check_ptr_align(w_gate_next, 16, "w_gate_next");
  if (rc) return rc;
  if (ws_bytes < dymoe_predict_ws_bytes(T, M, k_route))
    return fail(DYMOE_ERR_WORKSPACE, "ws_bytes: %zu < dymoe_predict_ws_bytes = %zu", ws_bytes,
                dymoe_predict_ws_bytes(T, M, k_route));
  const size_t TM = (size_t)T * M, TK = (size_t)T * k_route;
  char* b = reinterpret_cast<char*>(ws);
  float* logits = logits_out ? logits_out : reinterpret_cast<float*>(b);
  int32_t* tidx = reinterpret_cast<int32_t*>(b + align_up(TM * 4));
  float* tw = reinterpret_cast<float*>(b + align_up(TM * 4) + align_up(TK * 4));
  float* probs = reinterpret_cast<float*>(b + align_up(TM * 4) + 2 * align_up(TK * 4));
  float* value = reinterpret_cast<float*>(b + 2 * align_up(TM * 4) + 2 * align_up(TK * 4));
  CHECK_LAUNCH(launch_predict_next(phase, h, w_gate_next, T, Hd, M, k_route, t, logits, tidx, tw,
                                   probs, value, experts, priority, n_out, S(stream)),
               "dymoe_predict_next");
  return ok();
}

int dymoe_renorm_weights(const int32_t* topk_idx, const float* topk_w, const uint8_t* bits, int T,
                         int k, int M, int renorm, float* w_out, dymoe_stream_t stream) {
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(k >= 1 && k <= 8, "k: must be in [1, 8]");
  CHECK_ARG(M >= 1 && M <= DYMOE_MAX_EXPERTS, "M: must be in [1, %d]", DYMOE_MAX_EXPERTS);
  if (T > 0) CHECK_ARG(topk_idx && topk_w && bits && w_out, "topk_idx/topk_w/bits/w_out: must not be NULL");
  CHECK_LAUNCH(launch_renorm_weights(topk_idx, topk_w, bits, T, k, renorm, w_out, S(stream)),
               "dymoe_renorm_weights");
  return ok();
}

// Prefill: experts with at most this many rows run on the decode GEMV kernels (0 = never).
// DYMOE_PREFILL_SMALL_ROWS overrides (measurement knob).
static int prefill_small_rows() {
  static const int v = getenv("DYMOE_PREFILL_SMALL_ROWS") ? atoi(getenv("DYMOE_PREFILL_SMALL_ROWS"))
                                                          : kPrefillSmallRows;
  return v;
}

// Splits the active list (list order kept) into experts with > small rows and those with
// 1..small rows.  One warp, 32 entries per ballot round.
__global__ void k_split_active(const int32_t* __restrict__ off, const int32_t* __restrict__ list,
                               int small, int32_t* __restrict__ large_list,
                               int32_t* __restrict__ small_list) {
  const int lane = threadIdx.x & 31;
  const int n = list[0];
  int nl = 0, ns = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const int e = i < n ? list[1 + i] : 0;
    const int rows = i < n ? off[e + 1] - off[e] : 0;
    const bool is_l = rows > small, is_s = rows > 0 && rows <= small;
    const unsigned bl = __ballot_sync(0xffffffffu, is_l), bs = __ballot_sync(0xffffffffu, is_s);
    const unsigned below = (1u << lane) - 1;
    if (is_l) large_list[1 + nl + __popc(bl & below)] = e;
    if (is_s) small_list[1 + ns + __popc(bs & below)] = e;
    nl += __popc(bl);
    ns += __popc(bs);
  }
  if (lane == 0) {
    large_list[0] = nl;
    small_list[0] = ns;
  }
}

static int run_ffn(const dymoe_layer* L, int mode, const uint16_t* x, int T, const uint8_t* bits,
                   const int32_t* expert_off, const int32_t* perm_token, const int32_t* active_list,
                   uint16_t* h, float* y_perm, float* y_part, int part_rows, int* parts_out,
                   uint32_t* status, cudaStream_t s, void* const* ev = nullptr) {
  // On return *parts_out = number of K-slice partials written to y_part ([parts][part_rows][Hd]),
  // or 0 if the result was written to y_perm directly.
  FfnArgs a{};
  a.experts = L->dev;
  a.M = L->M;
  a.k = L->k;
  a.Hd = L->Hd;
  a.F = L->F;
  a.x = x;
  a.T = T;
  a.bits = bits;
  a.expert_off = expert_off;
  a.perm_token = perm_token;
  a.active_list = active_list;
  a.h = h;
  a.y_perm = y_perm;
  a.y_part = y_part;
  a.part_rows = part_rows;
  a.status = status;
  // decode kernels write K-slice partials of W2; the prefill grouped GEMM writes y_perm directly
  *parts_out = mode == DYMOE_DECODE ? decode_w2_slices(L->F) : 0;
  if (T == 0) return DYMOE_OK;
  cudaError_t e;
  const int small = prefill_small_rows();
  if (mode == DYMOE_PREFILL && small > 0 && decode_w2_slices(L->F) == 1) {
    // Prefill with small experts split off (active_list has room for 3 lists of M + 1): experts
    // with <= `small` rows would fill a 256-token pair tile mostly with padding, so the GEMV
    // kernels stream their weights once per 8 tokens instead; the W2 GEMV (one K slice) writes
    // its rows of y_perm directly, after the grouped GEMM zeroed y_perm and added its own rows.
    int32_t* large_list = const_cast<int32_t*>(active_list) + (L->M + 1);
    int32_t* small_list = large_list + (L->M + 1);
    k_split_active<<<1, 32, 0, s>>>(expert_off, active_list, small, large_list, small_list);
    FfnArgs al = a;
    al.active_list = large_list;
    void* ev2[3] = {ev ? ev[0] : nullptr, ev ? ev[1] : nullptr, nullptr};
    e = launch_ffn_prefill(al, s, ev ? ev2 : nullptr);
    if (e == cudaSuccess) {
      FfnArgs as = a;
      as.active_list = small_list;
      as.y_part = y_perm;
      e = launch_ffn_decode(as, s, nullptr);
    }
    if (e == cudaSuccess && ev) record_ev(ev, 2, s);
  } else {
    e = mode == DYMOE_DECODE ? launch_ffn_decode(a, s, ev) : launch_ffn_prefill(a, s, ev);
  }
  if (e != cudaSuccess) return cuda_fail(e, "expert ffn");
  return DYMOE_OK;
}

// Builds the active list (experts with rows) from expert_off on device.
// One warp, 32 experts per ballot round, list order = expert order.
__global__ void k_active_from_off(const int32_t* __restrict__ off, int M, int32_t* list) {
  const int lane = threadIdx.x & 31;
  int n = 0;
  for (int e0 = 0; e0 < M; e0 += 32) {
    const int e = e0 + lane;
    const bool act = e < M && off[e + 1] > off[e];
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (act) list[1 + n + __popc(bal & ((1u << lane) - 1))] = e;
    n += __popc(bal);
  }
  if (lane == 0) list[0] = n;
}

}  // extern "C"

// dymoe_expert_ffn scratch: active lists (3 x (M + 1)), then the W2 K-slice partials (decode) or
// the expert-ordered token rows (prefill) -- the larger of the two.
size_t dymoe::ffn_ws_parts_bytes(const dymoe_layer* L, int rows) {
  const size_t dec = (size_t)decode_w2_slices(L->F) * rows * L->Hd * sizeof(float);
  const size_t pre = (size_t)rows * L->Hd * 2;
  return dec > pre ? dec : pre;
}

extern "C" size_t dymoe_expert_ffn_ws_bytes(const dymoe_layer* L, int T) {
  if (!L || T < 0) return 0;
  return align_up((size_t)3 * (L->M + 1) * sizeof(int32_t)) +
         align_up(ffn_ws_parts_bytes(L, (T > 0 ? T : 1) * L->k));
}

// The expert FFN on expert-ordered rows whose count lives on the device (expert_off[M]):
// `cap_rows` bounds it (workspace, descriptors); the kernels read the real count.  Shared by
// dymoe_expert_ffn and the expert-parallel layer (rows received from peers).
int dymoe::expert_ffn_rows(const dymoe_layer* L, int mode, const uint16_t* x, int cap_rows,
                    const uint8_t* bits, const int32_t* expert_off, const int32_t* perm_token,
                    uint16_t* h_ws, float* y_perm, uint32_t* status, void* ws, cudaStream_t s,
                    void* const* ev) {
  int32_t* active = reinterpret_cast<int32_t*>(ws);
  float* parts = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) +
                                          align_up((size_t)3 * (L->M + 1) * sizeof(int32_t)));
  k_active_from_off<<<1, 32, 0, s>>>(expert_off, L->M, active);
  int n_parts = 0;
  // run_ffn's rows = T * k: pass the capacity as T with the layer's k folded in
  int rc = run_ffn(L, mode, x, cap_rows / L->k, bits, expert_off, perm_token, active, h_ws,
                   y_perm, parts, cap_rows, &n_parts, status, s, ev);
  if (rc == DYMOE_OK && n_parts > 0) {
    cudaError_t e = launch_reduce_parts(parts, n_parts, cap_rows, cap_rows, L->Hd, y_perm, s,
                                        expert_off + L->M);
    if (e != cudaSuccess) rc = cuda_fail(e, "expert ffn");
  }
  return rc;
}

extern "C" {

int dymoe_expert_ffn(const dymoe_layer* L, int mode, const uint16_t* x, int T,
                     const uint8_t* bits, const int32_t* expert_off, const int32_t* perm_token,
                     uint16_t* h_ws, float* y_perm, uint32_t* status, void* ws, size_t ws_bytes,
                     dymoe_stream_t stream) {
  CHECK_ARG(L != nullptr, "layer: must not be NULL");
  CHECK_ARG(mode == DYMOE_PREFILL || mode == DYMOE_DECODE,
            "mode: must be DYMOE_PREFILL or DYMOE_DECODE");
  CHECK_ARG(T >= 0, "T: must be >= 0");
  if (T == 0) return ok();
  CHECK_ARG(x && bits && expert_off && perm_token && h_ws && y_perm,
            "x/bits/expert_off/perm_token/h_ws/y_perm: must not be NULL");
  CHECK_ARG(ws != nullptr, "ws: must not be NULL");
  int rc = check_ptr_align(x, 16, "x");
  if (rc) return rc;
  rc = check_ptr_align(ws, 256, "ws");
  if (rc) return rc;
  const size_t need = dymoe_expert_ffn_ws_bytes(L, T);
  if (ws_bytes < need)
    return fail(DYMOE_ERR_WORKSPACE, "ws_bytes: %zu < dymoe_expert_ffn_ws_bytes = %zu", ws_bytes, need);
  rc = expert_ffn_rows(L, mode, x, T * L->k, bits, expert_off, perm_token, h_ws, y_perm, status,
                       ws, S(stream), nullptr);
  if (rc) return rc;
  return ok();
}

// ------------------------------------------------------------------------------------------
size_t dymoe_workspace_size(const dymoe_layer* L, int T) {
  if (!L || T < 0) return 0;
  return ws_layout(L->M, L->k, L->Hd, L->F, T).total;
}

int dymoe_workspace_views(const dymoe_layer* L, int T, void* ws, dymoe_ws_views* v) {
  CHECK_ARG(L != nullptr, "layer: must not be NULL");
  CHECK_ARG(v != nullptr, "views: must not be NULL");
  CHECK_ARG(ws != nullptr, "workspace: must not be NULL");
  CHECK_ARG(T >= 0, "T: must be >= 0");
  const WsLayout W = ws_layout(L->M, L->k, L->Hd, L->F, T);
  char* b = reinterpret_cast<char*>(ws);
  v->topk_idx = reinterpret_cast<int32_t*>(b + W.topk_idx);
  v->topk_w = reinterpret_cast<float*>(b + W.topk_w);
  v->probs = reinterpret_cast<float*>(b + W.probs);
  v->importance = reinterpret_cast<float*>(b + W.importance);
  v->heavy = reinterpret_cast<int32_t*>(b + W.heavy);
  v->bits = reinterpret_cast<uint8_t*>(b + W.bits);
  v->active = reinterpret_cast<uint8_t*>(b + W.active);
  v->expert_off = reinterpret_cast<int32_t*>(b + W.expert_off);
  v->perm_token = reinterpret_cast<int32_t*>(b + W.perm_token);
  v->perm_slot = reinterpret_cast<int32_t*>(b + W.perm_slot);
  v->inv_row = reinterpret_cast<int32_t*>(b + W.inv_row);
  v->h = reinterpret_cast<uint16_t*>(b + W.h);
  v->y_perm = reinterpret_cast<float*>(b + W.y_perm);
  v->status = reinterpret_cast<uint32_t*>(b + W.status);
  v->score_scratch = b + W.score_scratch;
  return ok();
}

int dymoe_moe_forward(const dymoe_layer* L, const uint16_t* x, const float* logits, int T,
                      const dymoe_fwd_opts* o, void* y, void* ws, size_t ws_bytes,
                      dymoe_stream_t stream) {
  CHECK_ARG(L != nullptr, "layer: must not be NULL");
  CHECK_ARG(o != nullptr, "opts: must not be NULL");
  CHECK_ARG(T >= 0, "T: must be >= 0");
  CHECK_ARG(o->phase == DYMOE_PREFILL || o->phase == DYMOE_DECODE, "opts.phase: must be DYMOE_PREFILL or DYMOE_DECODE");
  CHECK_ARG(o->out_dtype == DYMOE_OUT_F32 || o->out_dtype == DYMOE_OUT_BF16, "opts.out_dtype: must be DYMOE_OUT_F32 or DYMOE_OUT_BF16");
  CHECK_ARG(o->ffn_mode == -1 || o->ffn_mode == DYMOE_PREFILL || o->ffn_mode == DYMOE_DECODE,
            "opts.ffn_mode: must be -1, DYMOE_PREFILL or DYMOE_DECODE");
  AssignParams ap{};
  int rc = assign_params(&o->ladder, L->M, L->k, o->layer, o->num_layers, ap);
  if (rc) {
    g_err = "opts." + g_err;
    return rc;
  }
  if (T == 0) return ok();
  CHECK_ARG(x != nullptr, "x: must not be NULL");
  CHECK_ARG(logits != nullptr, "logits: must not be NULL");
  CHECK_ARG(y != nullptr, "y: must not be NULL");
  CHECK_ARG(ws != nullptr, "workspace: must not be NULL");
  rc = check_ptr_align(x, 16, "x");
  if (rc) return rc;
  rc = check_ptr_align(ws, 256, "workspace");
  if (rc) return rc;
  if (o->residual != nullptr) {
    rc = check_ptr_align(o->residual, 16, "opts.residual");
    if (rc) return rc;
  }
  const WsLayout W = ws_layout(L->M, L->k, L->Hd, L->F, T);
  if (ws_bytes < W.total)
    return fail(DYMOE_ERR_WORKSPACE, "ws_bytes: %zu < dymoe_workspace_size() = %zu", ws_bytes, W.total);
  int k_tokens = o->k_tokens;
  if (o->phase == DYMOE_PREFILL) {
    CHECK_ARG(o->attn_mass != nullptr, "opts.attn_mass: must not be NULL in PREFILL");
    CHECK_ARG(o->heads >= 1, "opts.heads: must be >= 1");
    if (k_tokens == 0) k_tokens = (T + 4) / 5;
    CHECK_ARG(k_tokens >= 0 && k_tokens <= T, "opts.k_tokens: must satisfy 0 <= k_tokens <= T");
  }
  dymoe_ws_views v{};
  dymoe_workspace_views(L, T, ws, &v);
  int32_t* active_list = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + W.active_list);
  cudaStream_t s = S(stream);

  const uint8_t* bits = o->forced_bits;
  if (o->phase == DYMOE_DECODE && T <= kFrontDecodeMaxT) {
    // decode batch: route, score, assign and permute in one launch
    CHECK_LAUNCH(launch_front_decode(logits, T, L->M, L->k, ap, bits, v.topk_idx, v.topk_w, v.probs,
                                     v.importance, v.bits, v.active, v.expert_off, v.perm_token,
                                     v.perm_slot, v.inv_row, active_list, s),
                 "front");
    if (bits == nullptr) bits = v.bits;
  } else {
    CHECK_LAUNCH(launch_route(logits, T, L->M, L->k, v.topk_idx, v.topk_w, v.probs, s), "route");
    if (bits == nullptr) {
      if (o->phase == DYMOE_PREFILL) {
        CHECK_LAUNCH(launch_score_prefill(o->attn_mass, o->heads, v.topk_idx, T, L->M, L->k,
                                          k_tokens, v.importance, v.heavy,
                                          reinterpret_cast<float*>(v.score_scratch), s),
                     "score");
      } else {
        CHECK_LAUNCH(launch_score_decode(logits, T, L->M, v.importance, s), "score");
      }
      CHECK_LAUNCH(launch_assign(v.importance, nullptr, v.topk_idx, T, ap, v.bits, v.active, s),
                   "assign");
      bits = v.bits;
    }
    CHECK_LAUNCH(launch_permute(v.topk_idx, T, L->k, L->M, bits, v.expert_off, v.perm_token,
                                v.perm_slot, v.inv_row, active_list, s,
                                reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + W.perm_scratch)),
                 "permute");
  }
  const int mode = o->ffn_mode == -1 ? o->phase : o->ffn_mode;
  float* y_part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + W.y_part);
  int n_parts = 0;
  rc = run_ffn(L, mode, x, T, bits, v.expert_off, v.perm_token, active_list, v.h, v.y_perm,
               y_part, T * L->k, &n_parts, v.status, s, o->prof_events);
  if (rc) return rc;
  CHECK_LAUNCH(launch_combine(n_parts > 0 ? y_part : v.y_perm, n_parts > 0 ? n_parts : 1, T * L->k,
                              v.inv_row, v.topk_w, T, L->k, L->Hd, o->ladder.renorm_on_skip,
                              o->out_dtype, y, s, o->residual),
               "combine");
  return ok();
}

int dymoe_check_status(const dymoe_layer* L, int T, void* ws, uint32_t* bits_out,
                       dymoe_stream_t stream) {
  CHECK_ARG(L != nullptr, "layer: must not be NULL");
  CHECK_ARG(ws != nullptr, "workspace: must not be NULL");
  const WsLayout W = ws_layout(L->M, L->k, L->Hd, L->F, T);
  uint32_t word = 0;
  uint32_t* dptr = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ws) + W.status);
  cudaError_t e = cudaMemcpyAsync(&word, dptr, 4, cudaMemcpyDeviceToHost, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  if (e == cudaSuccess) e = cudaMemsetAsync(dptr, 0, 4, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "dymoe_check_status");
  if (bits_out) *bits_out = word;
  if (word) return fail(DYMOE_ERR_DEVICE, "device status word 0x%x (bit 1: an assigned width is not resident)", word);
  return ok();
}

}  // extern "C"

// TMA descriptor helper for the kernels' launchers (C++ linkage, outside the C ABI)
bool dymoe::encode_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t d0,
                           uint64_t d1, uint64_t stride1, uint32_t b0, uint32_t b1,
                           CUtensorMapSwizzle swz) {
  const uint64_t dims[2] = {d0, d1}, str[1] = {stride1};
  const uint32_t box[2] = {b0, b1};
  return encode(m, dt, base, 2, dims, str, box, swz);
}

int dymoe::set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
void dymoe::clear_error() { g_err.clear(); }

cudaError_t dymoe::preload_api() { return preload_kernels(k_split_active, k_active_from_off); }
