// ko_api.cpp — the C ABI of libko.so (include/ko.h): host validation, workspace layout, and the
// orchestration of the sm_100a kernels in ko_kernels.cu.  No allocation happens in a call; every
// launch goes on the caller's stream.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "ko.h"
#include "ko_internal.h"

namespace {
// NVTX range around every compute entry point (and each routed plan position), so an nsys /
// ncu --nvtx timeline shows the library's calls; header-only NVTX3: a no-op without a tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

namespace {

thread_local std::string g_err;
thread_local cudaEvent_t g_trace_begin = nullptr, g_trace_end = nullptr;
thread_local int32_t g_launches = 0;  // kernels launched by the last compute call (ko_last_launch_count)

ko_status fail(ko_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
ko_status fail(ko_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

// a kernel launch of this library: counted for ko_last_launch_count, then checked
#define KO_LAUNCH(expr)                                                                \
  do {                                                                                 \
    ++g_launches;                                                                      \
    KO_CUDA(expr);                                                                     \
  } while (0)

#define KO_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e__ = (expr);                                                          \
    if (e__ != cudaSuccess) return fail(KO_ECUDA, "%s: %s", #expr, cudaGetErrorString(e__)); \
  } while (0)

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// external variant: margins supplied by the caller (keep‰ = 0, layer_cut = 0), e.g. an
// embedding-similarity stage from ko_embed_scores
inline bool is_external(const ko_variant& v) { return v.keep_permille == 0 && v.layer_cut == 0; }

int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

ko_status validate_kv(const ko_kv_cache* kv) {
  if (!kv) return fail(KO_EINVAL, "kv is NULL");
  if (!kv->kv_pool || !kv->page_indptr || !kv->page_ids || !kv->seq_len)
    return fail(KO_EINVAL, "kv: NULL pool/page_indptr/page_ids/seq_len");
  if (kv->head_dim != 64 && kv->head_dim != 128)
    return fail(KO_EINVAL, "head_dim %d not in {64,128}", kv->head_dim);
  if (kv->n_layers < 1 || kv->n_kv_heads < 1 || kv->gqa_group < 1 || kv->n_q < 1)
    return fail(KO_EINVAL, "kv: n_layers/n_kv_heads/gqa_group/n_q must be >= 1");
  if (kv->n_tuples < 0 || kv->n_pages < 0) return fail(KO_EINVAL, "kv: negative sizes");
  if (kv->n_tuples > 0x7fffffffll) return fail(KO_EUNSUPPORTED, "n_tuples > 2^31-1");
  if (((uintptr_t)kv->kv_pool & 15) != 0) return fail(KO_EINVAL, "kv_pool not 16-byte aligned");
  return KO_OK;
}

ko_status validate_ops(const ko_kv_cache* kv, const ko_operator* ops, int32_t n_ops) {
  if (!ops || n_ops < 1 || n_ops > KO_MAX_OPS)
    return fail(KO_EINVAL, "n_ops %d outside [1,%d]", n_ops, KO_MAX_OPS);
  for (int o = 0; o < n_ops; ++o) {
    if (!ops[o].q || !ops[o].w || !ops[o].b) return fail(KO_EINVAL, "op %d: NULL q/w/b", o);
    if (ops[o].n_classes < 1) return fail(KO_EINVAL, "op %d: n_classes < 1", o);
    if (ops[o].n_classes > KO_MAX_CLASSES)
      return fail(KO_EUNSUPPORTED, "op %d: n_classes %d > %d", o, ops[o].n_classes, KO_MAX_CLASSES);
  }
  if ((int64_t)kv->gqa_group * kv->n_q > KO_MAX_ROWS)
    return fail(KO_EUNSUPPORTED, "gqa_group*n_q = %d > %d", kv->gqa_group * kv->n_q, KO_MAX_ROWS);
  return KO_OK;
}

ko_status validate_variants(const ko_kv_cache* kv, const ko_variant* v, int32_t n) {
  if (!v || n < 1 || n > KO_MAX_VARIANTS)
    return fail(KO_EINVAL, "n_variants %d outside [1,%d]", n, KO_MAX_VARIANTS);
  for (int i = 0; i < n; ++i) {
    if (v[i].keep_permille == 0 && v[i].layer_cut == 0) continue;  // external (caller's margins)
    if (v[i].keep_permille < 1 || v[i].keep_permille > 1000)
      return fail(KO_EINVAL, "variant %d: keep_permille %d outside [1,1000]", i, v[i].keep_permille);
    if (v[i].layer_cut < 1 || v[i].layer_cut > kv->n_layers)
      return fail(KO_EINVAL, "variant %d: layer_cut %d outside [1,%d]", i, v[i].layer_cut,
                  kv->n_layers);
  }
  return KO_OK;
}

ko_status validate_plan(const ko_plan* P, int g, const int32_t* n_classes, int32_t n_ops,
                        int32_t n_variants) {
  if (P->n_stages < 1 || P->n_stages > KO_MAX_STAGES)
    return fail(KO_EINVAL, "plan %d: n_stages %d outside [1,%d]", g, P->n_stages, KO_MAX_STAGES);
  int final_at[KO_MAX_OPS];
  for (int o = 0; o < KO_MAX_OPS; ++o) final_at[o] = -2;  // -2: unreferenced, -1: no final yet
  for (int s = 0; s < P->n_stages; ++s) {
    const ko_stage& st = P->stage[s];
    if (st.op < 0 || st.op >= n_ops) return fail(KO_EINVAL, "plan %d stage %d: op %d", g, s, st.op);
    if (st.variant < 0 || st.variant >= n_variants)
      return fail(KO_EINVAL, "plan %d stage %d: variant %d", g, s, st.variant);
    if (!(st.theta_lo <= st.theta_hi))
      return fail(KO_EINVAL, "plan %d stage %d: theta_lo > theta_hi (or NaN)", g, s);
    if (final_at[st.op] >= 0)
      return fail(KO_EINVAL, "plan %d stage %d: op %d has a stage after its final stage", g, s,
                  st.op);
    if (final_at[st.op] == -2) final_at[st.op] = -1;
    if (st.is_final) {
      if (n_classes[st.op] <= 1 && st.theta_lo != st.theta_hi)
        return fail(KO_EINVAL, "plan %d stage %d: final filter stage needs theta_lo == theta_hi",
                    g, s);
      final_at[st.op] = s;
    }
  }
  for (int o = 0; o < n_ops; ++o)
    if (final_at[o] == -1) return fail(KO_EINVAL, "plan %d: op %d has no final stage", g, o);
  return KO_OK;
}

struct Workspace {
  unsigned long long* unit_counter;
  unsigned long long* worklist_len;
  unsigned long long* round_len;  // [KO_MAX_VARIANTS] worklist lengths of the routed rounds
  int32_t* done;
  float* part;
  uint4* qfrag;
  uint4* wfrag;
  uint32_t* tuple_state;
  int32_t* worklist;
  int32_t* round_wl;              // [KO_MAX_STAGES][n_tuples] per-position worklists
  ko_plan* gplans;                // [KO_MAX_PLANS] device copy of the plans
  uint32_t* tuple_done;           // [n_tuples]
  int* lpt_hist;                  // [4097] longest-first counting sort (grid mode)
  int32_t* lpt_perm;              // [n_work] the work list in longest-first order
  float* rstate;                  // [n_ops groups][n_tuples][n_layers][Hkv][8][rstate_w]
  int rstate_w;
  size_t rstate_group;            // floats per group slice
  size_t total;
};

// Saved softmax state of one lane group for a table of NT W·V tiles: M[2], den[2], acc[2·NT],
// padded to whole 32-byte sectors (the kernel writes every record as whole sectors: partially
// written sectors cost the routed C4 round 0 ≈ 1 % — profiles/r02_ab/rstate).
constexpr int rstate_record_floats(int nt) { return (4 + 2 * nt + 7) / 8 * 8; }

// Layout: [counters 256 B][done][part][qfrag][wfrag][tuple_state][worklist][position
// worklists][tuple_done][rstate]
Workspace layout(const ko_kv_cache* kv, int max_cls, int max_ent, int32_t n_ops, int32_t n_variants,
                 int64_t n_work, uint8_t* base) {
  Workspace w{};
  const int CPR = pow2_at_least(max_cls);
  const int KS = kv->head_dim / 16;
  const int NT = 2 * CPR;
  const size_t nt = (size_t)std::max<int64_t>(kv->n_tuples, 1);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return base ? base + o : nullptr;
  };
  uint8_t* ctr = take(256);
  w.unit_counter = (unsigned long long*)ctr;
  w.worklist_len = ctr ? (unsigned long long*)(ctr + 8) : nullptr;
  w.round_len = ctr ? (unsigned long long*)(ctr + 64) : nullptr;
  w.done = (int32_t*)take(sizeof(int32_t) * (size_t)std::max<int64_t>(n_work, 1));
  // partials: per work slot (grid) or per tuple (walk: they persist across the rounds of a call)
  // (walk mode: per tuple and layer·kv-head, n_variants whole-sector blocks of n_ops·CPR floats)
  w.part = (float*)take(sizeof(float) * (size_t)std::max<int64_t>(std::max<int64_t>(n_work, kv->n_tuples), 1) *
                        kv->n_layers * kv->n_kv_heads * n_variants * ko::walk_part_blk(n_ops, CPR));
  w.qfrag = (uint4*)take(sizeof(uint4) * (size_t)kv->n_layers * kv->n_kv_heads * KS * 32);
  w.wfrag = (uint4*)take(sizeof(uint4) * (size_t)kv->n_layers * kv->n_kv_heads * NT * KS * 32);
  w.tuple_state = (uint32_t*)take(sizeof(uint32_t) * nt);
  w.worklist = (int32_t*)take(sizeof(int32_t) * nt);
  w.round_wl = (int32_t*)take(sizeof(int32_t) * nt * KO_MAX_STAGES);
  w.gplans = (ko_plan*)take(sizeof(ko_plan) * KO_MAX_PLANS);
  w.tuple_done = (uint32_t*)take(sizeof(uint32_t) * nt);
  w.lpt_hist = (int*)take(sizeof(int) * 4097);
  w.lpt_perm = (int32_t*)take(sizeof(int32_t) * (size_t)std::max<int64_t>(n_work, 1));
  // saved softmax states of the routed rounds: a group's table needs ≤ pow2(max entries per row)
  // tiles, so rstate_record_floats(that) floats per lane group bound every group's record
  w.rstate_w = rstate_record_floats(std::min(ko::kMaxTNT, pow2_at_least(std::max(max_ent, 1))));
  w.rstate_group = nt * kv->n_layers * kv->n_kv_heads * 8 * (size_t)w.rstate_w;
  w.rstate = (float*)take(sizeof(float) * w.rstate_group * n_ops);
  w.total = off;
  return w;
}

int max_classes(const ko_operator* ops, int n_ops) {
  int m = 1;
  for (int o = 0; o < n_ops; ++o) m = std::max(m, (int)ops[o].n_classes);
  return m;
}
// W·V entries of one row of the table packing: classes, ×2 for fp32 readouts (hi + lo)
int max_entries(const ko_operator* ops, int n_ops) {
  int m = 1;
  for (int o = 0; o < n_ops; ++o) m = std::max(m, (int)ops[o].n_classes * (ops[o].w_is_bf16 ? 1 : 2));
  return m;
}

// TMA descriptor of the pool: 5-D bf16 view, innermost first: (head_dim, 16 tokens, kv-head,
// 2·layer + {K,V}, page); box (64, 16, 1, 2, 1) = the K and V rows of one kv-head of one layer of
// one page for 64 head dims; SWIZZLE_128B (conflict-free fragment reads, see ko_kernels.cu).
// cuTensorMapEncodeTiled through the runtime's driver entry point (libko.so does not link libcuda,
// so the host-only parts of the ABI load on machines without a driver); bf16, 128B swizzle
ko_status encode_tmap(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims,
                      const cuuint64_t* strides, const cuuint32_t* box, bool swizzle = true) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
      return fail(KO_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
    encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KO_ECUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return KO_OK;
}

ko_status make_tmap(CUtensorMap* map, const ko_kv_cache* kv) {
  const cuuint64_t D = (cuuint64_t)kv->head_dim;
  cuuint64_t dims[5] = {D, 16, (cuuint64_t)kv->n_kv_heads, (cuuint64_t)(2 * kv->n_layers),
                        (cuuint64_t)std::max<int64_t>(kv->n_pages, 1)};
  cuuint64_t strides[4] = {D * 2, 16 * D * 2, (cuuint64_t)kv->n_kv_heads * 16 * D * 2,
                           (cuuint64_t)(2 * kv->n_layers) * kv->n_kv_heads * 16 * D * 2};
  cuuint32_t box[5] = {64, 16, 1, 2, 1};
  return encode_tmap(map, kv->kv_pool, 5, dims, strides, box);
}

// Table packing (every scoring launch).  Lane group g owns S rows g (half 0) and g + 8 (half 1); W·V tile tt
// gives it slot (tt, hr) = A row g + 8·hr, which always accumulates with S-row half hr.  So each
// half of a lane group offers NT slots.  An S row (op, gqa member, query row) of a C-class op needs
// C entries (2C for fp32 W: bf16 hi and lo).  A row with ≤ NT entries takes one half; a row with
// NT < e ≤ 2·NT entries is duplicated into both halves of a lane group (the same query in S rows g
// and g + 8) and its entries are split between them.  Smallest NT ∈ {1, 2, 4, 8} that fits, big
// rows first; returns 0 if none fits.
int pack_table(const ko_operator* ops, const int* order, int n_sel, int rows_per_op,
               ko::ScoreParams& sp, ko::PrepParams& pp) {
  struct Row { int i, rem, e; };
  Row rows[16];
  int nr = 0;
  for (int i = 0; i < n_sel; ++i)
    for (int r = 0; r < rows_per_op; ++r) {
      if (nr == 16) return 0;
      rows[nr++] = {i, r, (int)ops[order[i]].n_classes * (ops[order[i]].w_is_bf16 ? 1 : 2)};
    }
  std::stable_sort(rows, rows + nr, [](const Row& a, const Row& b) { return a.e > b.e; });
  for (int NT : {1, 2, 4, 8}) {
    int at[8][2];  // row index (into rows[]) at (lane group, half), −1 free
    for (int b = 0; b < 8; ++b) at[b][0] = at[b][1] = -1;
    bool ok = true;
    for (int k = 0; k < nr && ok; ++k) {
      const int e = rows[k].e;
      if (e > 2 * NT) { ok = false; break; }
      bool placed = false;
      if (e > NT) {  // both halves of a free lane group
        for (int b = 0; b < 8 && !placed; ++b)
          if (at[b][0] < 0 && at[b][1] < 0) { at[b][0] = at[b][1] = k; placed = true; }
      } else {
        for (int b = 0; b < 8 && !placed; ++b)
          for (int hs = 0; hs < 2 && !placed; ++hs)
            if (at[b][hs] < 0) { at[b][hs] = k; placed = true; }
      }
      ok = placed;
    }
    if (!ok) continue;
    for (int r = 0; r < 16; ++r) { sp.slot_op[r] = -1; pp.slot_op[r] = -1; pp.slot_rem[r] = 0; }
    for (int b = 0; b < 8; ++b) {
      for (int k = 0; k < 16; ++k) { sp.tbl_tgt[b][k] = -1; pp.tbl_w[b][k] = -1; }
      for (int hs = 0; hs < 2; ++hs) {
        if (at[b][hs] < 0) continue;
        const Row& R = rows[at[b][hs]];
        sp.slot_op[hs * 8 + b] = R.i;
        pp.slot_op[hs * 8 + b] = R.i;
        pp.slot_rem[hs * 8 + b] = R.rem;
        const ko_operator& op = ops[order[R.i]];
        const int nlo = op.w_is_bf16 ? 1 : 2;
        const bool dup = at[b][0] == at[b][1];
        const int e0 = dup ? (R.e + 1) / 2 : R.e;  // entries on half 0 (all of them if not split)
        const int lo_e = dup && hs == 1 ? e0 : 0, hi_e = dup && hs == 0 ? e0 : R.e;
        for (int ent = lo_e, tt = 0; ent < hi_e; ++ent, ++tt) {
          const int c = ent / nlo, lo = ent % nlo;
          pp.tbl_w[b][2 * tt + hs] = R.i | (R.rem << 3) | (c << 8) | (lo << 12);
          sp.tbl_tgt[b][2 * tt + hs] = (int8_t)(R.i * 8 + c);
        }
      }
    }
    return NT;
  }
  return 0;
}

// Fill the kv/op/variant part of ScoreParams and the matching PrepParams for the selected ops
// (caller indices op_sel[0..n_sel)) and variants: local ops in descending class count, the table
// packing of their rows (NT, returned; 0 = does not fit) and the partial class stride CPR
// (pow2 ≥ the largest class count, returned).
void fill_common(ko::ScoreParams& sp, ko::PrepParams& pp, const ko_kv_cache* kv,
                 const ko_operator* ops, const int* op_sel, int n_sel, const ko_variant* variants,
                 const int* var_sel, int n_vsel, int32_t n_ops_total, int32_t n_var_total,
                 const Workspace& ws, int* CPR, int* NT) {
  std::memset(&sp, 0, sizeof(sp));
  std::memset(&pp, 0, sizeof(pp));
  sp.pool = (const uint16_t*)kv->kv_pool;
  sp.page_elems = (int64_t)kv->n_layers * 2 * kv->n_kv_heads * KO_PAGE_TOKENS * kv->head_dim;
  sp.page_indptr = kv->page_indptr;
  sp.page_ids = kv->page_ids;
  sp.seq_len = kv->seq_len;
  sp.n_tuples = kv->n_tuples;
  sp.n_pages = kv->n_pages;
  sp.n_layers = kv->n_layers;
  sp.n_kv_heads = kv->n_kv_heads;
  sp.gqa = kv->gqa_group;
  sp.n_q = kv->n_q;
  sp.n_ops = n_sel;
  sp.rows_per_op = kv->gqa_group * kv->n_q;
  sp.n_ops_total = n_ops_total;
  sp.n_var_total = n_var_total;
  for (int o = 0; o < n_ops_total; ++o) {
    sp.op_classes_g[o] = ops[o].n_classes;
    sp.bias_g[o] = ops[o].b;
  }
  int n_l = 1;
  sp.n_var = n_vsel;
  for (int i = 0; i < KO_MAX_VARIANTS; ++i) sp.var_local[i] = -1;
  for (int i = 0; i < n_vsel; ++i) {
    const ko_variant& v = variants[var_sel[i]];
    sp.keep[i] = v.keep_permille;
    sp.cut[i] = v.layer_cut;
    sp.var_ids[i] = var_sel[i];
    sp.var_local[var_sel[i]] = i;
    n_l = std::max(n_l, (int)v.layer_cut);
  }
  sp.n_l = n_l;
  // local op order: descending class count (stable)
  int order[KO_MAX_OPS];
  for (int i = 0; i < n_sel; ++i) order[i] = op_sel[i];
  std::stable_sort(order, order + n_sel,
                   [&](int a, int b) { return ops[a].n_classes > ops[b].n_classes; });
  int max_cls = 1;
  for (int i = 0; i < n_sel; ++i) {
    const ko_operator& op = ops[order[i]];
    sp.op_ids[i] = order[i];
    sp.op_classes[i] = op.n_classes;
    sp.bias[i] = op.b;
    pp.q[i] = (const uint16_t*)op.q;
    pp.w[i] = op.w_is_bf16 ? nullptr : (const float*)op.w;
    pp.w_bf16[i] = op.w_is_bf16 ? (const uint16_t*)op.w : nullptr;
    pp.op_classes[i] = op.n_classes;
    max_cls = std::max(max_cls, (int)op.n_classes);
  }
  // table packing: S rows → lane groups, (row, class[, hi/lo]) entries → W·V tile slots
  *NT = pack_table(ops, order, n_sel, sp.rows_per_op, sp, pp);
  *CPR = pow2_at_least(max_cls);
  pp.tbl_nt = *NT;
  sp.qfrag = ws.qfrag;
  sp.wfrag = ws.wfrag;
  sp.part = ws.part;
  sp.done = ws.done;
  sp.unit_counter = ws.unit_counter;
  sp.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)kv->head_dim));
  // Work-unit size: a unit streams HG kv-heads of one (tuple, layer) back-to-back, HG chosen so
  // a unit is ~64 pages (estimated from the pool's average pages per tuple and the largest
  // keep‰), which hides the per-unit start-up latency behind the stream for short tuples.
  {
    int max_keep = 1;
    for (int i = 0; i < n_vsel; ++i) max_keep = std::max(max_keep, (int)variants[var_sel[i]].keep_permille);
    const double ppu = kv->n_tuples > 0
                           ? (double)kv->n_pages / (double)kv->n_tuples * max_keep / 1000.0
                           : 32.0;
    static const int hg_env = [] {  // tuning knob for A/B measurements
      const char* e = std::getenv("KO_HEADS_PER_UNIT");
      return e ? std::atoi(e) : 0;
    }();
    static const double unit_pages = [] {  // tuning knob (A/B): target pages per work unit
      const char* e = std::getenv("KO_UNIT_PAGES");
      return e ? std::atof(e) : 64.0;
    }();
    int hg = 1;
    while (hg * 2 <= kv->n_kv_heads && kv->n_kv_heads % (hg * 2) == 0 &&
           (hg * 2) * ppu <= unit_pages)
      hg *= 2;
    if (hg_env > 0 && kv->n_kv_heads % hg_env == 0) hg = hg_env;
    sp.heads_per_unit = hg;
  }
  pp.n_l = n_l;
  pp.n_kv_heads = kv->n_kv_heads;
  pp.gqa = kv->gqa_group;
  pp.n_q = kv->n_q;
  pp.n_layers = kv->n_layers;
  pp.head_dim = kv->head_dim;
  pp.n_ops = n_sel;
  pp.rows_per_op = sp.rows_per_op;
  pp.qfrag = ws.qfrag;
  pp.wfrag = ws.wfrag;
}

}  // namespace

extern "C" {

const char* ko_last_error(void) { return g_err.c_str(); }

void ko_set_trace_events(void* ev_begin, void* ev_end) {
  g_trace_begin = (cudaEvent_t)ev_begin;
  g_trace_end = (cudaEvent_t)ev_end;
}

int32_t ko_last_launch_count(void) { return g_launches; }

const char* ko_version(void) { return "ko 0.1 (sm_100a, mma.sync bf16 W-folded paged attention)"; }

size_t ko_workspace_size(const ko_kv_cache* kv, const ko_operator* ops, int32_t n_ops,
                         int32_t n_variants, int64_t n_work) {
  if (validate_kv(kv) != KO_OK || validate_ops(kv, ops, n_ops) != KO_OK) return 0;
  if (n_variants < 1 || n_variants > KO_MAX_VARIANTS || n_work < 0) return 0;
  return layout(kv, max_classes(ops, n_ops), max_entries(ops, n_ops), n_ops, n_variants, n_work,
                nullptr).total;
}

ko_status ko_score_batch(const ko_kv_cache* kv, const ko_operator* ops, int32_t n_ops,
                         const ko_variant* variants, int32_t n_variants, const int32_t* tuple_idx,
                         int64_t n_idx, float* margins, int32_t* classes, const ko_plan* plans,
                         int32_t n_plans, const uint8_t* gold, int64_t* counts, void* workspace,
                         size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("ko_score_batch");
  g_launches = 0;
  ko_status st;
  if ((st = validate_kv(kv)) != KO_OK) return st;
  if ((st = validate_ops(kv, ops, n_ops)) != KO_OK) return st;
  if ((st = validate_variants(kv, variants, n_variants)) != KO_OK) return st;
  if (n_plans < 0 || n_plans > KO_MAX_PLANS) return fail(KO_EINVAL, "n_plans %d outside [0,64]", n_plans);
  if (n_plans > 0 && !plans) return fail(KO_EINVAL, "plans is NULL with n_plans > 0");
  int32_t ncls[KO_MAX_OPS] = {1, 1, 1, 1};
  for (int o = 0; o < n_ops; ++o) ncls[o] = ops[o].n_classes;
  for (int g = 0; g < n_plans; ++g) {
    if ((st = validate_plan(&plans[g], g, ncls, n_ops, n_variants)) != KO_OK) return st;
    for (int i = 0; i < plans[g].n_stages; ++i)
      if (is_external(variants[plans[g].stage[i].variant]) && ncls[plans[g].stage[i].op] > 1)
        return fail(KO_EUNSUPPORTED, "plan %d stage %d: external variant on a map operator", g, i);
  }
  if (n_plans > 0 && !counts) return fail(KO_EINVAL, "counts is NULL with plans");
  if (tuple_idx && n_idx < 0) return fail(KO_EINVAL, "n_idx < 0");
  const bool routed = n_plans == 1;
  if (!routed && !margins) return fail(KO_EINVAL, "margins may be NULL only in routed mode");
  const int64_t n_work = tuple_idx ? n_idx : kv->n_tuples;
  if (n_work > kv->n_tuples) return fail(KO_EINVAL, "n_idx > n_tuples");
  const int maxc = max_classes(ops, n_ops);
  if (!routed && (int64_t)n_ops * kv->gqa_group * kv->n_q > KO_MAX_ROWS)
    return fail(KO_EUNSUPPORTED, "n_ops*gqa_group*n_q = %d > %d rows per kv-head",
                n_ops * kv->gqa_group * kv->n_q, KO_MAX_ROWS);
  if (!workspace) return fail(KO_EINVAL, "workspace is NULL");
  if (((uintptr_t)workspace & 255) != 0) return fail(KO_EINVAL, "workspace not 256-byte aligned");
  Workspace ws = layout(kv, maxc, max_entries(ops, n_ops), n_ops, n_variants, n_work,
                        (uint8_t*)workspace);
  if (workspace_bytes < ws.total)
    return fail(KO_EWORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, ws.total);
  cudaStream_t s = (cudaStream_t)stream;
  if (n_work == 0) return KO_OK;

  if (!routed) {
    // ---- grid / profiling mode: all ops × all variants in one read, every plan per tuple
    int op_sel[KO_MAX_OPS], var_sel[KO_MAX_VARIANTS], n_int = 0, ext[KO_MAX_VARIANTS], n_ext = 0;
    for (int i = 0; i < n_ops; ++i) op_sel[i] = i;
    for (int i = 0; i < n_variants; ++i) {
      if (is_external(variants[i])) ext[n_ext++] = i; else var_sel[n_int++] = i;
    }
    if (n_int == 0) return fail(KO_EINVAL, "no KV variant to score (all variants external)");
    int CPR = 1, NT = 0;
    ko::ScoreParams sp;
    ko::PrepParams pp;
    fill_common(sp, pp, kv, ops, op_sel, n_ops, variants, var_sel, n_int, n_ops, n_variants,
                ws, &CPR, &NT);
    if (NT <= 0)
      return fail(KO_EUNSUPPORTED, "operators need more than %d W·V tiles per kv-head row tile",
                  ko::kMaxTNT);
    sp.n_ext = n_ext;
    for (int i = 0; i < n_ext; ++i) sp.ext_ids[i] = ext[i];
    if ((st = make_tmap(&sp.tmap, kv)) != KO_OK) return st;
    // longest-first work order (varlen tail balance; identity for a fixed-length batch)
    KO_LAUNCH(ko::launch_lpt_order(tuple_idx, n_work, kv->seq_len, ws.lpt_hist, ws.lpt_perm, s));
    g_launches += 2;  // launch_lpt_order: 3 kernels
    sp.work = ws.lpt_perm;
    sp.work_len_host = n_work;
    sp.work_len_dev = nullptr;
    sp.margins = margins;
    sp.classes = classes;
    sp.mode = ko::MODE_GRID;
    sp.n_plans = n_plans;
    sp.gold = gold;
    sp.counts = (unsigned long long*)counts;
    for (int g = 0; g < n_plans; ++g) sp.plans[g] = plans[g];
    sp.gplans = ws.gplans;
    pp.gplans = ws.gplans;
    pp.n_plans = n_plans;
    for (int g = 0; g < n_plans; ++g) pp.plans[g] = plans[g];
    // Tuple finaliser: its own launch once the scan is long enough for the idle rings it saves
    // to outweigh one more launch (C5 / C3: −0.4 / −0.6 % per step; C2's 10 k tuples: flat;
    // C1's 64 tuples: +20 µs), else inside the scoring kernel.  Both are bit-identical
    // (tests/test_grid_final_gpu.py).  KO_GRID_FIN_KERNEL=0/1 forces one (A/B knob).
    static const int fin_env = [] {
      const char* e = std::getenv("KO_GRID_FIN_KERNEL");
      return e ? std::atoi(e) : -1;
    }();
    sp.fin_kernel = fin_env >= 0 ? fin_env : (n_work >= 8192 ? 1 : 0);
    KO_LAUNCH(ko::launch_prep(pp, s));
    KO_CUDA(cudaMemsetAsync(ws.unit_counter, 0, 16, s));
    if (!sp.fin_kernel) KO_CUDA(cudaMemsetAsync(ws.done, 0, sizeof(int32_t) * (size_t)n_work, s));
    if (g_trace_begin) KO_CUDA(cudaEventRecord(g_trace_begin, s));
    KO_LAUNCH(ko::launch_score(sp, kv->head_dim, CPR, NT, n_work * sp.n_l * kv->n_kv_heads, s));
    if (g_trace_end) KO_CUDA(cudaEventRecord(g_trace_end, s));
    if (sp.fin_kernel) KO_LAUNCH(ko::launch_grid_final(sp, CPR, s));
    return KO_OK;
  }

  // ---- routed mode (cascade execution): only tuples reaching a stage are scored
  const ko_plan& P = plans[0];
  ko::RouteParams rp;
  std::memset(&rp, 0, sizeof(rp));
  rp.plan = P;
  rp.n_ops = n_ops;
  rp.n_variants = n_variants;
  rp.n_tuples = kv->n_tuples;
  for (int o = 0; o < n_ops; ++o) rp.n_classes[o] = ops[o].n_classes;
  rp.subset = tuple_idx;
  rp.n_subset = n_work;
  rp.tuple_state = ws.tuple_state;
  rp.worklist = ws.worklist;
  rp.worklist_len = ws.worklist_len;
  rp.gold = gold;
  rp.counts = (unsigned long long*)counts;

  // Operator groups: the referenced ops fused into ONE read while their rows fit one 16-row tile
  // and the table packing stays within 4 W·V tiles (a speculative op costs tensor-core work on
  // bytes the read moves anyway, never extra bytes); otherwise a new group starts.  KO_FUSE=0
  // (A/B knob): only filters are fused, each map is a group of its own.
  const int rows_per_op = kv->gqa_group * kv->n_q;
  static const int fuse_all = [] {
    const char* e = std::getenv("KO_FUSE");
    return e ? std::atoi(e) : 1;
  }();
  int group_of_op[KO_MAX_OPS] = {-1, -1, -1, -1};
  int group_ops[KO_MAX_OPS][KO_MAX_OPS], group_n[KO_MAX_OPS] = {0, 0, 0, 0}, n_groups = 0;
  // fusing stays within 4 W·V tiles; an operator alone may take up to kMaxTNT (e.g. an 8-class
  // fp32 map on 16 rows)
  auto packs = [&](const int* sel, int n, int max_nt) {
    if (n * rows_per_op > KO_MAX_ROWS) return false;
    ko::ScoreParams tsp;
    ko::PrepParams tpp;
    const int nt = pack_table(ops, sel, n, rows_per_op, tsp, tpp);
    return nt > 0 && nt <= max_nt;
  };
  for (int i = 0; i < P.n_stages; ++i) {
    const int o = P.stage[i].op;
    if (group_of_op[o] >= 0) continue;
    int g = -1;
    for (int c = n_groups - 1; c >= 0 && g < 0; --c) {
      const bool maps_alone = !fuse_all && (ops[o].n_classes > 1 || ops[group_ops[c][0]].n_classes > 1);
      if (maps_alone) continue;
      int sel[KO_MAX_OPS];
      for (int k = 0; k < group_n[c]; ++k) sel[k] = group_ops[c][k];
      sel[group_n[c]] = o;
      if (packs(sel, group_n[c] + 1, 4)) g = c;
    }
    if (g < 0) {
      g = n_groups++;
      if (!packs(&o, 1, ko::kMaxTNT))
        return fail(KO_EUNSUPPORTED, "routed mode: op %d needs more than %d W·V tiles (%d classes, %s W)",
                    o, ko::kMaxTNT, ops[o].n_classes, ops[o].w_is_bf16 ? "bf16" : "fp32");
    }
    group_of_op[o] = g;
    group_ops[g][group_n[g]++] = o;
  }
  // Variant ranks: the plan's distinct KV variants ordered by extent (keep‰ · layers); a launch of
  // round r streams the extents of ranks ≤ r.  A variant's margin is complete (available) after
  // the first round r at which, for every layer l < its cut, some variant of rank ≤ r with cut > l
  // keeps at least as many tokens — then every snapshot it needs was taken by a round ≤ r.
  int pv[KO_MAX_VARIANTS], n_pv = 0;
  bool seen_v[KO_MAX_VARIANTS] = {false};
  for (int i = 0; i < P.n_stages; ++i)
    if (!seen_v[P.stage[i].variant] && !is_external(variants[P.stage[i].variant])) {
      seen_v[P.stage[i].variant] = true;
      pv[n_pv++] = P.stage[i].variant;
    }
  std::stable_sort(pv, pv + n_pv, [&](int a, int b) {
    const int64_t ea = (int64_t)variants[a].keep_permille * variants[a].layer_cut;
    const int64_t eb = (int64_t)variants[b].keep_permille * variants[b].layer_cut;
    return ea < eb;
  });
  int avail[KO_MAX_VARIANTS];
  for (int k = 0; k < n_pv; ++k) {
    const ko_variant& v = variants[pv[k]];
    avail[k] = k;
    for (int r = 0; r <= k; ++r) {
      bool ok = true;
      for (int l = 0; l < v.layer_cut && ok; ++l) {
        bool cov = false;
        for (int u = 0; u <= r && !cov; ++u)
          cov = variants[pv[u]].layer_cut > l && variants[pv[u]].keep_permille >= v.keep_permille;
        ok = cov;
      }
      if (ok) { avail[k] = r; break; }
    }
  }
  int var_rank[KO_MAX_VARIANTS];  // caller's variant → round after which its margin is available
  for (int v = 0; v < KO_MAX_VARIANTS; ++v) var_rank[v] = (v < n_variants && is_external(variants[v])) ? -1 : 0;
  for (int k = 0; k < n_pv; ++k) var_rank[pv[k]] = avail[k];
  if (!margins) {
    for (int i = 0; i < P.n_stages; ++i)
      if (is_external(variants[P.stage[i].variant]))
        return fail(KO_EINVAL, "routed plan uses an external variant but margins is NULL");
  }
  int pos_group[KO_MAX_STAGES], pos_round[KO_MAX_STAGES];
  for (int q = 0; q < P.n_stages; ++q) {
    pos_group[q] = group_of_op[P.stage[q].op];
    pos_round[q] = var_rank[P.stage[q].variant];
  }

  // One launch per plan position (= stage): tuples are queued by their own plan walk to the
  // first later position that computes what they need, so one pass in plan order suffices.
  // A position whose (group, round) is covered by position 0 never receives a tuple (position 0
  // processes every tuple), so it is not launched.
  KO_CUDA(cudaMemsetAsync(ws.round_len, 0, sizeof(unsigned long long) * KO_MAX_STAGES, s));
  // Launched positions.  A stage on an external variant (e.g. the embedding pre-filter) streams
  // nothing: position 0 on one only walks every tuple (deciding it from the caller's margins and
  // queueing the survivors), and a later one never receives a tuple (its margin is always
  // available).  A KV position whose (group, round) position 0 already streamed is covered.
  auto covered = [&](int pos) {
    if (pos == 0) return false;
    if (pos_round[pos] < 0) return true;
    return pos_round[0] >= 0 && pos_group[pos] == pos_group[0] && pos_round[pos] <= pos_round[0];
  };
  // Which positions can receive tuples at all: a walk after position w queues a tuple only to
  // the FIRST later position computing the (group, rank) of the stage it stopped at, and only
  // for a (group, rank) not yet computed for it — w's own group up to w's rank and position 0's
  // group up to its rank are (position 0 processes every tuple).  A superset of the real
  // traffic, so skipping the rest never drops a tuple (C4: positions 3 and 5 repeat position
  // 1's (group, rank 1) and would only ever run empty).
  bool receives[KO_MAX_STAGES] = {false};
  receives[0] = true;
  for (int w = 0; w < P.n_stages; ++w) {
    if (!receives[w] || covered(w)) continue;
    for (int s2 = 0; s2 < P.n_stages; ++s2) {
      const int g2 = pos_group[s2], rk = pos_round[s2];
      if (rk < 0) continue;                                        // external: always there
      if (pos_round[w] >= 0 && g2 == pos_group[w] && rk <= pos_round[w]) continue;
      if (pos_round[0] >= 0 && g2 == pos_group[0] && rk <= pos_round[0]) continue;
      int q = w + 1;
      while (q < P.n_stages && !(pos_group[q] == g2 && pos_round[q] >= rk)) ++q;
      if (q < P.n_stages) receives[q] = true;
    }
  }
  auto launched = [&](int pos) { return !covered(pos) && receives[pos]; };
  int last_launch = 0, prepped_group = -1;
  for (int pos = 0; pos < P.n_stages; ++pos)
    if (launched(pos)) last_launch = pos;
  for (int pos = 0; pos < P.n_stages; ++pos) {
    if (!launched(pos)) continue;
    char nv_name[48];
    std::snprintf(nv_name, sizeof(nv_name), "ko_score_batch/routed position %d", pos);
    NvtxRange nvtx_pos(nv_name);
    const int g = pos_group[pos];
    const bool walk_only = pos_round[pos] < 0;  // external stage at position 0
    const int r = std::max(pos_round[pos], 0);
    int CPR = 1, NT = 0;
    ko::ScoreParams sp;
    ko::PrepParams pp;
    fill_common(sp, pp, kv, ops, group_ops[g], group_n[g], variants, pv, n_pv, n_ops, n_variants,
                ws, &CPR, &NT);
    if (NT <= 0) return fail(KO_EUNSUPPORTED, "routed mode: table packing failed");
    if ((st = make_tmap(&sp.tmap, kv)) != KO_OK) return st;
    int n_l = 1;
    for (int k = 0; k <= r && k < n_pv; ++k) n_l = std::max(n_l, (int)variants[pv[k]].layer_cut);
    sp.n_l = n_l;
    sp.n_lh_all = kv->n_layers * kv->n_kv_heads;
    sp.part_cpr = pow2_at_least(maxc);  // the workspace's partial class stride
    sp.save_state = 0;
    for (int q = 0; q < P.n_stages; ++q)
      if (pos_group[q] == g && pos_round[q] > r) sp.save_state = 1;
    sp.rstate = ws.rstate + (size_t)g * ws.rstate_group;
    sp.rstate_w = rstate_record_floats(NT);  // this group's record (≤ the workspace bound)
    if (sp.rstate_w > ws.rstate_w) return fail(KO_EWORKSPACE, "routed mode: state record %d > %d", sp.rstate_w, ws.rstate_w);
    sp.pos = pos;
    sp.n_pos = P.n_stages;
    sp.group = walk_only ? -1 : g;  // −1: the walk records no computed round
    sp.round = r;
    for (int q = 0; q < P.n_stages; ++q) {
      sp.pos_group[q] = pos_group[q];
      sp.pos_round[q] = pos_round[q];
      sp.wl[q] = ws.round_wl + (size_t)q * std::max<int64_t>(kv->n_tuples, 1);
      sp.wl_len[q] = ws.round_len + q;
    }
    for (int o = 0; o < KO_MAX_OPS; ++o) sp.group_of_op[o] = group_of_op[o];
    for (int v = 0; v < KO_MAX_VARIANTS; ++v) sp.var_rank[v] = var_rank[v];
    if (pos == 0) {
      sp.work = tuple_idx;
      sp.work_len_host = n_work;
      sp.work_len_dev = nullptr;
    } else {
      sp.work = sp.wl[pos];
      sp.work_len_host = 0;
      sp.work_len_dev = (const int64_t*)sp.wl_len[pos];
    }
    sp.margins = margins;
    sp.classes = classes;
    sp.mode = ko::MODE_WALK;
    sp.n_plans = 1;
    sp.plans[0] = P;
    sp.tuple_state = ws.tuple_state;
    sp.tuple_done = ws.tuple_done;
    sp.counts = (unsigned long long*)counts;
    if (g_trace_begin && pos == 0) KO_CUDA(cudaEventRecord(g_trace_begin, s));
    if (!walk_only) {
      if (g != prepped_group) {  // the fragments depend only on the group (all plan layers)
        KO_LAUNCH(ko::launch_prep(pp, s));
        prepped_group = g;
      }
      KO_CUDA(cudaMemsetAsync(ws.unit_counter, 0, 8, s));
      KO_LAUNCH(ko::launch_score(sp, kv->head_dim, CPR, NT, n_work * sp.n_l * kv->n_kv_heads, s));
    }
    KO_LAUNCH(ko::launch_walk(sp, s));
    if (g_trace_end && pos == last_launch) KO_CUDA(cudaEventRecord(g_trace_end, s));
  }
  KO_LAUNCH(ko::launch_final_counts(rp, s));
  return KO_OK;
}

ko_status ko_route(const ko_plan* plan, const float* margins, const int32_t* classes,
                   const int32_t* n_classes, int32_t n_ops, int32_t n_variants, int64_t n_tuples,
                   int32_t stage, uint32_t* tuple_state, int32_t* worklist_out,
                   int64_t* worklist_len, const uint8_t* gold, int64_t* counts, void* stream) {
  NvtxRange nvtx_("ko_route");
  g_launches = 0;
  if (!plan || !margins || !n_classes || !tuple_state || !counts)
    return fail(KO_EINVAL, "ko_route: NULL plan/margins/n_classes/tuple_state/counts");
  if (n_ops < 1 || n_ops > KO_MAX_OPS) return fail(KO_EINVAL, "n_ops %d", n_ops);
  if (n_variants < 1 || n_variants > KO_MAX_VARIANTS) return fail(KO_EINVAL, "n_variants %d", n_variants);
  if (n_tuples < 0 || n_tuples > 0x7fffffffll) return fail(KO_EINVAL, "n_tuples %lld", (long long)n_tuples);
  for (int o = 0; o < n_ops; ++o)
    if (n_classes[o] < 1 || n_classes[o] > KO_MAX_CLASSES) return fail(KO_EINVAL, "n_classes[%d]", o);
  ko_status st;
  if ((st = validate_plan(plan, 0, n_classes, n_ops, n_variants)) != KO_OK) return st;
  if (stage < -1 || stage >= plan->n_stages) return fail(KO_EINVAL, "stage %d", stage);
  bool has_map = false;
  for (int s = 0; s < plan->n_stages; ++s) has_map |= n_classes[plan->stage[s].op] > 1;
  if (has_map && !classes) return fail(KO_EINVAL, "classes required for map operators");
  if ((worklist_out == nullptr) != (worklist_len == nullptr))
    return fail(KO_EINVAL, "worklist_out and worklist_len must both be set or both NULL");
  cudaStream_t s = (cudaStream_t)stream;
  ko::RouteParams rp;
  std::memset(&rp, 0, sizeof(rp));
  rp.plan = *plan;
  rp.margins = margins;
  rp.classes = classes;
  for (int o = 0; o < n_ops; ++o) rp.n_classes[o] = n_classes[o];
  rp.n_ops = n_ops;
  rp.n_variants = n_variants;
  rp.n_tuples = n_tuples;
  rp.tuple_state = tuple_state;
  rp.worklist = worklist_out;
  rp.worklist_len = (unsigned long long*)worklist_len;
  rp.gold = gold;
  rp.counts = (unsigned long long*)counts;
  if (n_tuples == 0) {
    if (worklist_len) KO_CUDA(cudaMemsetAsync(worklist_len, 0, 8, s));
    return KO_OK;
  }
  if (worklist_len) KO_CUDA(cudaMemsetAsync(worklist_len, 0, 8, s));
  if (stage == -1) {
    KO_LAUNCH(ko::launch_route_plan(rp, s));
    return KO_OK;
  }
  rp.stage = stage;
  KO_LAUNCH(ko::launch_route_apply(rp, s));
  if (worklist_out) {
    rp.stage = stage + 1;  // tuples reaching the next stage (none after the last)
    KO_LAUNCH(ko::launch_route_reach(rp, s));
  }
  return KO_OK;
}

ko_status ko_reduce_stats(const ko_plan* plans, int32_t n_plans, const float* margins,
                          const int32_t* classes, const int32_t* n_classes, int32_t n_ops,
                          int32_t n_variants, int64_t n_tuples, const uint8_t* gold,
                          int64_t* counts, void* stream) {
  NvtxRange nvtx_("ko_reduce_stats");
  g_launches = 0;
  if (!plans || !margins || !n_classes || !counts)
    return fail(KO_EINVAL, "ko_reduce_stats: NULL plans/margins/n_classes/counts");
  if (n_plans < 1 || n_plans > KO_MAX_PLANS) return fail(KO_EINVAL, "n_plans %d", n_plans);
  if (n_ops < 1 || n_ops > KO_MAX_OPS) return fail(KO_EINVAL, "n_ops %d", n_ops);
  if (n_variants < 1 || n_variants > KO_MAX_VARIANTS) return fail(KO_EINVAL, "n_variants %d", n_variants);
  if (n_tuples < 0) return fail(KO_EINVAL, "n_tuples < 0");
  for (int o = 0; o < n_ops; ++o)
    if (n_classes[o] < 1 || n_classes[o] > KO_MAX_CLASSES) return fail(KO_EINVAL, "n_classes[%d]", o);
  ko_status st;
  bool has_map = false;
  for (int g = 0; g < n_plans; ++g) {
    if ((st = validate_plan(&plans[g], g, n_classes, n_ops, n_variants)) != KO_OK) return st;
    for (int s = 0; s < plans[g].n_stages; ++s) has_map |= n_classes[plans[g].stage[s].op] > 1;
  }
  if (has_map && !classes) return fail(KO_EINVAL, "classes required for map operators");
  if (n_tuples == 0) return KO_OK;
  ko::ReduceParams rp;
  std::memset(&rp, 0, sizeof(rp));
  rp.n_plans = n_plans;
  rp.margins = margins;
  rp.classes = classes;
  for (int o = 0; o < n_ops; ++o) rp.n_classes[o] = n_classes[o];
  rp.n_ops = n_ops;
  rp.n_variants = n_variants;
  rp.n_tuples = n_tuples;
  rp.gold = gold;
  rp.counts = (unsigned long long*)counts;
  for (int g = 0; g < n_plans; ++g) rp.plans[g] = plans[g];
  KO_LAUNCH(ko::launch_reduce(rp, (cudaStream_t)stream));
  return KO_OK;
}

ko_status ko_embed_scores(const void* item_emb, int32_t dim, int64_t n_tuples, const void* op_emb,
                          int32_t n_emb, const int32_t* op_ids, int32_t n_ops, int32_t variant,
                          int32_t n_variants, const int32_t* tuple_idx, int64_t n_idx,
                          float* margins, void* stream) {
  NvtxRange nvtx_("ko_embed_scores");
  g_launches = 0;
  if (!item_emb || !op_emb || !op_ids || !margins) return fail(KO_EINVAL, "ko_embed_scores: NULL argument");
  if (dim < 8 || dim % 8 != 0 || dim > 1024) return fail(KO_EINVAL, "dim %d: multiple of 8 in [8,1024]", dim);
  if (n_emb < 1 || n_emb > KO_MAX_OPS) return fail(KO_EINVAL, "n_emb %d outside [1,%d]", n_emb, KO_MAX_OPS);
  if (n_ops < 1 || n_ops > KO_MAX_OPS) return fail(KO_EINVAL, "n_ops %d", n_ops);
  if (variant < 0 || variant >= n_variants || n_variants > KO_MAX_VARIANTS)
    return fail(KO_EINVAL, "variant %d / n_variants %d", variant, n_variants);
  if (n_tuples < 0 || (tuple_idx && n_idx < 0)) return fail(KO_EINVAL, "negative sizes");
  if (((uintptr_t)item_emb & 15) != 0) return fail(KO_EINVAL, "item_emb not 16-byte aligned");
  ko::EmbedParams ep;
  std::memset(&ep, 0, sizeof(ep));
  for (int i = 0; i < n_emb; ++i) {
    if (op_ids[i] < 0 || op_ids[i] >= n_ops) return fail(KO_EINVAL, "op_ids[%d] = %d", i, op_ids[i]);
    ep.op_ids[i] = op_ids[i];
  }
  ep.item_emb = (const uint16_t*)item_emb;
  ep.op_emb = (const uint16_t*)op_emb;
  ep.dim = dim;
  ep.n_e = n_emb;
  ep.variant = variant;
  ep.n_variants = n_variants;
  ep.n_tuples = n_tuples;
  ep.tuple_idx = tuple_idx;
  ep.n_idx = n_idx;
  ep.margins = margins;
  if ((tuple_idx ? n_idx : n_tuples) == 0) return KO_OK;
  ep.use_tmap = 0;
  static const int emb_tmap = [] {  // A/B knob: 2-D tensor-map loads for contiguous rows
    const char* e = std::getenv("KO_EMB_TMAP");
    return e ? std::atoi(e) : 1;
  }();
  if (emb_tmap && dim % 16 == 0 && dim <= 512 && n_tuples > 0 && n_tuples < (1ll << 31)) {
    // a 2-D tensor map over item_emb, 128B swizzle: contiguous rows in boxes of 64 dims × 16
    // rows; gathered rows (tuple_idx) with tile::gather4, whose box is 64 dims × 1 row
    cuuint64_t dims[2] = {(cuuint64_t)dim, (cuuint64_t)n_tuples};
    cuuint64_t strides[1] = {(cuuint64_t)dim * 2};
    cuuint32_t box[2] = {64, tuple_idx ? 1u : 16u};
    // on failure the per-lane copy path runs (the message of the failed encode is dropped)
    ep.use_tmap = encode_tmap(&ep.tmap, item_emb, 2, dims, strides, box) == KO_OK;
  }
  KO_LAUNCH(ko::launch_embed(ep, (cudaStream_t)stream));
  return KO_OK;
}

ko_status ko_build_importance_order(const ko_kv_cache* src, const float* mu, const float* sigma2,
                                    void* dst_pool, const int32_t* dst_page_ids, void* stream) {
  NvtxRange nvtx_("ko_build_importance_order");
  g_launches = 0;
  ko_status st;
  if ((st = validate_kv(src)) != KO_OK) return st;
  if (!mu || !sigma2 || !dst_pool || !dst_page_ids)
    return fail(KO_EINVAL, "ko_build_importance_order: NULL mu/sigma2/dst_pool/dst_page_ids");
  if (((uintptr_t)dst_pool & 15) != 0) return fail(KO_EINVAL, "dst_pool not 16-byte aligned");
  if (src->n_tuples == 0) return KO_OK;
  ko::BuildParams bp;
  std::memset(&bp, 0, sizeof(bp));
  bp.src_pool = (const uint16_t*)src->kv_pool;
  bp.indptr = src->page_indptr;
  bp.src_ids = src->page_ids;
  bp.seq_len = src->seq_len;
  bp.n_tuples = src->n_tuples;
  bp.n_layers = src->n_layers;
  bp.n_kv_heads = src->n_kv_heads;
  bp.head_dim = src->head_dim;
  bp.page_elems = (int64_t)src->n_layers * 2 * src->n_kv_heads * KO_PAGE_TOKENS * src->head_dim;
  bp.mu = mu;
  bp.sigma2 = sigma2;
  bp.dst_pool = (uint16_t*)dst_pool;
  bp.dst_ids = dst_page_ids;
  bp.inv_sqrt_d = 1.0 / std::sqrt((double)src->head_dim);
  bp.inv_2d = 1.0 / (2.0 * (double)src->head_dim);
  bp.n_pages = src->n_pages;
  {
    // 2-D views of both pools for the TMA loads, row gathers and stores (ko_build.cu)
    const int64_t rows = src->n_pages * 2 * src->n_layers * src->n_kv_heads * KO_PAGE_TOKENS;
    if (rows >= (1ll << 31))
      return fail(KO_EUNSUPPORTED, "pool of %lld rows: the builder's TMA row coordinates are int32",
                  (long long)rows);
    const cuuint64_t D = (cuuint64_t)src->head_dim;
    // score loads: 64-d × 16-row boxes, 128B swizzle (conflict-free per-token reads); row
    // gathers and chunk stores: whole rows, unswizzled (the gathered rows are only copied)
    struct { CUtensorMap* map; const void* base; cuuint32_t box_d, box_rows; bool swz; } views[3] = {
        {&bp.tm_src, src->kv_pool, 64, 16, true}, {&bp.tm_row, src->kv_pool, (cuuint32_t)D, 1, false},
        {&bp.tm_dst, dst_pool, (cuuint32_t)D, 16, false}};
    for (auto& v : views) {
      cuuint64_t dims[2] = {D, (cuuint64_t)std::max<int64_t>(rows, 1)};
      cuuint64_t strides[1] = {D * 2};
      cuuint32_t box[2] = {v.box_d, v.box_rows};
      if ((st = encode_tmap(v.map, v.base, 2, dims, strides, box, v.swz)) != KO_OK) return st;
    }
  }
  KO_LAUNCH(ko::launch_build(bp, (cudaStream_t)stream));
  ++g_launches;  // launch_build: two kernels (short / long tuples)
  return KO_OK;
}

size_t ko_soft_workspace_size(int32_t n_stages, int64_t n_tuples) {
  if (n_stages < 1 || n_stages > KO_MAX_STAGES || n_tuples < 0) return 0;
  // the soft kernel's per-CTA partial sums of every (direction, output) row
  return align256(sizeof(double) * (size_t)(3 * n_stages + 1) * 4 * (size_t)ko::soft_blocks(n_tuples));
}

ko_status ko_soft_stats(const ko_plan* plan, const double* pick_scores, const double* stage_cost,
                        double tau, const float* margins, const int32_t* classes,
                        const int32_t* n_classes, int32_t n_ops, int32_t n_variants,
                        int64_t n_tuples, const uint8_t* gold, double* out, void* workspace,
                        size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("ko_soft_stats");
  g_launches = 0;
  if (!plan || !pick_scores || !stage_cost || !margins || !n_classes || !out || !workspace)
    return fail(KO_EINVAL, "ko_soft_stats: NULL argument");
  if (n_ops < 1 || n_ops > KO_MAX_OPS) return fail(KO_EINVAL, "n_ops %d", n_ops);
  if (n_variants < 1 || n_variants > KO_MAX_VARIANTS) return fail(KO_EINVAL, "n_variants %d", n_variants);
  if (n_tuples < 0) return fail(KO_EINVAL, "n_tuples < 0");
  if (!(tau > 0.0) || !std::isfinite(tau)) return fail(KO_EINVAL, "tau must be > 0");
  ko_status st;
  if ((st = validate_plan(plan, 0, n_classes, n_ops, n_variants)) != KO_OK) return st;
  ko::SoftParams sp;
  std::memset(&sp, 0, sizeof(sp));
  for (int i = 0; i < plan->n_stages; ++i) {
    if (n_classes[plan->stage[i].op] > 1) {
      if (!classes) return fail(KO_EINVAL, "ko_soft_stats: stage %d is a map stage: classes required", i);
      sp.is_map[plan->stage[i].op] = 1;
    }
    if (!std::isfinite(pick_scores[i]) || !std::isfinite(stage_cost[i]))
      return fail(KO_EINVAL, "stage %d: non-finite pick score or cost", i);
    sp.pick[i] = pick_scores[i];
    sp.stage_cost[i] = stage_cost[i];
    sp.referenced[plan->stage[i].op] = 1;
  }
  if (workspace_bytes < ko_soft_workspace_size(plan->n_stages, n_tuples))
    return fail(KO_EWORKSPACE, "workspace %zu < %zu", workspace_bytes,
                ko_soft_workspace_size(plan->n_stages, n_tuples));
  sp.plan = *plan;
  sp.tau = tau;
  sp.margins = margins;
  sp.classes = classes;
  sp.n_ops = n_ops;
  sp.n_variants = n_variants;
  sp.n_tuples = n_tuples;
  sp.gold = gold;
  sp.partials = (double*)workspace;
  for (int o = 0; o < n_ops; ++o)  // compact slots in op-id order (same product order)
    if (sp.referenced[o]) {
      sp.slot_op[sp.n_slots] = o;
      sp.slot_is_map[sp.n_slots] = sp.is_map[o];
      ++sp.n_slots;
    }
  for (int i = 0; i < plan->n_stages; ++i) {
    for (int k = 0; k < sp.n_slots; ++k)
      if (sp.slot_op[k] == plan->stage[i].op) sp.stage_slot[i] = k;
    // parameters with an effect (ko.h: finals have only θ⁺, maps no θ⁻, a final map none)
    const bool fin = plan->stage[i].is_final != 0, map = sp.is_map[plan->stage[i].op] != 0;
    sp.dir_live[3 * i + 0] = !fin;
    sp.dir_live[3 * i + 1] = !fin && !map;
    sp.dir_live[3 * i + 2] = !(fin && map);
  }
  KO_LAUNCH(ko::launch_soft(sp, out, (cudaStream_t)stream));
  ++g_launches;  // launch_soft: two kernels (per-tuple values with CTA sums, in-order final sum)
  return KO_OK;
}

// ---- Bayesian lower bound (host): I^{-1}(1 − α; 1 + a, 1 + b) -------------------------------
// Regularized incomplete beta by its continued fraction evaluated with the modified Lentz method
// (textbook algorithm: W. H. Press et al., Numerical Recipes, 3rd ed., §6.4 "Incomplete Beta
// Function", routine betacf, whose variable names this follows; SPEC S:134 prescribes the same
// method with the symmetry split at x = (a+1)/(a+b+2)); inverse by bisection.
static double betacf(double a, double b, double x) {
  const double tiny = 1e-300, eps = 1e-16;
  double qab = a + b, qap = a + 1.0, qam = a - 1.0;
  double c = 1.0, d = 1.0 - qab * x / qap;
  if (std::fabs(d) < tiny) d = tiny;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= 100000; ++m) {
    const int m2 = 2 * m;
    double aa = m * (b - m) * x / ((qam + m2) * (a + m2));
    d = 1.0 + aa * d; if (std::fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c; if (std::fabs(c) < tiny) c = tiny;
    d = 1.0 / d; h *= d * c;
    aa = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
    d = 1.0 + aa * d; if (std::fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c; if (std::fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double del = d * c;
    h *= del;
    if (std::fabs(del - 1.0) < eps) break;
  }
  return h;
}

static double betainc_reg(double a, double b, double x) {
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double lbt = std::lgamma(a + b) - std::lgamma(a) - std::lgamma(b) + a * std::log(x) +
                     b * std::log1p(-x);
  if (x < (a + 1.0) / (a + b + 2.0)) return std::exp(lbt) * betacf(a, b, x) / a;
  return 1.0 - std::exp(lbt) * betacf(b, a, 1.0 - x) / b;
}

// x with I_x(a, b) = p (a, b > 0 real) by bisection: I is increasing in x.
static double betainc_inv(double a, double b, double p) {
  double lo = 0.0, hi = 1.0;
  for (int it = 0; it < 200 && hi - lo > 1e-16; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (betainc_reg(a, b, mid) < p) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

double ko_beta_lower_bound(int64_t a_cnt, int64_t b_cnt, double alpha) {
  if (a_cnt < 0 || b_cnt < 0 || !(alpha > 0.0 && alpha < 1.0)) return NAN;
  return betainc_inv(1.0 + (double)a_cnt, 1.0 + (double)b_cnt, 1.0 - alpha);
}

double ko_beta_lower_bound_real(double a_cnt, double b_cnt, double alpha, double* dl_da,
                                double* dl_db) {
  if (!(a_cnt >= 0.0) || !(b_cnt >= 0.0) || !std::isfinite(a_cnt) || !std::isfinite(b_cnt) ||
      !(alpha > 0.0 && alpha < 1.0))
    return NAN;
  const double A = 1.0 + a_cnt, B = 1.0 + b_cnt, p = 1.0 - alpha;
  const double x = betainc_inv(A, B, p);
  // Implicit differentiation of I_x(A, B) = p: dx/dA = −(∂I/∂A)/(∂I/∂x), with
  // ∂I/∂x the Beta(A, B) density at x and ∂I/∂A, ∂I/∂B central differences of I in the shape
  // (step 1e-5·max(1, shape)).  dA/da = dB/db = 1.
  if (dl_da || dl_db) {
    double da = 0.0, db = 0.0;
    if (x > 0.0 && x < 1.0) {
      const double log_dens = (A - 1.0) * std::log(x) + (B - 1.0) * std::log1p(-x) -
                              (std::lgamma(A) + std::lgamma(B) - std::lgamma(A + B));
      const double dens = std::exp(log_dens);
      if (dens > 0.0) {
        const double ha = 1e-5 * std::max(1.0, A), hb = 1e-5 * std::max(1.0, B);
        const double dIdA = (betainc_reg(A + ha, B, x) - betainc_reg(A - ha, B, x)) / (2.0 * ha);
        const double dIdB = (betainc_reg(A, B + hb, x) - betainc_reg(A, B - hb, x)) / (2.0 * hb);
        da = -dIdA / dens;
        db = -dIdB / dens;
      }
    }
    if (dl_da) *dl_da = da;
    if (dl_db) *dl_db = db;
  }
  return x;
}

ko_status ko_plan_loss(const double* stats, const double* jacobian, int32_t n_params,
                       double n_tuples, const double* stage_cost, int32_t n_stages,
                       const ko_loss_params* lp, double* out, double* grad) {
  g_launches = 0;
  if (!stats || !stage_cost || !lp || !out) return fail(KO_EINVAL, "ko_plan_loss: NULL argument");
  if (n_params < 0 || (n_params > 0 && !jacobian) || (grad && n_params > 0 && !jacobian))
    return fail(KO_EINVAL, "ko_plan_loss: n_params %d without a jacobian", n_params);
  if (n_stages < 1 || n_stages > KO_MAX_STAGES) return fail(KO_EINVAL, "n_stages %d", n_stages);
  if (!(n_tuples > 0.0)) return fail(KO_EINVAL, "n_tuples must be > 0");
  if (!(lp->alpha > 0.0 && lp->alpha < 1.0)) return fail(KO_EINVAL, "alpha outside (0,1)");
  if (!(lp->beta >= 0.0) || !std::isfinite(lp->beta)) return fail(KO_EINVAL, "beta must be >= 0");
  const double tp = stats[0], fp = stats[1], fn = stats[2], cost = stats[3];
  if (!(tp >= 0.0 && fp >= 0.0 && fn >= 0.0 && cost >= 0.0))
    return fail(KO_EINVAL, "ko_plan_loss: negative or NaN TP/FP/FN/cost");
  double csum = 0.0;  // Σ_i cost_{o_i} over the plan's stages (eqn:cost-loss)
  for (int i = 0; i < n_stages; ++i) {
    if (!(stage_cost[i] >= 0.0) || !std::isfinite(stage_cost[i]))
      return fail(KO_EINVAL, "stage_cost[%d] negative or non-finite", i);
    csum += stage_cost[i];
  }
  if (!(csum > 0.0)) return fail(KO_EINVAL, "sum of stage costs must be > 0");
  const double norm = n_tuples * csum;
  double dR_dtp, dR_dfn, dP_dtp, dP_dfp;
  const double lR = ko_beta_lower_bound_real(tp, fn, lp->alpha, &dR_dtp, &dR_dfn);
  const double lP = ko_beta_lower_bound_real(tp, fp, lp->alpha, &dP_dtp, &dP_dfp);
  const double L_cost = cost / norm;
  const double L_R = std::max(0.0, lp->target_recall - lR);
  const double L_P = std::max(0.0, lp->target_precision - lP);
  const bool act_R = lp->target_recall > lR, act_P = lp->target_precision > lP;
  out[0] = L_cost + lp->beta * L_P + lp->beta * L_R;
  out[1] = L_cost;
  out[2] = L_R;
  out[3] = L_P;
  out[4] = lR;
  out[5] = lP;
  // Target Met: achieved / target, achieved = the point recall / precision of the counts
  // (an empty output has precision 1, Q20); NaN for a zero target
  const double rec = tp + fn > 0.0 ? tp / (tp + fn) : 1.0;
  const double prec = tp + fp > 0.0 ? tp / (tp + fp) : 1.0;
  out[6] = rec;
  out[7] = prec;
  out[8] = lp->target_recall > 0.0 ? rec / lp->target_recall : NAN;
  out[9] = lp->target_precision > 0.0 ? prec / lp->target_precision : NAN;
  if (grad) {
    // dL/dp = (dcost/dp)/norm − β·[T_R > ℓ_R]·dℓ_R/dp − β·[T_P > ℓ_P]·dℓ_P/dp; the Jacobian rows
    // are (TP, FP, FN, cost) × n_params (ko_soft_stats' layout)
    const double* J_tp = jacobian;
    const double* J_fp = jacobian + n_params;
    const double* J_fn = jacobian + 2 * (size_t)n_params;
    const double* J_c = jacobian + 3 * (size_t)n_params;
    for (int k = 0; k < n_params; ++k) {
      double g = J_c[k] / norm;
      if (act_R) g -= lp->beta * (dR_dtp * J_tp[k] + dR_dfn * J_fn[k]);
      if (act_P) g -= lp->beta * (dP_dtp * J_tp[k] + dP_dfp * J_fp[k]);
      grad[k] = g;
    }
  }
  return KO_OK;
}

}  // extern "C"
