// ko_internal.h — host-side contract between ko_api.cpp (validation, workspace, dispatch) and
// ko_kernels.cu (device code + launchers).  Not part of the public ABI (that is include/ko.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "ko.h"

// Device-side checks of caller data (ko.h: "device-data errors are undefined behaviour" in the
// release build).  The KO_DEBUG build (lib/libko_debug.so, same ABI) traps on a page id outside
// [0, n_pages), seq_len < 1 or a tuple id outside [0, n_tuples), after printing the failed check.
#ifdef KO_DEBUG
#include <cstdio>
#define KO_DCHECK(cond)                                                                       \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("KO_DEBUG check failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,    \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                    \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define KO_DCHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace ko {

constexpr int kMaxOps = KO_MAX_OPS;
constexpr int kMaxVar = KO_MAX_VARIANTS;
constexpr int kMaxCls = KO_MAX_CLASSES;
constexpr int kMaxPlans = KO_MAX_PLANS;
constexpr int kCountsPerPlan = KO_COUNTS_PER_PLAN;
constexpr int kThreads = 128;  // score kernel CTA size (4 warps, one work unit per warp)
constexpr int kMaxTNT = 8;     // W·V tiles of the table-packed kernel (2·kMaxTNT slots per lane)

enum Mode : int32_t { MODE_GRID = 0, MODE_WALK = 2 };

// One launch of the scoring kernel.  "Local" op/variant indices are positions in this launch;
// op_ids / var_ids map them to the caller's indices (margins layout, plans, gold).
struct ScoreParams {
  // TMA descriptor of the pool viewed as 5-D bf16 [n_pages][2·n_layers][n_kv_heads][16][head_dim]
  // (innermost last), box 64 × 16 × 1 × 2 × 1, 128-byte swizzle
  alignas(64) CUtensorMap tmap;
  // paged KV store
  const uint16_t* pool;
  int64_t page_elems;  // bf16 elements per page = n_layers*2*n_kv_heads*16*head_dim
  const int64_t* page_indptr;
  const int32_t* page_ids;
  const int32_t* seq_len;
  int64_t n_tuples;
  int64_t n_pages;  // pool pages (KO_DEBUG bounds check of page ids)
  int32_t n_layers, n_kv_heads, gqa, n_q;
  // work list (tuple ids); NULL = identity.  Length from work_len_dev if non-NULL.
  const int32_t* work;
  int64_t work_len_host;
  const int64_t* work_len_dev;
  int32_t n_l;  // layers computed = max layer_cut over this launch's variants
  // operators of this launch
  int32_t n_ops;
  int32_t op_ids[kMaxOps];
  int32_t op_classes[kMaxOps];    // by local op
  int32_t op_classes_g[kMaxOps];  // by caller's op index
  const float* bias[kMaxOps];  // device fp32 [n_classes] per op
  const float* bias_g[kMaxOps];  // same, by caller's op index (routed walk)
  int32_t rows_per_op;  // gqa * n_q
  int32_t slot_op[16];  // row slot (half*8 + g) → local op, -1 = padding
  int32_t n_ops_total, n_var_total;
  int32_t n_ext;               // external variants (caller-supplied margins, keep‰ = 0)
  int32_t ext_ids[kMaxVar];
  // variants of this launch
  int32_t n_var;
  int32_t keep[kMaxVar], cut[kMaxVar], var_ids[kMaxVar];
  // prepared tensor-core fragments (workspace)
  const uint4* qfrag;  // [n_l*Hkv][KS][32]
  const uint4* wfrag;  // [n_l*Hkv][NT][KS][32]
  const ko_plan* gplans;  // device copy of plans[] (lanes read different plans: L1, not the
                          // constant bank, which serialises divergent reads)
  // scratch (workspace)
  float* part;                     // [n_work][n_l*Hkv][n_ops][n_var][CPR]
  int32_t* done;                   // [n_work]
  unsigned long long* unit_counter;
  // outputs
  float* margins;   // [n_ops_total][n_var_total][n_tuples] or NULL
  int32_t* classes;  // same or NULL
  float scale_log2;  // log2(e)/sqrt(head_dim)
  int32_t heads_per_unit;  // kv-heads one work unit streams back-to-back (divides n_kv_heads)
  // grid mode: per-tuple evaluation of every plan (indices are caller's = local here)
  int32_t mode;
  int32_t fin_kernel;   // grid mode: 1 = tuples finalised by grid_final_kernel after the launch
  int32_t n_plans;
  const uint8_t* gold;  // [n_ops_total][n_tuples] or NULL
  unsigned long long* counts;  // [n_plans][kCountsPerPlan] (int64 bit pattern)
  uint32_t* tuple_state;         // walk mode: per-tuple routing state (ko_route's bit layout)
  // walk mode (routed execution): launch = plan position pos = (operator group, variant rank)
  int32_t pos, n_pos, group, round;
  int32_t pos_group[KO_MAX_STAGES], pos_round[KO_MAX_STAGES];
  int32_t group_of_op[kMaxOps];  // caller's op → group
  int32_t var_rank[kMaxVar];     // caller's variant → rank (launches of rank r compute ranks ≤ r)
  int32_t var_local[kMaxVar];    // caller's variant → local index in this launch (-1: absent)
  int32_t* wl[KO_MAX_STAGES];                 // per-position worklists
  unsigned long long* wl_len[KO_MAX_STAGES];  // their lengths (device)
  uint32_t* tuple_done;          // per tuple: 4-bit (rank + 1) computed per group, 15 = none
  // walk mode, resumable extents: local variants are ALL the plan's KV variants in rank order
  // (local index = rank); this launch streams, per (tuple, layer), the tokens between the
  // extent of the tuple's previous rank for this group and the extent of rank `round`, resuming
  // the saved softmax state; partials persist per tuple (ko_walk_kernel finishes a variant's
  // margin once var_rank says it is complete).
  int32_t save_state;            // a later rank of this group exists: save the state at the end
  float* rstate;                 // [n_tuples][n_layers][Hkv][8][rstate_w] (this group's slice)
  int32_t rstate_w;              // floats per lane group: M[2], den[2], acc[2·NT], zero-padded
                                 // to whole 32-byte sectors (= the kernel's kRecW)
  int32_t n_lh_all;              // n_layers · Hkv (partials of walk mode are per tuple, all layers)
  int32_t part_cpr;              // class stride of walk-mode partials (same for every group)
                                 // walk-mode partials: [t][variant][layer·Hkv + h][block], block
                                 // = [op][part_cpr] padded to whole sectors (walk_part_blk)
  // table-driven row/class packing (template NT): per lane group g, W·V slot k = 2·tile + hr
  // (A-row half hr) accumulates with S row g + 8·hr into the local (op, class) target
  // tgt = op·8 + class (−1: unused)
  int8_t tbl_tgt[8][16];
  ko_plan plans[kMaxPlans];
};

// Floats per (tuple, layer·kv-head, variant) block of walk-mode partial logits: [op][cpr],
// padded to whole 32-byte sectors so a snapshot stores its block as whole sectors.
__host__ __device__ inline int walk_part_blk(int n_ops_total, int cpr) {
  return (n_ops_total * cpr + 7) / 8 * 8;
}

struct PrepParams {
  int32_t n_l, n_kv_heads, gqa, n_q, n_layers, head_dim;
  int32_t n_ops, rows_per_op;
  int32_t slot_op[16];   // row slot → local op (-1 = padding)
  int32_t slot_rem[16];  // row slot → row within the op (gqa member * n_q + query row)
  const uint16_t* q[kMaxOps];
  const float* w[kMaxOps];          // fp32 readout, or NULL when w_bf16 is given
  const uint16_t* w_bf16[kMaxOps];  // bf16 readout (ko_operator.w_is_bf16)
  // table packing: W entry of lane group g, slot k = 2·tile + A-row half:
  // −1 unused, else (local op) | rem << 3 | class << 8 | lo << 12 (lo: the fp32 residual part)
  int32_t tbl_nt;
  int32_t tbl_w[8][16];
  int32_t op_classes[kMaxOps];
  uint4* qfrag;
  uint4* wfrag;
  int32_t n_plans;
  ko_plan* gplans;  // prep copies plans[] here (device)
  ko_plan plans[kMaxPlans];
};

struct RouteParams {
  ko_plan plan;
  const float* margins;
  const int32_t* classes;
  int32_t n_classes[kMaxOps];
  int32_t n_ops, n_variants;
  int64_t n_tuples;
  const int32_t* subset;  // optional tuple subset (NULL = all)
  int64_t n_subset;
  int32_t stage;
  uint32_t* tuple_state;
  int32_t* worklist;
  unsigned long long* worklist_len;
  const uint8_t* gold;
  unsigned long long* counts;
};

struct ReduceParams {
  int32_t n_plans;
  const float* margins;
  const int32_t* classes;
  int32_t n_classes[kMaxOps];
  int32_t n_ops, n_variants;
  int64_t n_tuples;
  const uint8_t* gold;
  unsigned long long* counts;
  ko_plan plans[kMaxPlans];
};

// embedding-similarity stage
struct EmbedParams {
  alignas(64) CUtensorMap tmap;  // item_emb as 2-D bf16 [n_tuples][dim], box 64 × 16, 128B swizzle
  int32_t use_tmap;              // contiguous rows (tuple_idx == NULL): tensor-map loads
  const uint16_t* item_emb;  // bf16 [n_tuples][dim]
  const uint16_t* op_emb;    // bf16 [n_e][dim]
  int32_t dim, n_e;
  int32_t op_ids[kMaxOps];   // caller's op of each embedding
  int32_t variant, n_variants;
  int64_t n_tuples;
  const int32_t* tuple_idx;
  int64_t n_idx;
  float* margins;            // [n_ops][n_variants][n_tuples]
};
cudaError_t launch_embed(const EmbedParams& p, cudaStream_t s);

// importance-ordered cache builder (ko_build.cu)
struct BuildParams {
  // 2-D bf16 views [n_pages · 2·n_layers·n_kv_heads·16 rows][head_dim] of the pools:
  alignas(64) CUtensorMap tm_src;  // source, box 64 d × 16 rows, 128B swizzle (score loads)
  alignas(64) CUtensorMap tm_row;  // source, box D × 1 row, unswizzled (tile::gather4)
  alignas(64) CUtensorMap tm_dst;  // destination, box D × 16 rows, unswizzled (chunk stores)
  const uint16_t* src_pool;
  const int64_t* indptr;
  const int32_t* src_ids;
  const int32_t* seq_len;
  int64_t n_tuples;
  int32_t n_layers, n_kv_heads, head_dim;
  int64_t page_elems;
  const float* mu;      // [n_layers][n_kv_heads][head_dim]
  const float* sigma2;  // same
  uint16_t* dst_pool;
  const int32_t* dst_ids;
  double inv_sqrt_d, inv_2d;
  int64_t n_pages;  // pages of src and dst pools (KO_DEBUG bounds checks)
};
cudaError_t launch_build(const BuildParams& p, cudaStream_t s);

// soft relaxation of one plan (ko_soft.cu)
struct SoftParams {
  ko_plan plan;
  double pick[KO_MAX_STAGES];
  double stage_cost[KO_MAX_STAGES];
  double tau;
  const float* margins;  // [n_ops][n_variants][n_tuples]
  int32_t n_ops, n_variants;
  int64_t n_tuples;
  const uint8_t* gold;   // [n_ops][n_tuples] or NULL (filters 0/1, maps the class)
  const int32_t* classes;  // [n_ops][n_variants][n_tuples] argmax classes (maps) or NULL
  int32_t referenced[kMaxOps];
  int32_t is_map[kMaxOps];  // referenced op with n_classes > 1
  // compact operator slots: the plan's distinct operators in op-id order
  int32_t n_slots;
  int32_t slot_op[kMaxOps], slot_is_map[kMaxOps];
  int32_t stage_slot[KO_MAX_STAGES];
  int32_t dir_live[3 * KO_MAX_STAGES];  // direction 1 + 3i + f moves the outputs (0: exact zeros)
  double* partials;      // workspace [soft_blocks(n_tuples)][4·(3·S + 1)]: per-CTA sums
};
cudaError_t launch_soft(const SoftParams& p, double* out, cudaStream_t s);
int soft_blocks(int64_t n_tuples);  // CTAs of the soft tuple kernel (sizes the workspace)

// launchers (ko_kernels.cu); return cudaSuccess or the launch error
cudaError_t launch_prep(const PrepParams& p, cudaStream_t s);
// per-translation-unit instantiations of the scoring kernel (ko_score_d128.cu, ko_score_d64.cu)
cudaError_t launch_score_d128(const ScoreParams& p, int CPR, int NT, int64_t max_units, cudaStream_t s);
cudaError_t launch_score_d64(const ScoreParams& p, int CPR, int NT, int64_t max_units, cudaStream_t s);
// grid-mode tuple finaliser after launch_score (fin_kernel = 1): margins, every plan, counts
cudaError_t launch_grid_final(const ScoreParams& p, int CPR, cudaStream_t s);
// scoring kernel with NT table-packed W·V tiles; CPR = class stride of the grid-mode partials
cudaError_t launch_score(const ScoreParams& p, int head_dim, int CPR, int NT, int64_t max_units,
                         cudaStream_t s);
// routed round finaliser (margins, plan walk, counts, queueing) after a walk-mode launch_score
cudaError_t launch_walk(const ScoreParams& p, cudaStream_t s);
cudaError_t launch_route_reach(const RouteParams& p, cudaStream_t s);  // build worklist for stage
cudaError_t launch_route_apply(const RouteParams& p, cudaStream_t s);  // apply stage on margins
cudaError_t launch_route_plan(const RouteParams& p, cudaStream_t s);   // whole plan on margins
cudaError_t launch_route_init(uint32_t* state, int64_t n, cudaStream_t s);
cudaError_t launch_final_counts(const RouteParams& p, cudaStream_t s);  // TP/FP/FN from state
// longest-first order of a work list (tuple ids, or 0..n−1 when work is NULL) into perm:
// hist = workspace [4097] ints; 3 kernels (+ a memset)
cudaError_t launch_lpt_order(const int32_t* work, int64_t n_work, const int32_t* seq_len,
                             int* hist, int32_t* perm, cudaStream_t s);
cudaError_t launch_reduce(const ReduceParams& p, cudaStream_t s);
cudaError_t launch_fill_f32(float* p, float v, int64_t n, cudaStream_t s);

}  // namespace ko
