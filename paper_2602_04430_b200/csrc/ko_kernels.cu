// ko_kernels.cu — the sm_100a kernels around the scoring kernel (which lives in ko_score.cuh):
// Q/W fragment preparation, routing / reduction on precomputed margins (ko_route,
// ko_reduce_stats), the routed round finaliser (ko_walk_kernel), the embedding-similarity stage
// (ko_embed_scores) and their launchers.
#include "ko_device.cuh"

namespace ko {
namespace {
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack2(uint16_t lo, uint16_t hi) {
  return (uint32_t)lo | ((uint32_t)hi << 16);
}

__global__ void prep_kernel(const __grid_constant__ PrepParams p) {
  if (blockIdx.x == 0 && p.gplans)
    for (int i = threadIdx.x; i < p.n_plans * (int)(sizeof(ko_plan) / 4); i += blockDim.x)
      reinterpret_cast<uint32_t*>(p.gplans)[i] = reinterpret_cast<const uint32_t*>(p.plans)[i];
  const int KS = p.head_dim / 16;
  const int NT = p.tbl_nt;
  const int Hq = p.n_kv_heads * p.gqa;
  const int n_lh = p.n_l * p.n_kv_heads;
  const int64_t nq_items = (int64_t)n_lh * KS * 32;
  const int64_t nw_items = (int64_t)n_lh * NT * KS * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq_items + nw_items;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool isq = i < nq_items;
    int64_t r = isq ? i : i - nq_items;
    const int lane = (int)(r % 32); r /= 32;
    const int ks = (int)(r % KS); r /= KS;
    int tt = 0;
    if (!isq) { tt = (int)(r % NT); r /= NT; }
    const int lh = (int)r;
    const int l = lh / p.n_kv_heads, h = lh % p.n_kv_heads;
    const int g = lane >> 2, q = lane & 3;
    const int j = ks >> 1, e = ks & 1;
    const int d0 = 64 * (j >> 1) + 16 * q + 8 * (j & 1) + 4 * e;  // see frag_off in the kernel
    uint16_t vals[2][4];  // [row half 0/1 (A rows g / g+8)][d0..d0+3]
    if (isq) {
      for (int hr = 0; hr < 2; ++hr) {
        const int rho = hr * 8 + g;
        for (int k = 0; k < 4; ++k) {
          uint16_t b = 0;
          if (p.slot_op[rho] >= 0) {
            const int o = p.slot_op[rho], rem = p.slot_rem[rho];
            const int jj = h * p.gqa + rem / p.n_q, nq = rem % p.n_q;
            b = p.q[o][(((size_t)l * Hq + jj) * p.n_q + nq) * p.head_dim + d0 + k];
          }
          vals[hr][k] = b;
        }
      }
    } else {
      // table packing: A-row half hr of tile tt at lane group g = slot 2·tt + hr of the table
      for (int hr = 0; hr < 2; ++hr) {
        const int ent = p.tbl_w[g][2 * tt + hr];
        for (int k = 0; k < 4; ++k) {
          uint16_t b = 0;
          if (ent >= 0) {
            const int o = ent & 7, rem = (ent >> 3) & 31, c = (ent >> 8) & 15, lo = (ent >> 12) & 1;
            const int jj = h * p.gqa + rem / p.n_q, nq = rem % p.n_q;
            const size_t wi = ((((size_t)c * p.n_layers + l) * Hq + jj) * p.n_q + nq) * p.head_dim + d0 + k;
            if (p.w_bf16[o]) {
              b = lo ? 0 : p.w_bf16[o][wi];
            } else {
              const float w = p.w[o][wi];
              const __nv_bfloat16 hi = __float2bfloat16_rn(w);
              b = __bfloat16_as_ushort(lo ? __float2bfloat16_rn(w - __bfloat162float(hi)) : hi);
            }
          }
          vals[hr][k] = b;
        }
      }
    }
    uint4 out;
    out.x = pack2(vals[0][0], vals[0][1]);
    out.y = pack2(vals[1][0], vals[1][1]);
    out.z = pack2(vals[0][2], vals[0][3]);
    out.w = pack2(vals[1][2], vals[1][3]);
    if (isq) p.qfrag[((int64_t)lh * KS + ks) * 32 + lane] = out;
    else p.wfrag[(((int64_t)lh * NT + tt) * KS + ks) * 32 + lane] = out;
  }
}

// ------------------------------------------------------------------------------------------
// Routing / reduction kernels on precomputed margins (ko_route, ko_reduce_stats, and the staged
// executor of ko_score_batch's routed mode).
// ------------------------------------------------------------------------------------------
__global__ void route_init_kernel(uint32_t* state, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    state[i] = 1u;
}

// warp-aggregated append of tuple t (if pred) to the worklist
__device__ __forceinline__ void append(bool pred, int32_t t, int32_t* wl, unsigned long long* len) {
  const unsigned mask = __ballot_sync(0xffffffffu, pred);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(len, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
  if (pred) wl[base + __popc(mask & ((1u << lane) - 1))] = t;
}

// tuples reaching stage p.stage (alive ∧ op pending) → worklist
__global__ void route_reach_kernel(const __grid_constant__ RouteParams p) {
  const int64_t n = p.subset ? p.n_subset : p.n_tuples;
  const int64_t n_round = (n + 31) & ~31ll;
  const bool have = p.stage >= 0 && p.stage < p.plan.n_stages;
  const int o = have ? p.plan.stage[p.stage].op : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_round;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool pred = false;
    int32_t t = 0;
    if (i < n && have) {
      t = p.subset ? p.subset[i] : (int32_t)i;
      const uint32_t st = p.tuple_state[t];
      pred = (st & 1u) && op_status(st, o) == 0;
    }
    append(pred, t, p.worklist, p.worklist_len);
  }
}

// apply stage p.stage's decision (margins precomputed) to every tuple reaching it
__global__ void route_apply_kernel(const __grid_constant__ RouteParams p) {
  __shared__ int s_cnt[kCountsPerPlan];
  for (int i = threadIdx.x; i < kCountsPerPlan; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const ko_stage& st = p.plan.stage[p.stage];
  const int o = st.op;
  int* cnt = s_cnt + 5 + 4 * p.stage;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < p.n_tuples;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t state = p.tuple_state[t];
    if (!(state & 1u) || op_status(state, o) != 0) continue;
    const size_t idx = ((size_t)o * p.n_variants + st.variant) * p.n_tuples + t;
    const int d = decide(p.margins[idx], st, p.n_classes[o]);
    atomicAdd(&cnt[0], 1);
    if (d == D_ACCEPT || d == D_RESOLVED) {
      state |= 1u << (1 + 2 * o);
      if (d == D_RESOLVED) state |= ((uint32_t)p.classes[idx] & 15u) << (16 + 4 * o);
      atomicAdd(&cnt[1], 1);
    } else if (d == D_REJECT) {
      state = (state & ~1u) | (2u << (1 + 2 * o));
      atomicAdd(&cnt[2], 1);
    } else {
      atomicAdd(&cnt[3], 1);
    }
    p.tuple_state[t] = state;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4; i += blockDim.x)
    if (cnt[i]) atomicAdd(&p.counts[5 + 4 * p.stage + i], (unsigned long long)cnt[i]);
}

// whole plan on precomputed margins: final state, P_o worklist, full count row
__global__ void route_plan_kernel(const __grid_constant__ RouteParams p) {
  __shared__ int s_cnt[kCountsPerPlan];
  for (int i = threadIdx.x; i < kCountsPerPlan; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int64_t n_round = (p.n_tuples + 31) & ~31ll;  // whole warps reach the ballot in append()
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_round;
       t += (int64_t)gridDim.x * blockDim.x) {
    bool alive = false;
    if (t < p.n_tuples) {
      float ms[kMaxOps * kMaxVar];
      int32_t cs[kMaxOps * kMaxVar];
      for (int s = 0; s < p.plan.n_stages; ++s) {
        const int idx = p.plan.stage[s].op * p.n_variants + p.plan.stage[s].variant;
        const size_t gi = (size_t)idx * p.n_tuples + t;
        ms[idx] = p.margins[gi];
        cs[idx] = p.classes ? p.classes[gi] : 0;
      }
      const uint32_t st = eval_plan(p.plan, ms, cs, p.n_variants, p.n_classes, p.gold, p.n_tuples,
                                    t, s_cnt);
      if (p.tuple_state) p.tuple_state[t] = st;
      alive = st & 1u;
    }
    if (p.worklist) append(alive, (int32_t)t, p.worklist, p.worklist_len);
  }
  flush_counts(s_cnt, 1, p.counts, p.gold != nullptr);
}

// TP/FP/FN/|P_o|/|P_g| from the final tuple states of a routed execution
__global__ void final_counts_kernel(const __grid_constant__ RouteParams p) {
  __shared__ int s_cnt[kCountsPerPlan];
  for (int i = threadIdx.x; i < kCountsPerPlan; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  uint32_t referenced = 0;
  for (int s = 0; s < p.plan.n_stages; ++s) referenced |= 1u << p.plan.stage[s].op;
  const int64_t n = p.subset ? p.n_subset : p.n_tuples;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = p.subset ? p.subset[i] : i;
    const uint32_t st = p.tuple_state[t];
    const bool in_out = st & 1u;
    bool in_gold = p.gold != nullptr, maps_ok = true;
    if (p.gold) {
      for (int o = 0; o < kMaxOps; ++o) {
        if (!(referenced & (1u << o))) continue;
        const uint8_t gv = p.gold[(int64_t)o * p.n_tuples + t];
        if (p.n_classes[o] <= 1) {
          if (gv != 1) in_gold = false;
        } else if (((st >> (16 + 4 * o)) & 15u) != gv || op_status(st, o) != 1) {
          maps_ok = false;
        }
      }
    }
    if (in_out) atomicAdd(&s_cnt[KO_C_OUT], 1);
    if (in_gold) atomicAdd(&s_cnt[KO_C_GOLD], 1);
    if (in_out && in_gold && maps_ok) atomicAdd(&s_cnt[KO_C_TP], 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 5; k += blockDim.x) {
    long long v = s_cnt[k];
    if (k == KO_C_FP) v = p.gold ? (long long)s_cnt[KO_C_OUT] - s_cnt[KO_C_TP] : 0;
    if (k == KO_C_FN) v = p.gold ? (long long)s_cnt[KO_C_GOLD] - s_cnt[KO_C_TP] : 0;
    if (v) atomicAdd(&p.counts[k], (unsigned long long)v);
  }
}

// G-plan grid on precomputed margins: one warp per tuple, one lane per plan
// ko_reduce_stats: warp per tuple, lane per plan.  Latency-bound per warp (margin loads, then the
// plan walks), so CTAs are 32 warps wide: many tuples in flight per SM, while the per-CTA count
// flush (one global atomic per counter) stays at 2 CTAs per SM.
constexpr int kReduceThreads = 512;
__global__ void __launch_bounds__(kReduceThreads, 2) reduce_kernel(const __grid_constant__ ReduceParams p) {
  __shared__ int s_cnt[kMaxPlans * kCountsPerPlan];
  __shared__ ko_plan s_plans[kMaxPlans];  // lanes read different plans: smem, not the param bank
  for (int i = threadIdx.x; i < p.n_plans * (int)(sizeof(ko_plan) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s_plans)[i] = reinterpret_cast<const uint32_t*>(p.plans)[i];
  __shared__ float s_m[kReduceThreads / 32][kMaxOps * kMaxVar];
  __shared__ int32_t s_c[kReduceThreads / 32][kMaxOps * kMaxVar];
  for (int i = threadIdx.x; i < p.n_plans * kCountsPerPlan; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  __shared__ uint8_t s_g[kReduceThreads / 32][kMaxOps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int nmv = p.n_ops * p.n_variants;  // ≤ 32: one (op, variant) entry per lane
  const int64_t stride = (int64_t)gridDim.x * nw;
  // the next tuple's margins / classes / gold bytes are loaded while this one's plans run
  auto fetch = [&](int64_t t, float& m, int32_t& c, uint8_t& gv) {
    m = 0.f; c = 0; gv = 0;
    if (t >= p.n_tuples) return;
    if (lane < nmv) {
      m = p.margins[(size_t)lane * p.n_tuples + t];
      c = p.classes ? p.classes[(size_t)lane * p.n_tuples + t] : 0;
    }
    if (p.gold && lane < p.n_ops) gv = p.gold[(size_t)lane * p.n_tuples + t];
  };
  float nm;
  int32_t nc;
  uint8_t ng;
  int64_t t = (int64_t)blockIdx.x * nw + w;
  fetch(t, nm, nc, ng);
  for (; t < p.n_tuples; t += stride) {
    if (lane < nmv) { s_m[w][lane] = nm; s_c[w][lane] = nc; }
    if (lane < kMaxOps) s_g[w][lane] = ng;
    __syncwarp();
    fetch(t + stride, nm, nc, ng);
    // gold bytes from shared memory: [op][1] with n_tuples = 1, tuple 0
    for (int gp = lane; gp < p.n_plans; gp += 32)
      eval_plan(s_plans[gp], s_m[w], s_c[w], p.n_variants, p.n_classes,
                p.gold ? s_g[w] : nullptr, 1, 0, s_cnt + gp * kCountsPerPlan);
    __syncwarp();
  }
  flush_counts(s_cnt, p.n_plans, p.counts, p.gold != nullptr);
}

// Routed round finaliser (after each walk-mode scoring launch): ONE THREAD PER TUPLE of the round
// walks the plan from where the tuple stopped (Eqs. accept-i/reject-i/unsure-i, P:323-327;
// inter-op reach P:536-539), deciding every reached stage whose margin is available — computed on
// demand from the per-tuple partial logits (z_c = b_c + Σ_u partial, fp64, u ascending: the grid
// finaliser's arithmetic) and written out, since only reached entries are outputs (§8(b)) — and
// stops at the first stage whose margin is not yet available, queueing the tuple for the first
// LATER plan position that computes it.  Per-stage counts: shared-memory atomics flushed once per
// CTA; queue appends are warp-aggregated.
__device__ __forceinline__ float walk_margin(const ScoreParams& p, int64_t t, int o, int v,
                                             int32_t* cls_out) {
  const int CPR = p.part_cpr;  // one class stride for every group's partials
  const int PB = walk_part_blk(p.n_ops_total, CPR);
  const int nzg = PB;  // floats per (tuple, variant, layer·kv-head) block
  const int nu = min(p.cut[p.var_local[v]], p.n_layers) * p.n_kv_heads;  // l-major units
  const float* src =
      p.part + ((size_t)t * p.n_var_total + v) * p.n_lh_all * PB + (size_t)o * CPR;
  const int C = p.op_classes_g[o];
  float best = -CUDART_INF_F, second = -CUDART_INF_F;
  int bi = 0;
  for (int c = 0; c < C; ++c) {
    double acc = 0.0;
    int u = 0;
    for (; u + 4 <= nu; u += 4) {
      const float a0 = __ldcg(src + (size_t)(u + 0) * nzg + c), a1 = __ldcg(src + (size_t)(u + 1) * nzg + c);
      const float a2 = __ldcg(src + (size_t)(u + 2) * nzg + c), a3 = __ldcg(src + (size_t)(u + 3) * nzg + c);
      acc += (double)a0; acc += (double)a1; acc += (double)a2; acc += (double)a3;
    }
    for (; u < nu; ++u) acc += (double)__ldcg(src + (size_t)u * nzg + c);
    const float z = (float)((double)__ldg(p.bias_g[o] + c) + acc);
    if (C <= 1) {
      *cls_out = 0;
      return z;
    }
    if (z > best) {  // lowest class index on ties
      second = best;
      best = z;
      bi = c;
    } else if (z > second) {
      second = z;
    }
  }
  *cls_out = bi;
  return best - second;
}

constexpr int kWalkThreads = 256;
__global__ void __launch_bounds__(kWalkThreads) ko_walk_kernel(const __grid_constant__ ScoreParams p) {
  __shared__ int s_cnt[4 * KO_MAX_STAGES];
  for (int i = threadIdx.x; i < 4 * KO_MAX_STAGES; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t n_work = p.work_len_dev ? *p.work_len_dev : p.work_len_host;
  const ko_plan& P = p.plans[0];
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n_work;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = base + threadIdx.x;
    int qdest = -1;
    int64_t t = 0;
    if (w < n_work) {
      t = p.work ? (int64_t)p.work[w] : w;
      if (p.pos == 0 && p.margins) {
        // this call's tuples start with NaN KV-variant margins (only reached entries are
        // written, §8(b)); tuples outside the call's tuple_idx are not touched
        for (int o = 0; o < p.n_ops_total; ++o)
          for (int v = 0; v < p.n_var_total; ++v)
            if (p.var_rank[v] >= 0)
              p.margins[((size_t)o * p.n_var_total + v) * p.n_tuples + t] = CUDART_NAN_F;
      }
      uint32_t state = p.pos == 0 ? 1u : __ldcg(p.tuple_state + t);
      uint32_t done = p.pos == 0 ? 0xFFFFFFFFu : __ldcg(p.tuple_done + t);  // 4-bit round+1 per group
      if (p.group >= 0) {  // −1: a walk-only launch (external stage at position 0) computed nothing
        const uint32_t cur = (done >> (4 * p.group)) & 15u;
        const uint32_t mine = (uint32_t)p.round + 1u;
        if (cur == 15u || cur < mine) done = (done & ~(15u << (4 * p.group))) | (mine << (4 * p.group));
      }
      const int s_from = (int)((state >> kWalkStageShift) & 15u);
      int stop = P.n_stages;
      for (int s = s_from; s < P.n_stages; ++s) {
        const ko_stage& st = P.stage[s];
        const int o = st.op;
        if (!(state & 1u) || op_status(state, o) != 0) continue;  // not reached
        const int g = p.group_of_op[o];
        const int rk = p.var_rank[st.variant];
        const uint32_t have = (done >> (4 * g)) & 15u;      // 15: never computed
        if (rk >= 0 && (have == 15u || (int)have - 1 < rk)) {  // rk < 0: external, always there
          // the next position computing (g, ≥ rk) exists: stage s itself is one (s > pos)
          int q = p.pos + 1;
          while (q < p.n_pos && !(p.pos_group[q] == g && p.pos_round[q] >= rk)) ++q;
          if (q < p.n_pos) qdest = q;
          stop = s;
          break;
        }
        const size_t oi = ((size_t)o * p.n_var_total + st.variant) * p.n_tuples + t;
        float m;
        int32_t cls = 0;
        if (rk < 0) {                 // external variant: the caller's margin (filters only)
          m = __ldcg(p.margins + oi);
        } else {
          m = walk_margin(p, t, o, st.variant, &cls);
          if (p.margins) p.margins[oi] = m;
          if (p.classes) p.classes[oi] = cls;
        }
        const int d = decide(m, st, p.op_classes_g[o]);
        int k = 3;  // [n_in, n_acc, n_rej, n_uns] of stage s
        if (d == D_ACCEPT || d == D_RESOLVED) {
          state |= 1u << (1 + 2 * o);
          if (d == D_RESOLVED) state |= ((uint32_t)cls & 15u) << (16 + 4 * o);
          k = 1;
        } else if (d == D_REJECT) {
          state = (state & ~1u) | (2u << (1 + 2 * o));
          k = 2;
        }
        atomicAdd(&s_cnt[4 * s], 1);
        atomicAdd(&s_cnt[4 * s + k], 1);
      }
      p.tuple_state[t] = (state & ~(15u << kWalkStageShift)) | ((uint32_t)stop << kWalkStageShift);
      p.tuple_done[t] = done;
    }
    // warp-aggregated queue appends: lanes with the same destination share one atomic
    const unsigned act = __ballot_sync(0xffffffffu, qdest >= 0);
    if (qdest >= 0) {
      const unsigned same = __match_any_sync(act, qdest);
      const int leader = __ffs(same) - 1;
      unsigned long long at = 0;
      if (lane == leader) at = atomicAdd(p.wl_len[qdest], (unsigned long long)__popc(same));
      at = __shfl_sync(same, at, leader);
      p.wl[qdest][at + __popc(same & ((1u << lane) - 1u))] = (int32_t)t;
    }
  }
  // per-stage counts: shared-memory atomics per CTA, one global atomic per counter per CTA
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * KO_MAX_STAGES; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&p.counts[5 + i], (unsigned long long)s_cnt[i]);
}


// ------------------------------------------------------------------------------------------
// Embedding-similarity filter stage (Blip): cosine of each item
// embedding with each operator embedding.  One warp per tuple, 16-byte loads, fp32 accumulate;
// HBM-bound GEMV (the operator embeddings live in shared memory).
// ------------------------------------------------------------------------------------------
// Each lane owns 8 consecutive dims of every 256-dim chunk; the operator embeddings of its dims
// stay in registers, 4 tuples are in flight per warp, and one xor-tree per tuple and output
// finishes the dot products.
template <int CH>  // 256-dim chunks per embedding (dim ≤ 256·CH)
__global__ void __launch_bounds__(256) embed_kernel(const __grid_constant__ EmbedParams p) {
  const int lane = threadIdx.x & 31;
  const int dim = p.dim;
  float qv[KO_MAX_OPS][CH][8];
  float qn[KO_MAX_OPS];
#pragma unroll
  for (int o = 0; o < KO_MAX_OPS; ++o) {
    float acc = 0.f;
#pragma unroll
    for (int ch = 0; ch < CH; ++ch)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int d = ch * 256 + lane * 8 + k;
        const float x = (o < p.n_e && d < dim)
                            ? __bfloat162float(__ushort_as_bfloat16(p.op_emb[(size_t)o * dim + d]))
                            : 0.f;
        qv[o][ch][k] = x;
        acc = fmaf(x, x, acc);
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    qn[o] = sqrtf(acc);
  }
  constexpr int TB = 4;  // tuples per warp iteration
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n = p.tuple_idx ? p.n_idx : p.n_tuples;
  for (int64_t w0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * TB; w0 < n;
       w0 += nw * TB) {
    uint4 v[TB][CH];
    int64_t tt[TB];
#pragma unroll
    for (int b = 0; b < TB; ++b) {
      const int64_t w = w0 + b;
      tt[b] = w < n ? (p.tuple_idx ? (int64_t)p.tuple_idx[w] : w) : -1;
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        const int d0 = ch * 256 + lane * 8;
        v[b][ch] = (tt[b] >= 0 && d0 < dim)
                       ? __ldg(reinterpret_cast<const uint4*>(p.item_emb + (size_t)tt[b] * dim + d0))
                       : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int b = 0; b < TB; ++b) {
      float dot[KO_MAX_OPS] = {0.f, 0.f, 0.f, 0.f};
      float nn = 0.f;
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        const uint32_t wv[4] = {v[b][ch].x, v[b][ch].y, v[b][ch].z, v[b][ch].w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float x = __uint_as_float(k & 1 ? wv[k >> 1] & 0xFFFF0000u : wv[k >> 1] << 16);
          nn = fmaf(x, x, nn);
#pragma unroll
          for (int o = 0; o < KO_MAX_OPS; ++o) dot[o] = fmaf(x, qv[o][ch][k], dot[o]);
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        nn += __shfl_xor_sync(0xffffffffu, nn, off);
#pragma unroll
        for (int o = 0; o < KO_MAX_OPS; ++o)
          if (o < p.n_e) dot[o] += __shfl_xor_sync(0xffffffffu, dot[o], off);
      }
      if (tt[b] >= 0 && lane < p.n_e) {
        float d = dot[0], qq = qn[0];
#pragma unroll
        for (int o = 1; o < KO_MAX_OPS; ++o)
          if (lane == o) { d = dot[o]; qq = qn[o]; }
        const float den = sqrtf(nn) * qq;
        p.margins[((size_t)p.op_ids[lane] * p.n_variants + p.variant) * p.n_tuples + tt[b]] =
            den > 0.f ? __fdiv_rn(d, den) : 0.f;
      }
    }
  }
}

// Tensor-core path (dim a multiple of 16, ≤ 512): per warp a 3-stage shared-memory ring of
// 16-tuple blocks, each item row brought in by its own 1-D bulk copy (cp.async.bulk, one lane per
// row, tuple_idx gathers for free) into a row padded by 16 B so ldmatrix is conflict-free.  Per
// k-step of 16 dims one ldmatrix.x4 gives the A fragment X[16 tuples × 16 dims]; then
//   D = X · Qᵀ  (B = the ≤ 4 operator embeddings, fragments in registers)   — the dot products,
//   G = X · Xᵀ  (B = the A fragment itself: rows 0-7 = {a0, a2}, rows 8-15 = {a1, a3})
// whose diagonal holds the squared norms; fp32 accumulation (mma.sync m16n8k16 bf16).  The
// epilogue takes the diagonal (lane (g, g/2) holds ‖x_g‖² and ‖x_{g+8}‖²) and writes the cosines.
#ifndef KO_EMB_STAGES
#define KO_EMB_STAGES 3
#endif
constexpr int kEmbWarps = 4, kEmbStages = KO_EMB_STAGES, kEmbRows = 16;
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816b(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                          uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
               "{%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// KSM: k-steps of 16 dims (dim ≤ 16·KSM).  TM: tensor-map loads into 128B-swizzled 16-row boxes —
// contiguous rows as 64 × 16 boxes, or (G4) gathered rows (tuple_idx) with the sm_100 TMA row
// gather `tile::gather4`: one op brings 4 arbitrary rows × 64 dims, so a 16-row block at dim 256
// is 16 TMA ops instead of 512 per-lane cp.async copies, and the swizzled layout is the same as the
// contiguous path's.  !TM: per-lane cp.async copies into padded rows (fallback).
template <int KSM, bool TM, bool G4 = false>
__global__ void __launch_bounds__(kEmbWarps * 32) embed_mma_kernel(const __grid_constant__ EmbedParams p) {
  extern __shared__ __align__(128) uint8_t emb_sm[];
  __shared__ __align__(8) uint64_t bar[kEmbWarps][kEmbStages];
  __shared__ int32_t s_tl[kEmbWarps][kEmbStages][kEmbRows];  // G4: the stage's tuple ids
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int dim = p.dim, KS = dim / 16;
  // row layout of a stage: TM — NB boxes of 16 rows × 128 B (64 dims), 128B-swizzled; else rows
  // padded to dim·2 + 16 bytes (each row its own bulk copy)
  const int NB = (dim + 63) / 64;
  const int RS = dim * 2 + 16;                        // padded row stride (bytes), !TM
  const int SB = TM ? NB * kEmbRows * 128 : kEmbRows * RS;  // stage bytes
  uint8_t* base = TM ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(emb_sm) + 1023) &
                                                  ~static_cast<uintptr_t>(1023))  // swizzle atom
                     : emb_sm;
  uint8_t* ring = base + (size_t)warp * kEmbStages * SB;
  const uint32_t ring_s = smem_u32(ring);
  if (lane == 0) {  // TM: one arrival (lane 0's expect_tx) + bytes; gathers: one per lane
    for (int s = 0; s < kEmbStages; ++s) mbar_init(&bar[warp][s], TM ? 1 : 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // operator embeddings as B fragments: lane (g, q) holds op g's dims 16·ks + {2q, 2q+1} and
  // 16·ks + 8 + {2q, 2q+1} (zero for g ≥ n_e); and each op's norm
  uint32_t bq[KSM][2];
#pragma unroll
  for (int ks = 0; ks < KSM; ++ks) {
    bq[ks][0] = bq[ks][1] = 0u;
    if (ks < KS && g < p.n_e) {
      const uint16_t* e = p.op_emb + (size_t)g * dim + 16 * ks + 2 * q;
      bq[ks][0] = (uint32_t)e[0] | ((uint32_t)e[1] << 16);
      bq[ks][1] = (uint32_t)e[8] | ((uint32_t)e[9] << 16);
    }
  }
  float qn[KO_MAX_OPS];
#pragma unroll
  for (int o = 0; o < KO_MAX_OPS; ++o) {
    float acc = 0.f;
    if (o < p.n_e)
      for (int d = lane; d < dim; d += 32) {
        const float x = __bfloat162float(__ushort_as_bfloat16(p.op_emb[(size_t)o * dim + d]));
        acc = fmaf(x, x, acc);
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    qn[o] = sqrtf(acc);
  }
  // this lane's outputs: ops 2q and 2q + 1 (C fragment columns) — row pointer and 1/‖q‖
  float* out[2];
  float rq[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int o = 2 * q + e;
    float qo = qn[0];
#pragma unroll
    for (int o2 = 1; o2 < KO_MAX_OPS; ++o2)
      if (o == o2) qo = qn[o2];
    out[e] = o < p.n_e ? p.margins + ((size_t)p.op_ids[o] * p.n_variants + p.variant) * p.n_tuples
                       : nullptr;
    rq[e] = qo > 0.f ? 1.f / qo : 0.f;
  }
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

  const int64_t n = p.tuple_idx ? p.n_idx : p.n_tuples;
  const int64_t n_blk = (n + kEmbRows - 1) / kEmbRows;
  const int64_t nw = (int64_t)gridDim.x * kEmbWarps;
  int64_t next = (int64_t)blockIdx.x * kEmbWarps + warp;  // next block to issue
  uint32_t issued = 0, consumed = 0;
  const uint32_t row_bytes = (uint32_t)dim * 2;
  // gathers: lane r's tuple of the NEXT block to issue, loaded one issue ahead so the index
  // lookup is off the copy's critical path
  // (kept as the loaded int32: widening it at the load would wait for the load right there)
  auto load_tl = [&]() -> int32_t {
    const int64_t w = next * kEmbRows + lane;
    return ((!TM || G4) && next < n_blk && w < n) ? p.tuple_idx[w] : 0;
  };
  int32_t tl_next = load_tl();
  auto issue = [&]() {
    const int slot = issued % kEmbStages;
    const int64_t w0 = next * kEmbRows;
    const int rows = (int)(n - w0 < kEmbRows ? n - w0 : kEmbRows);
    if constexpr (TM && G4) {
      // 4 row groups × NB column boxes of gather4 (4 rows × 64 dims = 512 B each, at stage offset
      // box·2048 + group·512, i.e. where a 16-row box puts those rows); lane j < 4 issues group j.
      // Rows past the end of the list repeat the block's first tuple (loaded, never written out).
      int32_t tl = tl_next;
      const int32_t t0 = __shfl_sync(0xffffffffu, tl, 0);
      if (lane >= rows) tl = t0;
      if (lane < kEmbRows) s_tl[warp][slot][lane] = tl;
      int32_t r4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) r4[i] = __shfl_sync(0xffffffffu, tl, (4 * lane + i) & 31);
      if (lane == 0) mbar_expect_tx(&bar[warp][slot], (uint32_t)SB);
      __syncwarp();
      if (lane < 4)
        for (int b = 0; b < NB; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(ring_s + slot * SB + b * kEmbRows * 128 + lane * 512),
              "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(64 * b), "r"(r4[0]), "r"(r4[1]), "r"(r4[2]),
              "r"(r4[3]), "r"(smem_u32(&bar[warp][slot])), "l"(policy)
              : "memory");
      ++issued;
      next += nw;
      tl_next = load_tl();
      return;
    } else if constexpr (TM) {  // NB boxes (64 dims × 16 rows); out-of-range rows / dims are zero-filled
      if (lane == 0) {
        mbar_expect_tx(&bar[warp][slot], (uint32_t)SB);
        for (int b = 0; b < NB; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(ring_s + slot * SB + b * kEmbRows * 128),
              "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(64 * b), "r"((int)w0),
              "r"(smem_u32(&bar[warp][slot])), "l"(policy)
              : "memory");
      }
      ++issued;
      next += nw;
      return;
    }
    // gathered rows: every lane copies 16-byte chunks (cp.async) of the block's rows into the
    // padded stage, then arrives on the stage's mbarrier when its copies land (.noinc: the
    // barrier was initialised with one pending arrival per lane)
    const int cpr = (int)(row_bytes >> 4);  // 16-byte chunks per row (≤ 64)
    const int32_t tl = tl_next;
    for (int r = 0; r < rows; ++r) {  // row r: lanes copy chunks lane, lane + 32
      const uint32_t t = (uint32_t)__shfl_sync(0xffffffffu, tl, r);
      const uint16_t* src = p.item_emb + (size_t)t * dim;
      const uint32_t dst = ring_s + slot * SB + r * RS;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int k = lane + 32 * j;
        if (k < cpr)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * k), "l"(src + 8 * k)
                       : "memory");
      }
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar[warp][slot]))
                 : "memory");
    ++issued;
    next += nw;
    tl_next = load_tl();
  };
  for (int k = 0; k < kEmbStages && next < n_blk; ++k) issue();
  // ldmatrix row address of this lane inside a stage: matrix (lane / 8) = (rows +8·(m&1),
  // dims +8·(m>>1)); row (lane & 7)
  const uint32_t lrow = (uint32_t)((lane & 7) + 8 * ((lane >> 3) & 1)) * RS + 16 * (lane >> 4);
  for (int64_t blk = (int64_t)blockIdx.x * kEmbWarps + warp; blk < n_blk; blk += nw) {
    const int slot = consumed % kEmbStages;
    // output tuples of rows g, g + 8 (gathers: loaded before the wait, off the epilogue's path)
    const int64_t w0 = blk * kEmbRows;
    int32_t tout[2];  // int32 until used (see load_tl)
    if constexpr (G4) {  // the ids the issue staged in shared memory (no global load here)
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) tout[hr] = s_tl[warp][slot][g + 8 * hr];
    } else {
#pragma unroll
      for (int hr = 0; hr < 2; ++hr)
        tout[hr] = w0 + g + 8 * hr < n ? (p.tuple_idx ? p.tuple_idx[w0 + g + 8 * hr] : (int32_t)0) : 0;
    }
    mbar_wait(&bar[warp][slot], (consumed / kEmbStages) & 1u);
    const uint32_t st = ring_s + slot * SB + (TM ? 0u : lrow);
    auto ldsm_ks = [&](uint32_t (&a)[4], int ks) {
      if constexpr (TM) {
        // box ks/4, 16-byte chunk 2·(ks%4) + (matrix ≥ 2), XORed with the row (128B swizzle)
        const int r = (lane & 7) + 8 * ((lane >> 3) & 1);
        const int c = 2 * (ks & 3) + (lane >> 4);
        ldsm_x4(a, st + (ks >> 2) * (kEmbRows * 128) + r * 128 + ((c ^ (r & 7)) << 4));
      } else {
        ldsm_x4(a, st + 32 * ks);
      }
    };
    // two accumulator sets (even / odd k-steps) halve the MMA dependency chains
    float dd[2][4] = {}, g0[2][4] = {}, g1[2][4] = {};
    if constexpr (KSM <= 16 && (G4 || !TM)) {
      // gathered rows: the whole block's A fragments into registers first, so the stage goes
      // back to the copy engine before the MMAs and the ring keeps more bytes in flight per SM
      // (F = 0.5: 5.1 → 6.0 TB/s; the contiguous path ran 6.38 → 6.08 with it, so it keeps the
      // interleaved order)
      uint32_t af[KSM][4];
#pragma unroll
      for (int ks = 0; ks < KSM; ++ks)
        if (ks < KS) ldsm_ks(af[ks], ks);
      __syncwarp();
      ++consumed;
      if (next < n_blk) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue();
      }
#pragma unroll
      for (int ks = 0; ks < KSM; ++ks) {
        if (ks < KS) {
          mma16816b(dd[ks & 1], af[ks], bq[ks][0], bq[ks][1]);
          mma16816b(g0[ks & 1], af[ks], af[ks][0], af[ks][2]);
          mma16816b(g1[ks & 1], af[ks], af[ks][1], af[ks][3]);
        }
      }
    } else {
#pragma unroll
      for (int ks = 0; ks < KSM; ++ks) {
        if (ks < KS) {
          uint32_t a[4];
          ldsm_ks(a, ks);
          mma16816b(dd[ks & 1], a, bq[ks][0], bq[ks][1]);
          mma16816b(g0[ks & 1], a, a[0], a[2]);
          mma16816b(g1[ks & 1], a, a[1], a[3]);
        }
      }
      __syncwarp();
      ++consumed;
      if (next < n_blk) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue();
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dd[0][i] += dd[1][i];
      g0[0][i] += g0[1][i];
      g1[0][i] += g1[1][i];
    }
    // squared norms of tuples g and g + 8 sit in lane (g, g/2): G0[g][g], G1[g + 8][g + 8]
    const float gsel0 = (g & 1) ? g0[0][1] : g0[0][0];
    const float gsel1 = (g & 1) ? g1[0][3] : g1[0][2];
    const float n0 = __shfl_sync(0xffffffffu, gsel0, 4 * g + (g >> 1));
    const float n1 = __shfl_sync(0xffffffffu, gsel1, 4 * g + (g >> 1));
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int64_t w = w0 + g + 8 * hr;
      if (w >= n) continue;
      const int64_t t = p.tuple_idx ? (int64_t)(uint32_t)tout[hr] : w;
      const float n2 = hr ? n1 : n0;
      const float rn = n2 > 0.f ? rsqrtf(n2) : 0.f;  // 1/‖x‖ (≤ 2 ulp); 0 ⇒ cosine 0
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (out[e]) out[e][t] = dd[0][2 * hr + e] * rn * rq[e];
    }
  }
}

}  // namespace

cudaError_t launch_embed(const EmbedParams& p, cudaStream_t s) {
  const int64_t n = p.tuple_idx ? p.n_idx : p.n_tuples;
  if (p.dim % 16 == 0 && p.dim <= 512 && ((uintptr_t)p.item_emb & 15) == 0) {
    // tensor-core path: 3-stage ring of padded 16-row blocks per warp
    const int smem = p.use_tmap ? kEmbWarps * kEmbStages * ((p.dim + 63) / 64) * kEmbRows * 128 + 1024
                                : kEmbWarps * kEmbStages * kEmbRows * (p.dim * 2 + 16);
    const int64_t n_blk = (n + kEmbRows - 1) / kEmbRows;
    auto run = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int occ = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kEmbWarps * 32, smem);
      int64_t grid = (int64_t)num_sms() * std::max(occ, 1);
      grid = std::min<int64_t>(grid, (n_blk + kEmbWarps - 1) / kEmbWarps);
      kern<<<(unsigned)std::max<int64_t>(grid, 1), kEmbWarps * 32, smem, s>>>(p);
    };
    if (p.use_tmap && p.tuple_idx) {
      if (p.dim <= 128) run(embed_mma_kernel<8, true, true>);
      else if (p.dim <= 256) run(embed_mma_kernel<16, true, true>);
      else run(embed_mma_kernel<32, true, true>);
    } else if (p.use_tmap) {
      if (p.dim <= 128) run(embed_mma_kernel<8, true>);
      else if (p.dim <= 256) run(embed_mma_kernel<16, true>);
      else run(embed_mma_kernel<32, true>);
    } else {
      if (p.dim <= 128) run(embed_mma_kernel<8, false>);
      else if (p.dim <= 256) run(embed_mma_kernel<16, false>);
      else run(embed_mma_kernel<32, false>);
    }
    return cudaGetLastError();
  }
  int64_t blocks = (n + 31) / 32;  // 8 warps × 4 tuples
  blocks = std::min<int64_t>(blocks, (int64_t)num_sms() * 8);
  if (blocks < 1) blocks = 1;
  const int ch = (p.dim + 255) / 256;
  if (ch <= 1) embed_kernel<1><<<(unsigned)blocks, 256, 0, s>>>(p);
  else if (ch <= 2) embed_kernel<2><<<(unsigned)blocks, 256, 0, s>>>(p);
  else embed_kernel<4><<<(unsigned)blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_prep(const PrepParams& p, cudaStream_t s) {
  prep_kernel<<<num_sms() * 2, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_score(const ScoreParams& p, int head_dim, int CPR, int NT, int64_t max_units,
                         cudaStream_t s) {
  // the instantiations live in ko_score_d128.cu / ko_score_d64.cu
  if (head_dim == 128) return launch_score_d128(p, CPR, NT, max_units, s);
  if (head_dim == 64) return launch_score_d64(p, CPR, NT, max_units, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_walk(const ScoreParams& p, cudaStream_t s) {
  // grid-stride over the round's work list (its length is on the device)
  ko_walk_kernel<<<num_sms() * 4, kWalkThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_route_init(uint32_t* state, int64_t n, cudaStream_t s) {
  route_init_kernel<<<num_sms() * 4, 256, 0, s>>>(state, n);
  return cudaGetLastError();
}
cudaError_t launch_route_reach(const RouteParams& p, cudaStream_t s) {
  route_reach_kernel<<<num_sms() * 4, 256, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_route_apply(const RouteParams& p, cudaStream_t s) {
  route_apply_kernel<<<num_sms() * 4, 256, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_route_plan(const RouteParams& p, cudaStream_t s) {
  route_plan_kernel<<<num_sms() * 4, 256, 0, s>>>(p);
  return cudaGetLastError();
}
// ---- Longest-first work order (grid mode): a counting sort of the work list by streamed pages,
// descending, so the last work units a persistent kernel claims are short ones (the tail of a
// varlen batch is one short unit instead of up to a 4096-token one).  Bucket = min(pages, 4095),
// reversed; warp-aggregated atomics (a fixed-length batch has one bucket).  A batch with a single
// bucket keeps the caller's order (identity), so fixed-length configs are unaffected.
constexpr int kLptBuckets = 4096;
__device__ __forceinline__ int lpt_bucket(const int32_t* seq_len, int64_t t) {
  const int pages = (seq_len[t] + 15) >> 4;
  return kLptBuckets - 1 - min(pages, kLptBuckets - 1);  // longest first
}
__global__ void lpt_hist_kernel(const int32_t* work, int64_t n_work, const int32_t* seq_len,
                                int* hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - threadIdx.x < n_work;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool ok = i < n_work;
    const int b = ok ? lpt_bucket(seq_len, work ? work[i] : i) : -1;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (!ok) continue;
    const unsigned peers = __match_any_sync(act, b);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[b], __popc(peers));
  }
}
// one CTA: exclusive scan of the buckets in place; hist[kLptBuckets] = number of non-empty buckets
__global__ void __launch_bounds__(1024) lpt_scan_kernel(int* hist) {
  __shared__ int s_part[1024];
  __shared__ int s_ne[1024];
  constexpr int per = kLptBuckets / 1024;
  int v[per], sum = 0, ne = 0;
#pragma unroll
  for (int k = 0; k < per; ++k) {
    v[k] = hist[threadIdx.x * per + k];
    sum += v[k];
    ne += v[k] > 0;
  }
  s_part[threadIdx.x] = sum;
  s_ne[threadIdx.x] = ne;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan of the thread sums
    const int a = threadIdx.x >= off ? s_part[threadIdx.x - off] : 0;
    const int c = threadIdx.x >= off ? s_ne[threadIdx.x - off] : 0;
    __syncthreads();
    s_part[threadIdx.x] += a;
    s_ne[threadIdx.x] += c;
    __syncthreads();
  }
  int run = s_part[threadIdx.x] - sum;
#pragma unroll
  for (int k = 0; k < per; ++k) {
    hist[threadIdx.x * per + k] = run;
    run += v[k];
  }
  if (threadIdx.x == 1023) hist[kLptBuckets] = s_ne[1023];
}
__global__ void lpt_scatter_kernel(const int32_t* work, int64_t n_work, const int32_t* seq_len,
                                   int* offs, int32_t* perm) {
  const bool single = offs[kLptBuckets] <= 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - threadIdx.x < n_work;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool ok = i < n_work;
    const int32_t t = ok ? (work ? work[i] : (int32_t)i) : 0;
    if (single) {
      if (ok) perm[i] = t;
      continue;
    }
    const int b = ok ? lpt_bucket(seq_len, t) : -1;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (!ok) continue;
    const unsigned peers = __match_any_sync(act, b);
    const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
    int base = 0;
    if (lane == leader) base = atomicAdd(&offs[b], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    perm[base + __popc(peers & ((1u << lane) - 1))] = t;
  }
}

cudaError_t launch_lpt_order(const int32_t* work, int64_t n_work, const int32_t* seq_len,
                             int* hist, int32_t* perm, cudaStream_t s) {  // 3 launches
  cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(int) * (kLptBuckets + 1), s);
  if (e != cudaSuccess) return e;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n_work + 255) / 256, num_sms() * 4));
  lpt_hist_kernel<<<blocks, 256, 0, s>>>(work, n_work, seq_len, hist);
  lpt_scan_kernel<<<1, 1024, 0, s>>>(hist);
  lpt_scatter_kernel<<<blocks, 256, 0, s>>>(work, n_work, seq_len, hist, perm);
  return cudaGetLastError();
}

cudaError_t launch_final_counts(const RouteParams& p, cudaStream_t s) {
  final_counts_kernel<<<num_sms() * 2, 256, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_reduce(const ReduceParams& p, cudaStream_t s) {
  reduce_kernel<<<num_sms() * 2, kReduceThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ko
