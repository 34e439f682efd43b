// ko_kernels.cu — sm_100a kernels of the KV-cache semantic-operator scoring pass.
//
// Hot kernel: ko_score_kernel<D, CPR0, CPR1>.  One warp owns one work unit = (tuple t, layer l,
// kv-head h) and streams that unit's K and V rows (importance order, page by page) straight from
// HBM with 128-bit non-allocating loads, one page ahead.  Per 16-token page:
//   S = Q · Kᵀ        on tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate): the rows
//                     attending kv-head h (n_ops · gqa · n_q ≤ 16) are the M dimension, the
//                     page's tokens the N dimension, head_dim the K dimension;
//   U = W · Vᵀ        same shape: the readout W of every row/class is folded through V, so the
//                     logit contribution of a row is Σ_i softmax_i · U_i (linearity of
//                     z = b + W·O, DESIGN.md §"Kernel").  W is fp32 and enters as bf16 hi + lo
//                     (rows 0-7 / 8-15 of the same MMA);
//   online softmax    lane-local running (max, sum, Σ p·u) per row over the lane's own tokens,
//                     merged across the 4 lanes of a quad only at variant snapshots;
//   snapshots         tokens are in importance order, so every keep ratio is a prefix: the
//                     state is snapshot when the token index reaches each variant's n_kept, so
//                     one read serves every variant (nested prefixes, Q2); layer cuts select
//                     which units a variant sums.
// Partial logits per (unit, op, variant, class) go to a workspace; the warp that completes a
// tuple's last unit sums them in a FIXED order (bitwise-deterministic margins), derives margin
// and class, then either evaluates every plan of the grid (grid mode) or applies one cascade stage
// (stage mode), counting with shared-memory integer atomics flushed once per CTA.
//
// The key/value data layout, the d-permutation that lets one LDG.128 feed two MMA k-steps, and
// the roofline are in DESIGN.md §"Kernel".
#include <cuda_bf16.h>
#include <math_constants.h>

#include <algorithm>

#include "ko_internal.h"

namespace ko {
namespace {

enum { D_ACCEPT = 0, D_REJECT = 1, D_UNSURE = 2, D_RESOLVED = 3 };
// finite "no token yet" running max of the table-packed kernel: ex2(kNoMax − real) = 0 and
// ex2(kNoMax − kNoMax) = 1, so the online-softmax update needs no −∞ special cases
constexpr float kNoMax = -1e30f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t a0, const uint32_t a1,
                                         const uint32_t a2, const uint32_t a3, const uint32_t b0,
                                         const uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ int n_kept(int L, int keep) {  // Q3: max(1, floor(L·keep/1000))
  int n = (int)(((long long)L * keep) / 1000);
  return n < 1 ? 1 : n;
}

// Step-5 decision; identical semantics to the oracle (strict inequalities, Q5/Q6/Q13).
__device__ __forceinline__ int decide(float m, const ko_stage& st, int ncls) {
  if (ncls <= 1) {
    if (st.is_final) return m > st.theta_hi ? D_ACCEPT : D_REJECT;
    if (m > st.theta_hi) return D_ACCEPT;
    if (m < st.theta_lo) return D_REJECT;
    return D_UNSURE;
  }
  if (st.is_final) return D_RESOLVED;
  return m > st.theta_hi ? D_RESOLVED : D_UNSURE;
}

__device__ __forceinline__ int op_status(uint32_t st, int o) { return (st >> (1 + 2 * o)) & 3; }
// routed walk: the stage a tuple resumes at lives in the free bits 9..12 (bits 1..8 hold the
// op statuses, 16..31 the resolved classes of ops 0..3)
constexpr int kWalkStageShift = 9;

// Whole-plan evaluation for one tuple (Eqs. accept-i/reject-i/unsure-i, conjunctive
// inter-op semantics P:536-539, counts P:350-352).  ms/cs: margins/classes indexed
// [op * n_var + variant].  cnt: this plan's int32 counter row (shared memory).
// Returns the final tuple state (bit0 alive, 2-bit status per op, 4-bit class per op).
__device__ uint32_t eval_plan(const ko_plan& P, const float* ms, const int32_t* cs, int n_var,
                              const int32_t* ncls, const uint8_t* gold, int64_t n_tuples,
                              int64_t t, int* cnt) {
  uint32_t state = 1u;
  uint32_t referenced = 0;
  for (int s = 0; s < P.n_stages; ++s) referenced |= 1u << P.stage[s].op;
  for (int s = 0; s < P.n_stages; ++s) {
    const ko_stage& st = P.stage[s];
    const int o = st.op;
    if (!(state & 1u) || op_status(state, o) != 0) continue;
    if (cnt) atomicAdd(&cnt[5 + 4 * s], 1);
    const int idx = o * n_var + st.variant;
    const int d = decide(ms[idx], st, ncls[o]);
    if (d == D_ACCEPT || d == D_RESOLVED) {
      state |= 1u << (1 + 2 * o);
      if (d == D_RESOLVED) state |= ((uint32_t)cs[idx] & 15u) << (16 + 4 * o);
      if (cnt) atomicAdd(&cnt[6 + 4 * s], 1);
    } else if (d == D_REJECT) {
      state &= ~1u;
      state |= 2u << (1 + 2 * o);
      if (cnt) atomicAdd(&cnt[7 + 4 * s], 1);
    } else {
      if (cnt) atomicAdd(&cnt[8 + 4 * s], 1);
    }
  }
  if (cnt) {
    const bool in_out = state & 1u;
    bool in_gold = gold != nullptr, maps_ok = true;
    if (gold) {
      for (int o = 0; o < kMaxOps; ++o) {
        if (!(referenced & (1u << o))) continue;
        const uint8_t gv = gold[(int64_t)o * n_tuples + t];
        if (ncls[o] <= 1) {
          if (gv != 1) in_gold = false;
        } else if (((state >> (16 + 4 * o)) & 15u) != gv || op_status(state, o) != 1) {
          maps_ok = false;
        }
      }
    }
    if (in_out) atomicAdd(&cnt[KO_C_OUT], 1);
    if (in_gold) atomicAdd(&cnt[KO_C_GOLD], 1);
    if (in_out && in_gold && maps_ok) atomicAdd(&cnt[KO_C_TP], 1);
  }
  return state;
}

// Flush per-CTA int32 counters (FP/FN derived from n_out/n_gold/TP) into the int64 output.
__device__ void flush_counts(int* s_cnt, int n_rows, unsigned long long* counts) {
  __syncthreads();
  for (int i = threadIdx.x; i < n_rows * kCountsPerPlan; i += blockDim.x) {
    const int k = i % kCountsPerPlan;
    const int* row = s_cnt + (i - k);
    long long v = s_cnt[i];
    if (k == KO_C_FP) v = (long long)row[KO_C_OUT] - row[KO_C_TP];
    if (k == KO_C_FN) v = (long long)row[KO_C_GOLD] - row[KO_C_TP];
    if (v) atomicAdd(&counts[i], (unsigned long long)v);
  }
}

// ------------------------------------------------------------------------------------------
// The scoring kernel
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// TMA: one (64 d × 16 tokens × 1 head × {K,V}) box of page `page` → smem (128B-swizzled),
// completion counted on `bar`; L2 evict-first (the KV stream is read once).
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* map, int d0, int h,
                                             int kv0, int page, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(d0), "r"(0), "r"(h), "r"(kv0), "r"(page),
      "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr));
  return r;
}

template <int D>
struct Ring {
  static constexpr int kBoxBytes = 64 * 16 * 2 * 2;      // 64 d × 16 tokens × {K,V} × bf16
  static constexpr int kStageBytes = (D / 64) * kBoxBytes;
  static constexpr int kStages = D == 128 ? 3 : 6;       // per warp
  static constexpr int kWarpBytes = kStages * kStageBytes;
  static constexpr int kSmemBytes = (kThreads / 32) * kWarpBytes + 1024;  // + alignment slack
};

// ------------------------------------------------------------------------------------------
// Grid-mode tuple finaliser (run by the warp completing a tuple's last unit): margins/classes
// from the partial logits, then every plan of the grid per tuple.  zs / sm_w / sc_w: this warp's
// shared-memory scratch; s_cnt: the CTA's counters.  (Routed rounds: ko_walk_kernel.)
// ------------------------------------------------------------------------------------------
template <int CPR>
__device__ __forceinline__ void finalise_tuple(const ScoreParams& p, int64_t wslot, int64_t t,
                                               int lane, float* zs, float* sm_w, int32_t* sc_w,
                                               int* s_cnt) {

    // z = b + Σ_u partial_u over the units whose layer is inside the variant's cut, for every
    // (op, variant, class) entry: one lane per entry sums its units in a FIXED (ascending) order in
    // fp64, so margins stay bitwise reproducible.  This launch's partials per work slot, local
    // (op, variant).
    const int nz = p.n_ops * p.n_var * CPR;
    const int n_pu = p.n_l * p.n_kv_heads;  // partial slots per tuple (layer-major)
    const int nzg = nz;
    const float* tpart = p.part + (size_t)wslot * n_pu * nzg;
    for (int idx = lane; idx < nz; idx += 32) {
      const int c = idx % CPR, ov = idx / CPR;
      const int o = ov / p.n_var, v = ov - o * p.n_var;
      if (c >= p.op_classes[o]) continue;
      const float* src = tpart + idx;
      const int nu = min(p.cut[v], p.n_layers) * p.n_kv_heads;  // l-major: l < cut ⇔ u < cut·Hkv
      double acc = 0.0;
      int uu = 0;
      for (; uu + 4 <= nu; uu += 4) {
        const float a0 = __ldcg(src + (size_t)(uu + 0) * nzg), a1 = __ldcg(src + (size_t)(uu + 1) * nzg);
        const float a2 = __ldcg(src + (size_t)(uu + 2) * nzg), a3 = __ldcg(src + (size_t)(uu + 3) * nzg);
        acc += (double)a0; acc += (double)a1; acc += (double)a2; acc += (double)a3;
      }
      for (; uu < nu; ++uu) acc += (double)__ldcg(src + (size_t)uu * nzg);
      zs[idx] = (float)((double)__ldg(p.bias[o] + c) + acc);
    }
    __syncwarp();
    for (int idx = lane; idx < p.n_ops * p.n_var; idx += 32) {
      const int o = idx / p.n_var, v = idx % p.n_var;
      const float* zz = zs + idx * CPR;
      float m;
      int cls = 0;
      if (p.op_classes[o] <= 1) {
        m = zz[0];
      } else {
        for (int c = 1; c < p.op_classes[o]; ++c)
          if (zz[c] > zz[cls]) cls = c;  // lowest index on ties
        float second = -CUDART_INF_F;
        for (int c = 0; c < p.op_classes[o]; ++c)
          if (c != cls && zz[c] > second) second = zz[c];
        m = zz[cls] - second;
      }
      const size_t oi = ((size_t)p.op_ids[o] * p.n_var_total + p.var_ids[v]) * p.n_tuples + t;
      if (p.margins) p.margins[oi] = m;
      if (p.classes) p.classes[oi] = cls;
      sm_w[p.op_ids[o] * p.n_var_total + p.var_ids[v]] = m;  // caller's op and variant
      sc_w[p.op_ids[o] * p.n_var_total + p.var_ids[v]] = cls;
    }
    if (p.mode == MODE_GRID && p.n_ext) {
      // external variants (margins supplied by the caller, e.g. ko_embed_scores) join the plans
      for (int idx = lane; idx < p.n_ops_total * p.n_ext; idx += 32) {
        const int o = idx / p.n_ext, v = p.ext_ids[idx % p.n_ext];
        const size_t oi = ((size_t)o * p.n_var_total + v) * p.n_tuples + t;
        sm_w[o * p.n_var_total + v] = __ldcg(p.margins + oi);
        sc_w[o * p.n_var_total + v] = 0;
      }
    }
    __syncwarp();
    {
      for (int gp = lane; gp < p.n_plans; gp += 32)
        eval_plan(p.gplans[gp], sm_w, sc_w, p.n_var_total, p.op_classes_g, p.gold, p.n_tuples,
                  t, s_cnt + gp * kCountsPerPlan);
    }
}

// CPR0 / CPR1: classes per row slot in half 0 (A rows g) / half 1 (A rows g+8) of the row tile;
// CPR1 = 0 when at most 8 rows attend a kv-head; partial logits are stored with stride
// CPR = CPR0 (≥ every op's classes).  W·V tiles:
//   fp32 W (NOLO = false): bf16 hi in A rows 0-7 + lo in rows 8-15 of one tile per (half, class):
//     tile(h, c) = h ? CPR0 + c : c, u = C[e] + C[2+e];
//   bf16 W (NOLO = true, exact: no lo part): two classes per tile, class c in rows 0-7 (c even)
//     or 8-15 (c odd): tile(h, c) = (h ? ⌈CPR0/2⌉ : 0) + c/2, u = C[2(c&1) + e].
// TNT > 0 (table packing, every walk-mode launch): the W·V tiles are packed per lane group g
// from a host table — A-row half hr of tile tt at lane group g is slot k = 2·tt + hr, which
// accumulates with S row g + 8·hr for the (op, class) tgt[k]; a row with more entries than one
// half's TNT slots is duplicated into both halves.
template <int D, int CPR0, int CPR1, bool NOLO, int TNT>
__global__ void __launch_bounds__(kThreads, 2) ko_score_kernel(const __grid_constant__ ScoreParams p) {
  constexpr bool TBL = TNT > 0;
  constexpr int KS = D / 16;  // mma k-steps over head_dim
  constexpr int KP = D / 32;  // 128-bit fragment reads per token row per lane (2 k-steps each)
  constexpr int NH = TBL ? 2 : (CPR1 > 0 ? 2 : 1);
  constexpr int CPR = CPR0;
  constexpr int T0 = NOLO ? (CPR0 + 1) / 2 : CPR0;  // tiles of half 0
  constexpr int NT = TBL ? TNT : (NOLO ? T0 + (CPR1 + 1) / 2 : CPR0 + CPR1);
  constexpr int NSL = TBL ? 2 * TNT : 1;            // table slots per lane
  constexpr int WREG = NT <= 2 ? NT : 0;            // W·V tiles whose fragments stay in registers
  constexpr int S = Ring<D>::kStages;
  constexpr int STAGE = Ring<D>::kStageBytes;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;

  extern __shared__ uint8_t smem_dyn[];
  __shared__ int s_cnt[kMaxPlans * kCountsPerPlan];
  __shared__ float s_z[kThreads / 32][kMaxOps * kMaxVar * kMaxCls];
  __shared__ float s_m[kThreads / 32][kMaxOps * kMaxVar];
  __shared__ int32_t s_c[kThreads / 32][kMaxOps * kMaxVar];
  __shared__ __align__(8) uint64_t s_full[kThreads / 32][S];

  // per-warp ring of S stages (1024-byte aligned for the 128B swizzle atom)
  uint8_t* ring_base = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* ring = ring_base + warp * Ring<D>::kWarpBytes;
  const uint32_t ring_s = smem_u32(ring);

  const bool walk = p.mode == MODE_WALK;
  const int n_cnt_rows = p.mode == MODE_GRID ? p.n_plans : 0;  // walk: ko_walk_kernel counts
  for (int i = threadIdx.x; i < n_cnt_rows * kCountsPerPlan; i += blockDim.x) s_cnt[i] = 0;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&s_full[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
  __syncthreads();
  uint64_t policy = 0;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

  const int64_t n_work = p.work_len_dev ? *p.work_len_dev : p.work_len_host;
  const int Hkv = p.n_kv_heads;
  const int HG = p.heads_per_unit;  // kv-heads streamed back-to-back by one unit (same pages)
  const int upt = p.n_l * (Hkv / HG);  // work units per tuple: (layer, group of HG kv-heads)
  const int64_t n_units = n_work * upt;
  // variants whose extents this launch streams: grid = all; walk = ranks ≤ round
  const int v_hi = walk ? p.round : p.n_var - 1;

  // row slot → local op for this lane's two half-slots (legacy packing)
  int slot_op[NH];
#pragma unroll
  for (int hs = 0; hs < NH; ++hs) slot_op[hs] = p.slot_op[hs * 8 + g];
  // table packing: this lane group's slot k = 2·tile + hr (S-row half hr) → target op·8 + class
  int tgt[NSL];
#pragma unroll
  for (int k = 0; k < NSL; ++k) tgt[k] = -1;
  // snapshot reduction: lane j owns target j = op·8 + class, whose slots sit at positions
  // g·NSL + k of the warp's staging row; up to 4 positions are kept as a packed byte list (red_off,
  // red_n), more as a bit mask over all 8·NSL positions (red0/red1, bits 0-63 / 64-127)
  uint64_t red0 = 0, red1 = 0;
  uint32_t red_off = 0;
  int red_n = 0;
  if constexpr (TBL) {
#pragma unroll
    for (int k = 0; k < NSL; ++k) tgt[k] = p.tbl_tgt[g][k];
    for (int gg = 0; gg < 8; ++gg)
#pragma unroll
      for (int k = 0; k < NSL; ++k)
        if (p.tbl_tgt[gg][k] == lane) {
          const int i = gg * NSL + k;
          if (i < 64) red0 |= 1ull << i; else red1 |= 1ull << (i - 64);
          if (red_n < 4) red_off |= (uint32_t)i << (8 * red_n);
          ++red_n;
        }
  }

  // lane-constant smem offsets of this lane's fragment reads inside a stage: token row g (+8),
  // d-chunk (2q + (j & 1)) of box (j >> 1), XOR-swizzled by the row (= token mod 8)
  uint32_t frag_off[KP];
#pragma unroll
  for (int j = 0; j < KP; ++j)
    frag_off[j] = (j >> 1) * Ring<D>::kBoxBytes + g * 128 + ((((2 * q) + (j & 1)) ^ g) << 4);

  uint32_t issued = 0, consumed = 0;  // ring positions (warp-uniform, persistent across units)

  // Work units are consumed in claim order.  Their pages enter the ring through a producer cursor
  // that runs ahead of the consumer: once the current unit's pages are all issued, the producer
  // decodes the NEXT unit (claimed when the current one was decoded) and keeps issuing its pages,
  // so the ring stays full across the current unit's tail and its tuple finaliser.
  struct Unit {
    long long u;             // unit index (≥ n_units: none)
    int64_t wslot, t, pbase;
    int l, h0, L, s0, s1;    // layer, first kv-head, seq_len, streamed tokens [s0, s1)
    int n_str;               // pages the unit streams (HG kv-heads)
    int ih, ipg, nis;        // producer cursor: head offset, page, pages issued
    int pid_chunk, pid_reg;  // page-id cache (chunk of 32 ids, one per lane)
  };
  auto claim = [&]() {
    long long u = 0;
    if (lane == 0) u = (long long)atomicAdd(p.unit_counter, 1ull);
    return u;  // meaningful in lane 0 (broadcast by decode)
  };
  auto decode = [&](long long u0) {
    Unit U;
    U.u = __shfl_sync(0xffffffffu, u0, 0);
    U.nis = 0; U.ih = 0; U.s0 = 0; U.s1 = 0; U.pid_chunk = 0; U.pid_reg = 0;
    U.wslot = 0; U.t = 0; U.pbase = 0; U.l = 0; U.h0 = 0; U.L = 1; U.ipg = 0; U.n_str = 0;
    if (U.u >= n_units) return U;
    U.wslot = U.u / upt;
    const int unit = (int)(U.u - U.wslot * upt);
    U.l = unit / (Hkv / HG);
    U.h0 = (unit - U.l * (Hkv / HG)) * HG;
    U.t = p.work ? (int64_t)p.work[U.wslot] : U.wslot;
    U.L = p.seq_len[U.t];
    U.pbase = p.page_indptr[U.t];
    // tokens [s0, s1): s1 = the largest prefix among the streamed variants whose cut includes l;
    // walk mode resumes after the extent of the tuple's previous rank for this group (s0)
    int prev = -1;
    if (walk && p.pos > 0) {
      const uint32_t nib = (__ldcg(p.tuple_done + U.t) >> (4 * p.group)) & 15u;
      prev = nib == 15u ? -1 : (int)nib - 1;
    }
    for (int v = 0; v < p.n_var; ++v)
      if (p.cut[v] > U.l) {
        const int nk = n_kept(U.L, p.keep[v]);
        if (v <= v_hi) U.s1 = max(U.s1, nk);
        if (v <= prev) U.s0 = max(U.s0, nk);
      }
    U.ipg = U.s0 >> 4;
    U.n_str = U.s1 > U.s0 ? HG * (((U.s1 + 15) >> 4) - U.ipg) : 0;
    U.pid_chunk = U.ipg >> 5;
    const int idx = (U.pid_chunk << 5) + lane;
    if (idx < ((U.s1 + 15) >> 4)) U.pid_reg = __ldg(p.page_ids + U.pbase + idx);
    return U;
  };
  auto n_pages_of = [&](const Unit& U) {  // pages streamed per kv-head
    return U.s1 > U.s0 ? ((U.s1 + 15) >> 4) - (U.s0 >> 4) : 0;
  };
  // TMA issue of unit U's next stream page into the next ring slot (whole warp; lane 0 issues)
  auto issue = [&](Unit& U) {
    const int pg = U.ipg, pg1u = (U.s1 + 15) >> 4;
    const int chunk = pg >> 5;
    if (chunk != U.pid_chunk) {
      const int idx = (chunk << 5) + lane;
      U.pid_reg = idx < pg1u ? __ldg(p.page_ids + U.pbase + idx) : 0;
      U.pid_chunk = chunk;
    }
    const int pid = __shfl_sync(0xffffffffu, U.pid_reg, pg & 31);
    if (lane == 0) {
      const int slot = issued % S;
      uint64_t* bar = &s_full[warp][slot];
      mbar_expect_tx(bar, STAGE);
      uint8_t* dst = ring + slot * STAGE;
#pragma unroll
      for (int b = 0; b < D / 64; ++b)
        tma_load_box(dst + b * Ring<D>::kBoxBytes, &p.tmap, 64 * b, U.h0 + U.ih, 2 * U.l, pid, bar,
                     policy);
    }
    ++issued;
    ++U.nis;
    if (++U.ipg == pg1u) { U.ipg = U.s0 >> 4; ++U.ih; }
  };

  long long u_next = claim();
  Unit cur = decode(u_next);
  if (cur.u < n_units) u_next = claim();
  Unit nxt;
  bool have_nxt = false;
  // one ring slot was freed: issue the next page of the stream (current unit, else the next one)
  auto refill = [&]() {
    if (cur.nis < cur.n_str) {
      issue(cur);
      return;
    }
    if (!have_nxt) {
      nxt = decode(u_next);
      have_nxt = true;
      if (nxt.u < n_units) u_next = claim();
    }
    if (nxt.nis < nxt.n_str) issue(nxt);
  };

  while (cur.u < n_units) {
    // top up the ring with the unit's pages (some may already be in flight from the producer)
    while (cur.nis < cur.n_str && (int)(issued - consumed) < S) issue(cur);
    const int64_t wslot = cur.wslot, t = cur.t;
    const int l = cur.l, h0 = cur.h0, L = cur.L, s0 = cur.s0, s1 = cur.s1;
    // per-variant kept prefix at this layer (−1: the variant's cut excludes l) — computed once per
    // unit; the snapshot logic below only compares against these
    int nkv[kMaxVar];
#pragma unroll
    for (int v = 0; v < kMaxVar; ++v)
      nkv[v] = (v < p.n_var && p.cut[v] > l) ? n_kept(L, p.keep[v]) : -1;
    // snapshot points in (s0, s1]: any variant, any rank
    auto next_point = [&](int after) {
      int nx = 0x7fffffff;
#pragma unroll
      for (int v = 0; v < kMaxVar; ++v)
        if (nkv[v] > after) nx = min(nx, nkv[v]);
      return nx;
    };
    const int first_snap = next_point(s0);
    const int n_need = s1;
    const int pg0 = s0 >> 4;
    const int pg1 = (s1 + 15) >> 4;
    const int npu = n_pages_of(cur);  // pages streamed per kv-head

    // operator-query / readout fragments of (l, h): loaded for the unit's first head here and for
    // every later head right after the last page's MMAs of the previous one (latency hidden
    // behind that page's softmax work)
    uint32_t qa[KS][4];
    uint32_t wa1[WREG > 0 ? WREG : 1][KS][4];
    auto load_frags = [&](int h) {
      const int lh = l * Hkv + h;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint4 f = __ldg(p.qfrag + ((size_t)lh * KS + ks) * 32 + lane);
        qa[ks][0] = f.x; qa[ks][1] = f.y; qa[ks][2] = f.z; qa[ks][3] = f.w;
      }
#pragma unroll
      for (int tt = 0; tt < WREG; ++tt)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint4 f = __ldg(p.wfrag + (((size_t)lh * NT + tt) * KS + ks) * 32 + lane);
          wa1[tt][ks][0] = f.x; wa1[tt][ks][1] = f.y; wa1[tt][ks][2] = f.z; wa1[tt][ks][3] = f.w;
        }
    };
    if (npu > 0) load_frags(h0);

   for (int hh = 0; hh < (npu > 0 ? HG : 0); ++hh) {
    const int h = h0 + hh;
    const int unit_lh = l * Hkv + h;  // partial-logit slot of (layer, kv-head)
    int next_snap = first_snap;
    const uint4* wbase = p.wfrag + (size_t)unit_lh * NT * KS * 32 + lane;
    // saved state of (t, l, h) for this lane group (walk mode)
    float* rst = walk ? p.rstate + ((((size_t)t * p.n_layers + l) * Hkv + h) * 8 + g) * p.rstate_w
                      : nullptr;

    // lane-local online-softmax state per half-slot (log2 domain)
    float mx[NH], sm[NH], ac[TBL ? 1 : NH][CPR], at[NSL];
#pragma unroll
    for (int hs = 0; hs < NH; ++hs) {
      mx[hs] = TBL ? kNoMax : -CUDART_INF_F;
      sm[hs] = 0.f;
#pragma unroll
      for (int c = 0; c < CPR; ++c)
        if (!TBL) ac[TBL ? 0 : hs][c] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < NSL; ++k) at[k] = 0.f;
    if constexpr (TBL) {
      if (walk && s0 > 0 && q == 0) {  // resume: the quad's merged state enters through lane q = 0
        mx[0] = __ldcg(rst + 0);
        mx[1] = __ldcg(rst + 1);
        sm[0] = __ldcg(rst + 2);
        sm[1] = __ldcg(rst + 3);
#pragma unroll
        for (int k = 0; k < NSL; ++k) at[k] = __ldcg(rst + 4 + k);
      }
    }

    int snap_lo = s0;  // first token not yet folded into the running state

    for (int pg = pg0; pg < pg1; ++pg) {
      const int slot = consumed % S;
      mbar_wait(&s_full[warp][slot], (consumed / S) & 1u);
      const uint32_t stage = ring_s + slot * STAGE;
      // ---- tensor cores: S = Q·Kᵀ and U = W·Vᵀ for this page's 16 tokens
      const bool tail_page = pg * 16 + 16 > n_need;  // warp-uniform
      float Sacc[2][4];
      float U[NT][2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        uint4 kf[KP], vf[KP];
#pragma unroll
        for (int j = 0; j < KP; ++j) {
          const uint32_t a = stage + frag_off[j] + nt * 8 * 128;
          kf[j] = lds128(a);
          vf[j] = lds128(a + 16 * 128);  // V rows follow the 16 K rows of the box
        }
        if (tail_page) {  // tokens past the extent (unused slots may hold anything, even NaN)
          const bool valid = (pg * 16 + nt * 8 + g) < n_need;  // B-operand row = token nt*8+g
#pragma unroll
          for (int j = 0; j < KP; ++j)
            if (!valid) { kf[j] = make_uint4(0, 0, 0, 0); vf[j] = make_uint4(0, 0, 0, 0); }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) Sacc[nt][i] = 0.f;
#pragma unroll
        for (int tt = 0; tt < NT; ++tt)
#pragma unroll
          for (int i = 0; i < 4; ++i) U[tt][nt][i] = 0.f;
#pragma unroll
        for (int j = 0; j < KP; ++j) {
          mma16816(Sacc[nt], qa[2 * j][0], qa[2 * j][1], qa[2 * j][2], qa[2 * j][3], kf[j].x,
                   kf[j].y);
          mma16816(Sacc[nt], qa[2 * j + 1][0], qa[2 * j + 1][1], qa[2 * j + 1][2],
                   qa[2 * j + 1][3], kf[j].z, kf[j].w);
        }
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) {
#pragma unroll
          for (int j = 0; j < KP; ++j) {
            uint32_t a0[4], a1[4];
            if constexpr (WREG > 0) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                a0[i] = wa1[tt][2 * j][i];
                a1[i] = wa1[tt][2 * j + 1][i];
              }
            } else {
              const uint4 f0 = __ldg(wbase + ((size_t)tt * KS + 2 * j) * 32);
              const uint4 f1 = __ldg(wbase + ((size_t)tt * KS + 2 * j + 1) * 32);
              a0[0] = f0.x; a0[1] = f0.y; a0[2] = f0.z; a0[3] = f0.w;
              a1[0] = f1.x; a1[1] = f1.y; a1[2] = f1.z; a1[3] = f1.w;
            }
            mma16816(U[tt][nt], a0[0], a0[1], a0[2], a0[3], vf[j].x, vf[j].y);
            mma16816(U[tt][nt], a1[0], a1[1], a1[2], a1[3], vf[j].z, vf[j].w);
          }
        }
      }
      // the stage's bytes are in registers: hand the slot back to TMA for page pg + S
      __syncwarp();
      ++consumed;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      refill();
      // the fragments are dead after the last page's MMAs: fetch the next head's now
      if (pg + 1 == pg1 && hh + 1 < HG) load_frags(h + 1);
      // ---- per-lane token indices and values: k = nt*2 + e ↔ token pg*16 + nt*8 + 2q + e
      const int page_hi = min(pg * 16 + 16, n_need);
      for (;;) {
        const int seg_hi = min(next_snap, page_hi);
        // fold tokens [snap_lo, seg_hi) of this page into the lane-local state
        if constexpr (TBL) {
          // running max starts at a finite sentinel (kNoMax): corr and p need no −∞ guards
          float corr[2], ps[2][4];
          const bool full = pg * 16 >= snap_lo && pg * 16 + 16 <= seg_hi;  // warp-uniform
#pragma unroll
          for (int hs = 0; hs < 2; ++hs) {
            float x[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int nt = k >> 1, e = k & 1;
              x[k] = Sacc[nt][2 * hs + e] * p.scale_log2;
            }
            if (!full) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int tok = pg * 16 + (k >> 1) * 8 + 2 * q + (k & 1);
                if (!(tok >= snap_lo && tok < seg_hi)) x[k] = -CUDART_INF_F;
              }
            }
            const float mn = fmaxf(fmaxf(mx[hs], fmaxf(x[0], x[1])), fmaxf(x[2], x[3]));
            corr[hs] = ex2(mx[hs] - mn);
#pragma unroll
            for (int k = 0; k < 4; ++k) ps[hs][k] = ex2(x[k] - mn);
            sm[hs] = sm[hs] * corr[hs] + ((ps[hs][0] + ps[hs][1]) + (ps[hs][2] + ps[hs][3]));
            mx[hs] = mn;
          }
#pragma unroll
          for (int k = 0; k < NSL; ++k) {
            const int hr = k & 1;
            float a = at[k] * corr[hr];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              a = fmaf(ps[hr][kk], U[k >> 1][kk >> 1][2 * hr + (kk & 1)], a);
            at[k] = a;
          }
        } else {
#pragma unroll
        for (int hs = 0; hs < NH; ++hs) {
          float x[4];
          float xm = -CUDART_INF_F;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int nt = k >> 1, e = k & 1;
            const int tok = pg * 16 + nt * 8 + 2 * q + e;
            const bool in = tok >= snap_lo && tok < seg_hi;
            x[k] = in ? Sacc[nt][2 * hs + e] * p.scale_log2 : -CUDART_INF_F;
            xm = fmaxf(xm, x[k]);
          }
          const float mn = fmaxf(mx[hs], xm);
          if (mn != -CUDART_INF_F) {
            const float corr = ex2(mx[hs] - mn);
            float ps[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) ps[k] = ex2(x[k] - mn);
            sm[hs] = sm[hs] * corr + ((ps[0] + ps[1]) + (ps[2] + ps[3]));
#pragma unroll
            for (int c = 0; c < (hs == 0 ? CPR0 : CPR1); ++c) {
              const int tt = NOLO ? (hs == 0 ? 0 : T0) + c / 2 : (hs == 0 ? c : CPR0 + c);
              float a = ac[TBL ? 0 : hs][c] * corr;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int nt = k >> 1, e = k & 1;
                const float u = NOLO ? U[tt][nt][2 * (c & 1) + e] : U[tt][nt][e] + U[tt][nt][2 + e];
                a = fmaf(ps[k], u, a);
              }
              ac[TBL ? 0 : hs][c] = a;
            }
            mx[hs] = mn;
          }
        }
        }
        snap_lo = seg_hi;
        if (seg_hi == next_snap) {
          // ---- snapshot: merge the quad's lane states, reduce rows per op, emit partials
          float opv[kMaxOps][CPR];  // legacy packing: per-(op, class) partial (all lanes)
          if constexpr (TBL) {
            float Mq[2], f[2], den[2], rden[2];
#pragma unroll
            for (int hs = 0; hs < 2; ++hs) {
              float M = mx[hs];
              M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 1));
              M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 2));
              f[hs] = ex2(mx[hs] - M);
              float d = sm[hs] * f[hs];
              d += __shfl_xor_sync(0xffffffffu, d, 1);
              d += __shfl_xor_sync(0xffffffffu, d, 2);
              den[hs] = d;
              rden[hs] = __frcp_rn(d);
              Mq[hs] = M;
            }
            float accm[NSL], val[NSL];
#pragma unroll
            for (int k = 0; k < NSL; ++k) {
              float a = at[k] * f[k & 1];
              a += __shfl_xor_sync(0xffffffffu, a, 1);
              a += __shfl_xor_sync(0xffffffffu, a, 2);
              accm[k] = a;
              val[k] = a * rden[k & 1];
            }
            if (walk && p.save_state && next_snap == s1 && q == 0) {
              // end of this round's extent: save the merged state for a later round to resume
              rst[0] = Mq[0]; rst[1] = Mq[1]; rst[2] = den[0]; rst[3] = den[1];
#pragma unroll
              for (int k = 0; k < NSL; ++k) rst[4 + k] = accm[k];
            }
            // cross-lane-group sum per (op, class) target through shared memory: lane j adds
            // target j's slots in a fixed (ascending) order, then writes its partial
            float* sv = s_z[warp];
            if (q == 0) {
#pragma unroll
              for (int k = 0; k < NSL; ++k) sv[g * NSL + k] = val[k];
            }
            __syncwarp();
            float x = 0.f;
            if (red_n <= 4) {
#pragma unroll
              for (int r = 0; r < 4; ++r)
                if (r < red_n) x += sv[(red_off >> (8 * r)) & 255u];
            } else {
              for (uint64_t m = red0; m; m &= m - 1) x += sv[__ffsll((long long)m) - 1];
              for (uint64_t m = red1; m; m &= m - 1) x += sv[64 + __ffsll((long long)m) - 1];
            }
            __syncwarp();
            if (red_n > 0) {
              const int o = lane >> 3, c = lane & 7;
#pragma unroll
              for (int v = 0; v < kMaxVar; ++v)
                if (nkv[v] == next_snap) {
                  // walk: per tuple (persisting across rounds), caller's (op, variant); grid: per
                  // work slot, local (op, variant) — the grid finaliser's layout
                  const size_t at =
                      walk ? ((((size_t)t * p.n_lh_all + unit_lh) * p.n_ops_total + p.op_ids[o]) *
                                  p.n_var_total + p.var_ids[v]) * p.part_cpr + c
                           : ((((size_t)wslot * p.n_l * Hkv + unit_lh) * p.n_ops + o) * p.n_var + v) *
                                 CPR + c;
                  p.part[at] = x;
                }
            }
          } else {
          float val[NH][CPR];
#pragma unroll
          for (int hs = 0; hs < NH; ++hs) {
            float M = mx[hs];
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 1));
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 2));
            const float f = mx[hs] == -CUDART_INF_F ? 0.f : ex2(mx[hs] - M);
            float den = sm[hs] * f;
            den += __shfl_xor_sync(0xffffffffu, den, 1);
            den += __shfl_xor_sync(0xffffffffu, den, 2);
#pragma unroll
            for (int c = 0; c < CPR; ++c) {
              if (c >= (hs == 0 ? CPR0 : CPR1)) { val[hs][c] = 0.f; continue; }
              float a = ac[TBL ? 0 : hs][c] * f;
              a += __shfl_xor_sync(0xffffffffu, a, 1);
              a += __shfl_xor_sync(0xffffffffu, a, 2);
              val[hs][c] = __fdiv_rn(a, den);
            }
          }
#pragma unroll
          for (int o = 0; o < kMaxOps; ++o) {
#pragma unroll
            for (int c = 0; c < CPR; ++c) {
              float x = 0.f;
#pragma unroll
              for (int hs = 0; hs < NH; ++hs) x += slot_op[hs] == o ? val[hs][c] : 0.f;
              if (o < p.n_ops) {
                x += __shfl_xor_sync(0xffffffffu, x, 4);
                x += __shfl_xor_sync(0xffffffffu, x, 8);
                x += __shfl_xor_sync(0xffffffffu, x, 16);
              }
              opv[o][c] = x;
            }
          }
          }
          if (!TBL && lane == 0) {  // grid: partials per work slot, local (op, variant) indices
#pragma unroll
            for (int v = 0; v < kMaxVar; ++v) {
              if (nkv[v] != next_snap) continue;
#pragma unroll
              for (int o = 0; o < kMaxOps; ++o) {
                if (o >= p.n_ops) break;
                float* dst = p.part + ((((size_t)wslot * p.n_l * Hkv + unit_lh) * p.n_ops + o) * p.n_var + v) * CPR;
#pragma unroll
                for (int c = 0; c < CPR; ++c) dst[c] = opv[o][c];
              }
            }
          }
          next_snap = next_point(next_snap);  // the next larger snapshot point
        }
        if (snap_lo >= page_hi) break;
      }
    }

   }  // heads of the unit
    // ---- tuple completion (grid mode): the warp finishing the tuple's last unit finalises it;
    // routed rounds are finalised by ko_walk_kernel after the launch
    if (!walk) {
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        // release: this unit's partial logits (stored by this lane) are visible before the count
        uint32_t prev;
        asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;"
                     : "=r"(prev)
                     : "l"(p.done + wslot)
                     : "memory");
        last = prev == (uint32_t)(upt - 1);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();
        finalise_tuple<CPR>(p, wslot, t, lane, s_z[warp], s_m[warp], s_c[warp], s_cnt);
      }
    }
    // advance to the next unit (the producer may already have decoded it and issued its pages)
    if (!have_nxt) {
      nxt = decode(u_next);
      if (nxt.u < n_units) u_next = claim();
    }
    have_nxt = false;
    cur = nxt;
  }
  if (n_cnt_rows) flush_counts(s_cnt, n_cnt_rows, p.counts);
}

// ------------------------------------------------------------------------------------------
// Fragment preparation: Q (bf16) and W (fp32 → bf16 hi + lo) into the per-lane register layout
// of mma.m16n8k16 with the d-permutation of DESIGN.md §"Kernel":
//   k-step ks = 2j + e, lane (g, q): A regs {a0a1, a2a3, a4a5, a6a7} hold
//   (row g, d0, d0+1), (row g+8, d0, d0+1), (row g, d0+2, d0+3), (row g+8, d0+2, d0+3),
//   d0 = 64(j/2) + 16q + 8(j%2) + 4e — exactly the 8 consecutive bf16 of the 16-byte chunk
//   (2q + j%2) of 64-wide box j/2 that lane (g, q) reads from the swizzled TMA stage.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack2(uint16_t lo, uint16_t hi) {
  return (uint32_t)lo | ((uint32_t)hi << 16);
}

__global__ void prep_kernel(const __grid_constant__ PrepParams p) {
  if (blockIdx.x == 0 && p.gplans)
    for (int i = threadIdx.x; i < p.n_plans * (int)(sizeof(ko_plan) / 4); i += blockDim.x)
      reinterpret_cast<uint32_t*>(p.gplans)[i] = reinterpret_cast<const uint32_t*>(p.plans)[i];
  const int KS = p.head_dim / 16;
  const int NT = p.tbl_nt > 0 ? p.tbl_nt
               : p.nolo ? (p.CPR0 + 1) / 2 + (p.CPR1 + 1) / 2 : p.CPR0 + p.CPR1;
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
    } else if (p.tbl_nt > 0) {
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
    } else {
      if (!p.nolo) {
        // fp32 W: tile (half, class) holds bf16 hi in A rows 0-7 and the lo residual in 8-15
        const int hs = tt < p.CPR0 ? 0 : 1, c = tt < p.CPR0 ? tt : tt - p.CPR0;
        const int rho = hs * 8 + g;
        for (int k = 0; k < 4; ++k) {
          float w = 0.f;
          if (p.slot_op[rho] >= 0) {
            const int o = p.slot_op[rho], rem = p.slot_rem[rho];
            const int jj = h * p.gqa + rem / p.n_q, nq = rem % p.n_q;
            if (c < p.op_classes[o]) {
              const size_t wi = ((((size_t)c * p.n_layers + l) * Hq + jj) * p.n_q + nq) * p.head_dim + d0 + k;
              w = p.w_bf16[o] ? __bfloat162float(__ushort_as_bfloat16(p.w_bf16[o][wi])) : p.w[o][wi];
            }
          }
          const __nv_bfloat16 hi = __float2bfloat16_rn(w);
          const __nv_bfloat16 lo = __float2bfloat16_rn(w - __bfloat162float(hi));
          vals[0][k] = __bfloat16_as_ushort(hi);  // A rows 0-7: W_hi
          vals[1][k] = __bfloat16_as_ushort(lo);  // A rows 8-15: W_lo
        }
      } else {
        // bf16 W (exact): tile = (half, class pair); class 2τ' in A rows 0-7, 2τ'+1 in 8-15
        const int T0 = (p.CPR0 + 1) / 2;
        const int hs = tt < T0 ? 0 : 1, c0 = 2 * (tt < T0 ? tt : tt - T0);
        const int rho = hs * 8 + g;
        for (int hr = 0; hr < 2; ++hr)
          for (int k = 0; k < 4; ++k) {
            uint16_t b = 0;
            const int c = c0 + hr;
            if (p.slot_op[rho] >= 0) {
              const int o = p.slot_op[rho], rem = p.slot_rem[rho];
              const int jj = h * p.gqa + rem / p.n_q, nq = rem % p.n_q;
              if (c < p.op_classes[o])
                b = p.w_bf16[o][((((size_t)c * p.n_layers + l) * Hq + jj) * p.n_q + nq) * p.head_dim + d0 + k];
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
  flush_counts(s_cnt, 1, p.counts);
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
    if (k == KO_C_FP) v = (long long)s_cnt[KO_C_OUT] - s_cnt[KO_C_TP];
    if (k == KO_C_FN) v = (long long)s_cnt[KO_C_GOLD] - s_cnt[KO_C_TP];
    if (v) atomicAdd(&p.counts[k], (unsigned long long)v);
  }
}

// G-plan grid on precomputed margins: one warp per tuple, one lane per plan
__global__ void reduce_kernel(const __grid_constant__ ReduceParams p) {
  __shared__ int s_cnt[kMaxPlans * kCountsPerPlan];
  __shared__ ko_plan s_plans[kMaxPlans];  // lanes read different plans: smem, not the param bank
  for (int i = threadIdx.x; i < p.n_plans * (int)(sizeof(ko_plan) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s_plans)[i] = reinterpret_cast<const uint32_t*>(p.plans)[i];
  __shared__ float s_m[8][kMaxOps * kMaxVar];
  __shared__ int32_t s_c[8][kMaxOps * kMaxVar];
  for (int i = threadIdx.x; i < p.n_plans * kCountsPerPlan; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int nmv = p.n_ops * p.n_variants;
  for (int64_t t = (int64_t)blockIdx.x * nw + w; t < p.n_tuples; t += (int64_t)gridDim.x * nw) {
    for (int idx = lane; idx < nmv; idx += 32) {
      s_m[w][idx] = p.margins[(size_t)idx * p.n_tuples + t];
      s_c[w][idx] = p.classes ? p.classes[(size_t)idx * p.n_tuples + t] : 0;
    }
    __syncwarp();
    for (int gp = lane; gp < p.n_plans; gp += 32)
      eval_plan(s_plans[gp], s_m[w], s_c[w], p.n_variants, p.n_classes, p.gold, p.n_tuples, t,
                s_cnt + gp * kCountsPerPlan);
    __syncwarp();
  }
  flush_counts(s_cnt, p.n_plans, p.counts);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
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
  const int nzg = p.n_ops_total * p.n_var_total * CPR;
  const int nu = min(p.cut[p.var_local[v]], p.n_layers) * p.n_kv_heads;  // l-major units
  const float* src = p.part + (size_t)t * p.n_lh_all * nzg + (size_t)(o * p.n_var_total + v) * CPR;
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
      uint32_t state = p.pos == 0 ? 1u : __ldcg(p.tuple_state + t);
      uint32_t done = p.pos == 0 ? 0xFFFFFFFFu : __ldcg(p.tuple_done + t);  // 4-bit round+1 per group
      {
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

template <int D, int CPR0, int CPR1, bool NOLO, int TNT>
cudaError_t launch_score_t(const ScoreParams& p, int64_t max_units, cudaStream_t s) {
  static int occ = 0;
  constexpr int smem = Ring<D>::kSmemBytes;
  auto* kern = ko_score_kernel<D, CPR0, CPR1, NOLO, TNT>;
  if (!occ) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t warps_needed = max_units > 0 ? max_units : 1;
  int64_t grid = (int64_t)num_sms() * occ;
  const int64_t need = (warps_needed + (kThreads / 32) - 1) / (kThreads / 32);
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, smem, s>>>(p);
  return cudaGetLastError();
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

template <int KSM, bool TM>  // k-steps of 16 dims (dim ≤ 16·KSM); TM: tensor-map loads
__global__ void __launch_bounds__(kEmbWarps * 32) embed_mma_kernel(const __grid_constant__ EmbedParams p) {
  extern __shared__ __align__(128) uint8_t emb_sm[];
  __shared__ __align__(8) uint64_t bar[kEmbWarps][kEmbStages];
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
  if (lane == 0) {
    for (int s = 0; s < kEmbStages; ++s) mbar_init(&bar[warp][s], 1);
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
  auto tuple_of = [&](int64_t w) -> int64_t { return p.tuple_idx ? (int64_t)p.tuple_idx[w] : w; };
  auto issue = [&]() {
    const int slot = issued % kEmbStages;
    const int64_t w0 = next * kEmbRows;
    const int rows = (int)(n - w0 < kEmbRows ? n - w0 : kEmbRows);
    if constexpr (TM) {  // NB boxes (64 dims × 16 rows); out-of-range rows / dims are zero-filled
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
    // gathered rows: one 1-D bulk copy per row, all issued by lane 0 (a bulk copy takes uniform
    // operands; lanes issuing their own rows would be serialised by the compiler anyway)
    const int64_t tl = lane < rows ? tuple_of(w0 + lane) : 0;
    if (lane == 0) mbar_expect_tx(&bar[warp][slot], row_bytes * rows);
    for (int r = 0; r < rows; ++r) {
      const int64_t t = __shfl_sync(0xffffffffu, tl, r);
      if (lane == 0)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
            "%2, [%3], %4;" ::"r"(ring_s + slot * SB + r * RS),
            "l"(p.item_emb + (size_t)t * dim), "r"(row_bytes), "r"(smem_u32(&bar[warp][slot])),
            "l"(policy)
            : "memory");
    }
    ++issued;
    next += nw;
  };
  for (int k = 0; k < kEmbStages && next < n_blk; ++k) issue();
  // ldmatrix row address of this lane inside a stage: matrix (lane / 8) = (rows +8·(m&1),
  // dims +8·(m>>1)); row (lane & 7)
  const uint32_t lrow = (uint32_t)((lane & 7) + 8 * ((lane >> 3) & 1)) * RS + 16 * (lane >> 4);
  for (int64_t blk = (int64_t)blockIdx.x * kEmbWarps + warp; blk < n_blk; blk += nw) {
    const int slot = consumed % kEmbStages;
    mbar_wait(&bar[warp][slot], (consumed / kEmbStages) & 1u);
    const uint32_t st = ring_s + slot * SB + (TM ? 0u : lrow);
    // two accumulator sets (even / odd k-steps) halve the MMA dependency chains
    float dd[2][4] = {}, g0[2][4] = {}, g1[2][4] = {};
#pragma unroll
    for (int ks = 0; ks < KSM; ++ks) {
      if (ks < KS) {
        uint32_t a[4];
        if constexpr (TM) {
          // box ks/4, 16-byte chunk 2·(ks%4) + (matrix ≥ 2), XORed with the row (128B swizzle)
          const int r = (lane & 7) + 8 * ((lane >> 3) & 1);
          const int c = 2 * (ks & 3) + (lane >> 4);
          ldsm_x4(a, st + (ks >> 2) * (kEmbRows * 128) + r * 128 + ((c ^ (r & 7)) << 4));
        } else {
          ldsm_x4(a, st + 32 * ks);
        }
        mma16816b(dd[ks & 1], a, bq[ks][0], bq[ks][1]);
        mma16816b(g0[ks & 1], a, a[0], a[2]);
        mma16816b(g1[ks & 1], a, a[1], a[3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dd[0][i] += dd[1][i];
      g0[0][i] += g0[1][i];
      g1[0][i] += g1[1][i];
    }
    __syncwarp();
    ++consumed;
    if (next < n_blk) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue();
    }
    // squared norms of tuples g and g + 8 sit in lane (g, g/2): G0[g][g], G1[g + 8][g + 8]
    const float gsel0 = (g & 1) ? g0[0][1] : g0[0][0];
    const float gsel1 = (g & 1) ? g1[0][3] : g1[0][2];
    const float n0 = __shfl_sync(0xffffffffu, gsel0, 4 * g + (g >> 1));
    const float n1 = __shfl_sync(0xffffffffu, gsel1, 4 * g + (g >> 1));
    const int64_t w0 = blk * kEmbRows;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int64_t w = w0 + g + 8 * hr;
      if (w >= n) continue;
      const int64_t t = tuple_of(w);
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
    if (p.use_tmap) {
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

cudaError_t launch_score(const ScoreParams& p, int head_dim, int CPR0, int CPR1, bool nolo,
                         int tnt, int64_t max_units, cudaStream_t s) {
#define KO_DISPATCH(DD, C0, C1)                                                       \
  if (head_dim == DD && CPR0 == C0 && CPR1 == C1 && !nolo && tnt == 0)               \
    return launch_score_t<DD, C0, C1, false, 0>(p, max_units, s);
#define KO_DISPATCH_NOLO(DD, C0, C1)                                                  \
  if (head_dim == DD && CPR0 == C0 && CPR1 == C1 && nolo && tnt == 0)                \
    return launch_score_t<DD, C0, C1, true, 0>(p, max_units, s);
#define KO_DISPATCH_TBL(DD, C0, T)                                                    \
  if (head_dim == DD && CPR0 == C0 && tnt == T)                                      \
    return launch_score_t<DD, C0, 0, false, T>(p, max_units, s);
#define KO_DISPATCH_D(DD)                                                                  \
  KO_DISPATCH(DD, 1, 0) KO_DISPATCH(DD, 1, 1) KO_DISPATCH(DD, 2, 0) KO_DISPATCH(DD, 2, 1)   \
  KO_DISPATCH(DD, 2, 2) KO_DISPATCH(DD, 4, 0) KO_DISPATCH(DD, 4, 1) KO_DISPATCH(DD, 4, 2)   \
  KO_DISPATCH(DD, 4, 4) KO_DISPATCH(DD, 8, 0) KO_DISPATCH(DD, 8, 1) KO_DISPATCH(DD, 8, 2)   \
  KO_DISPATCH(DD, 8, 4) KO_DISPATCH(DD, 8, 8)                                              \
  KO_DISPATCH_NOLO(DD, 2, 0) KO_DISPATCH_NOLO(DD, 4, 0) KO_DISPATCH_NOLO(DD, 8, 0)          \
  KO_DISPATCH_NOLO(DD, 2, 1) KO_DISPATCH_NOLO(DD, 4, 1) KO_DISPATCH_NOLO(DD, 8, 1)          \
  KO_DISPATCH_TBL(DD, 1, 1) KO_DISPATCH_TBL(DD, 1, 2) KO_DISPATCH_TBL(DD, 1, 4)             \
  KO_DISPATCH_TBL(DD, 2, 1) KO_DISPATCH_TBL(DD, 2, 2) KO_DISPATCH_TBL(DD, 2, 4)             \
  KO_DISPATCH_TBL(DD, 4, 2) KO_DISPATCH_TBL(DD, 4, 4) KO_DISPATCH_TBL(DD, 4, 8)             \
  KO_DISPATCH_TBL(DD, 8, 4) KO_DISPATCH_TBL(DD, 8, 8)
  KO_DISPATCH_D(64)
  KO_DISPATCH_D(128)
#undef KO_DISPATCH_D
#undef KO_DISPATCH_TBL
#undef KO_DISPATCH_NOLO
#undef KO_DISPATCH
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
cudaError_t launch_final_counts(const RouteParams& p, cudaStream_t s) {
  final_counts_kernel<<<num_sms() * 2, 256, 0, s>>>(p);
  return cudaGetLastError();
}
cudaError_t launch_reduce(const ReduceParams& p, cudaStream_t s) {
  reduce_kernel<<<num_sms() * 2, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ko
