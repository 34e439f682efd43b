// ko_score.cuh — the hot kernel ko_score_kernel<D, CPR, NT> and its launcher
// template; instantiated per head_dim and packing family in ko_score_*.cu so the instantiations
// compile in parallel.
//
// One warp owns one work unit = (tuple t, layer l, HG kv-heads) and streams that unit's K and V
// rows (importance order, page by page) from HBM through a per-warp TMA ring
// (cp.async.bulk.tensor, 128B swizzle, mbarrier completion).  Per 16-token page:
//   S = Q · Kᵀ        on tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate): the rows
//                     attending a kv-head (n_ops · gqa · n_q ≤ 16) are the M dimension, the
//                     page's tokens N, head_dim K;
//   U = W · Vᵀ        same shape: the readout W of every row/class is folded through V, so the
//                     logit contribution of a row is Σ_i softmax_i · U_i (linearity of
//                     z = b + W·O); fp32 W enters as bf16 hi + lo;
//   online softmax    lane-local running (max, sum, Σ p·u) per row over the lane's own tokens,
//                     merged across the 4 lanes of a quad only at variant snapshots;
//   snapshots         tokens are in importance order, so every keep ratio is a prefix: the
//                     state is snapshot when the token index reaches each variant's n_kept, so
//                     one read serves every variant (nested prefixes, Q2); layer cuts select
//                     which units a variant sums.
// Grid mode: the warp completing a tuple's last unit sums the partial logits in a FIXED order
// (bitwise-deterministic margins) and evaluates every plan.  Walk (routed) mode: a round streams
// only the tokens past the tuple's previous extent, resuming the saved softmax state, and
// ko_walk_kernel finishes the round.  Layout, packings and roofline: DESIGN.md §4.
#pragma once

#include "ko_device.cuh"

namespace ko {
namespace {

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

// Table packing: the W·V tiles are packed per lane group g from a host table — A-row half hr of
// tile tt at lane group g is slot k = 2·tt + hr, which accumulates with S row g + 8·hr for the
// (op, class) tgt[k]; a row with more entries than one half's NT slots is duplicated into both
// halves.  CPR: class stride of the grid-mode partials (pow2 ≥ every op's
// classes); NT: W·V tiles.
template <int D, int CPR, int NT>
__global__ void __launch_bounds__(kThreads, 2) ko_score_kernel(const __grid_constant__ ScoreParams p) {
  constexpr int KS = D / 16;  // mma k-steps over head_dim
  constexpr int KP = D / 32;  // 128-bit fragment reads per token row per lane (2 k-steps each)
  constexpr int NSL = 2 * NT;                       // table slots per lane
  constexpr int kRecW = (4 + NSL + 7) / 8 * 8;      // saved-state record (walk), whole sectors
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
  // walk: ko_walk_kernel counts; grid with fin_kernel: grid_final_kernel counts
  const int n_cnt_rows = p.mode == MODE_GRID && !p.fin_kernel ? p.n_plans : 0;
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
  {
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

  // walk-mode partial blocks ([op][part_cpr], whole sectors): lane j < wblk owns position j =
  // (caller's op og, class c) — its value is the target sum of lane (local op)·8 + c; zero for
  // classes past the op's count and for the padding; ops outside this launch: not written
  const int wblk = walk ? walk_part_blk(p.n_ops_total, p.part_cpr) : 0;
  int wsrc = 0;
  bool wown = false, wzero = false;
  if (lane < wblk) {
    const int og = lane / p.part_cpr, c = lane - og * p.part_cpr;
    if (og >= p.n_ops_total) {
      wown = wzero = true;
    } else {
      for (int ol = 0; ol < p.n_ops; ++ol)
        if (p.op_ids[ol] == og) {
          wown = true;
          wzero = c >= p.op_classes[ol];
          wsrc = wzero ? 0 : ol * 8 + c;
        }
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
    KO_DCHECK(U.t >= 0 && U.t < p.n_tuples);
    U.L = p.seq_len[U.t];
    KO_DCHECK(U.L >= 1);
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
    KO_DCHECK(U.pid_reg >= 0 && U.pid_reg < p.n_pages);
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
      KO_DCHECK(U.pid_reg >= 0 && U.pid_reg < p.n_pages);
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
    KO_DCHECK(!walk || p.rstate_w == kRecW);
    float* rst = walk ? p.rstate + ((((size_t)t * p.n_layers + l) * Hkv + h) * 8 + g) * kRecW
                      : nullptr;

    // lane-local online-softmax state per half-slot (log2 domain)
    float mx[2], sm[2], at[NSL];
#pragma unroll
    for (int hs = 0; hs < 2; ++hs) {
      mx[hs] = kNoMax;
      sm[hs] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < NSL; ++k) at[k] = 0.f;
    if (walk && s0 > 0 && q == 0) {  // resume: the quad's merged state enters through lane q = 0
      mx[0] = __ldcg(rst + 0);
      mx[1] = __ldcg(rst + 1);
      sm[0] = __ldcg(rst + 2);
      sm[1] = __ldcg(rst + 3);
#pragma unroll
      for (int k = 0; k < NSL; ++k) at[k] = __ldcg(rst + 4 + k);
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
      // kEarly (one W·V tile, registers to spare): both n-tiles' K/V fragments are read first and
      // the stage goes back to the TMA before the MMAs; otherwise one n-tile at a time, the
      // stage handed back once the second n-tile's fragments are read
      constexpr bool kEarly = NT == 1;
      uint4 kfa[kEarly ? 2 : 1][KP], vfa[kEarly ? 2 : 1][KP];
      auto read_frags = [&](int nt, uint4* kf, uint4* vf) {
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
      };
      if constexpr (kEarly) {
        read_frags(0, kfa[0], vfa[0]);
        read_frags(1, kfa[1], vfa[1]);
        __syncwarp();
        ++consumed;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        refill();
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        uint4* kf = kfa[kEarly ? nt : 0];
        uint4* vf = vfa[kEarly ? nt : 0];
        if constexpr (!kEarly) {
          read_frags(nt, kf, vf);
          if (nt == 1) {  // the stage's last reads are issued: hand it back before these MMAs
            __syncwarp();
            ++consumed;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            refill();
          }
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
      // the fragments are dead after the last page's MMAs: fetch the next head's now
      if (pg + 1 == pg1 && hh + 1 < HG) load_frags(h + 1);
      // ---- per-lane token indices and values: k = nt*2 + e ↔ token pg*16 + nt*8 + 2q + e
      const int page_hi = min(pg * 16 + 16, n_need);
      for (;;) {
        const int seg_hi = min(next_snap, page_hi);
        // fold tokens [snap_lo, seg_hi) of this page into the lane-local state
        {
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
        }
        snap_lo = seg_hi;
        if (seg_hi == next_snap) {
          // ---- snapshot: merge the quad's lane states, reduce rows per op, emit partials
          {
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
            if (walk && p.save_state && next_snap == s1) {
              // end of this round's extent: save the merged state for a later round to resume.
              // The quad's 4 lanes hold the same merged values: lane q stores floats 8i + 2q and
              // 8i + 2q + 1 of the record (zero-padded to kRecW), so each warp store writes whole
              // 32-byte sectors (partial sectors cost DRAM write amplification)
              float rec[kRecW];
              rec[0] = Mq[0]; rec[1] = Mq[1]; rec[2] = den[0]; rec[3] = den[1];
#pragma unroll
              for (int k = 0; k < NSL; ++k) rec[4 + k] = accm[k];
#pragma unroll
              for (int k = 4 + NSL; k < kRecW; ++k) rec[k] = 0.f;
#pragma unroll
              for (int i = 0; i < kRecW / 8; ++i) {
                float a = rec[8 * i], b = rec[8 * i + 1];
                if (q == 1) { a = rec[8 * i + 2]; b = rec[8 * i + 3]; }
                if (q == 2) { a = rec[8 * i + 4]; b = rec[8 * i + 5]; }
                if (q == 3) { a = rec[8 * i + 6]; b = rec[8 * i + 7]; }
                *reinterpret_cast<float2*>(rst + 8 * i + 2 * q) = make_float2(a, b);
              }
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
            if (walk) {
              // per tuple (persisting across rounds), caller's (op, variant): lane j stores
              // position j of the variant's whole-sector block (value of lane wsrc, or zero)
              const float xv = __shfl_sync(0xffffffffu, x, wsrc);
              if (wown) {
#pragma unroll
                for (int v = 0; v < kMaxVar; ++v)
                  if (nkv[v] == next_snap)
                    p.part[(((size_t)t * p.n_var_total + p.var_ids[v]) * p.n_lh_all + unit_lh) * wblk +
                           lane] = wzero ? 0.f : xv;
              }
            } else if (red_n > 0) {
              // per work slot, local (op, variant): the grid finaliser's layout
              const int o = lane >> 3, c = lane & 7;
#pragma unroll
              for (int v = 0; v < kMaxVar; ++v)
                if (nkv[v] == next_snap)
                  p.part[((((size_t)wslot * p.n_l * Hkv + unit_lh) * p.n_ops + o) * p.n_var + v) *
                             CPR + c] = x;
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
    if (!walk && !p.fin_kernel) {
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
  if (n_cnt_rows) flush_counts(s_cnt, n_cnt_rows, p.counts, p.gold != nullptr);
}

// ------------------------------------------------------------------------------------------
// Fragment preparation: Q (bf16) and W (fp32 → bf16 hi + lo) into the per-lane register layout
// of mma.m16n8k16 with the d-permutation of DESIGN.md §"Kernel":
//   k-step ks = 2j + e, lane (g, q): A regs {a0a1, a2a3, a4a5, a6a7} hold
//   (row g, d0, d0+1), (row g+8, d0, d0+1), (row g, d0+2, d0+3), (row g+8, d0+2, d0+3),
//   d0 = 64(j/2) + 16q + 8(j%2) + 4e — exactly the 8 consecutive bf16 of the 16-byte chunk
//   (2q + j%2) of 64-wide box j/2 that lane (g, q) reads from the swizzled TMA stage.

template <int D, int CPR, int NT>
cudaError_t launch_score_t(const ScoreParams& p, int64_t max_units, cudaStream_t s) {
  // the smem attribute and the occupancy are per device: cached per device ordinal
  static std::atomic<int> occ_of[64];
  constexpr int smem = Ring<D>::kSmemBytes;
  auto* kern = ko_score_kernel<D, CPR, NT>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 63;
  int occ = occ_of[dev].load(std::memory_order_relaxed);
  if (!occ) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    if (occ < 1) occ = 1;
    occ_of[dev].store(occ, std::memory_order_relaxed);
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
// Grid-mode tuple finaliser as its own launch (fin_kernel = 1): one warp per work slot runs
// finalise_tuple on the partials the scoring launch left per work slot, so the scoring kernel's
// warps only stream (the routed mode's ko_walk_kernel split).  Same arithmetic,
// same fixed summation order: margins and counts are bitwise those of the in-kernel finaliser.
// ------------------------------------------------------------------------------------------
constexpr int kFinWarps = 16;
template <int CPR>
__global__ void __launch_bounds__(kFinWarps * 32) grid_final_kernel(const __grid_constant__ ScoreParams p) {
  __shared__ int s_cnt[kMaxPlans * kCountsPerPlan];
  __shared__ float s_z[kFinWarps][kMaxOps * kMaxVar * kMaxCls];
  __shared__ float s_m[kFinWarps][kMaxOps * kMaxVar];
  __shared__ int32_t s_c[kFinWarps][kMaxOps * kMaxVar];
  for (int i = threadIdx.x; i < p.n_plans * kCountsPerPlan; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n_work = p.work_len_host;
  for (int64_t w = (int64_t)blockIdx.x * kFinWarps + warp; w < n_work;
       w += (int64_t)gridDim.x * kFinWarps) {
    const int64_t t = p.work ? (int64_t)p.work[w] : w;
    finalise_tuple<CPR>(p, w, t, lane, s_z[warp], s_m[warp], s_c[warp], s_cnt);
  }
  flush_counts(s_cnt, p.n_plans, p.counts, p.gold != nullptr);
}

template <int CPR>
cudaError_t launch_grid_final_t(const ScoreParams& p, cudaStream_t s) {
  // latency-bound (L2 loads of the partials, gold, per-tuple plan walks): as many warps as fit
  static std::atomic<int> occ_of[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 63;
  int occ = occ_of[dev].load(std::memory_order_relaxed);
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_final_kernel<CPR>, kFinWarps * 32, 0);
    if (occ < 1) occ = 1;
    occ_of[dev].store(occ, std::memory_order_relaxed);
  }
  const int64_t need = (p.work_len_host + kFinWarps - 1) / kFinWarps;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)num_sms() * occ));
  grid_final_kernel<CPR><<<(unsigned)grid, kFinWarps * 32, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace
}  // namespace ko
