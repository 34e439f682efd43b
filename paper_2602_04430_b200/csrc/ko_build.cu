// ko_build.cu — offline importance-ordered KV-cache builder (NEXT-4).
//
// The paper prefills every item once and compresses its cache with query-agnostic Expected
// Attention.  The variant knob of this library (keep‰ = a prefix) needs each tuple's
// tokens stored in descending expected attention per (layer, kv-head) (Q2).  This kernel builds
// such a store from a cache in natural token order.  A persistent CTA takes one unit =
// (tuple, layer, kv-head) at a time; every byte moves through the tensor-memory accelerator:
//   1. score: the unit's K rows come in by TMA (2-D view of the pool, box 64 d × 16 tokens,
//      128B swizzle) into a ring of 8 page slots, loaded L2 evict_last so step 3 can find them
//      in L2; one thread per token computes s_i = (Σ_d μ_d k_d)/√D + (Σ_d σ²_d k_d²)/(2D) in fp64,
//      d ascending, one rounding per operation (__dmul_rn/__dadd_rn, no fused multiply-add), so
//      the order is decided exactly as the oracle decides it (Q25); the swizzle makes the 8
//      threads of a quarter-warp read 8 distinct bank groups;
//   2. bitonic sort of (s desc, index asc) in shared memory (L ≤ 4096);
//   3. gather: destination page chunk (16 ranks × one of K/V) ← 4 TMA row gathers
//      (tile::gather4, 4 whole source rows per op, unswizzled) into a ring slot, then one TMA
//      store of the 16-row box into the destination page — lane 0 of each of 4 warps drives 2
//      slots, one chunk ahead; K chunks go first, newest-scored pages first (most L2 hits); a
//      last partial page is written row by row (slots past L are not written).
// Every phase's copies are asynchronous; the CTA is small (≈ 47 KB of shared memory), so 4 CTAs
// per SM overlap each other's score, sort and gather phases.  TMA cost is per operation, so the
// ops are as large as the layout allows.  Measured variants: DESIGN.md §4c.
// Two launches sized by token count (≤ 1024, ≤ 4096): the sort keys' shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdio>

#include "ko_device.cuh"
#include "ko_internal.h"

namespace ko {
namespace {

constexpr int kBuildThreads = 256;
constexpr int kBuildMaxTokens = 4096;
constexpr int kBuildSmallTokens = 1024;
constexpr int kBuildSlotBytes = 4096;    // 16 rows × 128 d × bf16 (D = 64 uses half)

__device__ __forceinline__ double bf16_to_double(uint32_t b) {
  return (double)__uint_as_float(b << 16);
}

// a precedes b: higher score first, then lower original index
__device__ __forceinline__ bool precedes(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int x, int y0,
                                            int y1, int y2, int y3, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y0), "r"(y1), "r"(y2), "r"(y3),
      "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, uint32_t src,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::
          "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(src), "l"(policy)
      : "memory");
}

template <int MAXT, int SLOTS>
constexpr size_t build_smem_bytes() {
  return 1024 /* swizzle-atom alignment slack */ + (size_t)SLOTS * kBuildSlotBytes +
         (size_t)MAXT * (sizeof(double) + sizeof(int)) + 2 * sizeof(double) * 128 +
         2 * sizeof(int) * (MAXT / 16);
}

// this kernel's units: MINT < L ≤ MAXT; SLOTS ring slots (one 16-token page of one head each)
// (256, 4): the 64-register budget of 4 CTAs per SM; without the minimum ptxas kept 48 registers
// and spilled two loop counters (same-box A/B: 6.59 → 6.43 ms)
template <int MAXT, int MINT, int SLOTS, int kGatherWarps>
__global__ void __launch_bounds__(kBuildThreads, 4) build_kernel(const __grid_constant__ BuildParams p) {
  constexpr int kGatherSlots = SLOTS / kGatherWarps;  // per gather warp
  constexpr int kGatherAhead = kGatherSlots / 2;      // chunks a gather warp issues ahead
  extern __shared__ uint8_t bsm_raw[];
  __shared__ __align__(8) uint64_t sbar;               // score rounds
  __shared__ __align__(8) uint64_t gbar[SLOTS];  // gather chunks, one per ring slot
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(bsm_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const uint32_t ring_s = smem_u32(ring);
  double* key = reinterpret_cast<double*>(ring + SLOTS * kBuildSlotBytes);  // [MAXT]
  int* idx = reinterpret_cast<int*>(key + MAXT);                                 // [MAXT]
  double* s_mu = reinterpret_cast<double*>(idx + MAXT);                          // [D]
  double* s_s2 = s_mu + 128;                                                     // [D]
  int* s_src = reinterpret_cast<int*>(s_s2 + 128);                               // [MAXT/16]
  int* s_dst = s_src + MAXT / 16;                                                // [MAXT/16]

  const int D = p.head_dim, H = p.n_kv_heads, Lyr = p.n_layers;
  const int NB = D / 64;                 // 64-d boxes per row (D ∈ {64, 128})
  const int RP = 2 * Lyr * H * 16;       // rows (of D elements) per page in the 2-D view
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, n_warps = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&sbar, 1);
    for (int s = 0; s < SLOTS; ++s) mbar_init(&gbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t keep, stream;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(stream));
  uint32_t sphase = 0;  // parity of sbar's current phase
  uint32_t gq = 0;      // gather chunks this warp has issued (its slot g % S, parity (g / S) & 1)

  const int64_t n_units = p.n_tuples * Lyr * H;
#ifdef KO_BUILD_PROF
  long long tp[5] = {0, 0, 0, 0, 0}, t0c = clock64(), nu = 0;
#define PROF_MARK(i) do { long long c_ = clock64(); tp[i] += c_ - t0c; t0c = c_; } while (0)
#else
#define PROF_MARK(i) do {} while (0)
#endif
  __shared__ int s_first;
  for (int64_t u0 = blockIdx.x;;) {
    // this CTA's next unit (stride gridDim.x) whose tuple this launch builds — MINT < L ≤ MAXT;
    // the other launch's (or > 4096: documented, skipped) are passed over 256 candidates per
    // round, one seq_len load per thread, instead of one dependent load per unit
    int64_t u = -1;
    for (int64_t base = u0; base < n_units && u < 0;
         base += (int64_t)kBuildThreads * gridDim.x) {
      const int64_t c = base + (int64_t)threadIdx.x * gridDim.x;
      bool ok = false;
      if (c < n_units) {
        const int Lc = p.seq_len[c / (Lyr * H)];
        KO_DCHECK(Lc >= 1);
        ok = Lc > MINT && Lc <= MAXT;
      }
      __syncthreads();  // the previous round's s_first is read (and the previous unit is done)
      if (threadIdx.x == 0) s_first = 0x7fffffff;
      __syncthreads();
      if (ok) atomicMin(&s_first, (int)threadIdx.x);
      __syncthreads();
      if (s_first != 0x7fffffff) u = base + (int64_t)s_first * gridDim.x;
    }
    if (u < 0) break;
    u0 = u + gridDim.x;
    const int64_t t = u / (Lyr * H);
    const int l = (int)((u / H) % Lyr), h = (int)(u % H);
    const int L = p.seq_len[t];
    const int n_pg = (L + 15) >> 4;
    __syncthreads();  // the previous unit's keys / page ids are dead
    const int64_t pbase = p.indptr[t];
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      s_mu[d] = (double)p.mu[((size_t)l * H + h) * D + d];
      s_s2[d] = (double)p.sigma2[((size_t)l * H + h) * D + d];
    }
    for (int i = threadIdx.x; i < n_pg; i += blockDim.x) {
      s_src[i] = p.src_ids[pbase + i];
      s_dst[i] = p.dst_ids[pbase + i];
      KO_DCHECK(s_src[i] >= 0 && s_src[i] < p.n_pages && s_dst[i] >= 0 && s_dst[i] < p.n_pages);
    }
    __syncthreads();
    const int row_k = (2 * l * H + h) * 16, row_v = ((2 * l + 1) * H + h) * 16;  // in-page rows
    PROF_MARK(0);

    // ---- 1. scores, R pages (16·R tokens) per round, one thread per token
    int N = 64;  // ≥ one warp segment (padding sorts last)
    while (N < L) N <<= 1;
    for (int pg0 = 0; pg0 < n_pg; pg0 += SLOTS) {
      const int np = min(SLOTS, n_pg - pg0);
      if (threadIdx.x == 0) {
        // the ring's previous contents were read through the generic proxy (scores, partial
        // pages) or by bulk stores (drained at the end of the gather): order those reads
        // before the async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sbar, (uint32_t)(np * NB * 2048));
        for (int j = 0; j < np; ++j)
          for (int b = 0; b < NB; ++b)
            tma_load_2d(ring_s + j * kBuildSlotBytes + b * 2048, &p.tm_src, 64 * b,
                        s_src[pg0 + j] * RP + row_k, &sbar, keep);
      }
      // one warp polls the round's barrier; the rest sleep in the CTA barrier instead of
      // spinning on try_wait (the spin took 5 % of the issue slots the other CTAs need)
      if (warp == 0) mbar_wait(&sbar, sphase);
      __syncthreads();
      sphase ^= 1u;
      PROF_MARK(4);
      const int i = pg0 * 16 + threadIdx.x;
      if (threadIdx.x < np * 16 && i < L) {
        const int j = threadIdx.x >> 4, r = threadIdx.x & 15;
        const uint32_t rowa = ring_s + j * kBuildSlotBytes + r * 128;
        double a = 0.0, bq = 0.0;
        for (int b = 0; b < NB; ++b) {
          uint4 vv[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) vv[c] = lds128(rowa + b * 2048 + ((c ^ (r & 7)) << 4));
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int d = 64 * b + 8 * c;
            const uint32_t w[4] = {vv[c].x, vv[c].y, vv[c].z, vv[c].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const double x = bf16_to_double(e & 1 ? w[e >> 1] >> 16 : w[e >> 1] & 0xFFFFu);
              a = __dadd_rn(a, __dmul_rn(s_mu[d + e], x));
              bq = __dadd_rn(bq, __dmul_rn(s_s2[d + e], __dmul_rn(x, x)));
            }
          }
        }
        key[i] = __dadd_rn(__dmul_rn(a, p.inv_sqrt_d), __dmul_rn(bq, p.inv_2d));
        idx[i] = i;
      }
      __syncthreads();  // the ring slots are free for the next round
    }
    for (int i = L + threadIdx.x; i < N; i += blockDim.x) {
      key[i] = -CUDART_INF;
      idx[i] = 0x7fffffff;
    }
    __syncthreads();
    PROF_MARK(1);

    // ---- 2. bitonic sort: final order has precedes(i, i+1).  Phases whose pairs lie inside a
    // 64-element segment (j ≤ 32) run in registers, one warp per segment, lane holding elements
    // lane and lane + 32 (j = 32: in-lane, j < 32: shuffles); only the j ≥ 64 phases go through
    // shared memory with a CTA barrier — 6 barriers at N = 512 instead of 45.
    auto seg_phases = [&](int k_lo, int k_hi, int j_top) {  // levels k_lo..k_hi, first j ≤ j_top
      for (int seg = warp; seg < (N >> 6); seg += n_warps) {
        const int base = seg << 6;
        double kk[2] = {key[base + lane], key[base + lane + 32]};
        int ii[2] = {idx[base + lane], idx[base + lane + 32]};
        for (int k = k_lo; k <= k_hi; k <<= 1)
          for (int j = min(k >> 1, j_top); j > 0; j >>= 1) {
            if (j == 32) {  // pair (lane, lane + 32): both here, element lane is the lower
              const bool up = ((base + lane) & k) == 0;
              const bool swap = up ? precedes(kk[1], ii[1], kk[0], ii[0])
                                   : precedes(kk[0], ii[0], kk[1], ii[1]);
              if (swap) {
                const double tk = kk[0]; kk[0] = kk[1]; kk[1] = tk;
                const int ti = ii[0]; ii[0] = ii[1]; ii[1] = ti;
              }
            } else {
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int i = base + lane + 32 * hh;
                const double ko = __shfl_xor_sync(0xffffffffu, kk[hh], j);
                const int io = __shfl_xor_sync(0xffffffffu, ii[hh], j);
                const bool up = (i & k) == 0, lower = (lane & j) == 0;
                // the lower position keeps the element that comes first (up) / second (down)
                const bool other_first = precedes(ko, io, kk[hh], ii[hh]);
                if (lower == (up == other_first) && (ko != kk[hh] || io != ii[hh])) {
                  kk[hh] = ko;
                  ii[hh] = io;
                }
              }
            }
          }
        key[base + lane] = kk[0]; key[base + lane + 32] = kk[1];
        idx[base + lane] = ii[0]; idx[base + lane + 32] = ii[1];
      }
      __syncthreads();
    };
    seg_phases(2, 64, 32);  // every level up to 64 lies inside segments
    for (int k = 128; k <= N; k <<= 1) {
      for (int j = k >> 1; j >= 64; j >>= 1) {
        for (int q = threadIdx.x; q < (N >> 1); q += blockDim.x) {  // one thread per pair
          const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1)), ixj = i | j;  // bit j of i clear
          const bool up = (i & k) == 0;  // this pair must end in `precedes` order
          const double ka = key[i], kb = key[ixj];
          const int ia = idx[i], ib = idx[ixj];
          const bool swap = up ? precedes(kb, ib, ka, ia) : precedes(ka, ia, kb, ib);
          if (swap) {
            key[i] = kb; key[ixj] = ka;
            idx[i] = ib; idx[ixj] = ia;
          }
        }
        __syncthreads();
      }
      seg_phases(k, k, 32);
    }

    // ---- 3. gather: chunk c = (destination page, K or V) — order below.  All threads
    // first resolve every chunk's 16 source rows (rank r ← token idx[r]) into the dead key array;
    // then lane 0 of each of kGatherWarps warps runs its chunks (c ≡ warp mod kGatherWarps)
    // through kGatherSlots ring slots of its own: 4 gather4 ops bring the 16 whole rows in
    // (unswizzled: the rows are only copied), one TMA store of the 16-row box writes them out
    // kGatherAhead chunks later.  TMA cost is per operation, so the ops are as large as allowed.
    PROF_MARK(2);
    // chunk order: K of the full pages newest-loaded first (the score pass left them in L2),
    // then V of the full pages, then the last page's K and V (the last two chunks, so their
    // slots are not reused when the page is partial)
    auto chunk_of = [&](int c, int& pg, int& which) {
      const int nf = n_pg - 1;
      if (c < nf) { pg = nf - 1 - c; which = 0; }
      else if (c < 2 * nf) { pg = c - nf; which = 1; }
      else { pg = nf; which = c - 2 * nf; }
    };
    int* crow = reinterpret_cast<int*>(key);  // [2·n_pg][16] source rows (2·MAXT/16·16 ≤ 2·MAXT)
    const int n_ch = 2 * n_pg;
    for (int e = threadIdx.x; e < n_ch * 16; e += blockDim.x) {
      int pg, which;
      chunk_of(e >> 4, pg, which);
      const int rank = pg * 16 + (e & 15);
      const int tok = idx[rank < L ? rank : pg * 16];  // past L: any loaded row (never stored)
      crow[e] = s_src[tok >> 4] * RP + (which ? row_v : row_k) + (tok & 15);
    }
    __syncthreads();
    if (warp < kGatherWarps) {
      const int nk = (n_ch - warp + kGatherWarps - 1) / kGatherWarps;  // this warp's chunks
      if (lane == 0) {
        for (int k = 0; k < nk + kGatherAhead; ++k) {
          if (k < nk) {
            const int c = warp + k * kGatherWarps;
            const uint32_t g = gq + k, slot = warp * kGatherSlots + g % kGatherSlots;
            // the slot's previous store (this warp's chunk g − S) must have read its smem: the
            // stores of chunks ≤ g − kGatherAhead − 1 are issued (one bulk group each)
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kGatherSlots - kGatherAhead - 1)
                         : "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&gbar[slot], (uint32_t)(32 * D));
            const int4* rr = reinterpret_cast<const int4*>(crow + c * 16);
            for (int q = 0; q < 4; ++q) {  // rows 4q..4q+3, whole rows (unswizzled: no compute)
              const int4 r4 = rr[q];
              tma_gather4(ring_s + slot * kBuildSlotBytes + q * 8 * D, &p.tm_row, 0, r4.x, r4.y,
                          r4.z, r4.w, &gbar[slot], stream);
            }
          }
          const int kj = k - kGatherAhead;
          if (kj >= 0 && kj < nk) {
            const int c = warp + kj * kGatherWarps;
            int pg, which;
            chunk_of(c, pg, which);
            const uint32_t g = gq + kj, slot = warp * kGatherSlots + g % kGatherSlots;
            if (pg * 16 + 16 <= L) {
              mbar_wait(&gbar[slot], (g / kGatherSlots) & 1u);
              tma_store_2d(&p.tm_dst, 0, s_dst[pg] * RP + (which ? row_v : row_k),
                           ring_s + slot * kBuildSlotBytes, stream);
            }  // a partial last page is written by the whole warp below
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // (maybe empty) group
          }
        }
      }
      __syncwarp();
      // last partial page (its K and V chunks are the last two, so their slots were not reused):
      // rows < nv through registers — slots past L are not written
      const int nv = L - (n_pg - 1) * 16;
      if (nv < 16) {
        for (int c = n_ch - 2; c < n_ch; ++c) {
          if (c % kGatherWarps != warp) continue;
          const int kc = c / kGatherWarps, which = c - (n_ch - 2);
          const uint32_t g = gq + kc, slot = warp * kGatherSlots + g % kGatherSlots;
          mbar_wait(&gbar[slot], (g / kGatherSlots) & 1u);
          const int cpr = D / 8;  // 16-byte chunks per row
          uint16_t* dst = p.dst_pool + (size_t)s_dst[n_pg - 1] * p.page_elems +
                          (size_t)(which ? row_v : row_k) * D;
          for (int w = lane; w < nv * cpr; w += 32) {
            const int r = w / cpr, cc = w % cpr;
            const uint4 v = lds128(ring_s + slot * kBuildSlotBytes + r * 2 * D + cc * 16);
            __stcs(reinterpret_cast<uint4*>(dst + (size_t)r * D + cc * 8), v);
          }
        }
      }
      // the next unit's score loads reuse the ring: the stores must have read their slots
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      gq += (uint32_t)nk;
    }
    PROF_MARK(3);
#ifdef KO_BUILD_PROF
    ++nu;
#endif
  }
#ifdef KO_BUILD_PROF
  if ((blockIdx.x == 0 || blockIdx.x == 1) && (threadIdx.x == 0 || threadIdx.x == 32 * kGatherWarps))
    printf("blk %d thr %d units %lld: setup %lld load-wait %lld score %lld sort %lld gather %lld (cycles/unit)\n",
           blockIdx.x, threadIdx.x, nu, tp[0] / max(nu, 1ll), tp[4] / max(nu, 1ll), tp[1] / max(nu, 1ll),
           tp[2] / max(nu, 1ll), tp[3] / max(nu, 1ll));
#endif
  if (warp < kGatherWarps && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MAXT, int MINT, int SLOTS, int GW>
cudaError_t launch_build_t(const BuildParams& p, cudaStream_t s) {
  auto kern = build_kernel<MAXT, MINT, SLOTS, GW>;
  constexpr size_t smem = build_smem_bytes<MAXT, SLOTS>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBuildThreads, smem);
  const int64_t units = p.n_tuples * p.n_layers * p.n_kv_heads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)num_sms() * std::max(occ, 1)));
  kern<<<grid, kBuildThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_build(const BuildParams& p, cudaStream_t s) {  // 2 launches
  // A/B on C2 geometry (2000 × 512 tokens, profiles/r02_build.md): 8 slots with 4 gather warps
  // (4 CTAs/SM) 6.58 ms; 12 slots 7.22; 16 slots (2 CTAs/SM, K re-read all from L2) 8.03; 4–6
  // slots or 1–2 gather warps 6.9–8.2; score loads or gather through registers 7.6–9.5
  cudaError_t e = launch_build_t<kBuildSmallTokens, 0, 8, 4>(p, s);
  if (e != cudaSuccess) return e;
  return launch_build_t<kBuildMaxTokens, kBuildSmallTokens, 8, 4>(p, s);
}

}  // namespace ko
