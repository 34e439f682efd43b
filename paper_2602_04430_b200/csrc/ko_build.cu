// ko_build.cu — offline importance-ordered KV-cache builder (NEXT-4).
//
// The paper prefills every item once and compresses its cache with query-agnostic Expected
// Attention.  The variant knob of this library (keep‰ = a prefix) needs each tuple's
// tokens stored in descending expected attention per (layer, kv-head) (Q2).  This kernel builds
// such a store from a cache in natural token order: one CTA per (tuple, layer, kv-head)
//   1. s_i = (Σ_d μ_d k_d)/√D + (Σ_d σ²_d k_d²)/(2D) for every token (Q25), fp64, left to right,
//      one rounding per operation (__dmul_rn/__dadd_rn: no fused multiply-add), so the order is
//      decided exactly as the oracle decides it;
//   2. bitonic sort of (s desc, index asc) in shared memory (L ≤ 4096);
// Two launches sized by token count: units with L ≤ 1024 go to a kernel with ~14 KB of shared
// memory, so several CTAs share an SM (their score / sort / gather phases overlap each other's memory
// traffic); the rare longer ones to the 4096-token kernel (51 KB).  Each skips the other's units.
//   3. gather: the K and V rows of rank r go to slot r % 16 of logical page r / 16 of the
//      destination CSR, 16-byte copies through registers.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>

#include "ko_device.cuh"
#include "ko_internal.h"

namespace ko {
namespace {

constexpr int kBuildThreads = 256;
constexpr int kBuildMaxTokens = 4096;
constexpr int kBuildSmallTokens = 1024;
// sort keys (doubles) of a MAXT kernel
template <int MAXT>
__host__ __device__ constexpr int key_slots() { return MAXT; }

__device__ __forceinline__ double bf16_to_double(uint16_t b) {
  return (double)__uint_as_float((uint32_t)b << 16);
}

// a precedes b: higher score first, then lower original index
__device__ __forceinline__ bool precedes(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

template <int MAXT, int MINT>  // this kernel's units: MINT < L ≤ MAXT
__global__ void __launch_bounds__(kBuildThreads) build_kernel(const __grid_constant__ BuildParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* key = reinterpret_cast<double*>(smem);                  // [key_slots]
  int* idx = reinterpret_cast<int*>(key + key_slots<MAXT>());     // [MAXT]
  double* s_mu = reinterpret_cast<double*>(idx + MAXT);           // [D] (exact fp32 → fp64)
  double* s_s2 = s_mu + p.head_dim;                                 // [D]
  const int D = p.head_dim, H = p.n_kv_heads, Lyr = p.n_layers;
  const int64_t n_units = p.n_tuples * Lyr * H;
  for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const int64_t t = u / (Lyr * H);
    const int l = (int)((u / H) % Lyr), h = (int)(u % H);
    const int L = p.seq_len[t];
    KO_DCHECK(L >= 1);
    if (L <= MINT || L > MAXT) continue;  // the other launch's (or > 4096: documented, skipped)
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      s_mu[d] = (double)p.mu[((size_t)l * H + h) * D + d];
      s_s2[d] = (double)p.sigma2[((size_t)l * H + h) * D + d];
    }
    __syncthreads();
    const int64_t pbase = p.indptr[t];
    // element offset of (layer l, K/V, kv-head h, slot 0) inside a page; slot s adds s·D
    const int off_k = ((l * 2 + 0) * H + h) * 16 * D, off_v = ((l * 2 + 1) * H + h) * 16 * D;
    auto src_row = [&](int which, int i) -> const uint16_t* {
      const int64_t page = p.src_ids[pbase + (i >> 4)];
      KO_DCHECK(page >= 0 && page < p.n_pages);
      return p.src_pool + (size_t)page * p.page_elems + (which ? off_v : off_k) + (i & 15) * D;
    };
    int N = 64;  // ≥ one warp segment (padding sorts last)
    while (N < L) N <<= 1;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      if (i < L) {
        const uint16_t* k = src_row(0, i);
        double a = 0.0, b = 0.0;
        for (int d0 = 0; d0 < D; d0 += 32) {  // 4 row loads in flight, then their 32 terms in order
          uint4 vv[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) vv[c] = __ldg(reinterpret_cast<const uint4*>(k + d0 + 8 * c));
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int d = d0 + 8 * c;
            const uint32_t w[4] = {vv[c].x, vv[c].y, vv[c].z, vv[c].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const double x = bf16_to_double((uint16_t)(e & 1 ? w[e >> 1] >> 16 : w[e >> 1] & 0xFFFFu));
              a = __dadd_rn(a, __dmul_rn(s_mu[d + e], x));
              b = __dadd_rn(b, __dmul_rn(s_s2[d + e], __dmul_rn(x, x)));
            }
          }
        }
        key[i] = __dadd_rn(__dmul_rn(a, p.inv_sqrt_d), __dmul_rn(b, p.inv_2d));
        idx[i] = i;
      } else {
        key[i] = -CUDART_INF;
        idx[i] = 0x7fffffff;
      }
    }
    __syncthreads();
    // bitonic sort: final order has precedes(i, i+1).  Phases whose pairs lie inside a 64-element
    // segment (j ≤ 32) run in registers, one warp per segment, lane holding elements lane and
    // lane + 32 (j = 32: in-lane, j < 32: shuffles); only the j ≥ 64 phases go through shared
    // memory with a CTA barrier — 6 barriers at N = 512 instead of 45.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, n_warps = blockDim.x >> 5;
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
              for (int h = 0; h < 2; ++h) {
                const int i = base + lane + 32 * h;
                const double ko = __shfl_xor_sync(0xffffffffu, kk[h], j);
                const int io = __shfl_xor_sync(0xffffffffu, ii[h], j);
                const bool up = (i & k) == 0, lower = (lane & j) == 0;
                // the lower position keeps the element that comes first (up) / second (down)
                const bool other_first = precedes(ko, io, kk[h], ii[h]);
                if (lower == (up == other_first) && (ko != kk[h] || io != ii[h])) {
                  kk[h] = ko;
                  ii[h] = io;
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
    // gather: rank r ← token idx[r], 16-byte chunks through registers — each thread issues 4
    // loads, then stores them; no shared-memory stage and no CTA barrier, so warps stream
    // independently (the barrier after a staged pass was the top stall: ncu, 20 % of samples)
    const int chunks = D / 8;  // a power of two (D ∈ {64, 128}): shifts, not divisions
    const int cs = chunks == 16 ? 4 : 3;
    const int n_c = L * 2 * chunks;  // K and V row chunks of every rank
    constexpr int kU = 4;  // A/B: 2 → 8.49 ms, 4 → 7.58 ms, 8 → 7.77 ms (C2, 2000 tuples)
    for (int w0 = threadIdx.x; w0 < n_c; w0 += kU * blockDim.x) {
      uint4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int w = w0 + u * blockDim.x;
        if (w < n_c) {
          const int r = w >> (cs + 1), which = (w >> cs) & 1, ch = w & (chunks - 1);
          v[u] = __ldcs(reinterpret_cast<const uint4*>(src_row(which, idx[r]) + ch * 8));
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int w = w0 + u * blockDim.x;
        if (w < n_c) {
          const int r = w >> (cs + 1), which = (w >> cs) & 1, ch = w & (chunks - 1);
          const int64_t page = p.dst_ids[pbase + (r >> 4)];
          uint16_t* dst = p.dst_pool + (size_t)page * p.page_elems + (which ? off_v : off_k) +
                          (r & 15) * D + ch * 8;
          __stcs(reinterpret_cast<uint4*>(dst), v[u]);
        }
      }
    }
  }
}

template <int MAXT>
size_t build_smem_bytes(int head_dim) {
  return (size_t)key_slots<MAXT>() * sizeof(double) + (size_t)MAXT * sizeof(int) +
         2 * sizeof(double) * head_dim;
}

template <int MAXT, int MINT>
cudaError_t launch_build_t(const BuildParams& p, cudaStream_t s) {
  auto kern = build_kernel<MAXT, MINT>;
  const size_t smem = build_smem_bytes<MAXT>(p.head_dim);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBuildThreads, smem);
  const int64_t units = p.n_tuples * p.n_layers * p.n_kv_heads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)num_sms() * std::max(occ, 1)));
  kern<<<grid, kBuildThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_build(const BuildParams& p, cudaStream_t s) {  // 2 launches
  cudaError_t e = launch_build_t<kBuildSmallTokens, 0>(p, s);
  if (e != cudaSuccess) return e;
  return launch_build_t<kBuildMaxTokens, kBuildSmallTokens>(p, s);
}

}  // namespace ko
