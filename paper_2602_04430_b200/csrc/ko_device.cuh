// ko_device.cuh — device helpers shared by the sm_100a kernels of libko (decisions, plan
// evaluation, counters, mbarrier / TMA / shared-memory primitives).  Internal (not the ABI).
#pragma once

#include <atomic>
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
// Without labels (has_gold false) TP/FP/FN/|P_g| stay 0 (ko.h: execution on unlabelled data).
__device__ void flush_counts(int* s_cnt, int n_rows, unsigned long long* counts, bool has_gold) {
  __syncthreads();
  for (int i = threadIdx.x; i < n_rows * kCountsPerPlan; i += blockDim.x) {
    const int k = i % kCountsPerPlan;
    const int* row = s_cnt + (i - k);
    long long v = s_cnt[i];
    if (k == KO_C_FP) v = has_gold ? (long long)row[KO_C_OUT] - row[KO_C_TP] : 0;
    if (k == KO_C_FN) v = has_gold ? (long long)row[KO_C_GOLD] - row[KO_C_TP] : 0;
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

// SM count of the CURRENT device, cached per device ordinal (a process may drive several GPUs)
inline int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 63;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

}  // namespace
}  // namespace ko
