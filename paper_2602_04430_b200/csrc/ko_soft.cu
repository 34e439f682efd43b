// ko_soft.cu — continuous relaxation of a plan on precomputed margins (NEXT-1):
// soft TP / FP / FN / cost sums over the labelled sample and their exact derivatives with respect
// to every stage's pick score s_i and thresholds θ⁻_i, θ⁺_i — the quantities the paper's
// gradient-based optimizer (Adam on the loss of P:424-447) needs every iteration.
//
// Per tuple the relaxed cascade is a short chain of scalar operations; derivatives are taken in
// forward mode with dual numbers, one pass per parameter (3·S ≤ 24) over stage values computed
// once per tuple.  Each (direction, output) value is summed over the CTA right away — a fixed
// warp-shuffle tree, then the 4 warps in order into a per-CTA fp64 accumulator — and a second
// kernel adds the CTAs' partial sums in a fixed order, so results are bitwise reproducible and
// nothing per tuple goes to memory (r01 wrote every (direction, output, tuple) item to a
// workspace and summed it in two more launches).  Equations (same order as oracle/soft.py):
//   σ_i = sigmoid(s_i/τ) (finals: 1);  π_i = softmax([m − θ⁺, θ⁻ − m, 0]/τ) (finals: 2-way
//   sigmoid((m − θ⁺)/τ));  a_i = a + u σ π_acc, r_i = r + u σ π_rej, u = 1 − a − r per op;
//   cost += σ_i c_i u_{op_i} Π_{o'≠op_i}(1 − r_{o'});  A = Π_o a_o;  TP = Σ T g, FP = Σ (A − T g),
//   FN = Σ (g − T g) with g = Π_filters gold_o and T = Π_filters a_o · Π_maps κ_o.
// Map-classify stages (output-tuple selection; maps never reject, Q13): a non-final
// stage resolves u σ_i ρ_i, ρ_i = sigmoid((m − θ⁺)/τ) (finals: σ = ρ = 1), and the op's correct
// mass κ_o gains that amount when the stage's class equals the gold class (a wrong value is one
// FP and one FN).  For filter-only plans T = A and the sums reduce to A g, A(1−g), (1−A) g.
#include <algorithm>
#include <type_traits>

#include "ko_internal.h"

namespace ko {
namespace {

struct Dual {
  double v, d;
};
__device__ __forceinline__ Dual mk(double v, double d = 0.0) { return Dual{v, d}; }
__device__ __forceinline__ Dual operator+(Dual a, Dual b) { return {a.v + b.v, a.d + b.d}; }
__device__ __forceinline__ Dual operator-(Dual a, Dual b) { return {a.v - b.v, a.d - b.d}; }
__device__ __forceinline__ Dual operator*(Dual a, Dual b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
__device__ __forceinline__ Dual operator*(double a, Dual b) { return {a * b.v, a * b.d}; }
__device__ __forceinline__ Dual dsigmoid(Dual x) {
  // numerically stable logistic and its derivative σ(1 − σ)
  const double e = exp(-fabs(x.v));
  const double s = x.v >= 0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
  return {s, s * (1.0 - s) * x.d};
}
// softmax over (z0, z1, 0): returns p0, p1
__device__ __forceinline__ void dsoftmax3(Dual z0, Dual z1, Dual* p0, Dual* p1) {
  const double mx = fmax(fmax(z0.v, z1.v), 0.0);
  const double e0 = exp(z0.v - mx), e1 = exp(z1.v - mx), e2 = exp(-mx);
  const double den = e0 + e1 + e2;
  const double q0 = e0 / den, q1 = e1 / den;
  // d p_k = p_k (d z_k − Σ_j p_j d z_j), z2 ≡ 0
  const double dm = q0 * z0.d + q1 * z1.d;
  *p0 = {q0, q0 * (z0.d - dm)};
  *p1 = {q1, q1 * (z1.d - dm)};
}

// One thread per tuple.  Every stage's relaxed quantities (σ_i, π_acc,i, π_rej,i) and their local
// derivatives w.r.t. (s_i, θ⁻_i, θ⁺_i) are computed once — all the exp() calls — and kept in
// registers; then the cheap recurrence runs once per parameter direction (forward mode, dual
// numbers seeded at that parameter's stage; k = 0: values, k = 1 + 3i + f: field f of stage i).
// Local derivatives (the closed forms of the dual-number rules):
//   σ = sigmoid(s/τ):            ∂σ/∂s = σ(1 − σ)/τ                         (finals: σ = 1)
//   (π_a, π_r) = softmax3((m − θ⁺)/τ, (θ⁻ − m)/τ, 0):
//       ∂π_a/∂θ⁺ = −π_a(1 − π_a)/τ,  ∂π_r/∂θ⁺ = π_a π_r/τ,
//       ∂π_a/∂θ⁻ = −π_a π_r/τ,       ∂π_r/∂θ⁻ = π_r(1 − π_r)/τ
//   finals: π_a = sigmoid((m − θ⁺)/τ), π_r = 1 − π_a: ∂π_a/∂θ⁺ = −π_a(1 − π_a)/τ = −∂π_r/∂θ⁺.
constexpr int kSoftThreads = 128;
// SM ≥ the plan's stages; NO = the plan's distinct operators, in compact slots 0..NO-1 (slot
// order = operator order, so every product runs in the same order as over all op ids)
template <int SM, int NO>
__global__ void __launch_bounds__(kSoftThreads) soft_tuple_kernel(const __grid_constant__ SoftParams p) {
  __shared__ double s_acc[4 * (3 * SM + 1)];         // this CTA's sums, row = direction·4 + output
  __shared__ double s_w[kSoftThreads / 32][4];        // per-warp sums of one direction
  const int S = p.plan.n_stages;
  const int P = 3 * S + 1;
  const double itau = 1.0 / p.tau;
  const int64_t n = p.n_tuples;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4 * P; i += blockDim.x) s_acc[i] = 0.0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t iters = (n + stride - 1) / stride;  // the same for every thread (block sums)
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t t = it * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = t < n;
    double vs[SM], va[SM], vr[SM], ds[SM], dalo[SM], dahi[SM], drlo[SM], drhi[SM];
    bool ok[SM];  // map stages: the stage's class equals the gold class
#pragma unroll
    for (int i = 0; i < SM; ++i) {
      vs[i] = 1.0; va[i] = vr[i] = ds[i] = dalo[i] = dahi[i] = drlo[i] = drhi[i] = 0.0;
      ok[i] = false;
      if (i >= S || !valid) continue;
      const ko_stage& st = p.plan.stage[i];
      const size_t mi = ((size_t)st.op * p.n_variants + st.variant) * n + t;
      const double m = (double)p.margins[mi];
      const double hi = (double)st.theta_hi, lo = (double)st.theta_lo;
      if (p.is_map[st.op]) {
        ok[i] = p.gold && p.classes[mi] == (int32_t)p.gold[(size_t)st.op * n + t];
        if (st.is_final) {
          va[i] = 1.0;                                         // resolves all that reaches it
        } else {
          const Dual sg = dsigmoid(itau * mk(p.pick[i], 1.0));  // seeded in s
          vs[i] = sg.v; ds[i] = sg.d;
          const Dual pa = dsigmoid(itau * (mk(m) - mk(hi, 1.0)));  // ρ, seeded in θ⁺
          va[i] = pa.v; dahi[i] = pa.d;
        }
      } else if (st.is_final) {
        const Dual pa = dsigmoid(itau * (mk(m) - mk(hi, 1.0)));  // seeded in θ⁺
        va[i] = pa.v; vr[i] = 1.0 - pa.v; dahi[i] = pa.d; drhi[i] = -pa.d;
      } else {
        const Dual sg = dsigmoid(itau * mk(p.pick[i], 1.0));  // seeded in s
        vs[i] = sg.v; ds[i] = sg.d;
        Dual pa, pr;
        dsoftmax3(itau * (mk(m) - mk(hi, 1.0)), itau * (mk(lo) - mk(m)), &pa, &pr);  // θ⁺
        va[i] = pa.v; vr[i] = pr.v; dahi[i] = pa.d; drhi[i] = pr.d;
        dsoftmax3(itau * (mk(m) - mk(hi)), itau * (mk(lo, 1.0) - mk(m)), &pa, &pr);  // θ⁻
        dalo[i] = pa.d; drlo[i] = pr.d;
      }
    }
    double g = 1.0;
#pragma unroll
    for (int so = 0; so < NO; ++so)
      if (valid && !p.slot_is_map[so])
        g *= p.gold ? (double)(p.gold[(size_t)p.slot_op[so] * n + t] == 1) : 0.0;
    // Directions whose parameter has no effect (s and θ⁻ of a final stage, θ⁻ of a map stage,
    // a final map stage: p.dir_live) would add exact zeros: skipped.  (Starting each direction
    // at its seeded stage from a saved prefix state was measured slower: 24.7 → 30.8 µs.)
    for (int k = 0; k < P; ++k) {
      if (k > 0 && !p.dir_live[k - 1]) continue;  // uniform
      const int seed_stage = k == 0 ? -1 : (k - 1) / 3, seed_field = k == 0 ? -1 : (k - 1) % 3;
      Dual a[NO], r[NO], kap[NO];
#pragma unroll
      for (int o = 0; o < NO; ++o) { a[o] = mk(0.0); r[o] = mk(0.0); kap[o] = mk(0.0); }
      Dual cost = mk(0.0);
#pragma unroll
      for (int i = 0; i < SM; ++i) {
        if (i >= S) continue;
        const int o = p.stage_slot[i];
        const bool sd = seed_stage == i;
        const Dual sig = mk(vs[i], sd && seed_field == 0 ? ds[i] : 0.0);
        const Dual pa = mk(va[i], sd ? (seed_field == 1 ? dalo[i] : seed_field == 2 ? dahi[i] : 0.0) : 0.0);
        const Dual pr = mk(vr[i], sd ? (seed_field == 1 ? drlo[i] : seed_field == 2 ? drhi[i] : 0.0) : 0.0);
        // a / r indexed by compile-time op slots (selects, not a local-memory array)
        Dual ao = mk(0.0), ro = mk(0.0), alive = mk(1.0);
#pragma unroll
        for (int o2 = 0; o2 < NO; ++o2) {
          if (o2 == o) { ao = a[o2]; ro = r[o2]; }
          else alive = alive * (mk(1.0) - r[o2]);
        }
        const Dual u = mk(1.0) - ao - ro;
        cost = cost + p.stage_cost[i] * (sig * u * alive);
        const Dual res = u * sig * pa;
        const Dual na = ao + res, nr = ro + u * sig * pr;
#pragma unroll
        for (int o2 = 0; o2 < NO; ++o2)
          if (o2 == o) {
            a[o2] = na;
            r[o2] = nr;
            if (ok[i]) kap[o2] = kap[o2] + res;
          }
      }
      Dual A = mk(1.0), T = mk(1.0);
#pragma unroll
      for (int o = 0; o < NO; ++o) {
        A = A * a[o];
        T = T * (p.slot_is_map[o] ? kap[o] : a[o]);
      }
      const Dual tg = g * T;
      const bool val = k == 0;
      double v4[4] = {val ? tg.v : tg.d, val ? A.v - tg.v : A.d - tg.d, val ? g - tg.v : -tg.d,
                      val ? cost.v : cost.d};
      // CTA sum of this direction's 4 outputs in a fixed order: shuffle tree, then warps 0..3
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!valid) v4[q] = 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v4[q] += __shfl_down_sync(0xffffffffu, v4[q], off);
      }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) s_w[warp][q] = v4[q];
      }
      __syncthreads();
      if (threadIdx.x < 4) {
        double a = s_w[0][threadIdx.x];
        for (int w = 1; w < kSoftThreads / 32; ++w) a += s_w[w][threadIdx.x];
        s_acc[k * 4 + threadIdx.x] += a;
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < 4 * P; i += blockDim.x)
    p.partials[(size_t)blockIdx.x * 4 * P + i] = s_acc[i];
}

// The CTAs' partial sums, one warp per output row: lane j adds CTAs j, j + 32, ... in order,
// then a fixed shuffle tree.  Bitwise reproducible (the grid size depends only on n_tuples).
__global__ void soft_final_kernel(const double* part, int n_blocks, double* out, int n_rows, int S) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= n_rows) return;
  double a = 0.0;
  for (int b = lane; b < n_blocks; b += 32) a += part[(size_t)b * n_rows + row];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) a += __shfl_down_sync(0xffffffffu, a, off);
  if (lane == 0) {
    const int k = row / 4, q = row % 4;
    out[k == 0 ? q : 4 + q * 3 * S + (k - 1)] = a;
  }
}

}  // namespace

int soft_blocks(int64_t n_tuples) {  // the tuple kernel's grid: a function of n_tuples only
  const int64_t b = std::min<int64_t>((n_tuples + kSoftThreads - 1) / kSoftThreads, 148 * 8);
  return (int)std::max<int64_t>(b, 1);
}

cudaError_t launch_soft(const SoftParams& p, double* out, cudaStream_t s) {  // 2 launches
  const int S = p.plan.n_stages;
  const int P = 3 * S + 1;
  const int blocks = soft_blocks(p.n_tuples);
  auto run = [&](auto sm_tag) {
    constexpr int SM = decltype(sm_tag)::value;
    switch (p.n_slots) {
      case 1: soft_tuple_kernel<SM, 1><<<blocks, kSoftThreads, 0, s>>>(p); break;
      case 2: soft_tuple_kernel<SM, 2><<<blocks, kSoftThreads, 0, s>>>(p); break;
      case 3: soft_tuple_kernel<SM, 3><<<blocks, kSoftThreads, 0, s>>>(p); break;
      default: soft_tuple_kernel<SM, 4><<<blocks, kSoftThreads, 0, s>>>(p); break;
    }
  };
  static_assert(kMaxOps == 4, "soft kernel instantiations cover 1..4 operator slots");
  if (S <= 2) run(std::integral_constant<int, 2>{});
  else if (S <= 4) run(std::integral_constant<int, 4>{});
  else run(std::integral_constant<int, 8>{});
  soft_final_kernel<<<(4 * P + 3) / 4, 128, 0, s>>>(p.partials, blocks, out, 4 * P, S);
  return cudaGetLastError();
}

}  // namespace ko
