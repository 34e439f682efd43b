// ko_soft.cu — continuous relaxation of a plan on precomputed margins (NEXT-1):
// soft TP / FP / FN / cost sums over the labelled sample and their exact derivatives with respect
// to every stage's pick score s_i and thresholds θ⁻_i, θ⁺_i — the quantities the paper's
// gradient-based optimizer (Adam on the loss of P:424-447) needs every iteration.
//
// Per tuple the relaxed cascade is a short chain of scalar operations; derivatives are taken in
// forward mode with dual numbers, one pass per parameter (3·S ≤ 24), each work item = (tuple,
// parameter).  Per-item results go to a workspace and are summed per output in a fixed order
// (fp64), so results are bitwise reproducible.  Equations (same order as oracle/soft.py):
//   σ_i = sigmoid(s_i/τ) (finals: 1);  π_i = softmax([m − θ⁺, θ⁻ − m, 0]/τ) (finals: 2-way
//   sigmoid((m − θ⁺)/τ));  a_i = a + u σ π_acc, r_i = r + u σ π_rej, u = 1 − a − r per op;
//   cost += σ_i c_i u_{op_i} Π_{o'≠op_i}(1 − r_{o'});  A = Π_o a_o;  TP = Σ A g, FP = Σ A(1−g),
//   FN = Σ (1−A) g with g = Π_o gold_o.
#include <algorithm>

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

__global__ void soft_items_kernel(const __grid_constant__ SoftParams p) {
  const int S = p.plan.n_stages;
  const int P = 3 * S + 1;  // item k = 0: value pass; k = 1 + 3i + f: derivative w.r.t. field f
  const int64_t n_items = p.n_tuples * P;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n_items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(it / p.n_tuples);
    const int64_t t = it - (int64_t)k * p.n_tuples;
    const int seed_stage = k == 0 ? -1 : (k - 1) / 3, seed_field = k == 0 ? -1 : (k - 1) % 3;
    Dual a[kMaxOps], r[kMaxOps];
    for (int o = 0; o < kMaxOps; ++o) { a[o] = mk(0.0); r[o] = mk(0.0); }
    Dual cost = mk(0.0);
    for (int i = 0; i < S; ++i) {
      const ko_stage& st = p.plan.stage[i];
      const int o = st.op;
      const double m = (double)p.margins[((size_t)o * p.n_variants + st.variant) * p.n_tuples + t];
      const Dual s = mk(p.pick[i], seed_stage == i && seed_field == 0 ? 1.0 : 0.0);
      const Dual lo = mk((double)st.theta_lo, seed_stage == i && seed_field == 1 ? 1.0 : 0.0);
      const Dual hi = mk((double)st.theta_hi, seed_stage == i && seed_field == 2 ? 1.0 : 0.0);
      const double itau = 1.0 / p.tau;
      Dual sig, pa, pr;
      if (st.is_final) {
        sig = mk(1.0);
        pa = dsigmoid(itau * (mk(m) - hi));
        pr = mk(1.0) - pa;
      } else {
        sig = dsigmoid(itau * s);
        dsoftmax3(itau * (mk(m) - hi), itau * (lo - mk(m)), &pa, &pr);
      }
      const Dual u = mk(1.0) - a[o] - r[o];
      Dual alive = mk(1.0);
      for (int o2 = 0; o2 < p.n_ops; ++o2)
        if (o2 != o && p.referenced[o2]) alive = alive * (mk(1.0) - r[o2]);
      cost = cost + p.stage_cost[i] * (sig * u * alive);
      a[o] = a[o] + u * sig * pa;
      r[o] = r[o] + u * sig * pr;
    }
    Dual A = mk(1.0);
    double g = 1.0;
    for (int o = 0; o < p.n_ops; ++o)
      if (p.referenced[o]) {
        A = A * a[o];
        g *= p.gold ? (double)(p.gold[(size_t)o * p.n_tuples + t] == 1) : 0.0;
      }
    double* dst = p.items + (size_t)k * 4 * p.n_tuples;
    const bool val = k == 0;
    dst[0 * p.n_tuples + t] = val ? A.v * g : A.d * g;
    dst[1 * p.n_tuples + t] = val ? A.v * (1.0 - g) : A.d * (1.0 - g);
    dst[2 * p.n_tuples + t] = val ? (1.0 - A.v) * g : -A.d * g;
    dst[3 * p.n_tuples + t] = val ? cost.v : cost.d;
  }
}

// one block per output row: fixed-order sum of n values (strided per thread, then a tree)
// row = 4k + q (item k, quantity q) → out[q] for k = 0, out[4 + q·3S + (k − 1)] otherwise
__global__ void soft_reduce_kernel(const double* items, int64_t n, double* out, int n_rows, int S) {
  __shared__ double sh[256];
  const int row = blockIdx.x;
  if (row >= n_rows) return;
  const double* src = items + (size_t)row * n;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += src[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  const int k = row / 4, q = row % 4;
  if (threadIdx.x == 0) out[k == 0 ? q : 4 + q * 3 * S + (k - 1)] = sh[0];
}

__global__ void fill_zero_kernel(double* out, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = 0.0;
}

}  // namespace

cudaError_t launch_soft(const SoftParams& p, double* out, cudaStream_t s) {
  const int S = p.plan.n_stages;
  const int P = 3 * S + 1;
  fill_zero_kernel<<<1, 128, 0, s>>>(out, 4 + 12 * S);
  const int64_t items = p.n_tuples * P;
  int blocks = (int)std::min<int64_t>((items + 255) / 256, 148 * 16);
  if (blocks < 1) blocks = 1;
  soft_items_kernel<<<blocks, 256, 0, s>>>(p);
  soft_reduce_kernel<<<4 * P, 256, 0, s>>>(p.items, p.n_tuples, out, 4 * P, S);
  return cudaGetLastError();
}

}  // namespace ko
