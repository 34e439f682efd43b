// ko_oracle.cpp — plain, slow, obviously-correct fp64 CPU ORACLE for the KV-cache scoring pass.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  It shares no code, header, table or helper
// with the CUDA path (paper_2602_04430_b200/); it defines its own structs.  Citations: P:n =
// /root/reference/PAPER.md line n (not available at run time); the readings of silent or garbled
// passages are the ones listed in DESIGN.md §"Readings" (SURVEY.md §8(c) Q1–Q24).
//
// What it computes (SURVEY.md §8(c) steps 1–9), in the paper's order:
//   score  : for tuple t, op o, variant v = (keep‰, layer cut):
//              n = max(1, floor(L_t·keep/1000))                        (Q3)
//              for l < cut, q-head j (kv-head h = j / G), query row r:   (Q15, Q16, Q18)
//                s_i = Σ_k Q[l][j][r][k]·K[l][h][i][k] / sqrt(d),  i < n
//                M = max_i s_i,  p_i = exp(s_i − M),  O = Σ_i p_i V_i / Σ_i p_i   (two-pass)
//              z_c = b_c + Σ_{l<cut} Σ_j Σ_r Σ_k W[c][l][j][r][k]·O[k]        (Q1)
//              filter: m = z_0 (yes−no log-odds);  map: class = argmax_c z_c
//              (lowest index on ties), m = z_(1) − z_(2)                      (Q13)
//   decide : thresholds, P:456 and P:471-472 with strict inequalities (Q5, Q6, Q13)
//   plans  : cascade recurrences Eqs (accept-i)/(reject-i)/(unsure-i), with
//            σ ∈ {0,1} and conjunctive inter-operator semantics P:536-539 (Q12)
//   counts : TP/FP/FN of Eqs (sample-tp/fp/fn), applied to the whole plan output
//            vs the gold plan, with map output-tuple semantics P:513-519;
//            per-stage n_in / n_acc / n_rej / n_uns (selectivities P:541-547, cost Eq. P:338).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

extern "C" {

typedef struct {
  int32_t n_layers, n_kv_heads, gqa, head_dim, n_q;
  const uint16_t* kv_pool;  // bf16 bits [n_pages][n_layers][2][n_kv_heads][16][head_dim]
  int64_t n_pages;
  const int64_t* page_indptr;  // [n_tuples+1]
  const int32_t* page_ids;     // logical page order = importance order
  const int32_t* seq_len;      // [n_tuples]
  int64_t n_tuples;
} or_kv;

typedef struct {
  int32_t n_classes;  // 1 = filter, >= 2 map-classify
  const uint16_t* q;  // bf16 bits [n_layers][Hq][n_q][head_dim]
  const float* w;     // [n_classes][n_layers][Hq][n_q][head_dim]
  const float* b;     // [n_classes]
} or_op;

typedef struct {
  int32_t keep_permille, layer_cut;
} or_variant;

typedef struct {
  int32_t op, variant;
  float theta_lo, theta_hi;
  int32_t is_final;
} or_stage;

#define OR_MAX_STAGES 8
#define OR_COUNTS_PER_PLAN (5 + 4 * OR_MAX_STAGES)

typedef struct {
  int32_t n_stages;
  or_stage stage[OR_MAX_STAGES];
} or_plan;

}  // extern "C"

namespace {

double bf16_to_double(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return (double)f;
}

int64_t n_kept(int32_t L, int32_t keep_permille) {  // Q3
  int64_t n = ((int64_t)L * keep_permille) / 1000;
  return n < 1 ? 1 : n;
}

// K (kv = 0) or V (kv = 1) vector of logical token i of tuple t at (layer l, kv-head h)
const uint16_t* kv_row(const or_kv* kv, int64_t t, int32_t l, int32_t which, int32_t h, int64_t i) {
  int64_t page = kv->page_ids[kv->page_indptr[t] + i / 16];
  int64_t slot = i % 16;
  size_t off = ((((size_t)page * kv->n_layers + l) * 2 + which) * kv->n_kv_heads + h) * 16 + slot;
  return kv->kv_pool + off * kv->head_dim;
}

// z_c for (tuple t, op, variant): steps 1–4 of SURVEY §8(c)
void score_one(const or_kv* kv, const or_op* op, const or_variant* v, int64_t t, double* z) {
  const int32_t D = kv->head_dim, G = kv->gqa, Hq = kv->n_kv_heads * kv->gqa, NQ = kv->n_q;
  const int64_t n = n_kept(kv->seq_len[t], v->keep_permille);
  const double scale = 1.0 / std::sqrt((double)D);
  std::vector<double> s(n), O(D), q(D), kk(D);
  for (int c = 0; c < op->n_classes; ++c) z[c] = (double)op->b[c];
  for (int32_t l = 0; l < v->layer_cut; ++l)
    for (int32_t j = 0; j < Hq; ++j) {
      const int32_t h = j / G;
      for (int32_t r = 0; r < NQ; ++r) {
        const uint16_t* qrow = op->q + (((size_t)l * Hq + j) * NQ + r) * D;
        for (int k = 0; k < D; ++k) q[k] = bf16_to_double(qrow[k]);
        // scores
        double M = -INFINITY;
        for (int64_t i = 0; i < n; ++i) {
          const uint16_t* krow = kv_row(kv, t, l, 0, h, i);
          double acc = 0.0;
          for (int k = 0; k < D; ++k) acc += q[k] * bf16_to_double(krow[k]);
          s[i] = acc * scale;
          if (s[i] > M) M = s[i];
        }
        // two-pass softmax and weighted sum of V
        double den = 0.0;
        for (int k = 0; k < D; ++k) O[k] = 0.0;
        for (int64_t i = 0; i < n; ++i) {
          double p = std::exp(s[i] - M);
          den += p;
          const uint16_t* vrow = kv_row(kv, t, l, 1, h, i);
          for (int k = 0; k < D; ++k) O[k] += p * bf16_to_double(vrow[k]);
        }
        for (int k = 0; k < D; ++k) O[k] /= den;
        // linear readout
        for (int c = 0; c < op->n_classes; ++c) {
          const float* wrow =
              op->w + ((((size_t)c * kv->n_layers + l) * Hq + j) * NQ + r) * D;
          double acc = 0.0;
          for (int k = 0; k < D; ++k) acc += (double)wrow[k] * O[k];
          z[c] += acc;
        }
      }
    }
}

// margin and class from logits (step 4)
void margin_of(const double* z, int32_t C, double* m, int32_t* cls) {
  if (C <= 1) {
    *m = z[0];
    *cls = 0;
    return;
  }
  int32_t a = 0;
  for (int c = 1; c < C; ++c)
    if (z[c] > z[a]) a = c;  // lowest index on ties
  double second = -INFINITY;
  for (int c = 0; c < C; ++c)
    if (c != a && z[c] > second) second = z[c];
  *cls = a;
  *m = z[a] - second;
}

enum { D_ACCEPT = 0, D_REJECT = 1, D_UNSURE = 2, D_RESOLVED = 3 };

// step 5: stage decision (θ fp32 widened to fp64)
int decide(double m, const or_stage* st, int32_t n_classes) {
  const double lo = (double)st->theta_lo, hi = (double)st->theta_hi;
  if (n_classes <= 1) {
    if (st->is_final) return m > hi ? D_ACCEPT : D_REJECT;  // Q6: tie rejects
    if (m > hi) return D_ACCEPT;                             // Q5: strict
    if (m < lo) return D_REJECT;
    return D_UNSURE;
  }
  if (st->is_final) return D_RESOLVED;  // maps never reject
  return m > hi ? D_RESOLVED : D_UNSURE;
}

}  // namespace

extern "C" {

// margins/classes: [n_ops][n_variants][n]; z (optional): [n_ops][n_variants][n][zstride]
int oracle_score(const or_kv* kv, const or_op* ops, int32_t n_ops, const or_variant* variants,
                 int32_t n_variants, const int64_t* tuples, int64_t n, double* margins,
                 int32_t* classes, double* z_out, int32_t zstride, int32_t n_threads) {
  if (n_threads < 1) n_threads = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < n_threads; ++w)
    th.emplace_back([&, w]() {
      std::vector<double> z(64);
      for (int64_t i = w; i < n; i += n_threads) {
        const int64_t t = tuples ? tuples[i] : i;
        for (int32_t o = 0; o < n_ops; ++o)
          for (int32_t v = 0; v < n_variants; ++v) {
            score_one(kv, &ops[o], &variants[v], t, z.data());
            double m;
            int32_t c;
            margin_of(z.data(), ops[o].n_classes, &m, &c);
            const size_t idx = ((size_t)o * n_variants + v) * n + i;
            if (margins) margins[idx] = m;
            if (classes) classes[idx] = c;
            if (z_out)
              for (int k = 0; k < ops[o].n_classes && k < zstride; ++k) z_out[idx * zstride + k] = z[k];
          }
      }
    });
  for (auto& x : th) x.join();
  return 0;
}

// Steps 6–9.  margins/classes [n_ops][n_variants][n] (fp64), n_classes[n_ops], gold [n_ops][n]
// (filters 0/1, maps class) or NULL.  counts [n_plans][OR_COUNTS_PER_PLAN] are ACCUMULATED.
// final_alive (optional) [n_plans][n] receives the end state (1 = in P_o).
// stage_out (optional) [n_plans][OR_MAX_STAGES][n] receives each stage's outcome per tuple:
// 0 = not reached (unsure_{t,i-1} = 0), 1 = accept, 2 = reject, 3 = unsure, 4 = map resolved.
int oracle_run_plans(const or_plan* plans, int32_t n_plans, const double* margins,
                     const int32_t* classes, const int32_t* n_classes, int32_t n_ops,
                     int32_t n_variants, int64_t n, const uint8_t* gold, int64_t* counts,
                     uint8_t* final_alive, int8_t* stage_out) {
  for (int32_t g = 0; g < n_plans; ++g) {
    const or_plan* P = &plans[g];
    if (P->n_stages < 1 || P->n_stages > OR_MAX_STAGES) return 1;
    bool referenced[64] = {false};
    for (int s = 0; s < P->n_stages; ++s) {
      const or_stage* st = &P->stage[s];
      if (st->op < 0 || st->op >= n_ops || st->variant < 0 || st->variant >= n_variants) return 1;
      if (!(st->theta_lo <= st->theta_hi)) return 1;
      referenced[st->op] = true;
    }
    int64_t* cnt = counts + (size_t)g * OR_COUNTS_PER_PLAN;
    for (int64_t t = 0; t < n; ++t) {
      bool alive = true;
      int status[64];  // 0 pending, 1 accepted/resolved, 2 rejected
      int cls[64];
      for (int o = 0; o < n_ops; ++o) { status[o] = 0; cls[o] = -1; }
      for (int s = 0; s < P->n_stages; ++s) {
        const or_stage* st = &P->stage[s];
        const int o = st->op;
        int8_t* so = stage_out ? stage_out + ((size_t)g * OR_MAX_STAGES + s) * n + t : nullptr;
        if (so) *so = 0;
        if (!(alive && status[o] == 0)) continue;  // not reached: unsure_{t,i-1} = 0
        cnt[5 + 4 * s] += 1;                        // n_in
        const size_t idx = ((size_t)o * n_variants + st->variant) * n + t;
        const int dcs = decide(margins[idx], st, n_classes[o]);
        if (so) *so = dcs == D_ACCEPT ? 1 : dcs == D_REJECT ? 2 : dcs == D_RESOLVED ? 4 : 3;
        if (dcs == D_ACCEPT) { status[o] = 1; cnt[6 + 4 * s] += 1; }
        else if (dcs == D_RESOLVED) { status[o] = 1; cls[o] = classes[idx]; cnt[6 + 4 * s] += 1; }
        else if (dcs == D_REJECT) { alive = false; status[o] = 2; cnt[7 + 4 * s] += 1; }
        else cnt[8 + 4 * s] += 1;  // unsure: stays pending
      }
      bool in_out = alive;
      bool in_gold = true, maps_ok = true;
      if (gold) {
        for (int o = 0; o < n_ops; ++o) {
          if (!referenced[o]) continue;
          const uint8_t gv = gold[(size_t)o * n + t];
          if (n_classes[o] <= 1) {
            if (gv != 1) in_gold = false;
          } else if (cls[o] != (int)gv) {
            maps_ok = false;
          }
        }
      } else {
        in_gold = false;
      }
      if (in_out) cnt[3] += 1;
      if (in_gold) cnt[4] += 1;
      if (in_out && in_gold && maps_ok) cnt[0] += 1;
      if (final_alive) final_alive[(size_t)g * n + t] = in_out ? 1 : 0;
    }
    // FP = |P_o| − TP, FN = |P_g| − TP (accumulated form: recompute from running totals).
    // Without labels (gold == NULL) TP/FP/FN/|P_g| are undefined and stay 0 (ko.h contract,
    // SURVEY §8(b)); only |P_o| and the per-stage counts are produced.
    cnt[1] = gold ? cnt[3] - cnt[0] : 0;
    cnt[2] = gold ? cnt[4] - cnt[0] : 0;
  }
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// Offline importance-ordered cache builder (NEXT-4; KV caches are created
// offline and compressed with query-agnostic Expected Attention, "select tokens based on their
// expected contribution to attention across potential future queries").  Reading (DESIGN
// §2, Q25): with a Gaussian query model q ~ N(μ, diag σ²) per (layer, kv-head), the log expected
// un-normalised attention of key k is
//     s(k) = (Σ_d μ_d k_d) / sqrt(D) + (Σ_d σ²_d k_d²) / (2 D),
// evaluated in fp64, left to right, one rounding per operation (no fused multiply-add), so the
// GPU builder takes identical decisions.  Tokens are stored in descending s (ties: lower original
// index first); token of rank r goes to slot r % 16 of logical page r / 16.
// ---------------------------------------------------------------------------------------------
extern "C" int oracle_build_order(const or_kv* kv, const float* mu, const float* sigma2,
                                  uint16_t* dst_pool, const int32_t* dst_page_ids,
                                  int32_t n_threads) {
  const int32_t D = kv->head_dim, H = kv->n_kv_heads, Lyr = kv->n_layers;
  const double inv_sqrt_d = 1.0 / std::sqrt((double)D), inv_2d = 1.0 / (2.0 * (double)D);
  if (n_threads < 1) n_threads = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < n_threads; ++w)
    th.emplace_back([&, w]() {
      std::vector<double> sc;
      std::vector<int32_t> order;
      for (int64_t t = w; t < kv->n_tuples; t += n_threads) {
        const int32_t L = kv->seq_len[t];
        for (int32_t l = 0; l < Lyr; ++l)
          for (int32_t h = 0; h < H; ++h) {
            const float* m = mu + ((size_t)l * H + h) * D;
            const float* s2 = sigma2 + ((size_t)l * H + h) * D;
            sc.assign(L, 0.0);
            order.resize(L);
            for (int32_t i = 0; i < L; ++i) {
              const uint16_t* k = kv_row(kv, t, l, 0, h, i);
              double a = 0.0, b = 0.0;
              for (int32_t d = 0; d < D; ++d) {
                const double x = bf16_to_double(k[d]);
                const double pa = (double)m[d] * x;
                a = a + pa;
                const double xx = x * x;
                const double pb = (double)s2[d] * xx;
                b = b + pb;
              }
              const double ta = a * inv_sqrt_d;
              const double tb = b * inv_2d;
              sc[i] = ta + tb;
              order[i] = i;
            }
            std::stable_sort(order.begin(), order.end(),
                             [&](int32_t x, int32_t y) { return sc[x] > sc[y]; });
            for (int32_t r = 0; r < L; ++r) {
              const int64_t page = dst_page_ids[kv->page_indptr[t] + r / 16];
              for (int which = 0; which < 2; ++which) {
                const uint16_t* src = kv_row(kv, t, l, which, h, order[r]);
                uint16_t* dst = dst_pool + (((((size_t)page * Lyr + l) * 2 + which) * H + h) * 16 + r % 16) * D;
                std::memcpy(dst, src, sizeof(uint16_t) * D);
              }
            }
          }
      }
    });
  for (auto& x : th) x.join();
  return 0;
}
