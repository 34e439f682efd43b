/* kogen.h — seeded, integer-only synthetic workload generator (test/bench FIXTURE).
 *
 * This module produces the INPUTS of the KV-cache scoring pass: bf16 KV pages, operator
 * queries Q, readouts W, tuple lengths, evidence positions and latent labels.  It holds
 * none of the method's arithmetic (no attention, no logits, no routing, no counts); both
 * the CPU oracle (oracle/) and the CUDA product path (paper_2602_04430_b200/) consume what
 * it produces, and neither imports the other.  The recipe is SURVEY.md §8(d), restated in
 * DESIGN.md §"Input recipe":
 *
 *   * H(...)      chained splitmix64 over (seed, tensor id, 4 indices); nrm(h) =
 *                 floor((Σ 4 low bytes − 510)·14189 / 2^16) ≈ N(0, 32²), |nrm| ≤ 110.
 *   * values      clamp(int, ±127)/32  — exact in bf16 (K, V, Q);  W = int/2^w_log2_den (default
 *                 4096; |int| ≤ 138, so exact in bf16 and fp32).  All divisions are FLOOR divisions (kg_fdiv).
 *   * shared query-agnostic direction μ[l][h] (same for all ops, the "Expected Attention"
 *     importance signal), per-op query direction qdir_o[l][h] and readout
 *     direction ρ_{o,c}[l][h]; K = noise + importance ramp ⌊8(L−i)μ/(32L)⌋ + evidence;
 *     V = noise + label-signed readout direction at the op's evidence tokens.
 *
 * Every function is integer-only, so the host (gen/kogen.c) and device (gen/kogen_gpu.cu)
 * twins produce bit-identical values.  Header-only, C99 / CUDA compatible.
 */
#ifndef KOGEN_H
#define KOGEN_H

#include <stdint.h>

#ifdef __CUDACC__
#define KG_HD __host__ __device__ __forceinline__
#else
#define KG_HD static inline
#endif

#define KG_MAX_OPS 4
#define KG_MAX_CLASSES 32
#define KG_PAGE 16

/* tensor ids: separate hash streams */
enum {
  KG_T_MU = 1, KG_T_QDIR = 2, KG_T_RHO = 3, KG_T_Q = 4, KG_T_W = 5,
  KG_T_K = 6, KG_T_V = 7, KG_T_EVID = 8, KG_T_LABEL = 9, KG_T_LEN = 10, KG_T_EMB = 11,
  KG_T_EDIR = 12
};

typedef struct {
  uint64_t seed;
  int32_t n_layers, n_kv_heads, gqa, head_dim, n_q;
  int32_t n_ops;
  int32_t op_classes[KG_MAX_OPS];      /* 1 = filter (binary label), K >= 2 = map-classify   */
  int32_t op_pi_permille[KG_MAX_OPS];  /* filters: P(label = +1) in permille                 */
  int32_t len_min, len_max;            /* len_min == len_max: fixed length; else octave
                                          log-uniform in [len_min, len_max), len_max/len_min
                                          a power of two                                    */
  int32_t n_evid;                      /* evidence tokens per (tuple, op), default 3         */
  int32_t k_ramp;                      /* importance ramp strength, default 8                */
  int32_t k_beta;                      /* K evidence strength, default 16                    */
  int32_t v_gamma;                     /* V evidence strength, default 10                    */
  int32_t w_log2_den;                  /* W = int / 2^w_log2_den, default 12 (= /4096)       */
} kg_cfg;

KG_HD uint64_t kg_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* H(seed, tensor, a, b, c, d): chained splitmix64 */
KG_HD uint64_t kg_h(uint64_t seed, uint64_t tensor, uint64_t a, uint64_t b, uint64_t c,
                    uint64_t d) {
  uint64_t h = kg_mix(seed);
  h = kg_mix(h ^ tensor);
  h = kg_mix(h ^ a);
  h = kg_mix(h ^ b);
  h = kg_mix(h ^ c);
  return kg_mix(h ^ d);
}

/* floor division, b > 0 */
KG_HD int32_t kg_fdiv(int32_t a, int32_t b) {
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}
KG_HD int64_t kg_fdiv64(int64_t a, int64_t b) {
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

KG_HD int32_t kg_clamp127(int32_t v) { return v > 127 ? 127 : (v < -127 ? -127 : v); }

/* ≈ N(0, 32²) from 4 uniform bytes */
KG_HD int32_t kg_nrm32(uint32_t x) {
  int32_t s = (int32_t)(x & 255u) + (int32_t)((x >> 8) & 255u) + (int32_t)((x >> 16) & 255u) +
              (int32_t)(x >> 24);
  return kg_fdiv((s - 510) * 14189, 65536);
}

/* element e of the noise row whose row hash is `base` */
KG_HD int32_t kg_nrm_at(uint64_t base, int32_t e) {
  uint64_t w = kg_mix(base ^ (uint64_t)(e >> 1));
  return kg_nrm32((e & 1) ? (uint32_t)(w >> 32) : (uint32_t)w);
}

/* ---------------- shared direction tables (small; per layer/kv-head/dim) ---------------- */
KG_HD int32_t kg_mu(const kg_cfg* c, int32_t l, int32_t h, int32_t d) {
  return kg_nrm_at(kg_h(c->seed, KG_T_MU, (uint64_t)l, (uint64_t)h, 0, 0), d);
}
KG_HD int32_t kg_qdir(const kg_cfg* c, int32_t o, int32_t l, int32_t h, int32_t d) {
  return kg_nrm_at(kg_h(c->seed, KG_T_QDIR, (uint64_t)o, (uint64_t)l, (uint64_t)h, 0), d);
}
KG_HD int32_t kg_rho(const kg_cfg* c, int32_t o, int32_t cls, int32_t l, int32_t h, int32_t d) {
  return kg_nrm_at(kg_h(c->seed, KG_T_RHO, (uint64_t)o, (uint64_t)cls, (uint64_t)l, (uint64_t)h),
                   d);
}

/* ---------------- operator query and readout (integers; Q = int/32, W = int/2^w_log2_den) */
/* q-head j uses kv-head h = j / gqa (HF repeat_kv convention) */
KG_HD int32_t kg_q_int(const kg_cfg* c, int32_t o, int32_t l, int32_t j, int32_t r, int32_t d) {
  int32_t h = j / c->gqa;
  int32_t n = kg_nrm_at(kg_h(c->seed, KG_T_Q, (uint64_t)o, (uint64_t)l, (uint64_t)j, (uint64_t)r), d);
  return kg_clamp127(kg_fdiv(n, 2) + kg_fdiv(16 * kg_mu(c, l, h, d), 32) +
                     kg_fdiv(kg_qdir(c, o, l, h, d), 2));
}
KG_HD int32_t kg_w_int(const kg_cfg* c, int32_t o, int32_t cls, int32_t l, int32_t j, int32_t r,
                       int32_t d) {
  int32_t h = j / c->gqa;
  int32_t n = kg_nrm_at(
      kg_h(c->seed, KG_T_W, (uint64_t)o, (uint64_t)cls, (uint64_t)l, (uint64_t)(j * 4096 + r)), d);
  return kg_fdiv(n, 4) + kg_rho(c, o, cls, l, h, d);
}

/* ---------------- per-tuple metadata ---------------- */
KG_HD int32_t kg_seq_len(const kg_cfg* c, int64_t t) {
  if (c->len_max <= c->len_min) return c->len_min;
  int32_t n_oct = 0;
  while ((c->len_min << (n_oct + 1)) <= c->len_max) ++n_oct;
  uint64_t h = kg_h(c->seed, KG_T_LEN, (uint64_t)t, 0, 0, 0);
  int32_t k = (int32_t)((uint32_t)h % (uint32_t)n_oct);
  uint64_t base = (uint64_t)c->len_min << k;
  return (int32_t)(base + (((h >> 32) * base) >> 32));
}

/* latent label: filters ±1 with P(+1) = pi; maps a class in [0, K) */
KG_HD int32_t kg_label(const kg_cfg* c, int64_t t, int32_t o) {
  uint64_t h = kg_h(c->seed, KG_T_LABEL, (uint64_t)t, (uint64_t)o, 0, 0);
  uint32_t u = (uint32_t)(h >> 11);
  if (c->op_classes[o] <= 1) return (int32_t)(u % 1000u) < c->op_pi_permille[o] ? 1 : -1;
  return (int32_t)(u % (uint32_t)c->op_classes[o]);
}

/* k-th evidence token position of op o in tuple t (skewed toward the important prefix) */
KG_HD int32_t kg_evidence(const kg_cfg* c, int64_t t, int32_t o, int32_t k, int32_t L) {
  uint64_t h = kg_h(c->seed, KG_T_EVID, (uint64_t)t, (uint64_t)o, (uint64_t)k, 0);
  uint32_t u1 = (uint32_t)h, u2 = (uint32_t)(h >> 32);
  uint64_t h2 = kg_mix(h);
  uint32_t x = (h2 & 1u) ? u1 : (u1 < u2 ? u1 : u2);
  return (int32_t)(((uint64_t)(uint32_t)L * (uint64_t)x) >> 32);
}

/* per-tuple context: evidence positions and labels, computed once per tuple */
typedef struct {
  int32_t L;
  int32_t evid[KG_MAX_OPS][8];
  int32_t label[KG_MAX_OPS];
} kg_tuple;

KG_HD void kg_tuple_init(const kg_cfg* c, int64_t t, kg_tuple* tp) {
  tp->L = kg_seq_len(c, t);
  for (int32_t o = 0; o < c->n_ops; ++o) {
    for (int32_t k = 0; k < c->n_evid && k < 8; ++k) tp->evid[o][k] = kg_evidence(c, t, o, k, tp->L);
    tp->label[o] = kg_label(c, t, o);
  }
}

KG_HD int32_t kg_is_evid(const kg_cfg* c, const kg_tuple* tp, int32_t o, int32_t i) {
  for (int32_t k = 0; k < c->n_evid && k < 8; ++k)
    if (tp->evid[o][k] == i) return 1;
  return 0;
}

/* row hash for the noise of K (kv=0) / V (kv=1) row (t, l, h, i) */
KG_HD uint64_t kg_kv_row_hash(const kg_cfg* c, int32_t kv, int64_t t, int32_t l, int32_t h,
                              int32_t i) {
  return kg_h(c->seed, kv ? KG_T_V : KG_T_K, (uint64_t)t, (uint64_t)l, (uint64_t)h, (uint64_t)i);
}

/* K element, given the row hash and the direction-table values at (l, h, d):
 * mu = μ[l][h][d], qdir[o] = qdir_o[l][h][d] */
KG_HD int32_t kg_k_int(const kg_cfg* c, const kg_tuple* tp, uint64_t row_hash, int32_t i,
                       int32_t d, int32_t mu, const int32_t* qdir) {
  int32_t v = kg_nrm_at(row_hash, d) + kg_fdiv(c->k_ramp * (tp->L - i) * mu, 32 * tp->L);
  for (int32_t o = 0; o < c->n_ops; ++o)
    if (kg_is_evid(c, tp, o, i)) v += kg_fdiv(c->k_beta * qdir[o], 32);
  return kg_clamp127(v);
}

/* V element; rho_lab[o] = ρ_{o,c}[l][h][d] for filters (c = 0) scaled by the ±1 label, or
 * for maps ρ_{o, label}[l][h][d] */
KG_HD int32_t kg_v_int(const kg_cfg* c, const kg_tuple* tp, uint64_t row_hash, int32_t i,
                       int32_t d, const int32_t* rho_lab) {
  int32_t v = kg_nrm_at(row_hash, d);
  for (int32_t o = 0; o < c->n_ops; ++o)
    if (kg_is_evid(c, tp, o, i)) v += kg_fdiv(c->v_gamma * rho_lab[o], 32);
  return kg_clamp127(v);
}

/* ---------------- item / operator embeddings (embedding-similarity stage, NEXT-3) --------
 * op embedding e_o[d] = clamp(edir_o[d])/32; item embedding of tuple t:
 * clamp(nrm + Σ_{filters o} ⌊γ_e · y_{t,o} · edir_o[d] / 32⌋)/32 with y = ±1 the latent label —
 * a weaker, noisier signal than the KV-cache operators (a cheap first stage). */
KG_HD int32_t kg_edir(const kg_cfg* c, int32_t o, int32_t d) {
  return kg_nrm_at(kg_h(c->seed, KG_T_EDIR, (uint64_t)o, 0, 0, 0), d);
}
KG_HD int32_t kg_emb_int(const kg_cfg* c, const kg_tuple* tp, int64_t t, int32_t d, int32_t gamma) {
  int32_t v = kg_nrm_at(kg_h(c->seed, KG_T_EMB, (uint64_t)t, 0, 0, 0), d);
  for (int32_t o = 0; o < c->n_ops; ++o)
    if (c->op_classes[o] <= 1) v += kg_fdiv(gamma * tp->label[o] * kg_edir(c, o, d), 32);
  return kg_clamp127(v);
}

/* int in [-127,127] / 32 → bf16 bits (exact: |v|/32 has ≤ 7 significant bits) */
KG_HD uint16_t kg_bf16_of_int32nd(int32_t v) {
  if (v == 0) return 0;
  uint32_t s = v < 0 ? 0x8000u : 0u;
  uint32_t a = (uint32_t)(v < 0 ? -v : v);
  int32_t e = 31;
  while (!(a & (1u << e))) --e;          /* a in [2^e, 2^(e+1)) */
  /* value = a * 2^-5 = 1.m * 2^(e-5); bf16: 8 exponent bits (bias 127), 7 mantissa bits */
  uint32_t exp = (uint32_t)(e - 5 + 127);
  uint32_t mant = (a << (7 - e)) & 0x7Fu; /* e ≤ 6 so shift is non-negative */
  return (uint16_t)(s | (exp << 7) | mant);
}

#endif /* KOGEN_H */
