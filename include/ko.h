/* ko.h — C ABI of libko.so: the KV-cache semantic-operator scoring → routing → count pass of
 * arXiv 2602.04430 ("Stretto"), built for B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n (section / equation named beside it).  The readings of silent
 * or garbled passages (Q1–Q24) are listed in DESIGN.md §Readings.
 *
 *   Operator (§"KV cache–enabled Operators / Online"): an operator "loads a collection
 *   of precomputed KV caches, appends an operator-specific query ..., and executes a single
 *   batched forward pass to produce one output per item".  Filters use the logits of tokens '1'
 *   and '0' and "compute the log-odds between these tokens, which the system uses to classify the
 *   item as accepted, rejected, or unsure based on optimized thresholds".
 *   Here the forward pass is the attention-only proxy of Q1: per layer l, q-head j (kv-head
 *   h = j / gqa_group) and query row r,
 *       s_i = <Q[l][j][r], K[l][h][i]> / sqrt(head_dim),  O = softmax(s) · V   (i < n_kept)
 *       z_c = b_c + Σ_{l < layer_cut} Σ_j Σ_r <W[c][l][j][r], O>
 *   filter margin m = z_0 (yes − no log-odds); map-classify: class = argmax z (lowest index on
 *   ties), m = z_(1) − z_(2).
 *   Variant ("profile"; compression ratio P:190-193): the tuple's tokens are
 *   stored in descending query-agnostic importance, so a compression ratio is the prefix
 *   n_kept = max(1, floor(L_t · keep_permille / 1000)) (Q2, Q3); layer_cut stands in for model
 *   size (Q2).
 *   Plan (Eqs. accept-i / reject-i / unsure-i at P:323-327): an ordered list of stages;
 *   a filter stage accepts iff m > theta_hi, rejects iff m < theta_lo, else unsure (
 *   strict, Q5); a final stage accepts iff m > theta (tie rejects, Q6); a map stage resolves iff
 *   m > theta_hi (final: always), maps never reject (Q13).  Tuple t reaches stage s iff it is
 *   alive and op_s is still pending (inter-operator semantics P:536-539, conjunctive, Q12).
 *   Counts: TP/FP/FN of Eqs. sample-tp/fp/fn on the whole plan output vs the gold
 *   plan (map values P:513-519), and per stage n_in / n_acc / n_rej / n_uns, from which
 *   cost Eq. and inter/intra selectivities derive on the host.
 *
 * Conventions (all entry points):
 *   - Every data pointer is DEVICE memory owned by the caller (e.g. a torch tensor), except the
 *     descriptor structs (ko_kv_cache, ko_operator, ko_variant, ko_plan), which are HOST structs
 *     read before the call returns.  Nothing is allocated inside a call; scratch lives in the
 *     caller's workspace (size from ko_workspace_size).
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).  Outputs
 *     are valid after the stream reaches the call.
 *   - Errors: host validation runs before any launch.  KO_EINVAL (bad argument), KO_EUNSUPPORTED
 *     (shape outside the compiled kernels), KO_EWORKSPACE (workspace too small) and KO_ECUDA (a
 *     launch or CUDA API failure) return without touching outputs past the failing launch;
 *     ko_last_error() returns a thread-local message.  Device-data errors (page id out of range,
 *     seq_len <= 0) are undefined behaviour.
 *   - Determinism: margins are bitwise reproducible for a given input regardless of tuple order,
 *     sharding or page placement (fixed-order per-tuple sums, no float atomics).  Counts are exact
 *     integers, ACCUMULATED (+=) into a caller-zeroed int64 buffer, so shards and resident
 *     batches add and multi-GPU is one all-reduce(SUM).
 */
#ifndef KO_H
#define KO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KO_OK = 0,
  KO_EINVAL = 1,
  KO_EUNSUPPORTED = 2,
  KO_ECUDA = 3,
  KO_EWORKSPACE = 4
} ko_status;

enum {
  KO_PAGE_TOKENS = 16,  /* tokens per KV page                                          */
  KO_MAX_OPS = 4,       /* operators per call                                          */
  KO_MAX_VARIANTS = 8,  /* variants per call                                           */
  KO_MAX_STAGES = 8,    /* stages per plan                                             */
  KO_MAX_PLANS = 64,    /* plans per grid call                                         */
  KO_MAX_CLASSES = 8,   /* classes of a map-classify operator                          */
  KO_MAX_ROWS = 16,     /* n_ops · gqa_group · n_q rows attending one kv-head          */
  KO_COUNTS_PER_PLAN = 5 + 4 * KO_MAX_STAGES
};

/* counts layout per plan g (int64, stride KO_COUNTS_PER_PLAN):
 *   [0] TP  [1] FP  [2] FN  [3] n_out = |P_o|  [4] n_gold = |P_g|
 *   then per stage s: [5+4s] n_in  [6+4s] n_acc  [7+4s] n_rej  [8+4s] n_uns           */
enum { KO_C_TP = 0, KO_C_FP = 1, KO_C_FN = 2, KO_C_OUT = 3, KO_C_GOLD = 4, KO_C_STAGE0 = 5 };

/* One importance-ordered paged KV store (device memory, caller-owned). */
typedef struct {
  int32_t n_layers;    /* layers stored                                                  */
  int32_t n_kv_heads;  /* kv heads                                                       */
  int32_t gqa_group;   /* q-heads per kv-head (q-head j uses kv-head j / gqa_group, Q18) */
  int32_t head_dim;    /* 64 or 128                                                      */
  int32_t n_q;         /* operator-query rows per q-head (>= 1)                          */
  const void* kv_pool; /* bf16 [n_pages][n_layers][2 (K,V)][n_kv_heads][16][head_dim],
                          16-byte aligned; K is post-RoPE (Q15)                          */
  int64_t n_pages;
  const int64_t* page_indptr; /* [n_tuples+1] CSR offsets into page_ids                  */
  const int32_t* page_ids;    /* logical page order = token importance order (Q2)        */
  const int32_t* seq_len;     /* [n_tuples] L_t >= 1; slots >= L_t of the last page are
                                 never read (they may hold anything, including NaN)       */
  int64_t n_tuples;
} ko_kv_cache;

/* One logical operator, shared by all tuples (device memory). */
typedef struct {
  int32_t n_classes; /* 1 = filter (z_0 = yes−no log-odds), 2..KO_MAX_CLASSES = map-classify */
  const void* q;     /* bf16 [n_layers][n_kv_heads*gqa_group][n_q][head_dim], post-RoPE       */
  const void* w;     /* readout [n_classes][n_layers][n_kv_heads*gqa_group][n_q][head_dim]:
                        fp32 (entered as bf16 hi + lo, error ≤ 2^-17 |w|) or, with w_is_bf16,
                        bf16 (exact; a K-class map then needs half the tensor-core tiles)      */
  const float* b;    /* fp32 [n_classes]                                                      */
  int32_t w_is_bf16; /* 0: w is fp32; 1: w is bf16                                            */
} ko_operator;

typedef struct {
  int32_t keep_permille; /* 1..1000: n_kept = max(1, floor(L·keep/1000)) (Q3)             */
  int32_t layer_cut;     /* 1..n_layers: layers l < layer_cut are consulted              */
} ko_variant;
/* A variant with keep_permille == 0 and layer_cut == 0 is EXTERNAL: its margins are supplied
 * by the caller in the margins array (e.g. an embedding-similarity stage, ko_embed_scores) and
 * plans may use it like any other (filters only).  ko_score_batch never overwrites them.      */

typedef struct {
  int32_t op, variant; /* indices into the call's ops[] and variants[]                   */
  float theta_lo;      /* θ⁻ (filters, non-final); ignored for maps                       */
  float theta_hi;      /* θ⁺; final filter stage: theta_lo == theta_hi == θ_f required    */
  int32_t is_final;    /* 1 = the op's last (gold-like) stage: resolves every tuple       */
} ko_stage;

typedef struct {
  int32_t n_stages;             /* 1..KO_MAX_STAGES, in execution order (Q23)           */
  ko_stage stage[KO_MAX_STAGES];
} ko_plan;

/* ko_score_batch — score tuples with every (op, variant), optionally route + count.
 *
 * kv, ops[n_ops], variants[n_variants]: as above.
 * tuple_idx: device int32 [n_idx] tuple ids to process (any order, no duplicates), or NULL = all
 *            n_tuples (n_idx ignored).  n_idx == 0 with a non-NULL tuple_idx is a no-op.
 * margins:   device fp32 [n_ops][n_variants][n_tuples], indexed by tuple id (may be NULL only in
 *            routed mode).  classes: device int32, same shape, argmax class (0 for filters); may
 *            be NULL; in routed mode only the reached (finite-margin) entries are written.
 * plans[n_plans]: host plan structs; NULL/0 = profiling only.
 *   - n_plans >= 2 or plans on a profiling call ("grid mode", P:281-286 profiling + the 64-point
 *     grid of BASELINE config 5): every (op, variant, tuple) margin is computed in ONE read of
 *     each tuple's cache (nested prefixes: the largest variant's bytes serve all), then every
 *     plan is evaluated per tuple (by a finaliser launch on the same stream, after the scan) and
 *     its counts accumulated.
 *   - n_plans == 1 ("routed mode", P:176-180 cascades): stages execute in order; only tuples
 *     reaching a stage are scored for it (the rest of the processed tuples' KV-variant margins
 *     are set to NaN; tuples outside tuple_idx and external variants are not touched), which is the
 *     runtime saving cascades exist for.  Each tuple's cache is read once, up to the
 *     largest extent its reached stages need: the plan's operators share one read while they fit
 *     one 16-row tile (an operator's margin may be computed for a tuple that never reaches its
 *     stage — never written, same bytes), and a later, larger variant resumes from the softmax
 *     state saved at the end of the earlier extent.  Margins are bitwise
 *     reproducible; they may differ in the last bits from grid mode's (different summation
 *     split), within the parity tolerance.
 * gold:      device uint8 [n_ops][n_tuples] (filter 0/1, map class) or NULL: then TP/FP/FN and
 *            n_gold stay 0 (execution on unlabelled data).
 * counts:    device int64 [n_plans][KO_COUNTS_PER_PLAN], accumulated (+=).
 * workspace: device scratch of >= ko_workspace_size(...) bytes, 256-byte aligned (per-tuple
 *            partial logits and, for routed mode, saved softmax states: O(n_tuples · n_layers ·
 *            n_kv_heads · n_ops · (n_variants · classes + 8·(4 + 2·tiles))) floats).  Its
 *            contents on entry do not matter: a call reads only what it wrote itself.
 * Errors: KO_EINVAL for NULL required pointers, head_dim not in {64,128}, keep_permille outside
 *   [1,1000], layer_cut outside [1,n_layers], theta_lo > theta_hi, a final filter stage with
 *   theta_lo != theta_hi, a referenced op with no final stage or a stage after its final stage,
 *   n_stages outside [1,8], n_plans > 64; KO_EUNSUPPORTED when n_ops·gqa_group·n_q > 16 or
 *   n_classes > 8.                                                                         */
ko_status ko_score_batch(const ko_kv_cache* kv, const ko_operator* ops, int32_t n_ops,
                         const ko_variant* variants, int32_t n_variants, const int32_t* tuple_idx,
                         int64_t n_idx, float* margins, int32_t* classes, const ko_plan* plans,
                         int32_t n_plans, const uint8_t* gold, int64_t* counts, void* workspace,
                         size_t workspace_bytes, void* stream);

/* ko_route — cascade routing (Eqs. accept-i / reject-i / unsure-i) on precomputed
 * margins/classes [n_ops][n_variants][n_tuples] (device).  n_classes: host int32 [n_ops].
 *   stage == -1: run the whole plan for every tuple; tuple_state ends in the final state,
 *                worklist_out receives P_o (the alive tuples) and counts get the plan's full
 *                count row (gold may be NULL).
 *   stage == s : apply stage s's decision to every tuple that reaches s (alive and op_s pending),
 *                update tuple_state and the stage-s counters, then write to worklist_out the
 *                tuples that reach stage s+1 (none when s is the last stage).
 * tuple_state: device uint32 [n_tuples] in/out.  bit 0 = alive; bits 1+2o..2+2o = status of op o
 *              (0 pending, 1 accepted/resolved, 2 rejected); bits 16+4o..19+4o = resolved class
 *              of map op o; bits 9..15 are reserved (the score_batch routed executor keeps its
 *              resume stage there).  Initialise to 1 (alive, all pending) before stage 0.
 * worklist_out: device int32 [n_tuples]; worklist_len: device int64 scalar (overwritten).  The
 *              order of the worklist is unspecified (compare as a set).                      */
ko_status ko_route(const ko_plan* plan, const float* margins, const int32_t* classes,
                   const int32_t* n_classes, int32_t n_ops, int32_t n_variants, int64_t n_tuples,
                   int32_t stage, uint32_t* tuple_state, int32_t* worklist_out,
                   int64_t* worklist_len, const uint8_t* gold, int64_t* counts, void* stream);

/* ko_reduce_stats — evaluate n_plans (<= 64) plans on the same precomputed margins and
 * accumulate each plan's count row (TP, FP, FN, |P_o|, |P_g|, per-stage n_in/acc/rej/uns).  This
 * is the profiling-matrix → counts step the optimizer consumes.        */
ko_status ko_reduce_stats(const ko_plan* plans, int32_t n_plans, const float* margins,
                          const int32_t* classes, const int32_t* n_classes, int32_t n_ops,
                          int32_t n_variants, int64_t n_tuples, const uint8_t* gold,
                          int64_t* counts, void* stream);

/* ko_embed_scores — the embedding-similarity filter stage ("a lightweight embedding-based
 * operator that computes similarities between data and query embeddings and applies a decision
 * threshold", P:456-458 two thresholds, Blip P:746; NEXT-3): for every tuple t (tuple_idx or all)
 * and every operator embedding e, margins[op_ids[e]][variant][t] = cos(item_emb[t], op_emb[e]).
 * item_emb: device bf16 [n_tuples][dim] (16-byte aligned); op_emb: device bf16 [n_emb][dim];
 * op_ids: host int32 [n_emb]; dim a multiple of 8 (≤ 1024); fp32 accumulation.  Use a variant
 * marked external (keep‰ = layer_cut = 0) to chain it into plans.                              */
ko_status ko_embed_scores(const void* item_emb, int32_t dim, int64_t n_tuples, const void* op_emb,
                          int32_t n_emb, const int32_t* op_ids, int32_t n_ops, int32_t variant,
                          int32_t n_variants, const int32_t* tuple_idx, int64_t n_idx,
                          float* margins, void* stream);

/* ko_build_importance_order — offline builder of the importance-ordered store the variants read
 * (NEXT-4; "KV Cache Creation", query-agnostic Expected Attention P:190-193).
 * For every tuple, layer and kv-head of `src` (any token order), the log expected un-normalised
 * attention of each key under a Gaussian query model N(mu, diag sigma2) (reading Q25),
 *     s(k) = (Σ_d mu_d k_d)/sqrt(D) + (Σ_d sigma2_d k_d²)/(2D)   (fp64, no fused multiply-add),
 * orders the tokens by descending s (ties: lower source index first) and writes their K and V
 * rows, rank r to slot r % 16 of logical page r / 16, into dst_pool at pages dst_page_ids (same
 * CSR offsets src->page_indptr; same page geometry).  Slots past L_t are not written.
 * mu, sigma2: device fp32 [n_layers][n_kv_heads][head_dim].  Tuples longer than 4096 tokens are
 * skipped (not supported).  Every byte moves by TMA over 2-D views of both pools
 * ([n_pages · 2·n_layers·n_kv_heads·16 rows][head_dim]); a pool whose view has ≥ 2^31 rows
 * returns KO_EUNSUPPORTED before any launch.  Asynchronous on `stream`.                       */
ko_status ko_build_importance_order(const ko_kv_cache* src, const float* mu, const float* sigma2,
                                    void* dst_pool, const int32_t* dst_page_ids, void* stream);

/* ko_soft_stats — the continuous relaxation of one plan (NEXT-1 of SURVEY §8(f)) on
 * precomputed margins: pick factors σ_i = sigmoid(s_i/τ) (final stages σ = 1), soft decisions
 * π_i = softmax([m − θ⁺, θ⁻ − m, 0]/τ) (final stages: accept = sigmoid((m − θ⁺)/τ)), the relaxed
 * recurrences of Eqs. accept-i / reject-i / unsure-i, plan accept mass = product over the plan's
 * operators, soft TP / FP / FN (Eqs. 5–7) and cost Σ σ_i c_i · (mass reaching stage i) — and the
 * exact derivatives of these four sums w.r.t. every stage's (s_i, θ⁻_i, θ⁺_i) at the plan's
 * thresholds.  Map-classify operators (output-tuple selection): a non-final map stage
 * resolves the mass u·σ_i·sigmoid((m − θ⁺)/τ) (finals: all of it) with the stage's argmax class;
 * maps never reject (Q13); TP counts a tuple's plan-output mass times, per map, the mass resolved
 * to its gold class, FP = output mass − TP, FN = gold mass − TP (a wrong value is one FP and one FN).
 * pick_scores, stage_cost: HOST double [plan->n_stages]; tau > 0; n_classes: host [n_ops].
 * classes: device int32 [n_ops][n_variants][n_tuples] argmax classes (required iff the plan has a
 *      map stage, else may be NULL); gold: device uint8 [n_ops][n_tuples] (filters 0/1, maps the
 *      class) or NULL.
 * out: DEVICE double [4 + 12·n_stages] = {TP, FP, FN, cost} then, for q in (TP, FP, FN, cost),
 *      d q / d(s_i, θ⁻_i, θ⁺_i) at index 4 + q·3·n_stages + 3i + {0,1,2} (finals: d/ds = d/dθ⁻ = 0,
 *      the threshold derivative is reported on θ⁺; map stages: d/dθ⁻ = 0; a final map stage has
 *      no parameters).  Sums are fp64 in a fixed order (bitwise reproducible).
 *      workspace: >= ko_soft_workspace_size(n_stages, n_tuples) bytes.                        */
ko_status ko_soft_stats(const ko_plan* plan, const double* pick_scores, const double* stage_cost,
                        double tau, const float* margins, const int32_t* classes,
                        const int32_t* n_classes, int32_t n_ops, int32_t n_variants,
                        int64_t n_tuples, const uint8_t* gold, double* out, void* workspace,
                        size_t workspace_bytes, void* stream);
size_t ko_soft_workspace_size(int32_t n_stages, int64_t n_tuples);

/* Bytes of device workspace ko_score_batch needs for this shape (n_work = number of tuples it
 * will process: n_idx, or n_tuples when tuple_idx is NULL).  Returns 0 on invalid arguments. */
size_t ko_workspace_size(const ko_kv_cache* kv, const ko_operator* ops, int32_t n_ops,
                         int32_t n_variants, int64_t n_work);

/* Host helper (not GPU work): Bayesian lower bound of Eqs. recall-lower-bound /
 * precision-lower-bound: the (1 − alpha) quantile of Beta(1 + a, 1 + b), i.e.
 * ℓ_α = I^{-1}(1 − α; 1 + a, 1 + b) (Q7).  recall: (a, b) = (TP, FN); precision: (TP, FP).
 * Returns NaN on invalid input (a < 0, b < 0, alpha outside (0,1)).                           */
double ko_beta_lower_bound(int64_t a, int64_t b, double alpha);

/* Host helper: ko_beta_lower_bound for real-valued (soft, relaxed) counts a, b >= 0 — the bound
 * the gradient loop differentiates — and its partial derivatives dℓ/da, dℓ/db (either
 * pointer may be NULL) by implicit differentiation of I_ℓ(1+a, 1+b) = 1 − α:
 * dℓ/da = −(∂I/∂a)/(∂I/∂x), ∂I/∂x the Beta density, ∂I/∂a central differences of I.
 * Returns NaN on invalid input. */
double ko_beta_lower_bound_real(double a, double b, double alpha, double* dl_da, double* dl_db);

/* Loss of the operator-selection objective (eqn:cost-loss … eqn:loss; NEXT-2):
 *   L_cost = cost / (|S| · Σ_i cost_{o_i}),   L_R = ReLU(T_R − ℓ_α^R),   L_P = ReLU(T_P − ℓ_α^P),
 *   L = L_cost + β·L_P + β·L_R,
 * ℓ_α^R = I^{-1}(1 − α; 1 + TP, 1 + FN), ℓ_α^P = I^{-1}(1 − α; 1 + TP, 1 + FP) (Eqs. 8–9, real
 * counts).  "The loss on precision and recall are only active (gradient ≠ 0) if the current
 * pipeline violates the respective target": at T = ℓ the constraint term contributes 0.
 * stats: HOST double [4] = {TP, FP, FN, cost} — hard counts (cost = Σ_s n_in[s]·stage_cost[s]) or
 *        ko_soft_stats' first four outputs (soft counts, σ-scaled cost).
 * jacobian: HOST double [4][n_params] = d{TP, FP, FN, cost}/d params (ko_soft_stats' layout, at
 *        out + 4 with n_params = 3·n_stages), or NULL with n_params = 0.
 * n_tuples: |S|; stage_cost: HOST double [n_stages] = cost_{o_i} of the plan's stages.
 * out: HOST double [10] = {L, L_cost, L_R, L_P, ℓ_R, ℓ_P, recall, precision, Target Met recall,
 *        Target Met precision}; Target Met = achieved / target (NaN for a zero target),
 *        achieved = TP/(TP+FN) and TP/(TP+FP) (1 when the denominator is 0, Q20).
 * grad: HOST double [n_params] = dL/d params by the chain rule through ℓ, or NULL.
 * Errors: KO_EINVAL (NULL/negative/NaN inputs, alpha outside (0,1), β < 0).  Host only.       */
typedef struct {
  double target_recall;    /* T_R (0 = no recall constraint)                                 */
  double target_precision; /* T_P (0 = no precision constraint)                              */
  double alpha;            /* credible level α of the lower bounds               */
  double beta;             /* constraint weight β of eqn:loss                                */
} ko_loss_params;
ko_status ko_plan_loss(const double* stats, const double* jacobian, int32_t n_params,
                       double n_tuples, const double* stage_cost, int32_t n_stages,
                       const ko_loss_params* lp, double* out, double* grad);

/* Tracing hook (runtime profiling): when ev_begin/ev_end (cudaEvent_t handles) are non-NULL,
 * every later ko_score_batch call on this thread records ev_begin on its stream immediately before
 * its first scoring-kernel launch and ev_end immediately after its last one, so a caller can time
 * the hot kernel alone with cudaEventElapsedTime.  Pass NULL, NULL to disable. */
void ko_set_trace_events(void* ev_begin, void* ev_end);

/* Number of kernels the last compute call on this thread (ko_score_batch, ko_route,
 * ko_reduce_stats, ko_embed_scores, ko_build_importance_order, ko_soft_stats) launched — how
 * bench.py counts the library's own launches inside its timed region. */
int32_t ko_last_launch_count(void);

/* Thread-local message describing the last non-OK status returned on this thread. */
const char* ko_last_error(void);

/* Library version string. */
const char* ko_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KO_H */
