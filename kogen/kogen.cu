// kogen.cu — host and device twins of the synthetic workload generator (FIXTURE, not product).
// Builds gen/libkogen.so.  All values come from the integer-only formulas in kogen.h, so the
// host fill (used to feed the CPU oracle) and the device fill (used to feed the CUDA path) are
// bit-identical; tests/test_gen.py checks that on sampled pages.
#include "kogen.h"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Tables {  // μ[l][h][d], qdir[o][l][h][d], ρ[o][c][l][h][d]
  std::vector<int32_t> mu, qdir, rho;
  int32_t C;     // max classes over ops (ρ stride)
};

Tables make_tables(const kg_cfg* c) {
  Tables t;
  const int32_t L = c->n_layers, H = c->n_kv_heads, D = c->head_dim;
  t.C = 1;
  for (int o = 0; o < c->n_ops; ++o) t.C = c->op_classes[o] > t.C ? c->op_classes[o] : t.C;
  t.mu.resize((size_t)L * H * D);
  t.qdir.resize((size_t)KG_MAX_OPS * L * H * D, 0);
  t.rho.resize((size_t)KG_MAX_OPS * t.C * L * H * D, 0);
  for (int l = 0; l < L; ++l)
    for (int h = 0; h < H; ++h)
      for (int d = 0; d < D; ++d) {
        t.mu[((size_t)l * H + h) * D + d] = kg_mu(c, l, h, d);
        for (int o = 0; o < c->n_ops; ++o) {
          t.qdir[(((size_t)o * L + l) * H + h) * D + d] = kg_qdir(c, o, l, h, d);
          for (int k = 0; k < c->op_classes[o]; ++k)
            t.rho[((((size_t)o * t.C + k) * L + l) * H + h) * D + d] = kg_rho(c, o, k, l, h, d);
        }
      }
  return t;
}

// ρ seen by V at op o for a tuple with latent label y: filters ±ρ_{o,0}; maps ρ_{o,y}
__host__ __device__ inline int32_t rho_for_label(const int32_t* rho, int32_t C, int32_t L,
                                                 int32_t H, int32_t D, int32_t o, int32_t ncls,
                                                 int32_t y, int32_t l, int32_t h, int32_t d) {
  if (ncls <= 1) return y * rho[((((size_t)o * C + 0) * L + l) * H + h) * D + d];
  return rho[((((size_t)o * C + y) * L + l) * H + h) * D + d];
}

// One page (16 token slots × all layers × K,V × heads × D) of tuple t, page index pi within
// the tuple, written to dst (bf16 bits).  Layout [Lyr][2][Hkv][16][D].
void fill_page_host(const kg_cfg* c, const Tables& tb, int64_t t, const kg_tuple& tp, int32_t pi,
                    uint16_t* dst, bool poison) {
  const int32_t L = c->n_layers, H = c->n_kv_heads, D = c->head_dim;
  int32_t qd[KG_MAX_OPS], rl[KG_MAX_OPS];
  for (int l = 0; l < L; ++l)
    for (int kv = 0; kv < 2; ++kv)
      for (int h = 0; h < H; ++h)
        for (int s = 0; s < KG_PAGE; ++s) {
          int32_t i = pi * KG_PAGE + s;
          uint16_t* row = dst + ((((size_t)l * 2 + kv) * H + h) * KG_PAGE + s) * D;
          if (i >= tp.L) {
            for (int d = 0; d < D; ++d) row[d] = poison ? 0x7FC0 : 0;
            continue;
          }
          uint64_t rh = kg_kv_row_hash(c, kv, t, l, h, i);
          for (int d = 0; d < D; ++d) {
            int32_t v;
            if (kv == 0) {
              for (int o = 0; o < c->n_ops; ++o) qd[o] = tb.qdir[(((size_t)o * L + l) * H + h) * D + d];
              v = kg_k_int(c, &tp, rh, i, d, tb.mu[((size_t)l * H + h) * D + d], qd);
            } else {
              for (int o = 0; o < c->n_ops; ++o)
                rl[o] = rho_for_label(tb.rho.data(), tb.C, L, H, D, o, c->op_classes[o], tp.label[o],
                                      l, h, d);
              v = kg_v_int(c, &tp, rh, i, d, rl);
            }
            row[d] = kg_bf16_of_int32nd(v);
          }
        }
}

struct DevCfg {
  kg_cfg c;
  int32_t C;
};

__global__ void fill_pool_kernel(DevCfg dc, int64_t t_begin, int64_t n_tuples,
                                 const int64_t* __restrict__ indptr,
                                 const int32_t* __restrict__ page_ids, uint16_t* __restrict__ pool,
                                 const int32_t* __restrict__ mu, const int32_t* __restrict__ qdir,
                                 const int32_t* __restrict__ rho, int poison) {
  const kg_cfg& c = dc.c;
  const int32_t L = c.n_layers, H = c.n_kv_heads, D = c.head_dim;
  const int64_t nnz = indptr[n_tuples] - indptr[0];
  __shared__ kg_tuple tp;
  __shared__ int64_t s_t;
  __shared__ int32_t s_pi;
  const size_t page_elems = (size_t)L * 2 * H * KG_PAGE * D;
  const int32_t chunks = (int32_t)(page_elems / 8);
  for (int64_t p = blockIdx.x; p < nnz; p += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t gp = indptr[0] + p;
      int64_t lo = 0, hi = n_tuples - 1;  // largest i with indptr[i] <= gp
      while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (indptr[mid] <= gp) lo = mid; else hi = mid - 1;
      }
      s_t = lo;
      s_pi = (int32_t)(gp - indptr[lo]);
      kg_tuple_init(&c, t_begin + lo, &tp);
    }
    __syncthreads();
    const int64_t t = t_begin + s_t;
    const int32_t pi = s_pi;
    uint16_t* dst = pool + (size_t)page_ids[indptr[0] + p] * page_elems;
    for (int32_t ch = threadIdx.x; ch < chunks; ch += blockDim.x) {
      size_t e0 = (size_t)ch * 8;
      int32_t d0 = (int32_t)(e0 % D);
      size_t r = e0 / D;  // row index over [L][2][H][16]
      int32_t s = (int32_t)(r % KG_PAGE);
      int32_t h = (int32_t)((r / KG_PAGE) % H);
      int32_t kv = (int32_t)((r / ((size_t)KG_PAGE * H)) % 2);
      int32_t l = (int32_t)(r / ((size_t)KG_PAGE * H * 2));
      int32_t i = pi * KG_PAGE + s;
      uint16_t vals[8];
      if (i >= tp.L) {
        for (int e = 0; e < 8; ++e) vals[e] = poison ? 0x7FC0 : 0;
      } else {
        uint64_t rh = kg_kv_row_hash(&c, kv, t, l, h, i);
        for (int e = 0; e < 8; ++e) {
          int32_t d = d0 + e;
          int32_t tmp[KG_MAX_OPS];
          int32_t v;
          if (kv == 0) {
            for (int o = 0; o < c.n_ops; ++o) tmp[o] = qdir[(((size_t)o * L + l) * H + h) * D + d];
            v = kg_k_int(&c, &tp, rh, i, d, mu[((size_t)l * H + h) * D + d], tmp);
          } else {
            for (int o = 0; o < c.n_ops; ++o)
              tmp[o] = rho_for_label(rho, dc.C, L, H, D, o, c.op_classes[o], tp.label[o], l, h, d);
            v = kg_v_int(&c, &tp, rh, i, d, tmp);
          }
          vals[e] = kg_bf16_of_int32nd(v);
        }
      }
      uint4 pk;
      pk.x = (uint32_t)vals[0] | ((uint32_t)vals[1] << 16);
      pk.y = (uint32_t)vals[2] | ((uint32_t)vals[3] << 16);
      pk.z = (uint32_t)vals[4] | ((uint32_t)vals[5] << 16);
      pk.w = (uint32_t)vals[6] | ((uint32_t)vals[7] << 16);
      *reinterpret_cast<uint4*>(dst + e0) = pk;
    }
  }
}

}  // namespace

extern "C" {

// Q_o as bf16 bits [n_layers][n_kv_heads*gqa][n_q][head_dim]
void kg_fill_q(const kg_cfg* c, int32_t o, uint16_t* q) {
  const int32_t Hq = c->n_kv_heads * c->gqa;
  size_t k = 0;
  for (int l = 0; l < c->n_layers; ++l)
    for (int j = 0; j < Hq; ++j)
      for (int r = 0; r < c->n_q; ++r)
        for (int d = 0; d < c->head_dim; ++d) q[k++] = kg_bf16_of_int32nd(kg_q_int(c, o, l, j, r, d));
}

// W_o = int / 2^w_log2_den as fp32 [n_classes][n_layers][n_kv_heads*gqa][n_q][head_dim]
void kg_fill_w(const kg_cfg* c, int32_t o, float* w) {
  const int32_t Hq = c->n_kv_heads * c->gqa;
  size_t k = 0;
  for (int cls = 0; cls < c->op_classes[o]; ++cls)
    for (int l = 0; l < c->n_layers; ++l)
      for (int j = 0; j < Hq; ++j)
        for (int r = 0; r < c->n_q; ++r)
          for (int d = 0; d < c->head_dim; ++d)
            w[k++] = (float)kg_w_int(c, o, cls, l, j, r, d) / (float)(1u << c->w_log2_den);
}

// seq_len[i] and latent labels[o][i] for tuples t0 .. t0+n-1 (labels: filters ±1, maps class)
void kg_fill_meta(const kg_cfg* c, int64_t t0, int64_t n, int32_t* seq_len, int32_t* labels) {
  for (int64_t i = 0; i < n; ++i) {
    if (seq_len) seq_len[i] = kg_seq_len(c, t0 + i);
    if (labels)
      for (int o = 0; o < c->n_ops; ++o) labels[(size_t)o * n + i] = kg_label(c, t0 + i, o);
  }
}

// evidence positions [n][n_ops][n_evid] (for tests of the recipe)
void kg_fill_evidence(const kg_cfg* c, int64_t t0, int64_t n, int32_t* ev) {
  for (int64_t i = 0; i < n; ++i) {
    kg_tuple tp;
    kg_tuple_init(c, t0 + i, &tp);
    for (int o = 0; o < c->n_ops; ++o)
      for (int k = 0; k < c->n_evid; ++k) ev[((size_t)i * c->n_ops + o) * c->n_evid + k] = tp.evid[o][k];
  }
}

// item embeddings bf16 [n][dim] of tuples t0..t0+n-1 and operator embeddings bf16 [n_ops][dim]
void kg_fill_embeddings(const kg_cfg* c, int64_t t0, int64_t n, int32_t dim, int32_t gamma,
                        uint16_t* item, uint16_t* op, int32_t n_threads) {
  std::vector<int32_t> edir((size_t)c->n_ops * dim);
  for (int o = 0; o < c->n_ops; ++o)
    for (int d = 0; d < dim; ++d) {
      edir[(size_t)o * dim + d] = kg_edir(c, o, d);
      if (op) op[(size_t)o * dim + d] = kg_bf16_of_int32nd(kg_clamp127(edir[(size_t)o * dim + d]));
    }
  if (!item) return;
  if (n_threads < 1) n_threads = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < n_threads; ++w)
    th.emplace_back([&, w]() {
      for (int64_t i = w; i < n; i += n_threads) {
        kg_tuple tp;
        kg_tuple_init(c, t0 + i, &tp);
        for (int d = 0; d < dim; ++d)
          item[(size_t)i * dim + d] = kg_bf16_of_int32nd(kg_emb_int(c, &tp, t0 + i, d, gamma));
      }
    });
  for (auto& x : th) x.join();
}

// Host fill of the pages of tuples tuple_ids[0..n): tuple tuple_ids[i] owns logical pages
// page_indptr[i] .. page_indptr[i+1] (ceil(L/16) of them) placed at physical page_ids[...].
// pool has room for max(page_ids)+1 pages.  Multi-threaded over tuples.
int kg_fill_pool_host(const kg_cfg* c, const int64_t* tuple_ids, int64_t n,
                      const int64_t* page_indptr, const int32_t* page_ids, uint16_t* pool,
                      int32_t poison, int32_t n_threads) {
  Tables tb = make_tables(c);
  const size_t page_elems = (size_t)c->n_layers * 2 * c->n_kv_heads * KG_PAGE * c->head_dim;
  if (n_threads < 1) n_threads = 1;
  std::vector<std::thread> th;
  for (int w = 0; w < n_threads; ++w)
    th.emplace_back([&, w]() {
      for (int64_t i = w; i < n; i += n_threads) {
        kg_tuple tp;
        kg_tuple_init(c, tuple_ids[i], &tp);
        int64_t np = page_indptr[i + 1] - page_indptr[i];
        for (int64_t pi = 0; pi < np; ++pi)
          fill_page_host(c, tb, tuple_ids[i], tp, (int32_t)pi,
                         pool + (size_t)page_ids[page_indptr[i] + pi] * page_elems, poison != 0);
      }
    });
  for (auto& x : th) x.join();
  return 0;
}

// Read-only HBM stream (measurement helper for bench.py's roofline context): every warp owns a
// 3-stage shared-memory ring of 16 KiB bulk copies (cp.async.bulk + mbarrier, L2 evict-first) and
// walks the buffer in warp-strided 16 KiB chunks, touching one word per chunk — the same
// TMA-into-smem read path as the scoring kernel, without its math.
__device__ __forceinline__ uint32_t rs_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int kRsStages = 3, kRsChunk = 16384;
__global__ void __launch_bounds__(128) read_stream_kernel(const uint8_t* __restrict__ p, int64_t n_chunks,
                                                          uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t rs_sm[];
  __shared__ __align__(8) uint64_t bar[4][kRsStages];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = rs_sm + warp * kRsStages * kRsChunk;
  if (lane == 0)
    for (int s = 0; s < kRsStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rs_su32(&bar[warp][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t nw = (int64_t)gridDim.x * 4;
  int64_t next = (int64_t)blockIdx.x * 4 + warp, issued = 0, consumed = 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&]() {
    if (lane == 0) {
      const int s = (int)(issued % kRsStages);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rs_su32(&bar[warp][s])),
                   "r"(kRsChunk) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
          "[%3], %4;" ::"r"(rs_su32(ring + s * kRsChunk)), "l"(p + next * kRsChunk), "r"(kRsChunk),
          "r"(rs_su32(&bar[warp][s])), "l"(pol) : "memory");
    }
    ++issued;
    next += nw;
  };
  for (int k = 0; k < kRsStages && next < n_chunks; ++k) issue();
  uint32_t acc = 0;
  while (consumed < issued) {
    const int s = (int)(consumed % kRsStages);
    const uint32_t par = (uint32_t)((consumed / kRsStages) & 1);
    uint32_t done = 0;
    do {
      asm volatile("{\n.reg .pred q;\nmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\nselp.u32 %0,1,0,q;\n}"
                   : "=r"(done) : "r"(rs_su32(&bar[warp][s])), "r"(par) : "memory");
    } while (!done);
    acc ^= *(volatile uint32_t*)(ring + s * kRsChunk + lane * 4);
    __syncwarp();
    ++consumed;
    if (next < n_chunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue();
    }
  }
  if (acc == 0x9e3779b9u) sink[blockIdx.x] = acc;  // practically never taken; keeps reads live
}

// Gathered-read stream: rows idx[0..n) of `row_bytes` each (16-byte multiple, ≤ 512) read
// once through a per-warp ring of bulk copies, 32 rows per stage (one per lane) — the ceiling of
// a kernel that reads a gathered row subset (ko_embed_scores with tuple_idx).
__global__ void __launch_bounds__(128) gather_stream_kernel(const uint8_t* __restrict__ base,
                                                            int row_bytes, const int32_t* __restrict__ idx,
                                                            int64_t n, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t gs_sm[];
  __shared__ __align__(8) uint64_t bar[4][kRsStages];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int stage_bytes = 32 * row_bytes;
  uint8_t* ring = gs_sm + warp * kRsStages * stage_bytes;
  if (lane == 0)
    for (int s = 0; s < kRsStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rs_su32(&bar[warp][s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t n_blk = (n + 31) / 32, nw = (int64_t)gridDim.x * 4;
  int64_t next = (int64_t)blockIdx.x * 4 + warp, issued = 0, consumed = 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&]() {
    const int s = (int)(issued % kRsStages);
    const int64_t w = next * 32 + lane;
    const int rows = (int)(n - next * 32 < 32 ? n - next * 32 : 32);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rs_su32(&bar[warp][s])),
                   "r"(rows * row_bytes) : "memory");
    __syncwarp();
    if (lane < rows)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
          "[%3], %4;" ::"r"(rs_su32(ring + s * stage_bytes + lane * row_bytes)),
          "l"(base + (int64_t)idx[w] * row_bytes), "r"(row_bytes), "r"(rs_su32(&bar[warp][s])), "l"(pol)
          : "memory");
    ++issued;
    next += nw;
  };
  for (int k = 0; k < kRsStages && next < n_blk; ++k) issue();
  uint32_t acc = 0;
  while (consumed < issued) {
    const int s = (int)(consumed % kRsStages);
    const uint32_t par = (uint32_t)((consumed / kRsStages) & 1);
    uint32_t done = 0;
    do {
      asm volatile("{\n.reg .pred q;\nmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\nselp.u32 %0,1,0,q;\n}"
                   : "=r"(done) : "r"(rs_su32(&bar[warp][s])), "r"(par) : "memory");
    } while (!done);
    acc ^= *(volatile uint32_t*)(ring + s * stage_bytes + lane * 4);
    __syncwarp();
    ++consumed;
    if (next < n_blk) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue();
    }
  }
  if (acc == 0x9e3779b9u) sink[blockIdx.x] = acc;  // practically never taken; keeps reads live
}

// Device fill: tuples t_begin .. t_begin+n_tuples-1 with device CSR (indptr has n_tuples+1
// entries, may start at a non-zero offset), pages written into the device pool.
int kg_fill_pool_device(const kg_cfg* c, int64_t t_begin, int64_t n_tuples, const int64_t* d_indptr,
                        const int32_t* d_page_ids, void* d_pool, int32_t poison, void* stream) {
  Tables tb = make_tables(c);
  int32_t *d_mu = nullptr, *d_qdir = nullptr, *d_rho = nullptr;
  if (cudaMalloc(&d_mu, tb.mu.size() * 4) != cudaSuccess) return 1;
  if (cudaMalloc(&d_qdir, tb.qdir.size() * 4) != cudaSuccess) return 1;
  if (cudaMalloc(&d_rho, tb.rho.size() * 4) != cudaSuccess) return 1;
  cudaMemcpy(d_mu, tb.mu.data(), tb.mu.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_qdir, tb.qdir.data(), tb.qdir.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_rho, tb.rho.data(), tb.rho.size() * 4, cudaMemcpyHostToDevice);
  DevCfg dc;
  dc.c = *c;
  dc.C = tb.C;
  cudaStream_t s = (cudaStream_t)stream;
  fill_pool_kernel<<<148 * 8, 256, 0, s>>>(dc, t_begin, n_tuples, d_indptr, d_page_ids,
                                           (uint16_t*)d_pool, d_mu, d_qdir, d_rho, poison);
  cudaError_t e = cudaGetLastError();
  cudaStreamSynchronize(s);
  cudaFree(d_mu);
  cudaFree(d_qdir);
  cudaFree(d_rho);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 2;
}

// Measurement helper (bench.py): one read-only pass over `bytes` (multiple of 16 KiB) of a device
// buffer through the bulk-copy ring above; its rate is the "read-stream peak" the scoring
// kernel's achieved GB/s is compared with besides the driver's read+write copy peak.
int kg_read_stream(const void* d_buf, int64_t bytes, uint32_t* d_sink, void* stream) {
  const int smem = 4 * kRsStages * kRsChunk;
  cudaFuncSetAttribute(read_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  read_stream_kernel<<<sms, 128, smem, (cudaStream_t)stream>>>((const uint8_t*)d_buf, bytes / kRsChunk,
                                                               d_sink);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int kg_gather_stream(const void* d_base, int32_t row_bytes, const int32_t* d_idx, int64_t n,
                     uint32_t* d_sink, void* stream) {
  if (row_bytes % 16 != 0 || row_bytes < 16 || row_bytes > 512) return 1;
  const int smem = 4 * kRsStages * 32 * row_bytes;
  cudaFuncSetAttribute(gather_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_stream_kernel, 128, smem);
  gather_stream_kernel<<<sms * (occ > 0 ? occ : 1), 128, smem, (cudaStream_t)stream>>>(
      (const uint8_t*)d_base, row_bytes, d_idx, n, d_sink);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // extern "C"
