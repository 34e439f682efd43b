// tools/mma_peak.cu — measured throughput of mma.sync.m16n8k16 bf16→fp32 on this GPU (the
// instruction the scoring kernel issues), to place the kernel's tensor-pipe utilisation on a
// measured rather than a nominal ceiling (DESIGN.md §4 roofline).  Every warp runs 8 independent
// accumulator chains; grid = SMs × 8 CTAs × 4 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak tools/mma_peak.cu && ./mma_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(128) mma_loop(int iters, float* out) {
  uint32_t a0 = threadIdx.x * 0x3f80u, a1 = a0 ^ 0x1234u, a2 = a0 + 7u, a3 = a1 + 3u;
  uint32_t b0 = a0 * 3u, b1 = a1 * 5u;
  float acc[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                   "{%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 20000, blocks = sms * 8;
  mma_loop<<<blocks, 128>>>(100, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    mma_loop<<<blocks, 128>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flop = 2.0 * 16 * 8 * 16 * 8.0 * iters * (double)blocks * 4;
  printf("{\"mma_sync_m16n8k16_bf16_tflops\": %.1f, \"sms\": %d, \"ms\": %.3f}\n",
         flop / (best / 1e3) / 1e12, sms, best);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
