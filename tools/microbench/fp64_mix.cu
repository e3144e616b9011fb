// Microbenchmark: do DFMA (CUDA-core FP64) and DMMA (FP64 tensor core, mma.sync m8n8k4) share one
// pipe on B200? Half the warps of each CTA run a DFMA loop, the other half a DMMA loop; compare
// the combined FLOP rate with each alone.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dfma_loop(int iters, double& x0, double& x1, double& x2, double& x3,
                                          double& x4, double& x5, double& x6, double& x7) {
  const double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
}
__device__ __forceinline__ void dmma_loop(int iters, double& c0, double& c1, double& d0, double& d1, double& e0,
                                          double& e1, double& f0, double& f1) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
    }
  }
}
// mode 0: all DFMA, 1: all DMMA, 2: half/half
__global__ void mix(double* out, int mode, int it_f, int it_m) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  const int warp = threadIdx.x >> 5;
  const bool do_f = mode == 0 || (mode == 2 && (warp & 1) == 0);
  if (do_f) dfma_loop(it_f, x0, x1, x2, x3, x4, x5, x6, x7);
  else dmma_loop(it_m, x0, x1, x2, x3, x4, x5, x6, x7);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 4 * 512);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 2;
  // per-warp flops: DFMA: it_f*64*32*2 ; DMMA: it_m*32*512 (8*8*4*2 flops per mma)
  const int it_f = 4096, it_m = 512;  // balanced so each half takes similar time
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<blocks, threads>>>(out, mode, 16, 4);
    cudaEventRecord(e0);
    mix<<<blocks, threads>>>(out, mode, it_f, it_m);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = (double)blocks * threads / 32;
    double ff = (double)it_f * 64 * 32 * 2, fm = (double)it_m * 32 * 512;
    double flops = mode == 0 ? warps * ff : mode == 1 ? warps * fm : warps / 2 * (ff + fm);
    printf("{\"mode\":\"%s\",\"ms\":%.3f,\"tflops\":%.2f}\n", mode == 0 ? "dfma" : mode == 1 ? "dmma" : "mixed", ms, flops / ms / 1e9);
  }
  return 0;
}
