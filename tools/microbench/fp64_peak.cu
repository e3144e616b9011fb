// Microbenchmark: device properties, FP64 FMA throughput (DFMA), FP64 tensor (DMMA m8n8k4)
// throughput, and a double2 streaming copy, on the B200 the bench runs on. Gives the "alu"
// roofline denominator DESIGN.md cites (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

__global__ void rmw_kernel(double2* __restrict__ a, size_t n, double s) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = a[i]; v.x *= s; v.y *= s; a[i] = v;
  }
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"mem_bytes\":%zu,\"smem_per_block_optin\":%zu,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"cc\":\"%d.%d\"}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.totalGlobalMem, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.major, p.minor);
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSm : {2, 4, 8}) {
    int iters = 4096, threads = 256, blocks = sms * blocksPerSm;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("{\"dfma_tflops\":%.2f,\"blocks_per_sm\":%d,\"ms\":%.3f}\n", flops / ms / 1e9, blocksPerSm, ms);
  }
  for (int blocksPerSm : {2, 4, 8}) {
    int iters = 2048, threads = 256, blocks = sms * blocksPerSm;
    dmma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 32.0 * iters * (double)blocks * threads / 32;
    printf("{\"dmma_tflops\":%.2f,\"blocks_per_sm\":%d,\"ms\":%.3f}\n", flops / ms / 1e9, blocksPerSm, ms);
  }
  size_t n = (size_t)1 << 28;  // 4 GiB of double2
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  for (int blocksPerSm : {4, 8, 16}) {
    int threads = 256, blocks = sms * blocksPerSm;
    copy_kernel<<<blocks, threads>>>(a, b, n);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); copy_kernel<<<blocks, threads>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"copy_gbs\":%.1f,\"blocks_per_sm\":%d}\n", 2.0 * n * 16 / best / 1e6, blocksPerSm);
    best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); rmw_kernel<<<blocks, threads>>>(a, n, 1.0); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"inplace_rmw_gbs\":%.1f,\"blocks_per_sm\":%d}\n", 2.0 * n * 16 / best / 1e6, blocksPerSm);
  }
  return 0;
}
