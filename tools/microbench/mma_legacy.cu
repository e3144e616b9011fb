// Throughput of legacy warp-level mma.sync on sm_100a for the complex64 dense-stage question:
// TF32 m16n8k8 and BF16 m16n8k16 (f32 accumulate) vs FP64 DMMA m8n8k4 (reference).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_legacy tools/microbench/mma_legacy.cu
#include <cstdio>
#include <cstdint>

__global__ void k_tf32(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_bf16(float* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f;
  float c[8];
  for (int j = 0; j < 8; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = fmaf(c[j], b, a);
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j];
  if (s == 1234.5f) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, double flops_per_iter_per_warp, int iters) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  const int blocks = sms * 4, threads = 256;
  kern<<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = flops_per_iter_per_warp * iters * (double)blocks * (threads / 32);
  printf("{\"kernel\":\"%s\",\"ms\":%.3f,\"tflops\":%.1f}\n", name, ms, flops / ms / 1e9);
  cudaFree(out);
}

int main() {
  run("mma.sync m16n8k8 tf32", k_tf32, 4.0 * 2 * 16 * 8 * 8, 20000);
  run("mma.sync m16n8k16 bf16", k_bf16, 4.0 * 2 * 16 * 8 * 16, 20000);
  run("ffma (3-reg)", k_ffma, 16.0 * 8 * 2 * 32, 20000);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
