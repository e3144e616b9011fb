// Microbenchmark: what bounds the dense FP64-MMA stage of kernels_reg.cu?
// A CTA of 256 threads owns a 2^11-amplitude complex128 tile in shared memory and runs S stages;
// each stage per warp: A fragments (16x16 complex variant matrix, 8 x 16 B per lane) from global
// (L1/L2), B fragments 8 x LDS.128, 64 DMMA m8n8k4, D 8 x STS.128, then __syncthreads().
// Flags switch parts off to see which one costs: MODE bit0 = A from global each stage (else
// registers once), bit1 = B/D through shared memory (else registers), bit2 = barrier per stage.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ds tools/microbench/dense_stage.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t swz(uint32_t t) { return t ^ (((t >> 3) ^ (t >> 6) ^ (t >> 9)) & 7u); }

template <int MODE>
__global__ void __launch_bounds__(256, 3) k_stage(const double2* __restrict__ gm, double* out, int stages, int reps) {
  __shared__ __align__(16) double2 tile[2048];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 2048; i += 256) tile[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double2 ue[2][4];
  const double2* U = gm + (blockIdx.x & 7) * 320;
#pragma unroll
  for (int mh = 0; mh < 2; ++mh)
#pragma unroll
    for (int kh = 0; kh < 4; ++kh) ue[mh][kh] = __ldg(U + (8 * mh + (lane >> 2)) * 20 + 4 * kh + (lane & 3));
  double b[2][8];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int k = 0; k < 8; ++k) b[nt][k] = 1e-3 * (lane + k + nt);
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    for (int s = 0; s < stages; ++s) {
      if (MODE & 1) {
        const double2* Us = gm + ((s * 37 + blockIdx.x * 11 + r * 5) & (MODE & 8 ? 255 : 7)) * 320;
#pragma unroll
        for (int mh = 0; mh < 2; ++mh)
#pragma unroll
          for (int kh = 0; kh < 4; ++kh) ue[mh][kh] = __ldg(Us + (8 * mh + (lane >> 2)) * 20 + 4 * kh + (lane & 3));
      }
      // per-stage register positions: rotate which tile bits form the 16-vector
      const uint32_t rot = (uint32_t)(s % 3);
      if (MODE & 2) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int kq = 0; kq < 4; ++kq) {
            const uint32_t t = ((uint32_t)warp << 8) | ((uint32_t)nt << 7) | ((uint32_t)(lane >> 2) << 4) |
                               ((uint32_t)(lane & 3) << 2) | kq;
            const double2 x = tile[swz((t << rot | t >> (11 - rot)) & 2047u)];
            b[nt][kq] = x.x;
            b[nt][kq + 4] = x.y;
          }
      }
      double d[4][2][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) d[mt][nt][0] = d[mt][nt][1] = 0.0;
#pragma unroll
      for (int mh = 0; mh < 2; ++mh)
#pragma unroll
        for (int kh = 0; kh < 4; ++kh) {
          const double2 e = ue[mh][kh];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            dmma(d[mh][nt][0], d[mh][nt][1], e.x, b[nt][kh]);
            dmma(d[mh + 2][nt][0], d[mh + 2][nt][1], e.y, b[nt][kh]);
          }
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            dmma(d[mh][nt][0], d[mh][nt][1], -e.y, b[nt][kh + 4]);
            dmma(d[mh + 2][nt][0], d[mh + 2][nt][1], e.x, b[nt][kh + 4]);
          }
        }
      if (MODE & 2) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int mh = 0; mh < 2; ++mh)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const uint32_t t = ((uint32_t)warp << 8) | ((uint32_t)nt << 7) | ((uint32_t)(lane >> 2) << 4) |
                                 ((uint32_t)(lane & 3) << 2) | (mh * 2 + v);
              tile[swz(t)] = make_double2(d[mh][nt][v], d[mh + 2][nt][v]);
            }
      } else {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            b[nt][k] = d[k & 3][nt][0] * 0.5;
            b[nt][k + 4] = d[k & 3][nt][1] * 0.5;
          }
      }
      if (MODE & 4) __syncthreads();
    }
  }
  for (int nt = 0; nt < 2; ++nt)
    for (int k = 0; k < 8; ++k) acc += b[nt][k];
  acc += tile[tid].x;
  if (acc == 12345.678) out[0] = acc;
}

template <int MODE>
void run(const double2* gm, double* out, int blocks_per_sm, int sms) {
  const int stages = 16, reps = 200;
  const int grid = sms * blocks_per_sm;
  k_stage<MODE><<<grid, 256>>>(gm, out, stages, 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_stage<MODE><<<grid, 256>>>(gm, out, stages, reps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = (double)grid * 8 * 64 * 512.0 * stages * reps;
  printf("{\"mode\":%d,\"a_l2\":%d,\"a_global\":%d,\"bd_smem\":%d,\"barrier\":%d,\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n",
         MODE, (MODE >> 3) & 1, MODE & 1, (MODE >> 1) & 1, (MODE >> 2) & 1, blocks_per_sm, ms, flops / ms / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double2* gm;
  double* out;
  cudaMalloc(&gm, 256 * 320 * sizeof(double2));
  cudaMemset(gm, 0, 256 * 320 * sizeof(double2));
  cudaMalloc(&out, 8);
  for (int bps : {2, 3}) {
    run<0>(gm, out, bps, sms);
    run<1>(gm, out, bps, sms);
    run<2>(gm, out, bps, sms);
    run<4>(gm, out, bps, sms);
    run<6>(gm, out, bps, sms);
    run<7>(gm, out, bps, sms);
    run<15>(gm, out, bps, sms);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
