// kernels_batch.cu — batch-mode expectation + adjoint gradient for small states (SURVEY §8(f)
// NEXT-1; "Gradient calculation in batch mode", Fig. 1).
//
// One CTA evaluates one parameter row completely: the whole 2^n-amplitude state (n <= 11) and its
// adjoint vector live in shared memory; the kernel applies the circuit, forms lambda = H psi and E,
// then runs the reverse sweep (overlap Re<lambda|D_k|psi> before un-applying each gate) and writes
// E and the gradient of its row. A batch of B rows is ONE launch of B CTAs: the latency-bound
// small-n evaluation (C1: 4 qubits, 8 gates) becomes throughput-bound. Reductions are block-level
// in a fixed order (deterministic); per-row gradient accumulation is sequential in gate order.
#include <cstdint>

#include "cx.cuh"
#include "sv_internal.h"

namespace sv {
namespace {

constexpr int kBT = 256;

__device__ __forceinline__ uint32_t ins0(uint32_t j, int p) { return ((j >> p) << (p + 1)) | (j & ((1u << p) - 1u)); }

// Block-wide fixed-order sum (result in all threads).
__device__ double bsum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += red[i];
  __syncthreads();
  return r;
}

// psi <- M psi on targets t0 (, t1) under control mask cm (k = 1 or 2; M row-major dim x dim).
// dag: apply M^dagger.
__device__ void bapply(double2* s, int n, const BatchOp& o, const double2* M, bool dag) {
  const uint32_t N = 1u << n, cm = (uint32_t)o.cmask;
  if (o.dim == 2) {
    const int p = o.t0;
    double2 m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];
    if (dag) {
      const double2 a = m01;
      m00 = make_double2(m00.x, -m00.y); m11 = make_double2(m11.x, -m11.y);
      m01 = make_double2(m10.x, -m10.y); m10 = make_double2(a.x, -a.y);
    }
    for (uint32_t j = threadIdx.x; j < (N >> 1); j += blockDim.x) {
      const uint32_t i0 = ins0(j, p), i1 = i0 | (1u << p);
      if ((i0 & cm) != cm) continue;
      const double2 a = s[i0], b = s[i1];
      s[i0] = cfma(m00, a, cmul(m01, b));
      s[i1] = cfma(m10, a, cmul(m11, b));
    }
  } else {
    const int pa = o.t0, pb = o.t1, lo = pa < pb ? pa : pb, hi = pa < pb ? pb : pa;
    for (uint32_t j = threadIdx.x; j < (N >> 2); j += blockDim.x) {
      const uint32_t i00 = ins0(ins0(j, lo), hi);
      if ((i00 & cm) != cm) continue;
      const uint32_t idx[4] = {i00, i00 | (1u << pa), i00 | (1u << pb), i00 | (1u << pa) | (1u << pb)};
      double2 x[4];
      for (int c = 0; c < 4; ++c) x[c] = s[idx[c]];
      for (int r = 0; r < 4; ++r) {
        double2 acc = make_double2(0.0, 0.0);
        for (int c = 0; c < 4; ++c) {
          double2 e = dag ? M[c * 4 + r] : M[r * 4 + c];
          if (dag) e.y = -e.y;
          acc = cfma(e, x[c], acc);
        }
        s[idx[r]] = acc;
      }
    }
  }
}

// Re <l| (Pi_C (x) G) |p> (this thread's share).
__device__ double boverlap(const double2* p, const double2* l, int n, const BatchOp& o, const double2* G) {
  const uint32_t N = 1u << n, cm = (uint32_t)o.cmask;
  double acc = 0.0;
  if (o.dim == 2) {
    const int q = o.t0;
    for (uint32_t j = threadIdx.x; j < (N >> 1); j += blockDim.x) {
      const uint32_t i0 = ins0(j, q), i1 = i0 | (1u << q);
      if ((i0 & cm) != cm) continue;
      acc += re_conj_mul(l[i0], cfma(G[0], p[i0], cmul(G[1], p[i1])));
      acc += re_conj_mul(l[i1], cfma(G[2], p[i0], cmul(G[3], p[i1])));
    }
  } else {
    const int pa = o.t0, pb = o.t1, lo = pa < pb ? pa : pb, hi = pa < pb ? pb : pa;
    for (uint32_t j = threadIdx.x; j < (N >> 2); j += blockDim.x) {
      const uint32_t i00 = ins0(ins0(j, lo), hi);
      if ((i00 & cm) != cm) continue;
      const uint32_t idx[4] = {i00, i00 | (1u << pa), i00 | (1u << pb), i00 | (1u << pa) | (1u << pb)};
      for (int r = 0; r < 4; ++r) {
        double2 t = make_double2(0.0, 0.0);
        for (int c = 0; c < 4; ++c) t = cfma(G[r * 4 + c], p[idx[c]], t);
        acc += re_conj_mul(l[idx[r]], t);
      }
    }
  }
  return acc;
}

__global__ void __launch_bounds__(kBT) k_batch_grad(const double2* __restrict__ psi0, int n, BatchArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << n;
  double2* p = reinterpret_cast<double2*>(smem_raw);
  double2* l = p + N;
  __shared__ double red[kBT / 32];
  const int row = blockIdx.x;
  const double2* mats = reinterpret_cast<const double2*>(a.mats) + (int64_t)row * a.row_stride;
  const double2* gens = reinterpret_cast<const double2*>(a.gens);
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) p[i] = psi0[i];
  __syncthreads();
  // forward
  for (int k = 0; k < a.nops; ++k) {
    bapply(p, n, a.ops[k], mats + a.ops[k].mat_off, false);
    __syncthreads();
  }
  // lambda = H psi (terms share the pass over the shared-memory state), E = Re<psi|lambda>
  double e_part = 0.0;
  for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int t = 0; t < a.nterms; ++t) {
      const uint64_t x = a.x[t], z = a.z[t];
      const uint32_t ip = i ^ (uint32_t)x;
      const double sg = (__popc(ip & (uint32_t)z) & 1) ? -1.0 : 1.0;
      const double2 c = reinterpret_cast<const double2*>(a.c)[t];
      acc = cfma(make_double2(sg * c.x, sg * c.y), p[ip], acc);
    }
    l[i] = acc;
    e_part += re_conj_mul(p[i], acc);
  }
  __syncthreads();
  const double E = bsum(e_part, red);
  if (threadIdx.x == 0) a.out_e[row] = E;
  double* grow = a.out_g + (int64_t)row * a.nparams;
  for (int q = threadIdx.x; q < a.nparams; q += blockDim.x) grow[q] = 0.0;
  __syncthreads();
  // reverse sweep
  for (int k = a.nops - 1; k >= 0; --k) {
    const BatchOp& o = a.ops[k];
    if (o.param >= 0) {
      const double d = bsum(boverlap(p, l, n, o, gens + o.gen_off), red);
      if (threadIdx.x == 0) grow[o.param] += o.coeff * 2.0 * d;
    }
    bapply(p, n, o, mats + o.mat_off, true);
    bapply(l, n, o, mats + o.mat_off, true);
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_batch_grad(const double* psi0, int n, const BatchArgs& a, int rows, cudaStream_t s) {
  const size_t smem = (size_t(32) << n);
  static std::atomic<uint64_t> attr{0};
  {
    cudaError_t e = once_per_device(
        attr, [] { return cudaFuncSetAttribute(k_batch_grad, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
    if (e != cudaSuccess) return e;
  }
  k_batch_grad<<<rows, kBT, smem, s>>>(reinterpret_cast<const double2*>(psi0), n, a);
  return cudaGetLastError();
}

}  // namespace sv
