// kernels_reg.cu — register-blocked fused tile pass (the main forward / adjoint kernel).
//
// One CTA (2^(k-NR) threads) owns a tile of 2^k amplitudes (complex128) in shared memory:
//   load    cp.async 16-byte copies, consecutive threads -> consecutive amplitudes of each
//           16*2^L-byte chunk (fully coalesced), into bank-swizzled slots;
//   stages  for each stage the host planned (StageDesc): every thread pulls its 2^NR amplitudes
//           (whose tile indices differ in the stage's NR register positions) into registers,
//           applies the stage's ops there — X-like swaps, Z-like scales, general 2x2 pairs and
//           4x4 quads (§3.1) with arbitrary controls (Fig. 1) — and writes
//           them back;
//   store   16-byte coalesced stores.
// Every gate of the pass is applied during ONE HBM read + write of the state. In the DUAL
// (adjoint) variant the same happens for psi and lambda together, and before un-applying a
// parametrised op each warp reduces its share of Re<lambda|D|psi> (shuffles) into a per-CTA,
// per-op accumulator: deterministic fixed-order partials, no floating-point atomics.
#include <cstdint>

#include "cx.cuh"
#include "sv_internal.h"

namespace sv {
namespace {

__device__ __forceinline__ uint32_t swz(uint32_t t) { return t ^ ((t >> 3 ^ t >> 6 ^ t >> 9 ^ t >> 12) & 7u); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

struct RegArgs {
  int32_t k, low, nops, nstages, n_outer, nmats, ngrad, grid;
  int8_t tq[kMaxTileQubits + 3];
  int8_t oq[64];
  int64_t ntiles;
  const DevOp* ops;
  const double* mats;
  const StageDesc* stages;
  double* partials;
};

// ---------------------------------------------------------------- register-resident op kernels

// Shared-memory load the compiler may not hoist or CSE (keeps 4x4 matrices out of registers).
__device__ __forceinline__ double2 lds(const double2* p) {
  double2 r;
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(r.x), "=d"(r.y) : "r"(a));
  return r;
}

template <int NR, int RB>
__device__ __forceinline__ void reg_m1(double2 (&v)[1 << NR], const double2* m, uint32_t cj) {
  const double2 m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    if ((j & cj) != cj) continue;
    const int j1 = j | (1 << RB);
    const double2 a = v[j], b = v[j1];
    v[j] = cfma(m00, a, cmul(m01, b));
    v[j1] = cfma(m10, a, cmul(m11, b));
  }
}

template <int NR, int RB>
__device__ __forceinline__ void reg_ax1(double2 (&v)[1 << NR], const double2* m, uint32_t cj) {
  const double2 a = m[0], b = m[1];  // X-like [[0,a],[b,0]]: new0 = a old1, new1 = b old0
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    if ((j & cj) != cj) continue;
    const int j1 = j | (1 << RB);
    const double2 x0 = v[j], x1 = v[j1];
    v[j] = cmul(a, x1);
    v[j1] = cmul(b, x0);
  }
}

template <int NR, int RA, int RB>
__device__ __forceinline__ void reg_m2(double2 (&v)[1 << NR], const double2* m, uint32_t cj) {
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & ((1 << RA) | (1 << RB))) continue;
    if ((j & cj) != cj) continue;
    const int idx[4] = {j, j | (1 << RA), j | (1 << RB), j | (1 << RA) | (1 << RB)};
    double2 x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = v[idx[c]];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2 acc = cmul(lds(m + r * 4), x[0]);
#pragma unroll
      for (int c = 1; c < 4; ++c) acc = cfma(lds(m + r * 4 + c), x[c], acc);
      v[idx[r]] = acc;
    }
  }
}

template <int NR, int RA, int RB>
__device__ __forceinline__ void reg_swap(double2 (&v)[1 << NR], uint32_t cj) {
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & ((1 << RA) | (1 << RB))) continue;
    if ((j & cj) != cj) continue;
    const int a = j | (1 << RA), b = j | (1 << RB);
    const double2 t = v[a];
    v[a] = v[b];
    v[b] = t;
  }
}

// Re <w| (Pi_C (x) G) |v> over this thread's amplitudes, G on register bit RB (2x2).
template <int NR, int RB>
__device__ __forceinline__ double reg_ov1(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], const double2* g,
                                          uint32_t cj) {
  const double2 g00 = g[0], g01 = g[1], g10 = g[2], g11 = g[3];
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    if ((j & cj) != cj) continue;
    const int j1 = j | (1 << RB);
    acc += re_conj_mul(w[j], cfma(g00, v[j], cmul(g01, v[j1])));
    acc += re_conj_mul(w[j1], cfma(g10, v[j], cmul(g11, v[j1])));
  }
  return acc;
}

template <int NR, int RA, int RB>
__device__ __forceinline__ double reg_ov2(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], const double2* g,
                                          uint32_t cj) {
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & ((1 << RA) | (1 << RB))) continue;
    if ((j & cj) != cj) continue;
    const int idx[4] = {j, j | (1 << RA), j | (1 << RB), j | (1 << RA) | (1 << RB)};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double2 t = cmul(lds(g + r * 4), v[idx[0]]);
#pragma unroll
      for (int c = 1; c < 4; ++c) t = cfma(lds(g + r * 4 + c), v[idx[c]], t);
      acc += re_conj_mul(w[idx[r]], t);
    }
  }
  return acc;
}

// Dispatch helpers: runtime register index -> compile-time template.
template <int NR>
__device__ __forceinline__ void disp_m1(double2 (&v)[1 << NR], int r, const double2* m, uint32_t cj) {
  switch (r) {
    case 0: reg_m1<NR, 0>(v, m, cj); break;
    case 1: reg_m1<NR, 1>(v, m, cj); break;
    case 2: reg_m1<NR, 2>(v, m, cj); break;
    default: if constexpr (NR > 3) reg_m1<NR, 3>(v, m, cj); break;
  }
}
template <int NR>
__device__ __forceinline__ void disp_ax1(double2 (&v)[1 << NR], int r, const double2* m, uint32_t cj) {
  switch (r) {
    case 0: reg_ax1<NR, 0>(v, m, cj); break;
    case 1: reg_ax1<NR, 1>(v, m, cj); break;
    case 2: reg_ax1<NR, 2>(v, m, cj); break;
    default: if constexpr (NR > 3) reg_ax1<NR, 3>(v, m, cj); break;
  }
}
template <int NR>
__device__ __forceinline__ void disp_m2(double2 (&v)[1 << NR], int ra, int rb, const double2* m, uint32_t cj) {
  const int key = ra * 4 + rb;  // ra < rb
  switch (key) {
    case 1: reg_m2<NR, 0, 1>(v, m, cj); break;
    case 2: reg_m2<NR, 0, 2>(v, m, cj); break;
    case 6: reg_m2<NR, 1, 2>(v, m, cj); break;
    default:
      if constexpr (NR > 3) {
        if (key == 3) reg_m2<NR, 0, 3>(v, m, cj);
        else if (key == 7) reg_m2<NR, 1, 3>(v, m, cj);
        else reg_m2<NR, 2, 3>(v, m, cj);
      }
      break;
  }
}
template <int NR>
__device__ __forceinline__ void disp_swap(double2 (&v)[1 << NR], int ra, int rb, uint32_t cj) {
  const int key = ra * 4 + rb;
  switch (key) {
    case 1: reg_swap<NR, 0, 1>(v, cj); break;
    case 2: reg_swap<NR, 0, 2>(v, cj); break;
    case 6: reg_swap<NR, 1, 2>(v, cj); break;
    default:
      if constexpr (NR > 3) {
        if (key == 3) reg_swap<NR, 0, 3>(v, cj);
        else if (key == 7) reg_swap<NR, 1, 3>(v, cj);
        else reg_swap<NR, 2, 3>(v, cj);
      }
      break;
  }
}
template <int NR>
__device__ __forceinline__ double disp_ov1(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], int r,
                                           const double2* g, uint32_t cj) {
  switch (r) {
    case 0: return reg_ov1<NR, 0>(v, w, g, cj);
    case 1: return reg_ov1<NR, 1>(v, w, g, cj);
    case 2: return reg_ov1<NR, 2>(v, w, g, cj);
    default: if constexpr (NR > 3) return reg_ov1<NR, 3>(v, w, g, cj); return 0.0;
  }
}
template <int NR>
__device__ __forceinline__ double disp_ov2(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], int ra, int rb,
                                           const double2* g, uint32_t cj) {
  const int key = ra * 4 + rb;
  switch (key) {
    case 1: return reg_ov2<NR, 0, 1>(v, w, g, cj);
    case 2: return reg_ov2<NR, 0, 2>(v, w, g, cj);
    case 6: return reg_ov2<NR, 1, 2>(v, w, g, cj);
    default:
      if constexpr (NR > 3) {
        if (key == 3) return reg_ov2<NR, 0, 3>(v, w, g, cj);
        if (key == 7) return reg_ov2<NR, 1, 3>(v, w, g, cj);
        return reg_ov2<NR, 2, 3>(v, w, g, cj);
      }
      return 0.0;
  }
}

// Bit of a target for register index j: register bit (ra >= 0), else thread / outer bit (tb).
__device__ __forceinline__ uint32_t tbit(int ra, int j, uint32_t tb) { return ra >= 0 ? ((uint32_t)j >> ra) & 1u : tb; }

template <int NR>
__device__ __forceinline__ void reg_apply(double2 (&v)[1 << NR], const DevOp& o, const double2* m, uint32_t tthr,
                                          uint64_t base) {
  const uint32_t cj = o.cj;
  switch (o.type) {
    case OP_M1: disp_m1<NR>(v, o.ra, m, cj); break;
    case OP_AX1: disp_ax1<NR>(v, o.ra, m, cj); break;
    case OP_M2: disp_m2<NR>(v, o.ra, o.rb, m, cj); break;
    case OP_SWAP: disp_swap<NR>(v, o.ra, o.rb, cj); break;
    case OP_D1: {
      const double2 f0 = m[0], f1 = m[1];
      const uint32_t tb = o.pa >= 0 ? (tthr >> o.pa) & 1u : (uint32_t)((base >> o.qa) & 1ull);
#pragma unroll
      for (int j = 0; j < (1 << NR); ++j) {
        if ((j & cj) != cj) continue;
        v[j] = cmul(tbit(o.ra, j, tb) ? f1 : f0, v[j]);
      }
      break;
    }
    case OP_D2: {
      const double2 f0 = m[0], f1 = m[1], f2 = m[2], f3 = m[3];
      const uint32_t ta = o.pa >= 0 ? (tthr >> o.pa) & 1u : (uint32_t)((base >> o.qa) & 1ull);
      const uint32_t tb = o.pb >= 0 ? (tthr >> o.pb) & 1u : (uint32_t)((base >> o.qb) & 1ull);
#pragma unroll
      for (int j = 0; j < (1 << NR); ++j) {
        if ((j & cj) != cj) continue;
        const uint32_t b0 = tbit(o.ra, j, ta), b1 = tbit(o.rb, j, tb);
        const double2 f = b1 ? (b0 ? f3 : f2) : (b0 ? f1 : f0);
        v[j] = cmul(f, v[j]);
      }
      break;
    }
  }
}

template <int NR>
__device__ __forceinline__ double reg_overlap(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], const DevOp& o,
                                              const double2* g, uint32_t tthr, uint64_t base) {
  const uint32_t cj = o.cj;
  if (o.gen_diag) {
    const uint32_t ta = o.pa >= 0 ? (tthr >> o.pa) & 1u : (uint32_t)((base >> o.qa) & 1ull);
    const uint32_t tb = (o.gen_dim == 4) ? (o.pb >= 0 ? (tthr >> o.pb) & 1u : (uint32_t)((base >> o.qb) & 1ull)) : 0u;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < (1 << NR); ++j) {
      if ((j & cj) != cj) continue;
      uint32_t idx = tbit(o.ra, j, ta);
      if (o.gen_dim == 4) idx |= tbit(o.rb, j, tb) << 1;
      acc += re_conj_mul(w[j], cmul(g[idx], v[j]));
    }
    return acc;
  }
  if (o.gen_dim == 2) return disp_ov1<NR>(v, w, o.ra, g, cj);
  return disp_ov2<NR>(v, w, o.ra, o.rb, g, cj);
}

// ---------------------------------------------------------------- the pass kernel

template <int NR, bool DUAL>
__global__ void __launch_bounds__(256, DUAL ? 1 : 2) k_pass_reg(double2* __restrict__ psi, double2* __restrict__ lam, RegArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << a.k;
  const int nthr = blockDim.x, tid = threadIdx.x, nwarps = nthr >> 5, warp = tid >> 5, lane = tid & 31;
  double2* tp = reinterpret_cast<double2*>(smem_raw);
  double2* tl = DUAL ? tp + N : nullptr;
  DevOp* s_ops = reinterpret_cast<DevOp*>(tp + (DUAL ? 2 * N : N));
  StageDesc* s_st = reinterpret_cast<StageDesc*>(s_ops + a.nops);
  double* s_mats = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(s_st + a.nstages) + 15) & ~uintptr_t(15));
  const int nhi = 1 << (a.k - a.low);
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(s_mats + a.nmats);
  double* s_acc = reinterpret_cast<double*>(s_hi + nhi);  // [ngrad][nwarps]

  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(a.ops);
    uint64_t* dst = reinterpret_cast<uint64_t*>(s_ops);
    for (int i = tid; i < a.nops * 8; i += nthr) dst[i] = src[i];
    const uint64_t* ss = reinterpret_cast<const uint64_t*>(a.stages);
    uint64_t* sd = reinterpret_cast<uint64_t*>(s_st);
    for (int i = tid; i < a.nstages * (int)(sizeof(StageDesc) / 8); i += nthr) sd[i] = ss[i];
    for (int i = tid; i < a.nmats; i += nthr) s_mats[i] = a.mats[i];
    for (int h = tid; h < nhi; h += nthr) {
      uint64_t off = 0;
      for (int b = 0; b < a.k - a.low; ++b)
        if ((h >> b) & 1) off |= 1ull << a.tq[a.low + b];
      s_hi[h] = off;
    }
    if (DUAL)
      for (int i = tid; i < a.ngrad * nwarps; i += nthr) s_acc[i] = 0.0;
  }
  __syncthreads();
  const uint32_t lowmask = (1u << a.low) - 1u;
  const int nthr_bits = a.k - NR;

  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    uint64_t base = 0;
    for (int j = 0; j < a.n_outer; ++j)
      if ((tile >> j) & 1) base |= 1ull << a.oq[j];
    // ---- load: HBM -> shared (cp.async, coalesced 16-byte) ----
    for (uint32_t e = tid; e < N; e += nthr) {
      const uint64_t gi = base | (e & lowmask) | s_hi[e >> a.low];
      cp_async16(tp + swz(e), psi + gi);
      if (DUAL) cp_async16(tl + swz(e), lam + gi);
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- stages ----
    for (int st = 0; st < a.nstages; ++st) {
      const StageDesc& S = s_st[st];
      uint32_t tthr = 0;
      for (int b = 0; b < nthr_bits; ++b)
        if ((tid >> b) & 1) tthr |= 1u << S.thrpos[b];
      const uint32_t A = swz(tthr);
      double2 v[1 << NR];
      double2 w[DUAL ? (1 << NR) : 1];
#pragma unroll
      for (int j = 0; j < (1 << NR); ++j) {
        v[j] = tp[A ^ S.swz_reg[j]];
        if constexpr (DUAL) w[j] = tl[A ^ S.swz_reg[j]];
      }
      for (int i = S.op_begin; i < S.op_end; ++i) {
        const DevOp& o = s_ops[i];
        const bool ok = ((base & o.couter) == o.couter) && ((tthr & (uint32_t)o.cthr) == (uint32_t)o.cthr);
        if constexpr (DUAL) {
          if (o.grad_slot >= 0) {
            double part = 0.0;
            if (ok) part = reg_overlap<NR>(v, w, o, reinterpret_cast<const double2*>(s_mats + o.gen_off), tthr, base);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            if (lane == 0) s_acc[o.grad_local * nwarps + warp] += part;
          }
        }
        if (!ok) continue;
        const double2* m = reinterpret_cast<const double2*>(s_mats + o.mat_off);
        reg_apply<NR>(v, o, m, tthr, base);
        if constexpr (DUAL) reg_apply<NR>(w, o, m, tthr, base);
      }
#pragma unroll
      for (int j = 0; j < (1 << NR); ++j) {
        tp[A ^ S.swz_reg[j]] = v[j];
        if constexpr (DUAL) tl[A ^ S.swz_reg[j]] = w[j];
      }
      __syncthreads();
    }
    // ---- store: shared -> HBM (coalesced 16-byte) ----
    for (uint32_t e = tid; e < N; e += nthr) {
      const uint64_t gi = base | (e & lowmask) | s_hi[e >> a.low];
      psi[gi] = tp[swz(e)];
      if (DUAL) lam[gi] = tl[swz(e)];
    }
    __syncthreads();
  }
  if (DUAL) {
    for (int i = tid; i < a.nops; i += nthr) {
      const DevOp& o = s_ops[i];
      if (o.grad_slot < 0) continue;
      double s = 0.0;
      for (int wi = 0; wi < nwarps; ++wi) s += s_acc[o.grad_local * nwarps + wi];
      a.partials[(int64_t)o.grad_slot * a.grid + blockIdx.x] = s;
    }
  }
}

size_t reg_smem_bytes(int k, int low, int nops, int nstages, int nmats, int ngrad, int nthr, bool dual) {
  size_t b = (size_t(16) << k) * (dual ? 2 : 1);
  b += (size_t)nops * sizeof(DevOp) + (size_t)nstages * sizeof(StageDesc) + 16;
  b += (size_t)nmats * 8 + (size_t(8) << (k - low));
  b += dual ? (size_t)ngrad * (nthr / 32) * 8 : 0;
  return b;
}

}  // namespace

cudaError_t launch_pass_reg(double* psi, double* lam, const PassLaunch& L, cudaStream_t s) {
  const PassDesc& pd = *L.pd;
  RegArgs a;
  a.k = pd.k;
  a.low = pd.low;
  a.nops = pd.op_end - pd.op_begin;
  a.nstages = pd.stage_end - pd.stage_begin;
  a.nmats = L.nmats;
  a.ngrad = pd.n_grad;
  a.grid = L.grid;
  for (int i = 0; i < kMaxTileQubits + 3; ++i) a.tq[i] = pd.tq[i];
  uint64_t tmask = 0;
  for (int p = 0; p < pd.k; ++p) tmask |= 1ull << pd.tq[p];
  a.n_outer = 0;
  for (int q = 0; q < L.n_local; ++q)
    if (!((tmask >> q) & 1ull)) a.oq[a.n_outer++] = (int8_t)q;
  a.ntiles = 1ll << (L.n_local - pd.k);
  a.ops = L.d_ops + pd.op_begin;
  a.mats = L.d_mats + pd.mat_begin;
  a.stages = L.d_stages + pd.stage_begin;
  a.partials = L.d_partials;
  const bool dual = lam != nullptr;
  const int nthr = 1 << (pd.k - pd.R);
  const size_t smem = reg_smem_bytes(a.k, a.low, a.nops, a.nstages, a.nmats, a.ngrad, nthr, dual);
  static bool attr_set[2] = {false, false};
  if (!attr_set[dual]) {
    cudaError_t e = dual ? cudaFuncSetAttribute(k_pass_reg<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)
                         : cudaFuncSetAttribute(k_pass_reg<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set[dual] = true;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (dual) {
    if (pd.R != 3) return cudaErrorInvalidValue;
    k_pass_reg<3, true><<<L.grid, nthr, smem, s>>>(reinterpret_cast<double2*>(psi), reinterpret_cast<double2*>(lam), a);
  } else {
    if (pd.R != 4) return cudaErrorInvalidValue;
    k_pass_reg<4, false><<<L.grid, nthr, smem, s>>>(reinterpret_cast<double2*>(psi), nullptr, a);
  }
  return cudaGetLastError();
}

}  // namespace sv
