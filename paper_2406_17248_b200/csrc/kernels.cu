// kernels.cu — sm_100a kernels of the state-vector hot path.
//
//  k_pass<DUAL=false>  fused forward gate pass: each CTA loads 2^k amplitudes of
//                      one tile into shared memory (contiguous 16*2^L-byte chunks, 16-byte
//                      coalesced loads), applies every op of the pass in order, writes the tile
//                      back: one HBM read + write of the state for all gates of the pass.
//  k_pass<DUAL=true>   fused adjoint pass (a6): the same on psi and lambda together; before
//                      un-applying a parametrised op it accumulates Re<lambda|D|psi> over the tile
//                      into a per-CTA partial (fixed order: deterministic).
//  k_pauli_group       one read pass per x-mask group of Pauli terms (a4/a5): pairs (i, i^x) read
//                      once, every term of the group evaluated from the index bits; optionally
//                      writes/accumulates lambda = H psi; per-CTA partials of <psi|H_group|psi>.
//  k_reduce_slots      fixed-order reduction of per-CTA partials (a7).
//
// Gate classes follow the paper (§3.1): X-like (anti-diagonal, "swap with scaling"),
// Z-like (diagonal, "no pairing"), general 2x2 pairs, two-qubit quads.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "cx.cuh"
#include "sv_internal.h"

namespace sv {
namespace {

__device__ __forceinline__ uint32_t insert_zero(uint32_t j, int p) {
  const uint32_t lo = j & ((1u << p) - 1u);
  return ((j >> p) << (p + 1)) | lo;
}
__device__ __forceinline__ uint64_t insert_zero64(uint64_t j, int p) {
  const uint64_t lo = j & ((1ull << p) - 1ull);
  return ((j >> p) << (p + 1)) | lo;
}

constexpr int kThreads = 256;

// Block-wide sum; result valid in thread 0. scratch: >= kThreads/32 doubles.
__device__ double block_sum(double v, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) scratch[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += scratch[i];
  }
  return r;
}

struct PassArgs {
  int32_t k, low, nops, n_outer;
  int8_t tq[kMaxTileQubits + 3];
  int8_t oq[64];
  int64_t ntiles;
  const DevOp* ops;
  const double* mats;
  int32_t nmats;
  double* partials;
  int32_t grid;
};

// Applies one op to a tile buffer t (2^k amplitudes in shared memory).
__device__ __forceinline__ void apply_op(double2* t, const DevOp& o, const double2* m, int k, uint64_t base) {
  const uint32_t N = 1u << k;
  const uint32_t ct = (uint32_t)o.ctile;
  switch (o.type) {
    case OP_M1: {
      const int p = o.pa;
      const double2 m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
      for (uint32_t j = threadIdx.x; j < (N >> 1); j += blockDim.x) {
        const uint32_t i0 = insert_zero(j, p), i1 = i0 | (1u << p);
        if ((i0 & ct) != ct) continue;
        const double2 v0 = t[i0], v1 = t[i1];
        t[i0] = cfma(m00, v0, cmul(m01, v1));
        t[i1] = cfma(m10, v0, cmul(m11, v1));
      }
      break;
    }
    case OP_AX1: {  // X-like: new[i0] = a old[i1], new[i1] = b old[i0]
      const int p = o.pa;
      const double2 a = m[0], b = m[1];
      for (uint32_t j = threadIdx.x; j < (N >> 1); j += blockDim.x) {
        const uint32_t i0 = insert_zero(j, p), i1 = i0 | (1u << p);
        if ((i0 & ct) != ct) continue;
        const double2 v0 = t[i0], v1 = t[i1];
        t[i0] = cmul(a, v1);
        t[i1] = cmul(b, v0);
      }
      break;
    }
    case OP_D1: {  // Z-like: per-amplitude scale, no pairing
      const double2 a = m[0], b = m[1];
      if (o.pa < 0) {
        const double2 f = ((base >> o.qa) & 1ull) ? b : a;
        for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
          if ((e & ct) != ct) continue;
          t[e] = cmul(f, t[e]);
        }
      } else {
        const int p = o.pa;
        for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
          if ((e & ct) != ct) continue;
          t[e] = cmul(((e >> p) & 1u) ? b : a, t[e]);
        }
      }
      break;
    }
    case OP_D2: {
      for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
        if ((e & ct) != ct) continue;
        const uint32_t b0 = o.pa >= 0 ? ((e >> o.pa) & 1u) : (uint32_t)((base >> o.qa) & 1ull);
        const uint32_t b1 = o.pb >= 0 ? ((e >> o.pb) & 1u) : (uint32_t)((base >> o.qb) & 1ull);
        t[e] = cmul(m[b0 | (b1 << 1)], t[e]);
      }
      break;
    }
    case OP_M2: {
      const int pa = o.pa, pb = o.pb;
      const int plo = pa < pb ? pa : pb, phi = pa < pb ? pb : pa;
      for (uint32_t j = threadIdx.x; j < (N >> 2); j += blockDim.x) {
        const uint32_t i00 = insert_zero(insert_zero(j, plo), phi);
        if ((i00 & ct) != ct) continue;
        const uint32_t idx[4] = {i00, i00 | (1u << pa), i00 | (1u << pb), i00 | (1u << pa) | (1u << pb)};
        double2 v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = t[idx[c]];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double2 acc = cmul(m[r * 4 + 0], v[0]);
#pragma unroll
          for (int c = 1; c < 4; ++c) acc = cfma(m[r * 4 + c], v[c], acc);
          t[idx[r]] = acc;
        }
      }
      break;
    }
    case OP_SWAP: {
      const int pa = o.pa, pb = o.pb;
      const int plo = pa < pb ? pa : pb, phi = pa < pb ? pb : pa;
      for (uint32_t j = threadIdx.x; j < (N >> 2); j += blockDim.x) {
        const uint32_t i00 = insert_zero(insert_zero(j, plo), phi);
        if ((i00 & ct) != ct) continue;
        const uint32_t i01 = i00 | (1u << pa), i10 = i00 | (1u << pb);
        const double2 v = t[i01];
        t[i01] = t[i10];
        t[i10] = v;
      }
      break;
    }
  }
}

// Re <lam| (Pi_C (x) G) |psi> over one tile, this thread's share.
__device__ __forceinline__ double overlap_op(const double2* ps, const double2* la, const DevOp& o, const double2* g,
                                             int k, uint64_t base) {
  const uint32_t N = 1u << k;
  const uint32_t ct = (uint32_t)o.ctile;
  double acc = 0.0;
  if (o.gen_diag) {
    for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
      if ((e & ct) != ct) continue;
      uint32_t idx = o.pa >= 0 ? ((e >> o.pa) & 1u) : (uint32_t)((base >> o.qa) & 1ull);
      if (o.gen_dim == 4) idx |= (o.pb >= 0 ? ((e >> o.pb) & 1u) : (uint32_t)((base >> o.qb) & 1ull)) << 1;
      acc += re_conj_mul(la[e], cmul(g[idx], ps[e]));
    }
  } else if (o.gen_dim == 2) {
    const int p = o.pa;
    for (uint32_t j = threadIdx.x; j < (N >> 1); j += blockDim.x) {
      const uint32_t i0 = insert_zero(j, p), i1 = i0 | (1u << p);
      if ((i0 & ct) != ct) continue;
      const double2 v0 = ps[i0], v1 = ps[i1];
      acc += re_conj_mul(la[i0], cfma(g[0], v0, cmul(g[1], v1)));
      acc += re_conj_mul(la[i1], cfma(g[2], v0, cmul(g[3], v1)));
    }
  } else {
    const int pa = o.pa, pb = o.pb;
    const int plo = pa < pb ? pa : pb, phi = pa < pb ? pb : pa;
    for (uint32_t j = threadIdx.x; j < (N >> 2); j += blockDim.x) {
      const uint32_t i00 = insert_zero(insert_zero(j, plo), phi);
      if ((i00 & ct) != ct) continue;
      const uint32_t idx[4] = {i00, i00 | (1u << pa), i00 | (1u << pb), i00 | (1u << pa) | (1u << pb)};
      double2 v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = ps[idx[c]];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double2 w = cmul(g[r * 4], v[0]);
#pragma unroll
        for (int c = 1; c < 4; ++c) w = cfma(g[r * 4 + c], v[c], w);
        acc += re_conj_mul(la[idx[r]], w);
      }
    }
  }
  return acc;
}

template <bool DUAL>
__global__ void __launch_bounds__(kThreads) k_pass(double2* __restrict__ psi, double2* __restrict__ lam, PassArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << a.k;
  double2* tp = reinterpret_cast<double2*>(smem_raw);
  double2* tl = DUAL ? tp + N : nullptr;
  DevOp* s_ops = reinterpret_cast<DevOp*>(tp + (DUAL ? 2 * N : N));
  double* s_mats = reinterpret_cast<double*>(s_ops + a.nops);
  const int nhi = 1 << (a.k - a.low);
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(s_mats + ((a.nmats + 1) & ~1));
  double* s_acc = reinterpret_cast<double*>(s_hi + nhi);  // per-op grad accumulators (DUAL)
  double* s_red = s_acc + (DUAL ? a.nops : 0);

  // ---- per-CTA setup: op list, matrices, high-offset table ----
  {
    const int op_words = a.nops * (int)(sizeof(DevOp) / 8);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(a.ops);
    uint64_t* dst = reinterpret_cast<uint64_t*>(s_ops);
    for (int i = threadIdx.x; i < op_words; i += blockDim.x) dst[i] = src[i];
    for (int i = threadIdx.x; i < a.nmats; i += blockDim.x) s_mats[i] = a.mats[i];
    for (int h = threadIdx.x; h < nhi; h += blockDim.x) {
      uint64_t off = 0;
      for (int b = 0; b < a.k - a.low; ++b)
        if ((h >> b) & 1) off |= 1ull << a.tq[a.low + b];
      s_hi[h] = off;
    }
    if (DUAL)
      for (int i = threadIdx.x; i < a.nops; i += blockDim.x) s_acc[i] = 0.0;
  }
  __syncthreads();
  const uint32_t lowmask = (1u << a.low) - 1u;

  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    uint64_t base = 0;
    for (int j = 0; j < a.n_outer; ++j)
      if ((tile >> j) & 1) base |= 1ull << a.oq[j];
    // ---- load (consecutive threads -> consecutive amplitudes of a 16*2^L-byte chunk) ----
    for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
      const uint64_t gi = base | (e & lowmask) | s_hi[e >> a.low];
      tp[e] = psi[gi];
      if (DUAL) tl[e] = lam[gi];
    }
    __syncthreads();
    // ---- ops ----
    for (int i = 0; i < a.nops; ++i) {
      const DevOp& o = s_ops[i];
      const bool outer_ok = (base & o.couter) == o.couter;
      if (DUAL && o.grad_slot >= 0) {
        double part = outer_ok ? overlap_op(tp, tl, o, reinterpret_cast<const double2*>(s_mats + o.gen_off), a.k, base)
                               : 0.0;
        part = block_sum(part, s_red);
        if (threadIdx.x == 0) s_acc[i] += part;
        __syncthreads();
      }
      if (!outer_ok) continue;
      const double2* m = reinterpret_cast<const double2*>(s_mats + o.mat_off);
      apply_op(tp, o, m, a.k, base);
      if (DUAL) apply_op(tl, o, m, a.k, base);
      __syncthreads();
    }
    // ---- store ----
    for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
      const uint64_t gi = base | (e & lowmask) | s_hi[e >> a.low];
      psi[gi] = tp[e];
      if (DUAL) lam[gi] = tl[e];
    }
    __syncthreads();
  }
  if (DUAL && threadIdx.x == 0) {
    for (int i = 0; i < a.nops; ++i)
      if (s_ops[i].grad_slot >= 0) a.partials[(int64_t)s_ops[i].grad_slot * a.grid + blockIdx.x] = s_acc[i];
  }
}


// ---- sharding helpers: global <-> local qubit swaps ----
// a[y0 | 2^l] <-> b[y0] for every y0 with bit l clear (virtual shards on one device).
__global__ void k_swap_halves(double2* __restrict__ a, double2* __restrict__ b, int nl, int l) {
  const int64_t half = 1ll << (nl - 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < half; i += stride) {
    const uint64_t y0 = insert_zero64((uint64_t)i, l);
    const uint64_t y1 = y0 | (1ull << l);
    const double2 t = a[y1];
    a[y1] = b[y0];
    b[y0] = t;
  }
}
// dst[i] = src[insert(off + i, l, h)] for i < count (pack == 1), or the reverse (pack == 0).
__global__ void k_pack_half(double2* __restrict__ shard, double2* __restrict__ buf, int l, int h, int64_t off,
                            int64_t count, int pack) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t y = insert_zero64((uint64_t)(off + i), l) | ((uint64_t)h << l);
    if (pack) buf[i] = shard[y];
    else shard[y] = buf[i];
  }
}

// Sampled-amplitude readout: out[j] = psi[idx[j]] for idx[j] != ~0, else 0 (an index another shard
// holds). T: double2 (complex128 state) or float2 (complex64 state).
template <typename T>
__global__ void k_gather(const T* __restrict__ psi, const uint64_t* __restrict__ idx, int64_t count,
                         double2* __restrict__ out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = idx[j];
    if (i == ~0ull) { out[j] = make_double2(0.0, 0.0); continue; }
    const T v = psi[i];
    out[j] = make_double2((double)v.x, (double)v.y);
  }
}

__global__ void k_init(double2* psi, int64_t n, bool one) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    psi[i] = make_double2((one && i == 0) ? 1.0 : 0.0, 0.0);
}

// mode 0: E partials only; 1: lam = H_g psi; 2: lam += H_g psi.
__global__ void __launch_bounds__(kThreads) k_pauli_group(const double2* __restrict__ psi, double2* __restrict__ lam,
                                                          int mode, int n, uint64_t x, const uint64_t* __restrict__ z,
                                                          const double2* __restrict__ c, int nterms,
                                                          double* __restrict__ partials) {
  __shared__ uint64_t s_z[256];
  __shared__ double2 s_c[256];
  __shared__ double s_red[kThreads / 32];
  for (int i = threadIdx.x; i < nterms; i += blockDim.x) { s_z[i] = z[i]; s_c[i] = c[i]; }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  if (x == 0) {
    const int64_t N = 1ll << n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += stride) {
      double2 C = make_double2(0.0, 0.0);
      for (int j = 0; j < nterms; ++j) {
        const double sg = (__popcll(i & s_z[j]) & 1) ? -1.0 : 1.0;
        C.x = fma(sg, s_c[j].x, C.x);
        C.y = fma(sg, s_c[j].y, C.y);
      }
      const double2 v = psi[i];
      const double2 w = cmul(C, v);
      acc += re_conj_mul(v, w);
      if (mode == 1) lam[i] = w;
      else if (mode == 2) { double2 l = lam[i]; l.x += w.x; l.y += w.y; lam[i] = l; }
    }
  } else {
    const int h = 63 - __clzll(x);
    const int64_t P = 1ll << (n - 1);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += stride) {
      const uint64_t i = insert_zero64((uint64_t)p, h), ip = i ^ x;
      double2 Ci = make_double2(0.0, 0.0), Cp = make_double2(0.0, 0.0);
      for (int j = 0; j < nterms; ++j) {
        // (P psi)[i] = c_j (-1)^{popc((i^x) & z)} psi[i^x]  (c_j includes i^{popc(x&z)})
        const double si = (__popcll(ip & s_z[j]) & 1) ? -1.0 : 1.0;
        const double sp = (__popcll(i & s_z[j]) & 1) ? -1.0 : 1.0;
        Ci.x = fma(si, s_c[j].x, Ci.x); Ci.y = fma(si, s_c[j].y, Ci.y);
        Cp.x = fma(sp, s_c[j].x, Cp.x); Cp.y = fma(sp, s_c[j].y, Cp.y);
      }
      const double2 vi = psi[i], vp = psi[ip];
      const double2 wi = cmul(Ci, vp), wp = cmul(Cp, vi);
      acc += re_conj_mul(vi, wi) + re_conj_mul(vp, wp);
      if (mode == 1) { lam[i] = wi; lam[ip] = wp; }
      else if (mode == 2) {
        double2 a = lam[i], b = lam[ip];
        a.x += wi.x; a.y += wi.y; b.x += wp.x; b.y += wp.y;
        lam[i] = a; lam[ip] = b;
      }
    }
  }
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}


// Cross-shard Pauli group (sharding, x-mask wider than a shard), one streamed CHUNK of the partner
// shard: partner[j - off] holds the partner's amplitudes j in [off, off + cnt) (cnt a power of two,
// off a multiple of cnt); this kernel adds the E partials of
//   sum_j conj(psi[j ^ xl]) C(j ^ xl) partner[j],  C(i) = sum_t c_t (-1)^{popc((i ^ xl) & z_t)},
// the partner's rank-bit signs folded into c_t by the host (so only a chunk-sized buffer is needed:
// a 34-qubit state on 2 GPUs leaves no room for a whole second shard). lam (optional) += C(i)
// partner[j] at i = j ^ xl. Partials accumulate into partials[blockIdx.x] across chunks (same grid).
__global__ void __launch_bounds__(kThreads) k_pauli_cross(const double2* __restrict__ psi,
                                                          const double2* __restrict__ partner, double2* __restrict__ lam,
                                                          int64_t off, int64_t cnt, uint64_t xl,
                                                          const uint64_t* __restrict__ z, const double2* __restrict__ c,
                                                          int nterms, double* __restrict__ partials, int first) {
  __shared__ uint64_t s_z[256];
  __shared__ double2 s_c[256];
  __shared__ double s_red[kThreads / 32];
  for (int i = threadIdx.x; i < nterms; i += blockDim.x) { s_z[i] = z[i]; s_c[i] = c[i]; }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jj < cnt; jj += stride) {
    const uint64_t j = (uint64_t)(off + jj);
    const uint64_t i = j ^ xl;
    double2 C = make_double2(0.0, 0.0);
    for (int t = 0; t < nterms; ++t) {
      const double sg = (__popcll(j & s_z[t]) & 1) ? -1.0 : 1.0;
      C.x = fma(sg, s_c[t].x, C.x);
      C.y = fma(sg, s_c[t].y, C.y);
    }
    const double2 w = cmul(C, partner[jj]);
    acc += re_conj_mul(psi[i], w);
    if (lam) { double2 l = lam[i]; l.x += w.x; l.y += w.y; lam[i] = l; }
  }
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) partials[blockIdx.x] = first ? acc : partials[blockIdx.x] + acc;
}


// ---- tiled multi-group Pauli pass (a4 / a5) ----
// One CTA loads a tile of 2^k amplitudes whose qubit set contains the x-masks of up to 32 Pauli
// groups; every element evaluates all those groups from the on-chip tile: one HBM read of psi (and
// one write / read-modify-write of lambda) for many groups instead of one pass per group.
//
// Geometry of the main path (2^12 tiles, 256 threads x 16 elements: the per-tile and per-entry setup
// of a thread is amortised over 16 elements; 8 warps per SM with 8 independent pairs each per term):
// element e = tid + 256 j of the tile, j < 16 in registers. The host orders the tile: positions 0..2
// = qubits 0..2 (128-byte HBM chunks; lanes on them read conflict-free 16-byte smem phases), 3..4
// (the other lane bits) = the two qubits least used by x-masks, 5..7 warp bits, 8..11 the register
// index j.
//
// Sign algebra (P = c i^{popc(x&z)} X^x Z^z, so (P psi)[e] = c' (-1)^{popc((e^x)&z)} psi[e^x]): per
// tile the outer-bit part (-1)^{popc(base & z_out)} and (-1)^{popc(x & z)} are folded into the
// coefficient (s_c); per element (-1)^{popc(e & z_tile)} = (-1)^{popc(tid & z)} (-1)^{popc(j & z_j)}:
// the first factor is a per-thread bit (computed once per kernel for each entry's first term), the second is bit
// j of the term's Walsh row walsh16(z_j) (uniform across the CTA).
//
// E only (mode 0): the host emits one entry per off-diagonal TERM (c' = c i^{popc(x&z)} is real or
// imaginary) plus one diagonal entry (all x = 0 terms). Off-diagonal entries use the Hermitian pair
// symmetry: the pair (e, e^x) contributes 2 Re[conj(psi_e) c' s(e) psi_{e^x}], so only one element
// of each pair (the "representative") is evaluated, and c' real / imaginary leaves one real product
// Re(conj(a) b) or Im(conj(a) b) per representative: 3 FP64 instructions and one 16-byte shared
// load per pair. Representatives: x has register bit JB -> the j with bit JB clear; x has warp bit
// w -> the j whose bit 0 equals bit w of tid (warp-uniform, no divergence, 8 of the 16 per thread);
// x inside the lane bits -> all elements without the factor 2. The diagonal entry uses |psi_j|^2,
// its 16-point Walsh-Hadamard transform W, and per register-part mask h one product
// (sum_t c_t (-1)^{popc(tid & z_t)}) * W[h].
// lambda modes (1: lam = H_pass psi, 2: lam += H_pass psi, 3: lam += H_pass psi and E = Re<psi|lam>):
// every element accumulates sum_g C_g(e) psi[e^x_g]; single-term groups with real / imaginary c'
// take 2 FMAs per element.
struct PauliTileArgs {
  int32_t k, low, n_outer, ngroups, nterms, mode;  // 0: E only; 1: lam = H_pass psi (+E); 2: lam += H_pass psi;
                                                   // 3: lam += H_pass psi, E = Re<psi|lam> (last tiled pass)
  int8_t tq[16];
  int8_t oq[64];
  int64_t ntiles;
  uint64_t xphys[32];
  uint32_t xtile[32];
  int32_t tbeg[32], tend[32];
  uint8_t gkind[32];    // bits 0-2: representative rule (PR_*); bits 3-4: PG_* type; bits 5-7: warp bit - 5
  int32_t diag_rb[17];  // E only: the diagonal entry's terms with register-part z mask h are [rb[h], rb[h+1])
  int32_t diag_g;       // E only: index of the diagonal entry (-1: none)
  int32_t cls_beg[11];  // E only: off-diagonal entries sorted by class (rule * 2 + imaginary): [cls_beg[c], cls_beg[c+1])
  uint32_t x16[32];     // E only: 16 * x_tile (byte-offset XOR of the partner element)
  uint32_t wrow[32];    // E only: Walsh row of the entry's register-part z mask
  uint64_t hsub[16];    // dep(i * 256 * PER): HBM offset of the copy / element index bits above the thread bits
  const uint64_t* z;
  const double2* c;
  double* partials;
};

__device__ __forceinline__ double2 amp(double2 v) { return v; }
__device__ __forceinline__ double2 amp(float2 v) { return make_double2((double)v.x, (double)v.y); }

constexpr int kPauliThreads = 1 << kPauliTileTidBits, kPauliTidBits = kPauliTileTidBits, kPauliEPT = 4096 / kPauliThreads;

// Walsh row of a 4-bit mask h: bit j (j < 16) = parity(j & h).
__device__ __forceinline__ uint32_t walsh16(uint32_t h) {
  uint32_t r = 0;
  if (h & 1u) r ^= 0xAAAAu;
  if (h & 2u) r ^= 0xCCCCu;
  if (h & 4u) r ^= 0xF0F0u;
  if (h & 8u) r ^= 0xFF00u;
  return r;
}

__device__ __forceinline__ double flip(double v, uint32_t neg) {  // neg ? -v : v (sign-bit xor)
  return __hiloint2double(__double2hiint(v) ^ (int)(neg << 31), __double2loint(v));
}

// Sum over the representatives j (bit JB of j == SEL; JB = 4: every j) of s_j Re(conj(v_j) p_j)
// (IM: Im(conj(v_j) p_j)); p_j is the partner element (tid + 512 j) ^ x of the tile, at byte offset
// q16 ^ (j * 16 * 512) with q16 = (16 tid) ^ (16 x); s_j = bit j of the Walsh row wr.
template <int JB, int SEL, bool IM, typename T>
__device__ __forceinline__ double pair_sum(const double2 (&v)[kPauliEPT], const char* __restrict__ tpb, uint32_t q16,
                                           uint32_t wr) {
  double s[4];
  int n = 0;
#pragma unroll
  for (int j = 0; j < kPauliEPT; ++j) {
    if (JB < 4 && (((j >> JB) & 1) != SEL)) continue;
    const double2 p = amp(*reinterpret_cast<const T*>(tpb + (q16 ^ ((uint32_t)j * (uint32_t)(sizeof(T) * kPauliThreads)))));
    const double q = flip(IM ? fma(v[j].x, p.y, -v[j].y * p.x) : fma(v[j].x, p.x, v[j].y * p.y), (wr >> j) & 1u);
    if (n < 4) s[n] = q;  // four independent chains, started from the first products
    else s[n & 3] += q;
    ++n;
  }
  return (s[0] + s[1]) + (s[2] + s[3]);
}

// The off-diagonal entries of one class [gb, ge) (compile-time representative rule and c' type).
// Entry g's term is term g of the pass (E-only layout); its coefficient s_c[g] is tile-folded.
template <int RULE, bool IM, typename T>
__device__ __forceinline__ double entry_class(const PauliTileArgs& a, int gb, int ge, const double2 (&v)[kPauliEPT],
                                              const char* __restrict__ tpb, const double2* __restrict__ s_c, uint32_t tid,
                                              uint32_t esg) {
  double acc = 0.0;
  for (int g = gb; g < ge; ++g) {
    const uint32_t q16 = (tid * (uint32_t)sizeof(T)) ^ (a.x16[g] >> (sizeof(T) == 16 ? 0 : 1));
    const uint32_t wr = a.wrow[g];
    const uint32_t nt = (esg >> g) & 1u;
    // the factor 2 of the pair-symmetric rules (representatives only) is in the host's coefficient
    double q;
    if (RULE < 4) {
      q = pair_sum<RULE, 0, IM, T>(v, tpb, q16, wr);
    } else if (RULE == PR_WARP) {
      const uint32_t sel = (tid >> (5 + (a.gkind[g] >> 5))) & 1u;
      q = sel ? pair_sum<0, 1, IM, T>(v, tpb, q16, wr) : pair_sum<0, 0, IM, T>(v, tpb, q16, wr);
    } else {
      q = pair_sum<4, 0, IM, T>(v, tpb, q16, wr);
    }
    // Re(c' q) = c'.x q (real c') or -c'.y q_im (imaginary c')
    acc = fma(IM ? flip(s_c[g].y, nt ^ 1u) : flip(s_c[g].x, nt), q, acc);
  }
  return acc;
}

template <typename T>  // T: double2 (complex128 state) or float2 (complex64 state, E only)
__global__ void __launch_bounds__(kPauliThreads, 1) k_pauli_tile(const T* __restrict__ psi, double2* __restrict__ lam,
                                                         PauliTileArgs a) {
  constexpr int EPT = kPauliEPT;
  constexpr uint32_t PER = sizeof(T) == 16 ? 1u : 2u;  // elements per 16-byte copy
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << a.k;
  T* tile_buf = reinterpret_cast<T*>(smem_raw);  // two tiles
  double2* s_c = reinterpret_cast<double2*>(tile_buf + 2 * N);   // folded coefficients (per tile)
  uint64_t* s_zo = reinterpret_cast<uint64_t*>(s_c + a.nterms);  // Z masks outside the tile (physical)
  uint32_t* s_zt = reinterpret_cast<uint32_t*>(s_zo + a.nterms); // tile-position Z masks | fixed fold parity << 31
  const int nhi = 1 << (a.k - a.low);
  uint64_t* s_hi = reinterpret_cast<uint64_t*>(s_zt + ((a.nterms + 1) & ~1));
  __shared__ uint64_t s_ob[4 * 64];  // tile base = OR of four 64-entry deposit tables over the outer qubits
  __shared__ double s_red[kPauliThreads / 32];
  uint64_t tmask = 0;
  for (int p = 0; p < a.k; ++p) tmask |= 1ull << a.tq[p];
  for (int g = 0; g < a.ngroups; ++g)
    for (int i = a.tbeg[g] + (int)threadIdx.x; i < a.tend[g]; i += blockDim.x) {
      const uint64_t z = a.z[i];
      s_zo[i] = z & ~tmask;
      uint32_t zt = 0;
      for (int p = 0; p < a.k; ++p)
        if ((z >> a.tq[p]) & 1ull) zt |= 1u << p;
      // the tile-independent part of the coefficient's sign, (-1)^{popc(x_tile & z_tile)}
      s_zt[i] = zt | ((uint32_t)(__popc(a.xtile[g] & zt) & 1) << 31);
    }
  for (int h = threadIdx.x; h < nhi; h += blockDim.x) {
    uint64_t off = 0;
    for (int b = 0; b < a.k - a.low; ++b)
      if ((h >> b) & 1) off |= 1ull << a.tq[a.low + b];
    s_hi[h] = off;
  }
  for (int h = threadIdx.x; h < 4 * 64; h += blockDim.x) {
    uint64_t off = 0;
    for (int b = 0; b < 6; ++b) {
      const int j = (h >> 6) * 6 + b;
      if (((h >> b) & 1) && j < a.n_outer) off |= 1ull << a.oq[j];
    }
    s_ob[h] = off;
  }
  const uint32_t tid = threadIdx.x;
  const uint32_t lowmask = (1u << a.low) - 1u;
  const int per_thread = (int)(N / blockDim.x);  // == EPT for 2^12-amplitude tiles, else smaller
  const bool fast = per_thread == EPT;
  // HBM offset of this thread's copies / elements within a tile (tile positions of the thread bits)
  uint64_t dep_t = 0;
  {
    const uint32_t e0 = tid * PER;
    for (int p = 0; p < a.k; ++p)
      if ((e0 >> p) & 1u) dep_t |= 1ull << a.tq[p];
  }
  __syncthreads();
  // per-thread sign bits (-1)^{popc(tid & z)} of the first term of each entry
  uint32_t esg = 0;
  for (int g = 0; g < a.ngroups; ++g) esg |= (uint32_t)(__popc(tid & s_zt[a.tbeg[g]] & 0x7fffffffu) & 1) << g;
  double acc = 0.0;
  auto tile_base = [&](int64_t tile) {
    uint64_t base = s_ob[tile & 63] | s_ob[64 + ((tile >> 6) & 63)] | s_ob[128 + ((tile >> 12) & 63)] |
                    s_ob[192 + ((tile >> 18) & 63)];
    for (int j = 24; j < a.n_outer; ++j)
      if ((tile >> j) & 1) base |= 1ull << a.oq[j];
    return base;
  };
  // 16-byte copies: one complex128 amplitude, or a complex64 pair (e, e + 1) — tile position 0 is
  // qubit 0, so the pair is contiguous in HBM too; double-buffered (cp.async streams tile i +
  // gridDim.x while tile i is evaluated)
  auto issue = [&](uint64_t base, T* dst) {
    if (fast) {
      const T* src = psi + (base | dep_t);
#pragma unroll
      for (int i = 0; i < EPT / (int)PER; ++i) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + tid * PER + (uint32_t)i * (kPauliThreads * PER));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + a.hsub[i]) : "memory");
      }
    } else {
      for (uint32_t e = threadIdx.x * PER; e < N; e += blockDim.x * PER) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(psi + (base | (e & lowmask) | s_hi[e >> a.low]))
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  uint64_t base_next = (int64_t)blockIdx.x < a.ntiles ? tile_base(blockIdx.x) : 0;
  if ((int64_t)blockIdx.x < a.ntiles) issue(base_next, tile_buf);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
    const uint64_t base = base_next;
    T* tp = tile_buf + (size_t)(it & 1) * N;
    __syncthreads();  // the other buffer's previous tile (and s_c) is fully consumed
    const int64_t next = tile + gridDim.x;
    const bool more = next < a.ntiles;
    if (more) {
      base_next = tile_base(next);
      issue(base_next, tile_buf + (size_t)((it + 1) & 1) * N);
    }
    // lambda modes 2 / 3: this tile's old lambda values are requested before the coefficient
    // fold, the tile wait and the barrier, so their HBM latency overlaps all three
    double2 l[EPT];
    if (fast && a.mode != 0) {
      const double2* lsrc = lam + (base | dep_t);
#pragma unroll
      for (int j = 0; j < EPT; ++j) l[j] = a.mode >= 2 ? lsrc[a.hsub[j]] : make_double2(0.0, 0.0);
    }
    // fold (-1)^{popc(base & z_out)} (outer part) and (-1)^{popc(xt & zt)} into the coefficients
    for (int t = (int)tid; t < a.nterms; t += blockDim.x) {
      const uint32_t neg = ((uint32_t)__popcll(base & s_zo[t]) ^ (s_zt[t] >> 31)) & 1u;
      const double2 c = a.c[t];
      s_c[t] = make_double2(flip(c.x, neg), flip(c.y, neg));
    }
    if (more) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if (fast && a.mode == 0) {
      // ---- E only: representatives of off-diagonal terms + the diagonal entry ----
      double2 v[EPT];
#pragma unroll
      for (int j = 0; j < EPT; ++j) v[j] = amp(tp[tid + (uint32_t)j * kPauliThreads]);
      if (a.diag_g >= 0) {
        // diagonal terms: Walsh transform of |psi_j|^2 over j; the terms with z_j = h give
        // (sum_t c_t (-1)^{popc(tid & z_t)}) * W[h]
        double W[EPT];
#pragma unroll
        for (int j = 0; j < EPT; ++j) W[j] = fma(v[j].x, v[j].x, v[j].y * v[j].y);
#pragma unroll
        for (int h = 1; h < EPT; h <<= 1)
#pragma unroll
          for (int j = 0; j < EPT; ++j)
            if (!(j & h)) {
              const double x0 = W[j], x1 = W[j | h];
              W[j] = x0 + x1;
              W[j | h] = x0 - x1;
            }
#pragma unroll
        for (int h = 0; h < EPT; ++h) {
          int t = a.diag_rb[h];
          const int te = a.diag_rb[h + 1];
          if (t == te) continue;
          double S = 0.0;
          for (; t < te; ++t) S += flip(s_c[t].x, __popc(tid & s_zt[t]) & 1u);  // x = 0: c' = c real
          acc = fma(S, W[h], acc);
        }
      }
      const char* tpb = reinterpret_cast<const char*>(tp);
      acc += entry_class<0, false, T>(a, a.cls_beg[0], a.cls_beg[1], v, tpb, s_c, tid, esg);
      acc += entry_class<0, true, T>(a, a.cls_beg[1], a.cls_beg[2], v, tpb, s_c, tid, esg);
      acc += entry_class<1, false, T>(a, a.cls_beg[2], a.cls_beg[3], v, tpb, s_c, tid, esg);
      acc += entry_class<1, true, T>(a, a.cls_beg[3], a.cls_beg[4], v, tpb, s_c, tid, esg);
      acc += entry_class<2, false, T>(a, a.cls_beg[4], a.cls_beg[5], v, tpb, s_c, tid, esg);
      acc += entry_class<2, true, T>(a, a.cls_beg[5], a.cls_beg[6], v, tpb, s_c, tid, esg);
      acc += entry_class<PR_WARP, false, T>(a, a.cls_beg[6], a.cls_beg[7], v, tpb, s_c, tid, esg);
      acc += entry_class<PR_WARP, true, T>(a, a.cls_beg[7], a.cls_beg[8], v, tpb, s_c, tid, esg);
      acc += entry_class<PR_ALL, false, T>(a, a.cls_beg[8], a.cls_beg[9], v, tpb, s_c, tid, esg);
      acc += entry_class<PR_ALL, true, T>(a, a.cls_beg[9], a.cls_beg[10], v, tpb, s_c, tid, esg);
    } else if (fast) {
      // ---- lambda modes: every element accumulates sum_g C_g(e) psi[e ^ x_g] ----
      // modes 2 / 3 (lambda += this pass' groups): l holds the old lambda values (requested
      // above); the sum is stored once
      for (int g = 0; g < a.ngroups; ++g) {
        const uint32_t gk = a.gkind[g];
        const uint32_t xt = a.xtile[g];
        const int tb = a.tbeg[g], te = a.tend[g];
        const uint32_t pb = tid ^ (xt & (kPauliThreads - 1u)), xj = xt >> kPauliTidBits;
        const uint32_t type = (gk >> 3) & 3u;
        if (type <= PG_SINGLE_IM) {
          // one term, c' real (l += w s_j p) or imaginary (l += i w s_j p)
          const uint32_t zt = s_zt[tb] & 0x7fffffffu;
          const uint32_t wr = walsh16(zt >> kPauliTidBits);
          const bool im = type == PG_SINGLE_IM;
          const double w = flip(im ? s_c[tb].y : s_c[tb].x, (esg >> g) & 1u);
#pragma unroll
          for (int j = 0; j < EPT; ++j) {
            const double2 p = amp(tp[pb + (((uint32_t)j ^ xj) << kPauliTidBits)]);
            const double ws = flip(w, (wr >> j) & 1u);
            if (im) {
              l[j].x = fma(-ws, p.y, l[j].x);
              l[j].y = fma(ws, p.x, l[j].y);
            } else {
              l[j].x = fma(ws, p.x, l[j].x);
              l[j].y = fma(ws, p.y, l[j].y);
            }
          }
          continue;
        }
        // several terms (or the diagonal group): the host sorts a group's terms by their
        // element-part mask zh = zt >> tid bits; a run of equal zh is summed once (per-thread signs
        // folded), then spread over the elements with compile-time Walsh signs
        double2 C[EPT];
#pragma unroll
        for (int j = 0; j < EPT; ++j) C[j] = make_double2(0.0, 0.0);
        double2 S = make_double2(0.0, 0.0);
        uint32_t cur = (s_zt[tb] & 0x7fffffffu) >> kPauliTidBits;
        auto spread = [&](uint32_t zh) {
#define SV_SPREAD(H)                                                  \
  case H:                                                             \
    _Pragma("unroll") for (int j = 0; j < EPT; ++j) {                 \
      if (__builtin_popcount(j & H) & 1) { C[j].x -= S.x; C[j].y -= S.y; } \
      else { C[j].x += S.x; C[j].y += S.y; }                           \
    }                                                                 \
    break;
          switch (zh & 15u) {
            SV_SPREAD(0) SV_SPREAD(1) SV_SPREAD(2) SV_SPREAD(3) SV_SPREAD(4) SV_SPREAD(5) SV_SPREAD(6) SV_SPREAD(7)
            SV_SPREAD(8) SV_SPREAD(9) SV_SPREAD(10) SV_SPREAD(11) SV_SPREAD(12) SV_SPREAD(13) SV_SPREAD(14) SV_SPREAD(15)
          }
#undef SV_SPREAD
        };
        for (int t = tb; t < te; ++t) {
          const uint32_t zt = s_zt[t] & 0x7fffffffu;
          const uint32_t zh = zt >> kPauliTidBits;
          if (zh != cur) {
            spread(cur);
            S = make_double2(0.0, 0.0);
            cur = zh;
          }
          const double2 c = s_c[t];
          const uint32_t neg = __popc(tid & zt) & 1u;
          S.x += flip(c.x, neg);
          S.y += flip(c.y, neg);
        }
        spread(cur);
        if (type == PG_DIAG) {  // the partner is the element itself
#pragma unroll
          for (int j = 0; j < EPT; ++j) l[j] = cfma(C[j], amp(tp[tid + (uint32_t)j * kPauliThreads]), l[j]);
        } else {
#pragma unroll
          for (int j = 0; j < EPT; ++j) l[j] = cfma(C[j], amp(tp[pb + (((uint32_t)j ^ xj) << kPauliTidBits)]), l[j]);
        }
      }
      double2* ldst = lam + (base | dep_t);
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        if (a.mode != 2) acc += re_conj_mul(amp(tp[tid + (uint32_t)j * kPauliThreads]), l[j]);  // mode 3: Re<psi|lambda> of all passes so far
        ldst[a.hsub[j]] = l[j];
      }
    } else {
      // small tiles (n < 12): one element at a time, every term of every group (mode 0 entries
      // are single terms here as well; no pair symmetry)
      for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
        double2 l = make_double2(0.0, 0.0);
        for (int g = 0; g < a.ngroups; ++g) {
          double2 C = make_double2(0.0, 0.0);
          for (int t = a.tbeg[g]; t < a.tend[g]; ++t) {
            const uint32_t neg = __popc(e & s_zt[t] & 0x7fffffffu) & 1u;
            const double2 c = s_c[t];
            C.x += flip(c.x, neg);
            C.y += flip(c.y, neg);
          }
          const double2 w = cmul(C, amp(tp[e ^ a.xtile[g]]));
          l.x += w.x;
          l.y += w.y;
        }
        const uint64_t gi = base | (e & lowmask) | s_hi[e >> a.low];
        if (a.mode >= 2) {
          const double2 o = lam[gi];
          l.x += o.x;
          l.y += o.y;
        }
        if (a.mode != 2) acc += re_conj_mul(amp(tp[e]), l);
        if (a.mode != 0) lam[gi] = l;
      }
    }
  }
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = acc;
}


// ---- sampling (NEXT-2: "Sampling Measurement", Fig. 1) ----
// Stage 1: probability mass of each block of 2^bl amplitudes (fixed-order block reduction).
__global__ void __launch_bounds__(kThreads) k_block_prob(const double2* __restrict__ psi, int bl, double* __restrict__ out) {
  __shared__ double s_red[kThreads / 32];
  const int64_t b0 = (int64_t)blockIdx.x << bl, B = 1ll << bl;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < B; i += blockDim.x) {
    const double2 v = psi[b0 + i];
    acc = fma(v.x, v.x, fma(v.y, v.y, acc));
  }
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
// Stage 2: one CTA per block holding draws: inclusive prefix of |psi|^2 over the block in chunks of
// blockDim amplitudes; draw r (target mass u_r - block start, sorted) resolves to the first index
// whose prefix reaches it.
__global__ void __launch_bounds__(kThreads) k_sample_block(const double2* __restrict__ psi, int bl,
                                                           const int64_t* __restrict__ blk, const int64_t* __restrict__ beg,
                                                           const double* __restrict__ target, int64_t* __restrict__ out) {
  __shared__ double s_scan[kThreads];
  __shared__ double s_carry;
  const int64_t b = blk[blockIdx.x], r0 = beg[blockIdx.x], r1 = beg[blockIdx.x + 1];
  const int64_t b0 = b << bl, B = 1ll << bl;
  if (threadIdx.x == 0) s_carry = 0.0;
  int64_t r = r0;  // next unresolved draw (uniform across the block)
  __syncthreads();
  for (int64_t off = 0; off < B && r < r1; off += blockDim.x) {
    double pv = 0.0;
    if (off + threadIdx.x < B) {
      const double2 v = psi[b0 + off + threadIdx.x];
      pv = fma(v.x, v.x, v.y * v.y);
    }
    s_scan[threadIdx.x] = pv;
    __syncthreads();
    if (threadIdx.x == 0) {  // sequential inclusive scan of the chunk (fixed order, exact reproducibility)
      double c = s_carry;
      for (int i = 0; i < (int)blockDim.x; ++i) { c += s_scan[i]; s_scan[i] = c; }
      s_carry = c;
    }
    __syncthreads();
    // resolve draws whose target falls in this chunk
    if (threadIdx.x == 0) {
      while (r < r1 && target[r] <= s_scan[blockDim.x - 1]) {
        int lo = 0, hi = (int)blockDim.x - 1;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_scan[mid] >= target[r]) hi = mid; else lo = mid + 1; }
        out[r] = b0 + off + lo;
        ++r;
      }
      s_scan[0] = (double)r;  // broadcast progress
    }
    __syncthreads();
    r = (int64_t)s_scan[0];
    __syncthreads();
  }
  // numerical tail (target beyond the block's accumulated mass by rounding): last index
  if (threadIdx.x == 0)
    for (; r < r1; ++r) out[r] = b0 + B - 1;
}


// ---- density matrix (NEXT-4, §3.2) ----
// tr(rho P) for the Pauli terms of one x-group: rho[r'][r] is stored at r' + (r << n), and
// (P rho)[r][r] = c' (-1)^{popc((r ^ x) & z)} rho[r ^ x][r]; E partial = Re sum_r sum_t (...).
__global__ void __launch_bounds__(kThreads) k_dm_trace(const double2* __restrict__ vec, int n, uint64_t x,
                                                       const uint64_t* __restrict__ z, const double2* __restrict__ c,
                                                       int nterms, double* __restrict__ partials) {
  __shared__ uint64_t s_z[256];
  __shared__ double2 s_c[256];
  __shared__ double s_red[kThreads / 32];
  for (int i = threadIdx.x; i < nterms; i += blockDim.x) { s_z[i] = z[i]; s_c[i] = c[i]; }
  __syncthreads();
  const int64_t N = 1ll << n, stride = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
    const uint64_t rp = (uint64_t)r ^ x;
    double2 C = make_double2(0.0, 0.0);
    for (int t = 0; t < nterms; ++t) {
      const double sg = (__popcll(rp & s_z[t]) & 1) ? -1.0 : 1.0;
      C.x = fma(sg, s_c[t].x, C.x);
      C.y = fma(sg, s_c[t].y, C.y);
    }
    const double2 v = vec[rp | ((uint64_t)r << n)];
    acc += fma(C.x, v.x, -C.y * v.y);
  }
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

// out[s] = sum_{j < per} partials[s*per + j], fixed order (strided per-thread sums, then a fixed tree).
// Re<a|b> over n amplitudes: per-CTA partials (fixed order; reduced by k_reduce_slots).
__global__ void __launch_bounds__(kThreads) k_redot(const double2* __restrict__ x, const double2* __restrict__ y, int64_t n,
                                                    double* __restrict__ partials) {
  __shared__ double s_red[kThreads / 32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += re_conj_mul(x[i], y[i]);
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(kThreads) k_reduce_slots(const double* __restrict__ partials, int per,
                                                           double* __restrict__ out) {
  __shared__ double s_red[kThreads / 32];
  const double* p = partials + (int64_t)blockIdx.x * per;
  double acc = 0.0;
  for (int j = threadIdx.x; j < per; j += blockDim.x) acc += p[j];
  acc = block_sum(acc, s_red);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

// out[i] = sum over g < n_cta of p[g * per + i], in g order (per-CTA contiguous partials)
__global__ void __launch_bounds__(kThreads) k_reduce_strided(const double* __restrict__ p, int64_t per, int n_cta,
                                                             double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int g = 0; g < n_cta; ++g) acc += p[(int64_t)g * per + i];
    out[i] = acc;
  }
}

size_t pass_smem_bytes(int k, int low, int nops, int nmats, bool dual) {
  const size_t N = size_t(1) << k;
  size_t b = N * 16 * (dual ? 2 : 1);
  b += (size_t)nops * sizeof(DevOp);
  b += (size_t)((nmats + 1) & ~1) * 8;
  b += (size_t(1) << (k - low)) * 8;
  b += (dual ? (size_t)nops * 8 : 0) + (kThreads / 32) * 8;
  return b;
}

std::atomic<int> g_num_sms[64];  // per device id (zero-initialised: static storage)
int num_sms() {
  const int dev = current_device() & 63;
  int v = g_num_sms[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    g_num_sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

}  // namespace

int device_sm_count() { return num_sms(); }

int pass_grid(int n_local, int k, bool dual) {
  const int64_t ntiles = 1ll << (n_local - k);
  const int64_t want = (int64_t)num_sms() * 2 * ((k <= 10) ? 2 : 1);
  return (int)(ntiles < want ? ntiles : want);
}

// One grid for every pass of a plan (the adjoint partials are laid out [slot][grid]): register
// passes run one persistent, double-buffered CTA per SM; shared-memory passes two or more.
static int plan_grid_uncached(const Plan& plan, int n_local);

int plan_grid(const Plan& plan, int n_local) {
  if (plan.grid_cache_n != n_local) {
    plan.grid_cache = plan_grid_uncached(plan, n_local);
    plan.grid_cache_n = n_local;
  }
  return plan.grid_cache;
}

static int plan_grid_uncached(const Plan& plan, int n_local) {
  plan.pass_grid.assign(plan.passes.size(), 1);
  if (plan.passes.empty()) return 1;
  const PassDesc& pd = plan.passes[0];
  if (pd.R > 0) {
    const int64_t ntiles = 1ll << (n_local - pd.k);
    // persistent grids sized by occupancy, pass by pass: forward passes run up to three 2^11-tile
    // CTAs per SM (their phases interleave: one CTA's MMA stage overlaps the others' shared-memory /
    // HBM phases), adjoint passes two 2^10-tile CTAs; fewer where a pass needs more shared memory.
    // The plan's grid (the stride of the adjoint partials) is the largest pass grid.
    const bool dual = plan.reverse;
    static const int dual_env = [] { const char* e = getenv("SV_DUAL_CTAS"); return e ? atoi(e) : 0; }();
    static const int fwd_env = [] { const char* e = getenv("SV_FWD_GRID_CTAS"); return e ? atoi(e) : 0; }();
    const int env = dual ? dual_env : fwd_env;
    int mx = 1;
    for (size_t i = 0; i < plan.passes.size(); ++i) {
      const PassDesc& p = plan.passes[i];
      const int64_t nt = 1ll << (n_local - p.k);
      const int ctas = env > 0 ? env : reg_pass_ctas_per_sm(plan, i, dual, n_local);
      const int64_t want = (int64_t)num_sms() * ctas;
      plan.pass_grid[i] = (int)(nt < want ? nt : want);
      mx = std::max(mx, plan.pass_grid[i]);
    }
    (void)ntiles;
    return mx;
  }
  const int g = pass_grid(n_local, pd.k, false);
  plan.pass_grid.assign(plan.passes.size(), g);
  return g;
}

cudaError_t launch_pass(double* psi, double* lam, const PassLaunch& L, cudaStream_t s) {
  const PassDesc& pd = *L.pd;
  if (pd.R > 0) return launch_pass_reg(psi, lam, L, s);
  PassArgs a;
  a.k = pd.k;
  a.low = pd.low;
  a.nops = pd.op_end - pd.op_begin;
  for (int i = 0; i < kMaxTileQubits + 3; ++i) a.tq[i] = pd.tq[i];
  uint64_t tmask = 0;
  for (int p = 0; p < pd.k; ++p) tmask |= 1ull << pd.tq[p];
  a.n_outer = 0;
  for (int q = 0; q < L.n_local; ++q)
    if (!((tmask >> q) & 1ull)) a.oq[a.n_outer++] = (int8_t)q;
  a.ntiles = 1ll << (L.n_local - pd.k);
  a.ops = L.d_ops + pd.op_begin;
  a.mats = L.d_mats + pd.mat_begin;
  a.nmats = L.nmats;
  a.partials = L.d_partials;
  a.grid = L.pstride > 0 ? L.pstride : L.grid;  // slot-row stride of the partials
  const bool dual = lam != nullptr;
  const size_t smem = pass_smem_bytes(a.k, a.low, a.nops, a.nmats, dual);
  static std::atomic<uint64_t> attr_set{0};
  {
    cudaError_t e = once_per_device(attr_set, [] {
      cudaError_t r = cudaFuncSetAttribute(k_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      return r == cudaSuccess ? cudaFuncSetAttribute(k_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) : r;
    });
    if (e != cudaSuccess) return e;
  }
  if (dual)
    k_pass<true><<<L.grid, kThreads, smem, s>>>(reinterpret_cast<double2*>(psi), reinterpret_cast<double2*>(lam), a);
  else
    k_pass<false><<<L.grid, kThreads, smem, s>>>(reinterpret_cast<double2*>(psi), nullptr, a);
  return cudaGetLastError();
}

cudaError_t launch_init_zero(double* psi, int64_t n_amps, bool one_at_zero, cudaStream_t s) {
  int64_t blocks = (n_amps + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_init<<<(int)blocks, kThreads, 0, s>>>(reinterpret_cast<double2*>(psi), n_amps, one_at_zero);
  return cudaGetLastError();
}

int pauli_grid(int n_local) {
  const int64_t work = (1ll << n_local) / kThreads / 4;
  const int64_t cap = (int64_t)num_sms() * 4;
  int64_t g = work < cap ? work : cap;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_pauli_group(const double* psi, double* lam, bool lam_accumulate, int n_local, uint64_t x,
                               const uint64_t* d_z, const double* d_c, int nterms, double* d_partials, int grid,
                               cudaStream_t s) {
  const int mode = lam == nullptr ? 0 : (lam_accumulate ? 2 : 1);
  k_pauli_group<<<grid, kThreads, 0, s>>>(reinterpret_cast<const double2*>(psi), reinterpret_cast<double2*>(lam), mode,
                                          n_local, x, d_z, reinterpret_cast<const double2*>(d_c), nterms, d_partials);
  return cudaGetLastError();
}

cudaError_t launch_redot(const double* x, const double* y, int64_t n, double* d_partials, int grid, cudaStream_t s) {
  k_redot<<<grid, kThreads, 0, s>>>(reinterpret_cast<const double2*>(x), reinterpret_cast<const double2*>(y), n, d_partials);
  return cudaGetLastError();
}

cudaError_t launch_reduce_strided(const double* d_partials, int64_t per, int n_cta, double* d_out, cudaStream_t s) {
  if (per <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((per + kThreads - 1) / kThreads, (int64_t)num_sms() * 4);
  k_reduce_strided<<<blocks, kThreads, 0, s>>>(d_partials, per, n_cta, d_out);
  return cudaGetLastError();
}

cudaError_t launch_reduce_slots(const double* d_partials, int n_slots, int per_slot, double* d_out, cudaStream_t s) {
  if (n_slots <= 0) return cudaSuccess;
  k_reduce_slots<<<n_slots, kThreads, 0, s>>>(d_partials, per_slot, d_out);
  return cudaGetLastError();
}

static int elementwise_grid(int64_t n) {
  int64_t blocks = (n + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

cudaError_t launch_gather(const void* psi, bool c64, const uint64_t* idx, int64_t count, double* out, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  if (c64)
    k_gather<float2><<<elementwise_grid(count), kThreads, 0, s>>>(static_cast<const float2*>(psi), idx, count,
                                                                  reinterpret_cast<double2*>(out));
  else
    k_gather<double2><<<elementwise_grid(count), kThreads, 0, s>>>(static_cast<const double2*>(psi), idx, count,
                                                                   reinterpret_cast<double2*>(out));
  return cudaGetLastError();
}

cudaError_t launch_swap_halves(double* a, double* b, int nl, int l, cudaStream_t s) {
  k_swap_halves<<<elementwise_grid(1ll << (nl - 1)), kThreads, 0, s>>>(reinterpret_cast<double2*>(a),
                                                                        reinterpret_cast<double2*>(b), nl, l);
  return cudaGetLastError();
}

cudaError_t launch_pack_half(double* shard, double* buf, int l, int h, int64_t off, int64_t count, bool pack,
                             cudaStream_t s) {
  k_pack_half<<<elementwise_grid(count), kThreads, 0, s>>>(reinterpret_cast<double2*>(shard),
                                                             reinterpret_cast<double2*>(buf), l, h, off, count,
                                                             pack ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_pauli_cross(const double* psi, const double* partner, double* lam, int64_t off, int64_t cnt,
                               uint64_t xl, const uint64_t* d_z, const double* d_c, int nterms, double* d_partials,
                               int grid, bool first, cudaStream_t s) {
  k_pauli_cross<<<grid, kThreads, 0, s>>>(reinterpret_cast<const double2*>(psi), reinterpret_cast<const double2*>(partner),
                                          reinterpret_cast<double2*>(lam), off, cnt, xl, d_z,
                                          reinterpret_cast<const double2*>(d_c), nterms, d_partials, first ? 1 : 0);
  return cudaGetLastError();
}

int pauli_tile_grid(int n_local, int k) {
  const int64_t ntiles = 1ll << (n_local - k);
  const int64_t want = (int64_t)num_sms();
  return (int)(ntiles < want ? ntiles : want);
}

static cudaError_t pauli_tile_impl(const void* psi, bool c64, double* lam, int mode, int n_local, const PauliPassDesc& pp,
                                   const uint64_t* d_z, const double* d_c, double* d_partials, int grid, cudaStream_t s) {
  PauliTileArgs a;
  std::memset(&a, 0, sizeof(a));
  a.k = pp.k;
  a.low = pp.low;
  a.ngroups = pp.ngroups;
  a.nterms = pp.nterms;
  a.mode = mode;
  for (int i = 0; i < 16; ++i) a.tq[i] = pp.tq[i];
  uint64_t tmask = 0;
  for (int p = 0; p < pp.k; ++p) tmask |= 1ull << pp.tq[p];
  a.n_outer = 0;
  for (int q = 0; q < n_local; ++q)
    if (!((tmask >> q) & 1ull)) a.oq[a.n_outer++] = (int8_t)q;
  a.ntiles = 1ll << (n_local - pp.k);
  for (int g = 0; g < pp.ngroups; ++g) {
    a.xphys[g] = pp.xphys[g];
    a.xtile[g] = pp.xtile[g];
    a.tbeg[g] = pp.tbeg[g];
    a.tend[g] = pp.tend[g];
    a.gkind[g] = pp.gkind[g];
  }
  for (int h = 0; h < 17; ++h) a.diag_rb[h] = pp.diag_rb[h];
  a.diag_g = pp.diag_g;
  for (int c = 0; c < 11; ++c) a.cls_beg[c] = pp.cls_beg[c];
  for (int g = 0; g < pp.ngroups; ++g) {
    a.x16[g] = pp.xtile[g] * 16u;
    uint32_t h = 0;
    for (int j = 0; j < 16; ++j)
      if (__builtin_popcount((uint32_t)j & (pp.zt_reg[g])) & 1) h |= 1u << j;
    a.wrow[g] = h;
  }
  {
    const uint32_t per = c64 ? 2u : 1u;
    for (int i = 0; i < 16; ++i) {
      const uint32_t e = (uint32_t)i * kPauliThreads * per;
      uint64_t off = 0;
      for (int p = 0; p < pp.k; ++p)
        if ((e >> p) & 1u) off |= 1ull << pp.tq[p];
      a.hsub[i] = off;
    }
  }
  a.z = d_z + pp.term_base;
  a.c = reinterpret_cast<const double2*>(d_c) + pp.term_base;
  a.partials = d_partials;
  size_t smem = (size_t(c64 ? 16 : 32) << pp.k) + (size_t)pp.nterms * 28 + 8 + (size_t(8) << (pp.k - pp.low));
  static std::atomic<uint64_t> attr{0};
  {
    cudaError_t e = once_per_device(attr, [] {
      cudaError_t r = cudaFuncSetAttribute(k_pauli_tile<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      return r == cudaSuccess ? cudaFuncSetAttribute(k_pauli_tile<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) : r;
    });
    if (e != cudaSuccess) return e;
  }
  if (c64) {
    if (lam || mode != 0 || pp.tq[0] != 0) return cudaErrorInvalidValue;  // E only; pairs need qubit 0 at position 0
    k_pauli_tile<float2><<<grid, kPauliThreads, smem, s>>>(reinterpret_cast<const float2*>(psi), nullptr, a);
  } else {
    k_pauli_tile<double2><<<grid, kPauliThreads, smem, s>>>(reinterpret_cast<const double2*>(psi), reinterpret_cast<double2*>(lam), a);
  }
  return cudaGetLastError();
}

cudaError_t launch_pauli_tile(const double* psi, double* lam, int mode, int n_local, const PauliPassDesc& pp,
                              const uint64_t* d_z, const double* d_c, double* d_partials, int grid, cudaStream_t s) {
  return pauli_tile_impl(psi, false, lam, mode, n_local, pp, d_z, d_c, d_partials, grid, s);
}

cudaError_t launch_pauli_tile_c64(const float* psi, int n_local, const PauliPassDesc& pp, const uint64_t* d_z,
                                  const double* d_c, double* d_partials, int grid, cudaStream_t s) {
  return pauli_tile_impl(psi, true, nullptr, 0, n_local, pp, d_z, d_c, d_partials, grid, s);
}



cudaError_t launch_block_prob(const double* psi, int n_local, int bl, double* out, cudaStream_t s) {
  k_block_prob<<<(unsigned)(1ll << (n_local - bl)), kThreads, 0, s>>>(reinterpret_cast<const double2*>(psi), bl, out);
  return cudaGetLastError();
}

cudaError_t launch_sample_blocks(const double* psi, int bl, int nblk, const int64_t* blk, const int64_t* beg,
                                 const double* target, int64_t* out, cudaStream_t s) {
  if (nblk <= 0) return cudaSuccess;
  k_sample_block<<<nblk, kThreads, 0, s>>>(reinterpret_cast<const double2*>(psi), bl, blk, beg, target, out);
  return cudaGetLastError();
}

cudaError_t launch_dm_trace(const double* vec, int n, uint64_t x, const uint64_t* d_z, const double* d_c, int nterms,
                            double* d_partials, int grid, cudaStream_t s) {
  k_dm_trace<<<grid, kThreads, 0, s>>>(reinterpret_cast<const double2*>(vec), n, x, d_z,
                                       reinterpret_cast<const double2*>(d_c), nterms, d_partials);
  return cudaGetLastError();
}

}  // namespace sv
