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
//
// Instruction economy (the pass is FP64-pipe bound once ~10 gates are fused): ops are 32-byte
// RegOps read with two 16-byte shared loads; the pair/quad loops are fully unrolled over
// compile-time register indices with a control-free fast path, so the FP64 pipe sees long runs of
// independent DFMAs; Z-like ops with a = 1 touch only half the amplitudes and CZ-type ops
// (a = 1, b = -1) are sign flips without FP64 work.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "cx.cuh"
#include "sv_internal.h"

#ifndef SV_DENSE_CTAS
#define SV_DENSE_CTAS 2  // k_pass_dense CTAs per SM (128 registers: the Gauss form's live set)
#endif
#ifndef SV_DENSE_NBUF
#define SV_DENSE_NBUF 2  // k_pass_dense tile ring depth (3: no gain measured)
#endif
#ifndef SV_DENSE_VT
#define SV_DENSE_VT 1
#endif
#ifndef SV_DA_R_3M
#define SV_DA_R_3M 1  // adjoint dense stages: R = sum psi lambda^H with three real products
#endif
#ifndef SV_DA_SHARED_A
#define SV_DA_SHARED_A 1  // adjoint dense stages: one A load and coefficient set for psi and lambda
#endif
#ifndef SV_DMMA_VOLATILE
#define SV_DMMA_VOLATILE 1
#endif
#ifndef SV_FWD_CTAS
#define SV_FWD_CTAS 2   // forward register passes: CTAs per SM (register budget 65536 / (256 * CTAs));
                        // 2 (128 registers) fits the dense stages' Gauss live set (3: 80, spills)
#endif
#ifndef SV_FWD_SEQ_CTAS
#define SV_FWD_SEQ_CTAS 3  // forward passes without dense stages (k_pass_reg<3, false, true>)
#endif
#ifndef SV_C64_CTAS
#define SV_C64_CTAS 3   // complex64 forward passes
#endif
#ifndef SV_DUAL_CTAS
#define SV_DUAL_CTAS 3  // adjoint-pass (2^10-tile, 128-thread) CTAs per SM (register cap 65536 / (128 * 3))
#endif
#ifndef SV_FWD_CTRL_SPLIT
#define SV_FWD_CTRL_SPLIT 0  // 1: forward register passes get separate code for ops with / without register controls
#endif
#ifndef SV_DUAL_CTRL_SPLIT
#define SV_DUAL_CTRL_SPLIT 0  // 1: separate DUAL op code for ops with / without register controls
#endif
#ifndef SV_DUAL_SB_CTAS
#define SV_DUAL_SB_CTAS 4  // single-buffered adjoint instantiation: CTAs per SM of its register cap
                           // (4: 128 registers, a few spills, still +3-7% over 3 at 168)
#endif
#ifndef SV_DUAL_RG_CTAS
#define SV_DUAL_RG_CTAS 4  // adjoint passes with L2 R accumulators: CTAs per SM of the register cap
                           // (4: 128 registers with spills, C4g 2.57 -> 2.62 over 3)
#endif
#ifndef SV_DUAL_SINGLE_BUF_MAX_N
#define SV_DUAL_SINGLE_BUF_MAX_N 64  // adjoint passes up to this many local qubits single-buffer
#endif

namespace sv {
namespace {

__host__ __device__ __forceinline__ uint32_t swz(uint32_t t) { return t ^ ((t >> 3 ^ t >> 6 ^ t >> 9 ^ t >> 12) & 7u); }
// complex64 tiles: 8-byte slots, 16 per 128-byte bank row -> 4-bit XOR fold
__host__ __device__ __forceinline__ uint32_t swz8(uint32_t t) { return t ^ ((t >> 4 ^ t >> 8 ^ t >> 12) & 15u); }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}

// Shared-memory load the compiler may not hoist or CSE (keeps 4x4 matrices out of registers).
__device__ __forceinline__ double2 lds(const double2* p) {
  double2 r;
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(r.x), "=d"(r.y) : "r"(a));
  return r;
}

__device__ __forceinline__ double2 cneg(double2 a) { return make_double2(-a.x, -a.y); }

struct RegArgs {
  int32_t k, low, nops, nstages, n_outer, nmats, ngrad, grid;
  int32_t n_da, pstride;  // pstride: slot-row stride of partials (>= grid)
  int32_t c64_terms;  // complex64 dense stages: 3 = hi/lo split products (default), 1 = hi only
  int32_t acc_thread; // adjoint: 1 = overlap partials per thread ([grad op][thread] in shared memory, summed
                      // once at the end), 0 = warp-shuffle reduced per op ([grad op][warp])
  int32_t single_buf; // adjoint: one (psi, lambda) tile buffer (more resident CTAs; passes with adjoint
                      // dense stages always)
  double* r_partials;  // adjoint dense stages: [da][warp][16 * 32][grid]
  int8_t tq[kMaxTileQubits + 3];
  int8_t oq[64];
  // element e = tid + i * nthr: dep(i << nthr_bits) and swz(i << nthr_bits) per i (host-computed;
  // kernel-parameter constants, no registers)
  uint64_t hsub[8];
  uint32_t zsub[8];
  int64_t ntiles;
  const RegOp* ops;
  const double* mats;
  const StageDesc* stages;
  double* partials;
};

// An op held as its raw words; fields are extracted where used (keeps register pressure low).
struct Op {
  uint32_t code, w1, w2, w3;
  uint64_t couter;
  __device__ __forceinline__ uint32_t type() const { return code & 15u; }
  __device__ __forceinline__ uint32_t ra() const { return (code >> 4) & 15u; }
  __device__ __forceinline__ uint32_t rb() const { return (code >> 8) & 15u; }
  __device__ __forceinline__ uint32_t cj() const { return (code >> 12) & 15u; }
  __device__ __forceinline__ uint32_t pa() const { return (code >> 16) & 31u; }
  __device__ __forceinline__ uint32_t pb() const { return (code >> 21) & 31u; }
  __device__ __forceinline__ uint32_t gen() const { return (code >> 26) & 3u; }
  __device__ __forceinline__ uint32_t gdiag() const { return (code >> 28) & 1u; }
  __device__ __forceinline__ uint32_t dfl() const { return code >> 29; }
  __device__ __forceinline__ uint32_t mat_off() const { return w1 & 0xffffu; }
  __device__ __forceinline__ uint32_t gen_off() const { return w1 >> 16; }
  __device__ __forceinline__ uint32_t cthr() const { return w2 & 0xffffu; }
  __device__ __forceinline__ int32_t grad_local() const { return (int32_t)(int16_t)(w2 >> 16); }
  __device__ __forceinline__ uint32_t qa() const { return w3 & 0xffu; }
  __device__ __forceinline__ uint32_t qb() const { return (w3 >> 8) & 0xffu; }
  __device__ __forceinline__ uint32_t run_len() const { return (w3 >> 16) & kRopRunMask; }
  __device__ __forceinline__ bool has_ctrl() const { return (w3 >> 31) != 0u; }  // kRopHasCtrl
};

__device__ __forceinline__ Op load_op(const RegOp* p) {
  const uint4 a = *reinterpret_cast<const uint4*>(p);
  const uint2 b = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint4*>(p) + 1);
  Op o;
  o.code = a.x;
  o.w1 = a.y;
  o.w2 = a.z;
  o.w3 = a.w;
  o.couter = (uint64_t)b.x | ((uint64_t)b.y << 32);
  return o;
}

// 16-byte aligned pointer into the dynamic shared block, derived from smem_raw by a byte offset
// (not through an integer round trip, which would hide the shared address space from the compiler
// and turn every access through it into a generic LD / ST)
template <typename T>
__device__ __forceinline__ T* smem_align16(unsigned char* smem_raw, const void* after) {
  const size_t off = (size_t)(reinterpret_cast<const unsigned char*>(after) - smem_raw);
  return reinterpret_cast<T*>(smem_raw + ((off + 15) & ~size_t(15)));
}

// ---------------------------------------------------------------- register-resident op kernels

#define SV_CTRL_SKIP(j) \
  if (CTRL && (((j) & cj) != cj)) continue;

template <int NR, int RB, bool CTRL>
__device__ __forceinline__ void reg_m1(double2 (&v)[1 << NR], const double2* m, uint32_t cj) {
  const double2 m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    SV_CTRL_SKIP(j)
    const int j1 = j | (1 << RB);
    const double2 a = v[j], b = v[j1];
    v[j] = cfma(m00, a, cmul(m01, b));
    v[j1] = cfma(m10, a, cmul(m11, b));
  }
}

// Real-structured rotations on register bit RB (no register controls): RX [[c, -is], [-is, c]],
// RY [[c, -s], [s, c]]; 4 FP64 instructions per amplitude.
template <int NR, int RB>
__device__ __forceinline__ void reg_rx(double2 (&v)[1 << NR], const double2* m) {
  const double c = m[0].x, s = -m[1].y;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    const int j1 = j | (1 << RB);
    const double2 a = v[j], b = v[j1];
    v[j] = make_double2(fma(c, a.x, s * b.y), fma(c, a.y, -s * b.x));
    v[j1] = make_double2(fma(c, b.x, s * a.y), fma(c, b.y, -s * a.x));
  }
}
template <int NR, int RB>
__device__ __forceinline__ void reg_ry(double2 (&v)[1 << NR], const double2* m) {
  const double c = m[0].x, s = -m[1].x;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    const int j1 = j | (1 << RB);
    const double2 a = v[j], b = v[j1];
    v[j] = make_double2(fma(c, a.x, -s * b.x), fma(c, a.y, -s * b.y));
    v[j1] = make_double2(fma(s, a.x, c * b.x), fma(s, a.y, c * b.y));
  }
}
// Overlaps of the rotation generators before un-applying (no register controls):
// RX: G = -(i/2) X -> Re<w|G|v> = (1/2) sum_pairs [Im(conj(w0) v1) + Im(conj(w1) v0)];
// RY: G = -(i/2) Y = [[0, -1/2], [1/2, 0]] -> (1/2) sum_pairs [Re(conj(w1) v0) - Re(conj(w0) v1)].
template <int NR, int RB>
__device__ __forceinline__ double reg_ov_rx(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR]) {
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    const int j1 = j | (1 << RB);
    a0 = fma(w[j].x, v[j1].y, fma(-w[j].y, v[j1].x, a0));
    a1 = fma(w[j1].x, v[j].y, fma(-w[j1].y, v[j].x, a1));
  }
  return 0.5 * (a0 + a1);
}
template <int NR, int RB>
__device__ __forceinline__ double reg_ov_ry(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR]) {
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    const int j1 = j | (1 << RB);
    a0 = fma(w[j1].x, v[j].x, fma(w[j1].y, v[j].y, a0));
    a1 = fma(w[j].x, v[j1].x, fma(w[j].y, v[j1].y, a1));
  }
  return 0.5 * (a0 - a1);
}

template <int NR, int RB, bool CTRL>
__device__ __forceinline__ void reg_ax1(double2 (&v)[1 << NR], const double2* m, uint32_t cj) {
  const double2 a = m[0], b = m[1];  // X-like [[0,a],[b,0]]: new0 = a old1, new1 = b old0
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    SV_CTRL_SKIP(j)
    const int j1 = j | (1 << RB);
    const double2 x0 = v[j], x1 = v[j1];
    v[j] = cmul(a, x1);
    v[j1] = cmul(b, x0);
  }
}

// Z-like diag(f0, f1) on register bit RB. dfl bit0: f0 == 1; bit1: f0 == 1 and f1 == -1.
template <int NR, int RB, bool CTRL>
__device__ __forceinline__ void reg_d1(double2 (&v)[1 << NR], const double2* m, uint32_t cj, uint32_t dfl) {
  if (dfl & 2u) {
#pragma unroll
    for (int j = 0; j < (1 << NR); ++j) {
      if (!(j & (1 << RB))) continue;
      SV_CTRL_SKIP(j)
      v[j] = cneg(v[j]);
    }
  } else if (dfl & 1u) {
    const double2 f1 = m[1];
#pragma unroll
    for (int j = 0; j < (1 << NR); ++j) {
      if (!(j & (1 << RB))) continue;
      SV_CTRL_SKIP(j)
      v[j] = cmul(f1, v[j]);
    }
  } else {
    const double2 f0 = m[0], f1 = m[1];
#pragma unroll
    for (int j = 0; j < (1 << NR); ++j) {
      SV_CTRL_SKIP(j)
      v[j] = cmul((j & (1 << RB)) ? f1 : f0, v[j]);
    }
  }
}

// Z-like op whose target is a thread or outer bit tb (uniform over the thread's amplitudes).
template <int NR, bool CTRL>
__device__ __forceinline__ void reg_d1_uniform(double2 (&v)[1 << NR], const double2* m, uint32_t cj, uint32_t dfl,
                                               uint32_t tb) {
  if ((dfl & 1u) && !tb) return;
  if (dfl & 2u) {
#pragma unroll
    for (int j = 0; j < (1 << NR); ++j) {
      SV_CTRL_SKIP(j)
      v[j] = cneg(v[j]);
    }
    return;
  }
  const double2 f = tb ? m[1] : m[0];
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    SV_CTRL_SKIP(j)
    v[j] = cmul(f, v[j]);
  }
}

template <int NR, int RA, int RB, bool CTRL>
__device__ __forceinline__ void reg_m2(double2 (&v)[1 << NR], const double2* m, uint32_t cj) {
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & ((1 << RA) | (1 << RB))) continue;
    SV_CTRL_SKIP(j)
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

template <int NR, int RA, int RB, bool CTRL>
__device__ __forceinline__ void reg_swap(double2 (&v)[1 << NR], uint32_t cj) {
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & ((1 << RA) | (1 << RB))) continue;
    SV_CTRL_SKIP(j)
    const int a = j | (1 << RA), b = j | (1 << RB);
    const double2 t = v[a];
    v[a] = v[b];
    v[b] = t;
  }
}

// Same with an anti-diagonal G (the generators of RX, RY: -i/2 X, -i/2 Y): half the products.
template <int NR, int RB, bool CTRL>
__device__ __forceinline__ double reg_ov1_anti(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR],
                                               const double2* g, uint32_t cj) {
  const double2 g01 = g[1], g10 = g[2];
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    SV_CTRL_SKIP(j)
    const int j1 = j | (1 << RB);
    acc0 += re_conj_mul(w[j], cmul(g01, v[j1]));
    acc1 += re_conj_mul(w[j1], cmul(g10, v[j]));
  }
  return acc0 + acc1;
}

// Re <w| (Pi_C (x) G) |v> over this thread's amplitudes, G on register bit RB (2x2).
template <int NR, int RB, bool CTRL>
__device__ __forceinline__ double reg_ov1(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], const double2* g,
                                          uint32_t cj) {
  const double2 g00 = g[0], g01 = g[1], g10 = g[2], g11 = g[3];
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & (1 << RB)) continue;
    SV_CTRL_SKIP(j)
    const int j1 = j | (1 << RB);
    acc0 += re_conj_mul(w[j], cfma(g00, v[j], cmul(g01, v[j1])));
    acc1 += re_conj_mul(w[j1], cfma(g10, v[j], cmul(g11, v[j1])));
  }
  return acc0 + acc1;
}

template <int NR, int RA, int RB, bool CTRL>
__device__ __forceinline__ double reg_ov2(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], const double2* g,
                                          uint32_t cj) {
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    if (j & ((1 << RA) | (1 << RB))) continue;
    SV_CTRL_SKIP(j)
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

// ---- runtime register index -> compile-time template dispatch ----
#define SV_DISP1(NR, r, CALL)                          \
  switch (r) {                                         \
    case 0: CALL(0); break;                            \
    case 1: CALL(1); break;                            \
    case 2: CALL(2); break;                            \
    default: if constexpr (NR > 3) { CALL(3); } break; \
  }
#define SV_DISP2(NR, ra, rb, CALL)                       \
  switch ((ra) * 4 + (rb)) {                             \
    case 1: CALL(0, 1); break;                           \
    case 2: CALL(0, 2); break;                           \
    case 6: CALL(1, 2); break;                           \
    case 3: if constexpr (NR > 3) { CALL(0, 3); } break; \
    case 7: if constexpr (NR > 3) { CALL(1, 3); } break; \
    default: if constexpr (NR > 3) { CALL(2, 3); } break; \
  }

template <int NR, bool CTRL>
__device__ __forceinline__ void reg_apply_c(double2 (&v)[1 << NR], const Op& o, const double2* m, uint32_t tthr,
                                            uint64_t base) {
  const uint32_t cj = o.cj();
  switch (o.type()) {
    case OP_M1: {
#define C1(R) reg_m1<NR, R, CTRL>(v, m, cj)
      SV_DISP1(NR, o.ra(), C1)
#undef C1
      break;
    }
    case OP_AX1: {
#define C1(R) reg_ax1<NR, R, CTRL>(v, m, cj)
      SV_DISP1(NR, o.ra(), C1)
#undef C1
      break;
    }
    case OP_RX: {
#define C1(R) reg_rx<NR, R>(v, m)
      SV_DISP1(NR, o.ra(), C1)
#undef C1
      break;
    }
    case OP_RY: {
#define C1(R) reg_ry<NR, R>(v, m)
      SV_DISP1(NR, o.ra(), C1)
#undef C1
      break;
    }
    case OP_M2: {
#define C2(A, B) reg_m2<NR, A, B, CTRL>(v, m, cj)
      SV_DISP2(NR, o.ra(), o.rb(), C2)
#undef C2
      break;
    }
    case OP_SWAP: {
#define C2(A, B) reg_swap<NR, A, B, CTRL>(v, cj)
      SV_DISP2(NR, o.ra(), o.rb(), C2)
#undef C2
      break;
    }
    case OP_D1: {
      if (o.ra() != 15u) {
#define C1(R) reg_d1<NR, R, CTRL>(v, m, cj, o.dfl())
        SV_DISP1(NR, o.ra(), C1)
#undef C1
      } else {
        const uint32_t tb = o.pa() != 31u ? (tthr >> o.pa()) & 1u : (uint32_t)((base >> o.qa()) & 1ull);
        reg_d1_uniform<NR, CTRL>(v, m, cj, o.dfl(), tb);
      }
      break;
    }
    case OP_D2: {
      const uint32_t ta = o.pa() != 31u ? (tthr >> o.pa()) & 1u : (uint32_t)((base >> o.qa()) & 1ull);
      const uint32_t tb = o.pb() != 31u ? (tthr >> o.pb()) & 1u : (uint32_t)((base >> o.qb()) & 1ull);
#pragma unroll
      for (int j = 0; j < (1 << NR); ++j) {
        SV_CTRL_SKIP(j)
        const uint32_t b0 = o.ra() != 15u ? ((uint32_t)j >> o.ra()) & 1u : ta;
        const uint32_t b1 = o.rb() != 15u ? ((uint32_t)j >> o.rb()) & 1u : tb;
        v[j] = cmul(lds(m + (b0 | (b1 << 1))), v[j]);
      }
      break;
    }
  }
}

template <int NR>
__device__ __forceinline__ void reg_apply(double2 (&v)[1 << NR], const Op& o, const double2* m, uint32_t tthr,
                                          uint64_t base) {
#if SV_FWD_CTRL_SPLIT
  if (o.cj()) reg_apply_c<NR, true>(v, o, m, tthr, base);
  else reg_apply_c<NR, false>(v, o, m, tthr, base);
#else
  reg_apply_c<NR, true>(v, o, m, tthr, base);  // one instantiation (cj = 0 never skips)
#endif
}

template <int NR, bool CTRL>
__device__ __forceinline__ double reg_overlap_c(const double2 (&v)[1 << NR], const double2 (&w)[1 << NR], const Op& o,
                                                const double2* g, uint32_t tthr, uint64_t base) {
  const uint32_t cj = o.cj();
  if (o.gdiag()) {
    // Re <w|G|v> with G diagonal: sum_j Re(g_{idx(j)} conj(w_j) v_j); the entries are read once
    // from shared memory and selected per amplitude (no per-element indexed loads)
    const uint32_t ta = o.pa() != 31u ? (tthr >> o.pa()) & 1u : (uint32_t)((base >> o.qa()) & 1ull);
    const uint32_t tb = o.pb() != 31u ? (tthr >> o.pb()) & 1u : (uint32_t)((base >> o.qb()) & 1ull);
    const double2 g0 = lds(g), g1 = lds(g + 1);
    const bool two = o.gen() == 2u;
    const double2 g2 = two ? lds(g + 2) : g0, g3 = two ? lds(g + 3) : g1;
    const uint32_t ra = o.ra(), rb = o.rb();
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < (1 << NR); ++j) {
      SV_CTRL_SKIP(j)
      const uint32_t b0 = ra != 15u ? ((uint32_t)j >> ra) & 1u : ta;
      const uint32_t b1 = two ? (rb != 15u ? ((uint32_t)j >> rb) & 1u : tb) : 0u;
      const double2 gs = b1 ? (b0 ? g3 : g2) : (b0 ? g1 : g0);
      const double2 p = make_double2(fma(w[j].x, v[j].x, w[j].y * v[j].y), fma(w[j].x, v[j].y, -w[j].y * v[j].x));
      acc += fma(gs.x, p.x, -gs.y * p.y);  // Re(gs * conj(w) v)
    }
    return acc;
  }
  double r = 0.0;
  if (o.gen() == 1u) {
#define C1(R) r = reg_ov1<NR, R, CTRL>(v, w, g, cj)
    SV_DISP1(NR, o.ra(), C1)
#undef C1
  } else {
#define C2(A, B) r = reg_ov2<NR, A, B, CTRL>(v, w, g, cj)
    SV_DISP2(NR, o.ra(), o.rb(), C2)
#undef C2
  }
  return r;
}


// DUAL diagonal op (Z-like, 1 or 2 targets) with compile-time target positions: RA / RB in
// [0, NR) are register bits, -1 a thread / outer bit whose value (ta / tb) is uniform over the
// thread's amplitudes (the entries are pre-selected once per op), -2 "no second target". Returns
// this thread's Re<w|(Pi_C (x) G)|v> (diagonal generator) before un-applying the op to v and w.
template <int NR, int RA, int RB, bool CTRL>
__device__ __forceinline__ double dual_diag(double2 (&v)[1 << NR], double2 (&w)[1 << NR], const double2* m,
                                            const double2* g, bool gen, bool g2, uint32_t cj, uint32_t ta,
                                            uint32_t tb, bool ok) {
  constexpr bool TWO = RB != -2;
  double2 d[4], q[4];
  d[0] = lds(m);
  d[1] = lds(m + 1);
  if (TWO) {
    d[2] = lds(m + 2);
    d[3] = lds(m + 3);
  }
  if (gen) {
    q[0] = lds(g);
    q[1] = lds(g + 1);
    q[2] = g2 ? lds(g + 2) : q[0];
    q[3] = g2 ? lds(g + 3) : q[1];
  } else {
    q[0] = q[1] = q[2] = q[3] = make_double2(0.0, 0.0);
  }
  if (!TWO) {
    d[2] = d[0];
    d[3] = d[1];
  }
  // uniform target bits: fold them into the entry index once
  if (RA == -1) {
    d[0] = ta ? d[1] : d[0];
    d[2] = ta ? d[3] : d[2];
    q[0] = ta ? q[1] : q[0];
    q[2] = ta ? q[3] : q[2];
  }
  if (RB == -1) {
    d[0] = tb ? d[2] : d[0];
    d[1] = tb ? d[3] : d[1];
    q[0] = tb ? q[2] : q[0];
    q[1] = tb ? q[3] : q[1];
  }
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // four independent chains (FP64 latency, few warps)
  if (!ok) return 0.0;
#pragma unroll
  for (int j = 0; j < (1 << NR); ++j) {
    SV_CTRL_SKIP(j)
    const int i0 = RA >= 0 ? ((j >> RA) & 1) : 0;
    const int i1 = RB >= 0 ? ((j >> RB) & 1) : 0;
    const int idx = i0 | (i1 << 1);
    if (gen) {
      const double2 p = make_double2(fma(w[j].x, v[j].x, w[j].y * v[j].y), fma(w[j].x, v[j].y, -w[j].y * v[j].x));
      acc[j & 3] = fma(q[idx].x, p.x, fma(-q[idx].y, p.y, acc[j & 3]));  // Re(g conj(w) v)
    }
    v[j] = cmul(d[idx], v[j]);
    w[j] = cmul(d[idx], w[j]);
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// DUAL (adjoint) op with ONE register-position dispatch: the overlap Re<w|(Pi_C (x) G)|v> of a
// parametrised op (before it is un-applied) and the un-application to v and w happen inside the same
// case, so the compiler keeps one register assignment for v and w per op instead of reshuffling
// both arrays at three separate switch joins.
template <int NR, bool CTRL>
__device__ __forceinline__ double dual_op_c(double2 (&v)[1 << NR], double2 (&w)[1 << NR], const Op& o, const double2* m,
                                            const double2* g, uint32_t tthr, uint64_t base, bool ok) {
  const uint32_t cj = o.cj();
  double part = 0.0;
  const bool gen = o.gen() != 0u;
  switch (o.type()) {
    case OP_M1: {
      bool anti = false;
      if (gen) {
        const double2 g00 = lds(g), g11 = lds(g + 3);
        anti = g00.x == 0.0 && g00.y == 0.0 && g11.x == 0.0 && g11.y == 0.0;
      }
#define C1(R)                                                   \
  {                                                             \
    if (gen && ok) part = anti ? reg_ov1_anti<NR, R, CTRL>(v, w, g, cj) : reg_ov1<NR, R, CTRL>(v, w, g, cj); \
    if (ok) {                                                   \
      reg_m1<NR, R, CTRL>(v, m, cj);                            \
      reg_m1<NR, R, CTRL>(w, m, cj);                            \
    }                                                           \
  }
      SV_DISP1(NR, o.ra(), C1)
#undef C1
      break;
    }
    case OP_RX: {
#define C1(R)                                       \
  {                                                 \
    if (ok) {                                       \
      if (gen) part = reg_ov_rx<NR, R>(v, w);       \
      reg_rx<NR, R>(v, m);                          \
      reg_rx<NR, R>(w, m);                          \
    }                                               \
  }
      SV_DISP1(NR, o.ra(), C1)
#undef C1
      break;
    }
    case OP_RY: {
#define C1(R)                                       \
  {                                                 \
    if (ok) {                                       \
      if (gen) part = reg_ov_ry<NR, R>(v, w);       \
      reg_ry<NR, R>(v, m);                          \
      reg_ry<NR, R>(w, m);                          \
    }                                               \
  }
      SV_DISP1(NR, o.ra(), C1)
#undef C1
      break;
    }
    case OP_M2: {
#define C2(A, B)                                                   \
  {                                                                \
    if (gen && ok) part = reg_ov2<NR, A, B, CTRL>(v, w, g, cj);    \
    if (ok) {                                                      \
      reg_m2<NR, A, B, CTRL>(v, m, cj);                            \
      reg_m2<NR, A, B, CTRL>(w, m, cj);                            \
    }                                                              \
  }
      SV_DISP2(NR, o.ra(), o.rb(), C2)
#undef C2
      break;
    }
    case OP_D1: {
      const uint32_t ta = o.pa() != 31u ? (tthr >> o.pa()) & 1u : (uint32_t)((base >> o.qa()) & 1ull);
      const bool g2 = o.gen() == 2u;
      switch (o.ra()) {
        case 0: part = dual_diag<NR, 0, -2, CTRL>(v, w, m, g, gen, g2, cj, ta, 0, ok); break;
        case 1: part = dual_diag<NR, 1, -2, CTRL>(v, w, m, g, gen, g2, cj, ta, 0, ok); break;
        case 2: part = dual_diag<NR, 2, -2, CTRL>(v, w, m, g, gen, g2, cj, ta, 0, ok); break;
        default: part = dual_diag<NR, -1, -2, CTRL>(v, w, m, g, gen, g2, cj, ta, 0, ok); break;
      }
      break;
    }
    case OP_D2: {
      const uint32_t ta = o.pa() != 31u ? (tthr >> o.pa()) & 1u : (uint32_t)((base >> o.qa()) & 1ull);
      const uint32_t tb = o.pb() != 31u ? (tthr >> o.pb()) & 1u : (uint32_t)((base >> o.qb()) & 1ull);
      const bool g2 = o.gen() == 2u;
      const uint32_t ra = o.ra() > 2u ? 3u : o.ra(), rb = o.rb() > 2u ? 3u : o.rb();
#define CD(A, B) part = dual_diag<NR, A, B, CTRL>(v, w, m, g, gen, g2, cj, ta, tb, ok)
      switch (ra * 4 + rb) {
        case 1: CD(0, 1); break;
        case 2: CD(0, 2); break;
        case 3: CD(0, -1); break;
        case 4: CD(1, 0); break;
        case 6: CD(1, 2); break;
        case 7: CD(1, -1); break;
        case 8: CD(2, 0); break;
        case 9: CD(2, 1); break;
        case 11: CD(2, -1); break;
        case 12: CD(-1, 0); break;
        case 13: CD(-1, 1); break;
        case 14: CD(-1, 2); break;
        default: CD(-1, -1); break;
      }
#undef CD
      break;
    }
    default: {
      if (gen && ok) part = reg_overlap_c<NR, CTRL>(v, w, o, g, tthr, base);
      if (ok) {
        reg_apply_c<NR, CTRL>(v, o, m, tthr, base);
        reg_apply_c<NR, CTRL>(w, o, m, tthr, base);
      }
    }
  }
  return part;
}

// ---------------------------------------------------------------- diagonal runs (DUAL)
//
// A run of consecutive diagonal ops (Z-like / two-qubit diagonal, no register controls) in an
// adjoint stage. For diagonal U, conj(U^+ lam)_e (U^+ psi)_e = conj(lam_e) psi_e, so every op of the
// run sees the same p_e = conj(lam_e) psi_e, and its overlap Re<lam|Pi_C G|psi> (G = i diag(gq),
// purely imaginary for RZ / RZZ / PS) is -sum_e gq(e) Im(p_e) over control-satisfied e. The run's
// un-application is one phase per amplitude: the product of the ops' entries, accumulated per thread
// in factor tables over the 3 register bits (U: ops on thread / outer bits only; A[r][b]: one
// register target r; B[pair][b_r + 2 b_s]: two register targets) and applied once to psi and lambda.
// psi and lambda are parked in their tile slots meanwhile (their registers carry the tables).
struct DiagTables {
  double2 U;
  double2 A[3][2];
  double2 B[3][4];  // pairs (0,1), (0,2), (1,2)
};

__device__ __forceinline__ void tab_one(double2& t) { t = make_double2(1.0, 0.0); }

// Sum over j of Im(p_j) with bit R of j equal to b (R compile-time)
template <int R>
__device__ __forceinline__ void half_sums(const double (&P)[8], double& s0, double& s1) {
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if ((j >> R) & 1) b += P[j];
    else a += P[j];
  }
  s0 = a;
  s1 = b;
}
// Quarter sums by (bit RA, bit RB) -> index bit_RA + 2 bit_RB
template <int RA, int RB>
__device__ __forceinline__ void quarter_sums(const double (&P)[8], double (&s)[4]) {
  s[0] = s[1] = s[2] = s[3] = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s[((j >> RA) & 1) | (((j >> RB) & 1) << 1)] += P[j];
}

// one op of a run: entries d[] (un-apply), generator imaginary parts gq[] (zero without gen)
template <int RA, int RB>  // register positions; -1: uniform (value ta / tb); RB = -2: one target
__device__ __forceinline__ double diag_run_op(DiagTables& T, const double (&P)[8], double Ptot, const double2* m,
                                              const double2* g, bool gen, uint32_t ta, uint32_t tb) {
  constexpr bool TWO = RB != -2;
  double2 d[4];
  double gq[4];
#pragma unroll
  for (int q = 0; q < (TWO ? 4 : 2); ++q) {
    d[q] = lds(m + q);
    gq[q] = gen ? lds(g + q).y : 0.0;
  }
  if constexpr (!TWO) {  // one target
    if constexpr (RA < 0) {
      T.U = cmul(T.U, d[ta]);
      return -gq[ta] * Ptot;
    } else {
      T.A[RA][0] = cmul(T.A[RA][0], d[0]);
      T.A[RA][1] = cmul(T.A[RA][1], d[1]);
      if (!gen) return 0.0;
      double s0, s1;
      half_sums<RA>(P, s0, s1);
      return -(gq[0] * s0 + gq[1] * s1);
    }
  } else if constexpr (RA < 0 && RB < 0) {  // two targets, both uniform
    T.U = cmul(T.U, d[ta | (tb << 1)]);
    return -gq[ta | (tb << 1)] * Ptot;
  } else if constexpr (RA < 0 || RB < 0) {  // one register target R, the other uniform (value u)
    constexpr int R = RA < 0 ? RB : RA;
    const uint32_t u = RA < 0 ? ta : tb;
    // entries with bit_R = 0 / 1 (index bit 0 <-> target a, bit 1 <-> target b)
    const int j0 = RA < 0 ? (int)u : (int)(u << 1), j1 = RA < 0 ? (int)u | 2 : (int)(u << 1) | 1;
    T.A[R][0] = cmul(T.A[R][0], d[j0]);
    T.A[R][1] = cmul(T.A[R][1], d[j1]);
    if (!gen) return 0.0;
    double s0, s1;
    half_sums<R>(P, s0, s1);
    return -(gq[j0] * s0 + gq[j1] * s1);
  } else {  // two register targets: table index b_LO + 2 b_HI, entry index b_RA + 2 b_RB
    constexpr int LO = RA < RB ? RA : RB, HI = RA < RB ? RB : RA;
    constexpr int PAIR = (LO == 0 && HI == 1) ? 0 : ((LO == 0) ? 1 : 2);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int blo = q & 1, bhi = q >> 1;
      const int e = RA < RB ? (blo | (bhi << 1)) : (bhi | (blo << 1));
      T.B[PAIR][q] = cmul(T.B[PAIR][q], d[e]);
    }
    if (!gen) return 0.0;
    double s[4];
    quarter_sums<RA, RB>(P, s);
    return -(gq[0] * s[0] + gq[1] * s[1] + gq[2] * s[2] + gq[3] * s[3]);
  }
}

// The run [ops, ops + len) of a DUAL stage on this thread's amplitudes v (psi), w (lambda); slots
// A ^ SR[...] hold them in the tile. Overlaps accumulate like single ops (per thread or per warp).
__device__ __forceinline__ void dual_diag_run(double2 (&v)[8], double2 (&w)[8], const RegOp* ops, int len,
                                              const double2* mats2, uint32_t tthr, uint64_t base, double2* tp,
                                              double2* tl, uint32_t A, const uint32_t (&SR)[3], double* s_acc,
                                              int nthr, int tid, int nwarps, int warp, int lane, bool acc_thread) {
  double P[8];
  double Ptot = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    P[j] = fma(w[j].x, v[j].y, -w[j].y * v[j].x);  // Im(conj(lambda) psi)
    Ptot += P[j];
  }
  uint32_t ad[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    ad[j] = A ^ ((j & 1) ? SR[0] : 0u) ^ ((j & 2) ? SR[1] : 0u) ^ ((j & 4) ? SR[2] : 0u);
    tp[ad[j]] = v[j];  // parked: their registers carry the tables during the run
    tl[ad[j]] = w[j];
  }
  DiagTables T;
  tab_one(T.U);
#pragma unroll
  for (int r = 0; r < 3; ++r) { tab_one(T.A[r][0]); tab_one(T.A[r][1]); }
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) tab_one(T.B[p][q]);
  for (int k = 0; k < len; ++k) {
    const Op o = load_op(ops + k);
    const bool ok = !o.has_ctrl() || (((base & o.couter) == o.couter) && ((tthr & o.cthr()) == o.cthr()));
    const bool gen = o.gen() != 0u;
    double part = 0.0;
    if (ok) {
      const uint32_t ta = o.pa() != 31u ? (tthr >> o.pa()) & 1u : (uint32_t)((base >> o.qa()) & 1ull);
      const uint32_t tb = o.pb() != 31u ? (tthr >> o.pb()) & 1u : (uint32_t)((base >> o.qb()) & 1ull);
      const double2* m = mats2 + o.mat_off();
      const double2* g = mats2 + o.gen_off();
      if (o.type() == OP_D1) {
        switch (o.ra()) {
          case 0: part = diag_run_op<0, -2>(T, P, Ptot, m, g, gen, ta, tb); break;
          case 1: part = diag_run_op<1, -2>(T, P, Ptot, m, g, gen, ta, tb); break;
          case 2: part = diag_run_op<2, -2>(T, P, Ptot, m, g, gen, ta, tb); break;
          default: part = diag_run_op<-1, -2>(T, P, Ptot, m, g, gen, ta, tb); break;
        }
      } else {
        const uint32_t ra = o.ra() > 2u ? 3u : o.ra(), rb = o.rb() > 2u ? 3u : o.rb();
#define CR(X, Y) part = diag_run_op<X, Y>(T, P, Ptot, m, g, gen, ta, tb)
        switch (ra * 4 + rb) {
          case 1: CR(0, 1); break;
          case 2: CR(0, 2); break;
          case 3: CR(0, -1); break;
          case 4: CR(1, 0); break;
          case 6: CR(1, 2); break;
          case 7: CR(1, -1); break;
          case 8: CR(2, 0); break;
          case 9: CR(2, 1); break;
          case 11: CR(2, -1); break;
          case 12: CR(-1, 0); break;
          case 13: CR(-1, 1); break;
          case 14: CR(-1, 2); break;
          default: CR(-1, -1); break;
        }
#undef CR
      }
    }
    if (gen) {
      if (acc_thread) {
        s_acc[o.grad_local() * nthr + tid] += part;
      } else {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
        if (lane == 0) s_acc[o.grad_local() * nwarps + warp] += part;
      }
    }
  }
  // phase of amplitude j = U A0[b0] A1[b1] A2[b2] B01[b0 + 2 b1] B02[b0 + 2 b2] B12[b1 + 2 b2], built bit by bit
  double2 q1[2], q2[4];
#pragma unroll
  for (int b0 = 0; b0 < 2; ++b0) q1[b0] = cmul(T.U, T.A[0][b0]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int b0 = i & 1, b1 = i >> 1;
    q2[i] = cmul(cmul(q1[b0], T.A[1][b1]), T.B[0][b0 | (b1 << 1)]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int b0 = j & 1, b1 = (j >> 1) & 1, b2 = j >> 2;
    const double2 ph = cmul(cmul(cmul(q2[j & 3], T.A[2][b2]), T.B[1][b0 | (b2 << 1)]), T.B[2][b1 | (b2 << 1)]);
    v[j] = cmul(ph, tp[ad[j]]);
    w[j] = cmul(ph, tl[ad[j]]);
  }
}

// ---------------------------------------------------------------- dense FP64-MMA stage
//
// The stage's ops were folded on the host into a 16x16 complex matrix U per variant, applied to the
// tile's 2^(k-4) vectors of 16 amplitudes X as mma.sync m8n8k4 f64 (DMMA) fragments with three
// real products instead of four (Gauss): with T = Ur (Xr + Xi),
//   Re Y = T + Cb Xi,  Cb = -(Ur + Ui),      Im Y = T + Cc Xr,  Cc = Ui - Ur,
// so 48 DMMAs per warp and stage instead of 64, one DADD per input element (Xr + Xi) and two per
// A entry (Cb, Cc: computed here; stored by the host after U, the extra A loads cost more than the
// DADDs), and T seeds both chains as the C operand of their first MMA (no output additions).
// Per warp 2 N-tiles of 8 vectors, 2 M-halves x 4 K-steps; both N-tiles advance together (4 T
// chains, then 8 Re / Im chains in flight). Fragment layouts (PTX m8n8k4 .f64):
// A[r = lane/4][c = lane%4], B[k = lane%4][n = lane/4], D[r = lane/4][c = 2 (lane%4) + {0,1}].
constexpr uint32_t kDenseRow = 16;  // double2 per stored variant-matrix row (plan.cpp kDenseStride)
constexpr uint32_t kDenseVar = 16u * kDenseRow;  // double2 per variant matrix

#if SV_DMMA_VOLATILE
#define SV_ASM_MMA asm volatile
#else
#define SV_ASM_MMA asm
#endif
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  SV_ASM_MMA("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// D = A B + C with C and D distinct registers (T seeds the Re and Im chains)
__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b, double c0, double c1) {
  SV_ASM_MMA("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// A operand of a dense stage for this lane: 8 entries (rows 8 mh + lane/4, columns 4 kh + lane%4)
// of the warp's variant matrix U (global, L2-resident)
struct DenseA {
  double2 u[2][4];
};

__device__ __forceinline__ void dense_load_u(const double2* __restrict__ U, int lane, DenseA& A) {
#pragma unroll
  for (int mh = 0; mh < 2; ++mh)
#pragma unroll
    for (int kh = 0; kh < 4; ++kh) {
      A.u[mh][kh] = __ldg(U + (8 * mh + (lane >> 2)) * kDenseRow + 4 * kh + (lane & 3));
    }
}

__device__ __forceinline__ void dense_load_a(const StageDesc& S, const double2* __restrict__ gmats2, uint64_t base,
                                             int warp, int lane, DenseA& A) {
  uint32_t var = S.warp_var[warp];
  for (int b = 0; b < S.m_outer; ++b) var |= (uint32_t)((base >> S.var_outer[b]) & 1ull) << (S.m_tile + b);
  dense_load_u(gmats2 + S.dense_off + var * kDenseVar, lane, A);
}

// 32-bit shared-window accesses: the swizzled offsets are XOR-linear in (nt, kq) and (nt, mh, v),
// so the 8 load and 8 store offsets are XORs of three basis values each (one LOP3 + one LEA per
// access)
__device__ __forceinline__ double2 lds_v2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double x) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(x) : "memory");
}

// Gauss coefficients of the A entries (two DADDs each)
struct DenseC {
  double cb[2][4], cc[2][4];
};
__device__ __forceinline__ void dense_coef(const DenseA& A, DenseC& C) {
#pragma unroll
  for (int mh = 0; mh < 2; ++mh)
#pragma unroll
    for (int kh = 0; kh < 4; ++kh) {
      C.cb[mh][kh] = -(A.u[mh][kh].x + A.u[mh][kh].y);
      C.cc[mh][kh] = A.u[mh][kh].y - A.u[mh][kh].x;
    }
}

// PRE: the coefficients come precomputed in *Cp (one set for the psi and lambda tiles of an adjoint
// dense stage); otherwise they are computed after the T chains are issued (measured faster than
// before them in the forward kernel)
// A dense stage's shared-memory offsets for this lane (swizzled slot indices, XOR-linear): B-load
// base and basis (kq bit 0, kq bit 1, nt), D-store base and basis (v, mh, nt)
struct DenseOff {
  uint32_t bB, Lk0, Lk1, Ln, bD, Sv, Sm, Sn;
};
__device__ __forceinline__ DenseOff dense_off(const StageDesc& S, int warp, int lane) {
  DenseOff o;
  const uint32_t wsw = S.warp_swz[warp];
  o.bB = wsw ^ (uint32_t)S.lane_b[lane];
  o.bD = wsw ^ (uint32_t)S.lane_d[lane];
  o.Lk0 = S.swz_reg[1];
  o.Lk1 = S.swz_reg[2];
  o.Ln = S.swz_reg[4];
  o.Sv = S.swz_reg[8 + 1];
  o.Sm = S.swz_reg[8 + 2];
  o.Sn = S.swz_reg[8 + 4];
  return o;
}

// tile element access on a 32-bit shared address: complex128 slots (16 bytes) or complex64 slots
// (8 bytes, widened to FP64 for the MMAs and rounded back on the store)
__device__ __forceinline__ double2 tile_lds(const double2*, uint32_t sb, uint32_t o) { return lds_v2(sb + (o << 4)); }
__device__ __forceinline__ double2 tile_lds(const float2*, uint32_t sb, uint32_t o) {
  float x, y;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];\n" : "=f"(x), "=f"(y) : "r"(sb + (o << 3)) : "memory");
  return make_double2((double)x, (double)y);
}
__device__ __forceinline__ void tile_sts(double2*, uint32_t sb, uint32_t o, double re, double im) {
  const uint32_t a = sb + (o << 4);
  sts_f64(a, re);
  sts_f64(a + 8, im);  // (ptxas fuses the halves into one 16-byte store)
}
__device__ __forceinline__ void tile_sts(float2*, uint32_t sb, uint32_t o, double re, double im) {
  asm volatile("st.shared.v2.f32 [%0], {%1,%2};\n" ::"r"(sb + (o << 3)), "f"((float)re), "f"((float)im) : "memory");
}

template <bool PRE = false, typename T>
__device__ __forceinline__ void dense_apply_o(T* tp, const DenseOff& O, const DenseA& A, const DenseC* Cp = nullptr) {
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(tp);
  double xr[2][4], xi[2][4];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      const double2 x = tile_lds(tp, sb, O.bB ^ (nt ? O.Ln : 0u) ^ ((kq & 1) ? O.Lk0 : 0u) ^ ((kq & 2) ? O.Lk1 : 0u));
      xr[nt][kq] = x.x;
      xi[nt][kq] = x.y;
    }
  double t[2][2][2];
#pragma unroll
  for (int kh = 0; kh < 4; ++kh)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const double sx = xr[nt][kh] + xi[nt][kh];
#pragma unroll
      for (int mh = 0; mh < 2; ++mh) {
        if (kh == 0) t[nt][mh][0] = t[nt][mh][1] = 0.0;
        dmma(t[nt][mh][0], t[nt][mh][1], A.u[mh][kh].x, sx);
      }
    }
  DenseC Cl;
  if (!PRE) dense_coef(A, Cl);
  const DenseC& C = PRE ? *Cp : Cl;
  double re[2][2][2], im[2][2][2];
#pragma unroll
  for (int kh = 0; kh < 4; ++kh)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int mh = 0; mh < 2; ++mh) {
        if (kh == 0) {
          dmma_c(re[nt][mh][0], re[nt][mh][1], C.cb[mh][0], xi[nt][0], t[nt][mh][0], t[nt][mh][1]);
          dmma_c(im[nt][mh][0], im[nt][mh][1], C.cc[mh][0], xr[nt][0], t[nt][mh][0], t[nt][mh][1]);
        } else {
          dmma(re[nt][mh][0], re[nt][mh][1], C.cb[mh][kh], xi[nt][kh]);
          dmma(im[nt][mh][0], im[nt][mh][1], C.cc[mh][kh], xr[nt][kh]);
        }
      }
  // stores: amps 8 mh + lane/4 of columns 2 (lane%4) + v
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int mh = 0; mh < 2; ++mh)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        tile_sts(tp, sb, O.bD ^ (nt ? O.Sn : 0u) ^ (mh ? O.Sm : 0u) ^ (v ? O.Sv : 0u), re[nt][mh][v], im[nt][mh][v]);
}

template <bool PRE = false>
__device__ __forceinline__ void dense_apply(double2* tp, const StageDesc& S, const DenseA& A, int warp, int lane,
                                            const DenseC* Cp = nullptr) {
  dense_apply_o<PRE>(tp, dense_off(S, warp, lane), A, Cp);
}

__device__ __forceinline__ void dense_stage(double2* tp, const StageDesc& S, const double2* __restrict__ gmats2,
                                            uint64_t base, int warp, int lane) {
  DenseA A;
  dense_load_a(S, gmats2, base, warp, lane, A);
  dense_apply(tp, S, A, warp, lane);
}

// complex64 tiles (NEXT-3): widened to FP64 in registers
__device__ __forceinline__ double2 tile_ld(const float2& v) { return make_double2((double)v.x, (double)v.y); }
__device__ __forceinline__ void tile_st(float2& d, double2 v) { d = make_float2((float)v.x, (float)v.y); }

// Adjoint dense stage (DUAL): accumulate R = sum_v psi_v lambda_v^H over the warp's 16 vectors at
// the stage start (FP64 MMAs with K = vectors) into the warp's private shared-memory accumulator,
// then un-apply the stage (dense U) to psi and lambda. The overlaps of the stage's parametrised
// ops follow on the host as tr(B_j R).
__device__ __forceinline__ void da_stage(double2* tp, double2* tl, const StageDesc& S, const double2* __restrict__ gmats2,
                                         uint64_t base, int warp, int lane, double* racc) {
#if SV_DA_SHARED_A
  DenseA A;  // one A operand for the psi and lambda applications, loaded before R (L2 latency hidden)
  dense_load_a(S, gmats2, base, warp, lane, A);
#endif
  const uint32_t wsw = S.warp_swz[warp];
  const uint32_t br = wsw ^ S.lane_r[lane];
  // fragments: A = Psi[a = 8 mt + lane/4][v = 4 kt + lane%4], B = Lambda[b = 8 nt + lane/4][v]
  double2 ps[2][4], la[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const uint32_t ad = br ^ S.off_r[mt * 4 + kt];
      ps[mt][kt] = tp[ad];
      la[mt][kt] = tl[ad];
    }
  double rre[2][2][2], rim[2][2][2];
#if SV_DA_R_3M
  // Re R = Pr Lr^T + Pi Li^T, Im R = Pi Lr^T - Pr Li^T with three products (Gauss):
  // T = (Pr + Pi) Lr^T, Re R = T - Pi (Lr - Li)^T, Im R = T - Pr (Lr + Li)^T
  double t[2][2][2];
#pragma unroll
  for (int kt = 0; kt < 4; ++kt)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const double sp = ps[mt][kt].x + ps[mt][kt].y;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        if (kt == 0) t[mt][nt][0] = t[mt][nt][1] = 0.0;
        dmma(t[mt][nt][0], t[mt][nt][1], sp, la[nt][kt].x);
      }
    }
#pragma unroll
  for (int kt = 0; kt < 4; ++kt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const double lm = la[nt][kt].x - la[nt][kt].y, lp = la[nt][kt].x + la[nt][kt].y;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        if (kt == 0) {
          dmma_c(rre[mt][nt][0], rre[mt][nt][1], -ps[mt][kt].y, lm, t[mt][nt][0], t[mt][nt][1]);
          dmma_c(rim[mt][nt][0], rim[mt][nt][1], -ps[mt][kt].x, lp, t[mt][nt][0], t[mt][nt][1]);
        } else {
          dmma(rre[mt][nt][0], rre[mt][nt][1], -ps[mt][kt].y, lm);
          dmma(rim[mt][nt][0], rim[mt][nt][1], -ps[mt][kt].x, lp);
        }
      }
    }
#else
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) rre[mt][nt][0] = rre[mt][nt][1] = rim[mt][nt][0] = rim[mt][nt][1] = 0.0;
#pragma unroll
  for (int kt = 0; kt < 4; ++kt)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        // Re R = Pr Lr^T + Pi Li^T ; Im R = Pi Lr^T - Pr Li^T
        dmma(rre[mt][nt][0], rre[mt][nt][1], ps[mt][kt].x, la[nt][kt].x);
        dmma(rim[mt][nt][0], rim[mt][nt][1], ps[mt][kt].y, la[nt][kt].x);
        dmma(rre[mt][nt][0], rre[mt][nt][1], ps[mt][kt].y, la[nt][kt].y);
        dmma(rim[mt][nt][0], rim[mt][nt][1], -ps[mt][kt].x, la[nt][kt].y);
      }
#endif
  // accumulate into the warp's slot: element e = ((mt * 2 + nt) * 2 + comp) * 2 + v, lane-contiguous
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        racc[((((mt * 2 + nt) * 2 + 0) * 2 + v) << 5) + lane] += rre[mt][nt][v];
        racc[((((mt * 2 + nt) * 2 + 1) * 2 + v) << 5) + lane] += rim[mt][nt][v];
      }
  __syncwarp();
#if SV_DA_SHARED_A
  DenseC C;
  dense_coef(A, C);
  dense_apply<true>(tp, S, A, warp, lane, &C);
  dense_apply<true>(tl, S, A, warp, lane, &C);
#else
  dense_stage(tp, S, gmats2, base, warp, lane);
  dense_stage(tl, S, gmats2, base, warp, lane);
#endif
}

// ---------------------------------------------------------------- the pass kernel

// SB (adjoint, compile-time): passes without adjoint dense stages — one (psi, lambda) tile buffer
// and no adjoint-dense-stage code, so the instantiation fits 128 registers and 4 CTAs per SM
// (C2 445 -> 476, C3 45.0 -> 46.6, C4g 2.41 -> 2.44 grad evals/s; a runtime single-buffer flag in
// the general kernel measured slower than this separate instantiation)
// RG (adjoint, compile-time): the adjoint dense stages' R accumulators live in the CTA's own
// L2-resident region of r_partials instead of shared memory (da_r_global: from 26 local qubits)
template <int NR, bool DUAL, bool SB = false, bool RG = false>
__global__ void __launch_bounds__(DUAL ? 128 : 256,
                                  DUAL ? (SB ? SV_DUAL_SB_CTAS : (RG ? SV_DUAL_RG_CTAS : SV_DUAL_CTAS))
                                       : (SB ? SV_FWD_SEQ_CTAS : SV_FWD_CTAS)) k_pass_reg(double2* __restrict__ psi, double2* __restrict__ lam,
                                                                  RegArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << a.k;
  const int nthr = blockDim.x, tid = threadIdx.x, nwarps = nthr >> 5, warp = tid >> 5, lane = tid & 31;
  const uint32_t NB = DUAL ? 2 * N : N;  // doubles2 per buffer (psi [+ lambda])
  double2* smem_tiles = reinterpret_cast<double2*>(smem_raw);
  double2* tp = smem_tiles;  // (setup-phase alias; the tile loop rebinds per buffer)
  RegOp* s_ops = reinterpret_cast<RegOp*>(smem_tiles + ((DUAL && (a.n_da > 0 || SB)) ? 1 : 2) * NB);
  StageDesc* s_st = reinterpret_cast<StageDesc*>(s_ops + a.nops);
  double* s_mats = smem_align16<double>(smem_raw, s_st + a.nstages);
  // tile index -> base offset of its outer qubits: four 64-entry deposit tables (tile bits
  // 6c .. 6c+5 -> their outer qubits), replacing a per-tile loop over n_outer bits
  uint64_t* s_ob = reinterpret_cast<uint64_t*>(s_mats + a.nmats);
  const int nacc = a.acc_thread ? nthr : nwarps;            // overlap accumulators per grad op
  double* s_acc = reinterpret_cast<double*>(s_ob + 4 * 64);  // [ngrad][nacc]
  // adjoint dense stages' R accumulators [n_da][nwarps][512]: shared memory, or (RG) this CTA's own
  // L2-resident region of r_partials ([grid][n_da][nwarps][512]), which frees their 16 KiB per slot
  // of shared memory for a third CTA
  double* s_racc = (DUAL && RG) ? a.r_partials + (size_t)blockIdx.x * ((size_t)a.n_da * nwarps * 512)
                                : s_acc + (DUAL ? a.ngrad * nacc : 0);

  {
    const uint4* src = reinterpret_cast<const uint4*>(a.ops);
    uint4* dst = reinterpret_cast<uint4*>(s_ops);
    for (int i = tid; i < a.nops * 2; i += nthr) dst[i] = src[i];
    const uint64_t* ss = reinterpret_cast<const uint64_t*>(a.stages);
    uint64_t* sd = reinterpret_cast<uint64_t*>(s_st);
    for (int i = tid; i < a.nstages * (int)(sizeof(StageDesc) / 8); i += nthr) sd[i] = ss[i];
    for (int i = tid; i < a.nmats; i += nthr) s_mats[i] = a.mats[i];
    for (int h = tid; h < 4 * 64; h += nthr) {
      uint64_t off = 0;
      for (int b = 0; b < 6; ++b) {
        const int j = (h >> 6) * 6 + b;
        if (((h >> b) & 1) && j < a.n_outer) off |= 1ull << a.oq[j];
      }
      s_ob[h] = off;
    }
    if (DUAL) {
      for (int i = tid; i < a.ngrad * nacc; i += nthr) s_acc[i] = 0.0;
      for (int i = tid; i < a.n_da * nwarps * 512; i += nthr) s_racc[i] = 0.0;
    }
  }
  __syncthreads();
  const int nthr_bits = a.k - NR;
  const double2* mats2 = reinterpret_cast<const double2*>(s_mats);
  // Element e = tid + i * nthr of the tile (i < 2^NR): its global index is base | dep(tid) | dep(i << nthr_bits)
  // and its shared slot swz(tid) ^ swz(i << nthr_bits) (dep and swz are XOR-linear), so the
  // per-element index work is one OR and one XOR with kernel-parameter constants.
  uint64_t dep_t = 0;
  for (int b = 0; b < nthr_bits; ++b)
    if ((tid >> b) & 1) dep_t |= 1ull << a.tq[b];
  const uint32_t swz_t = swz((uint32_t)tid);
  static_assert(NR == 3, "element split assumes 8 amplitudes per thread");

  // Double-buffered tiles: while the stages of tile i run from buffer (i & 1), cp.async streams
  // tile i + gridDim.x into the other buffer, so HBM reads overlap the FP64 work.
  auto tile_base = [&](int64_t tile) {
    uint64_t base = s_ob[tile & 63] | s_ob[64 + ((tile >> 6) & 63)] | s_ob[128 + ((tile >> 12) & 63)] |
                    s_ob[192 + ((tile >> 18) & 63)];
    for (int j = 24; j < a.n_outer; ++j)
      if ((tile >> j) & 1) base |= 1ull << a.oq[j];
    return base;
  };
  auto issue_load = [&](int64_t tile, int buf) {
    const uint64_t bt = tile_base(tile) | dep_t;
    double2* dp = tp + (size_t)buf * NB;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint64_t gi = bt | a.hsub[i];
      const uint32_t sl = swz_t ^ a.zsub[i];
      cp_async16(dp + sl, psi + gi);
      if (DUAL) cp_async16(dp + N + sl, lam + gi);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // Adjoint passes with adjoint dense stages keep ONE (psi, lambda) tile buffer: their R
  // accumulators need the shared memory, and a third CTA per SM hides the exposed load better than
  // a second buffer does (the other passes double-buffer).
  const bool dbuf = !(DUAL && (a.n_da > 0 || SB));
  if (dbuf && (int64_t)blockIdx.x < a.ntiles) issue_load(blockIdx.x, 0);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
    const int cur = dbuf ? (it & 1) : 0;
    const uint64_t base = tile_base(tile);
    const int64_t next = tile + gridDim.x;
    if (!dbuf) {
      issue_load(tile, 0);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    } else if (next < a.ntiles) {
      issue_load(next, cur ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    double2* tp = smem_tiles + (size_t)cur * NB;
    double2* tl = DUAL ? tp + N : nullptr;
    // ---- stages ----
    for (int st = 0; st < a.nstages; ++st) {
      const StageDesc& S = s_st[st];
      if constexpr (DUAL && !SB) {  // (single-buffered passes carry no adjoint dense stages)
        if (S.dense == 2) {
          uint32_t ov = 0;  // outer variant of this tile: its own R slot
          for (int b = 0; b < S.m_outer; ++b) ov |= (uint32_t)((base >> S.var_outer[b]) & 1ull) << b;
          da_stage(tp, tl, S, reinterpret_cast<const double2*>(a.mats), base, warp, lane,
                   s_racc + ((size_t)(S.da_index + ov) * nwarps + warp) * 512);
          __syncthreads();
          continue;
        }
      }
      if constexpr (!DUAL && !SB) {  // (SB forward instantiation: passes without dense stages)
        // L1 prefetch of the next dense stage's variant-matrix fragments (global, L2-resident):
        // the first MMA of that stage then finds its A operand in L1 instead of waiting on L2
        if (S.next_dense) {
          const StageDesc& Sn = s_st[st + S.next_dense];
          uint32_t var = Sn.warp_var[warp];
          for (int b = 0; b < Sn.m_outer; ++b) var |= (uint32_t)((base >> Sn.var_outer[b]) & 1ull) << (Sn.m_tile + b);
          const double2* U = reinterpret_cast<const double2*>(a.mats) + Sn.dense_off + var * kDenseVar;
          const double2* q = U + (lane >> 2) * kDenseRow + (lane & 3) * 4;  // one 64-byte line per lane covers 4 entries
          asm volatile("prefetch.global.L1 [%0];\n" ::"l"(q));
          asm volatile("prefetch.global.L1 [%0];\n" ::"l"(q + 8 * kDenseRow));
        }
        if (S.dense) {
          dense_stage(tp, S, reinterpret_cast<const double2*>(a.mats), base, warp, lane);
          __syncthreads();
          continue;
        }
      }
      uint32_t tthr = 0;
      for (int b = 0; b < nthr_bits; ++b)
        if ((tid >> b) & 1) tthr |= 1u << S.thrpos[b];
      const uint32_t A = swz(tthr);
      uint32_t SR[NR];
#pragma unroll
      for (int r = 0; r < NR; ++r) SR[r] = swz(1u << S.regpos[r]);
      double2 v[1 << NR];
      double2 w[DUAL ? (1 << NR) : 1];
#pragma unroll
      for (int j = 0; j < (1 << NR); ++j) {
        uint32_t ad = A;
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if ((j >> r) & 1) ad ^= SR[r];
        v[j] = tp[ad];
        if constexpr (DUAL) w[j] = tl[ad];
      }
      const int op_end = S.op_end;
      for (int i = S.op_begin; i < op_end; ++i) {
        const Op o = load_op(s_ops + i);
        if constexpr (DUAL) {
          const uint32_t rl = o.run_len();
          if (rl) {  // a run of diagonal ops, evaluated together
            dual_diag_run(v, w, s_ops + i, (int)rl, mats2, tthr, base, tp, tl, A, SR, s_acc, nthr, tid, nwarps, warp,
                          lane, a.acc_thread != 0);
            i += (int)rl - 1;
            continue;
          }
        }
        const bool ok = !o.has_ctrl() || (((base & o.couter) == o.couter) && ((tthr & o.cthr()) == o.cthr()));
        const double2* m = mats2 + o.mat_off();
        if constexpr (DUAL) {
          const double2* g = mats2 + o.gen_off();
#if SV_DUAL_CTRL_SPLIT
          double part = o.cj() ? dual_op_c<NR, true>(v, w, o, m, g, tthr, base, ok)
                               : dual_op_c<NR, false>(v, w, o, m, g, tthr, base, ok);
#else
          // one instantiation (register controls tested per amplitude; cj = 0 never skips): half the
          // DUAL code size (instruction-cache misses) and one switch join for v / w
          double part = dual_op_c<NR, true>(v, w, o, m, g, tthr, base, ok);
#endif
          if (o.gen()) {
            if (a.acc_thread) {
              s_acc[o.grad_local() * nthr + tid] += part;  // this thread's running sum over its tiles
            } else {
#pragma unroll
              for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
              if (lane == 0) s_acc[o.grad_local() * nwarps + warp] += part;
            }
          }
        } else {
          if (!ok) continue;
          reg_apply<NR>(v, o, m, tthr, base);
        }
      }
#pragma unroll
      for (int j = 0; j < (1 << NR); ++j) {
        uint32_t ad = A;
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if ((j >> r) & 1) ad ^= SR[r];
        tp[ad] = v[j];
        if constexpr (DUAL) tl[ad] = w[j];
      }
      __syncthreads();
    }
    // ---- store: shared -> HBM (coalesced 16-byte) ----
    {
      const uint64_t bt = base | dep_t;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint64_t gi = bt | a.hsub[i];
        const uint32_t sl = swz_t ^ a.zsub[i];
        psi[gi] = tp[sl];
        if (DUAL) lam[gi] = tl[sl];
      }
    }
    // no barrier: every thread reloads (cp.async) exactly the slots it just stored from, and the
    // last stage ended with one
  }
  if (DUAL) {
    if constexpr (!RG)
      for (int i = tid; i < a.n_da * nwarps * 512; i += nthr)
        a.r_partials[(int64_t)i * a.grid + blockIdx.x] = s_racc[i];
    for (int i = tid; i < a.nops; i += nthr) {
      const Op o = load_op(s_ops + i);
      if (!o.gen()) continue;
      double s = 0.0;
      for (int wi = 0; wi < nacc; ++wi) s += s_acc[o.grad_local() * nacc + wi];  // fixed order
      a.partials[(int64_t)s_ops[i].grad_slot * a.pstride + blockIdx.x] = s;
    }
  }
}

// ---------------------------------------------------------------- all-dense forward passes
//
// Most forward passes of deep circuits consist of dense stages only (C4: 53 of 58). For them a
// leaner kernel: no op list, no sequential-stage code, so the register budget of three CTAs per SM
// leaves room to load the next stage's A operand (its variant matrix, from L2) into registers
// before the barrier that ends the current stage, and the first stage's before the tile wait:
// the L2 latency overlaps barrier / load waits instead of stalling the first MMA of every stage.
// T = double2: complex128 state; T = float2: complex64 state (NEXT-3), 8-byte slots with the swz8
// fold, widened to FP64 for the Gauss DMMA stages and rounded back to FP32 once per stage.
template <typename T>
__device__ __forceinline__ uint32_t tile_swz(uint32_t t) { return sizeof(T) == 16 ? swz(t) : swz8(t); }

template <typename T>
__global__ void __launch_bounds__(256, SV_DENSE_CTAS) k_pass_dense(T* __restrict__ psi, RegArgs a) {
  constexpr bool C64 = sizeof(T) == 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << a.k;
  const int nthr = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  T* smem_tiles = reinterpret_cast<T*>(smem_raw);
  StageDesc* s_st = smem_align16<StageDesc>(smem_raw, smem_tiles + SV_DENSE_NBUF * N);
  uint64_t* s_ob = smem_align16<uint64_t>(smem_raw, s_st + a.nstages);
  // per stage, the variant-matrix offset contributed by the tile index: four 64-entry deposit
  // tables (tile bits 6c .. 6c+5 -> their outer qubits -> variant bits), so a stage's A operand
  // address costs four shared loads instead of a loop over its outer variant qubits
  uint32_t* s_vt = reinterpret_cast<uint32_t*>(s_ob + 4 * 64);
  // complex64: the stages' swz8 slot offsets (the StageDesc ones are for 16-byte slots), from the
  // stage's positions (XOR-linear, as plan.cpp make_dense builds them): per stage 8 warp bases,
  // 32 B-load and 32 D-store lane parts, 6 basis values
  uint16_t* s_o8 = reinterpret_cast<uint16_t*>(s_vt + a.nstages * 256);
  constexpr int kO8 = 8 + 32 + 32 + 8;
  {
    const uint64_t* ss = reinterpret_cast<const uint64_t*>(a.stages);
    uint64_t* sd = reinterpret_cast<uint64_t*>(s_st);
    for (int i = tid; i < a.nstages * (int)(sizeof(StageDesc) / 8); i += nthr) sd[i] = ss[i];
    for (int h = tid; h < 4 * 64; h += nthr) {
      uint64_t off = 0;
      for (int b = 0; b < 6; ++b) {
        const int j = (h >> 6) * 6 + b;
        if (((h >> b) & 1) && j < a.n_outer) off |= 1ull << a.oq[j];
      }
      s_ob[h] = off;
    }
    for (int e = tid; e < a.nstages * 256; e += nthr) {
      const StageDesc& S = *reinterpret_cast<const StageDesc*>(reinterpret_cast<const uint64_t*>(a.stages) +
                                                               (e >> 8) * (int)(sizeof(StageDesc) / 8));
      const int h = e & 255;
      uint32_t var = 0;
      for (int b = 0; b < 6; ++b) {
        const int jt = (h >> 6) * 6 + b;
        if (!((h >> b) & 1) || jt >= a.n_outer) continue;
        for (int t = 0; t < S.m_outer; ++t)
          if (S.var_outer[t] == a.oq[jt]) var |= 1u << (S.m_tile + t);
      }
      s_vt[e] = ((h >> 6) == 0 ? S.dense_off : 0u) + var * kDenseVar;  // summed over the 4 tables
    }
    if (C64)
      for (int e = tid; e < a.nstages * kO8; e += nthr) {
        const StageDesc& S = *reinterpret_cast<const StageDesc*>(reinterpret_cast<const uint64_t*>(a.stages) +
                                                                 (e / kO8) * (int)(sizeof(StageDesc) / 8));
        const int q = e % kO8;
        auto b8 = [&](int pos) { return pos >= 0 ? swz8(1u << pos) : 0u; };
        const uint32_t p0 = b8(S.regpos[0]), p1 = b8(S.regpos[1]), p2 = b8(S.regpos[2]), p3 = b8(S.regpos[3]);
        const uint32_t c0 = b8(S.thrpos[0]), c1 = b8(S.thrpos[1]), c2 = b8(S.thrpos[2]), n0 = b8(S.thrpos[3]);
        uint32_t v = 0;
        if (q < 8) {
          for (int bb = 0; bb < 3; ++bb)
            if ((q >> bb) & 1) v ^= b8(S.thrpos[4 + bb]);
        } else if (q < 40) {
          const int l = q - 8;
          v = (((l >> 2) & 1) ? c0 : 0u) ^ (((l >> 3) & 1) ? c1 : 0u) ^ (((l >> 4) & 1) ? c2 : 0u) ^ ((l & 1) ? p0 : 0u) ^
              ((l & 2) ? p1 : 0u);
        } else if (q < 72) {
          const int l = q - 40;
          v = (((l >> 2) & 1) ? p0 : 0u) ^ (((l >> 3) & 1) ? p1 : 0u) ^ (((l >> 4) & 1) ? p2 : 0u) ^ ((l & 1) ? c1 : 0u) ^
              ((l & 2) ? c2 : 0u);
        } else {
          const uint32_t basis[8] = {p2, p3, n0, c0, p3, n0, 0u, 0u};  // Lk0 Lk1 Ln | Sv Sm Sn
          v = basis[q - 72];
        }
        s_o8[e] = (uint16_t)v;
      }
  }
  __syncthreads();
  const int nthr_bits = a.k - 3;
  uint64_t dep_t = 0;
  for (int b = 0; b < nthr_bits; ++b)
    if ((tid >> b) & 1) dep_t |= 1ull << a.tq[b];
  const uint32_t swz_t = tile_swz<T>((uint32_t)tid);
  const double2* gm2 = reinterpret_cast<const double2*>(a.mats);
  auto tile_base = [&](int64_t tile) {
    uint64_t base = s_ob[tile & 63] | s_ob[64 + ((tile >> 6) & 63)] | s_ob[128 + ((tile >> 12) & 63)] |
                    s_ob[192 + ((tile >> 18) & 63)];
    for (int j = 24; j < a.n_outer; ++j)
      if ((tile >> j) & 1) base |= 1ull << a.oq[j];
    return base;
  };
  // a ring of SV_DENSE_NBUF tile buffers: tile i + NBUF - 1 streams in while tile i computes (every
  // iteration commits one cp.async group, empty past the end, so the wait count is constant)
  auto issue_load = [&](int64_t tile, int buf) {
    if (tile < a.ntiles) {
      const uint64_t bt = tile_base(tile) | dep_t;
      T* dp = smem_tiles + (size_t)buf * N;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (C64) cp_async8(dp + (swz_t ^ a.zsub[i]), psi + (bt | a.hsub[i]));
        else cp_async16(dp + (swz_t ^ a.zsub[i]), psi + (bt | a.hsub[i]));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
#pragma unroll
  for (int j = 0; j < SV_DENSE_NBUF - 1; ++j) issue_load(blockIdx.x + (int64_t)j * gridDim.x, j);
  DenseA ue;
  int it = 0, cur = 0;
  // A operand of stage st for a tile: warp part + tile part (tables; outer bits past 24 by loop)
  auto load_a = [&](int st, int64_t tile, uint64_t base) {
    const StageDesc& S = s_st[st];
    const uint32_t* vt = s_vt + st * 256;
    uint32_t off = vt[tile & 63] + vt[64 + ((tile >> 6) & 63)] + vt[128 + ((tile >> 12) & 63)] +
                   vt[192 + ((tile >> 18) & 63)];  // disjoint variant bits: sums are ORs
    if (a.n_outer > 24) {
      uint32_t var = 0;
      for (int b = 0; b < S.m_outer; ++b)
        for (int jt = 24; jt < a.n_outer; ++jt)
          if (a.oq[jt] == S.var_outer[b] && ((tile >> jt) & 1)) var |= 1u << (S.m_tile + b);
      off += var * kDenseVar;
    }
    dense_load_u(gm2 + off + (uint32_t)S.warp_var[warp] * kDenseVar, lane, ue);
  };
  if ((int64_t)blockIdx.x < a.ntiles) load_a(0, blockIdx.x, tile_base(blockIdx.x));
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
    const uint64_t base = tile_base(tile);
    const int64_t next = tile + gridDim.x;
    // the buffer tile - gridDim.x used (its stores are this thread's own slots, issued above)
    issue_load(tile + (int64_t)(SV_DENSE_NBUF - 1) * gridDim.x, cur == 0 ? SV_DENSE_NBUF - 1 : cur - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SV_DENSE_NBUF - 1) : "memory");
    __syncthreads();
    T* tp = smem_tiles + (size_t)cur * N;
    for (int st = 0; st < a.nstages; ++st) {
      if (C64) {
        const uint16_t* o8 = s_o8 + st * kO8;
        DenseOff O;
        O.bB = (uint32_t)o8[warp] ^ o8[8 + lane];
        O.bD = (uint32_t)o8[warp] ^ o8[40 + lane];
        O.Lk0 = o8[72];
        O.Lk1 = o8[73];
        O.Ln = o8[74];
        O.Sv = o8[75];
        O.Sm = o8[76];
        O.Sn = o8[77];
        dense_apply_o(tp, O, ue);
      } else {
        dense_apply_o(tp, dense_off(s_st[st], warp, lane), ue);
      }
      // the next A operand: this tile's next stage, or the next tile's first stage (its L2
      // latency then overlaps the barrier, the store and the next tile's wait)
#if SV_DENSE_VT
      if (st + 1 < a.nstages) load_a(st + 1, tile, base);
      else if (next < a.ntiles) load_a(0, next, 0);
#else
      if (st + 1 < a.nstages) dense_load_a(s_st[st + 1], gm2, base, warp, lane, ue);
      else if (next < a.ntiles) dense_load_a(s_st[0], gm2, tile_base(next), warp, lane, ue);
#endif
      __syncthreads();
    }
    {
      const uint64_t bt = base | dep_t;
#pragma unroll
      for (int i = 0; i < 8; ++i) psi[bt | a.hsub[i]] = tp[swz_t ^ a.zsub[i]];
    }
    // no barrier: every thread reloads (cp.async) exactly the slots it just stored from, and the
    // last stage ended with one
    cur = cur + 1 == SV_DENSE_NBUF ? 0 : cur + 1;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------- complex64 forward passes (NEXT-3)
//
// The state is complex64 in HBM and in the shared-memory tile (half the bytes of every pass): one
// 8-byte slot per amplitude, swizzled with a 4-bit XOR fold (16 slots per bank row), 8-byte
// cp.async copies in and 8-byte stores out; every address is derived in-kernel from the stage's
// positions. Register (sequential) stages widen the thread's 8 amplitudes to complex128 and run the
// same op code as the complex128 kernel (one rounding per stage); dense stages run on the TF32
// tensor cores with a 3-term split (dense_stage_tf32). Measured alternatives: FP32 FFMA on the CUDA
// cores and widening to the FP64 MMAs were both slower.

__constant__ uint32_t kPerm24[24] = {228, 180, 216, 120, 156, 108, 225, 177, 201, 57, 141, 45, 210, 114, 198, 54, 78, 30, 147, 99, 135, 39, 75, 27};  // plan.cpp make_dense order

// ---- complex64 dense stage on TF32 tensor cores with a 3-term split ("3xTF32") ----
// Y = [[Ur, -Ui], [Ui, Ur]] [Xr; Xi] as mma.sync m16n8k8 (TF32 in, FP32 accumulate): per warp
// 2 M-tiles (Re / Im out) x 2 N-tiles (its 16 vectors) x 4 K-steps. Every FP32 operand v is split
// into hi = tf32(v) and lo = tf32(v - hi); D += A_hi B_hi + A_hi B_lo + A_lo B_hi keeps ~21
// mantissa bits (the dropped A_lo B_lo term is ~2^-21 relative), i.e. near-FP32 accuracy at the
// TF32 tensor rate (measured 277 TF legacy mma.sync vs 37 TF for FP64). Fragment layouts (PTX
// m16n8k8 .tf32): A[g (+8)][t (+4)], B[k = t (+4)][n = g], D[g (+8)][2t (+1)]; g = lane/4, t = lane%4.
// hi keeps the top 10 mantissa bits (truncation: one LOP3; cvt.rna.tf32 is a multi-instruction
// sequence on sm_100a), lo = v - hi is exact in FP32 and the MMA reads its top 10 mantissa bits:
// together ~21 bits, the dropped remainder is <= 2^-21 relative.
#ifndef SV_TF32_RNA
#define SV_TF32_RNA 2  // 2: hi rounded to nearest by an integer add (measured 2.5x smaller error than
                       // truncation, +1% speed); 1: cvt.rna for hi and lo (same error, 10% slower)
#endif
__device__ __forceinline__ void split_tf32(float v, uint32_t& hi, uint32_t& lo) {
#if SV_TF32_RNA == 1
  // hi and lo rounded to nearest TF32 (cvt.rna): |v - hi - lo| <= 2^-22 |v| instead of the
  // truncation's lo read to 10 of its up to 13 bits
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(v));
  const float r = v - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
#elif SV_TF32_RNA == 2
  // hi rounded to nearest by integer add on the bit pattern (ties away; |v| << FLT_MAX here):
  // |lo| <= 2^-11 |v|, so the tensor core's 10-bit read of lo errs by <= 2^-21 |v|
  hi = (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;
  lo = __float_as_uint(v - __uint_as_float(hi));
#else
  hi = __float_as_uint(v) & 0xFFFFE000u;
  lo = __float_as_uint(v - __uint_as_float(hi));
#endif
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// The TF32 dense stage's swz8 slot offsets (XOR-linear in the positions): vector n = 8 nt + col (col
// bits -> the warp's first three vector positions in the host-chosen order StageDesc::c64_perm, nt ->
// the fourth), register index r (bit i -> regpos[i]). Entry q of the stage's 80: q < 8 warp part,
// 8 + lane B-load lane part (n col = g, in amp r = t), 40 + lane D-store lane part (out amp o = g,
// n col = 2 t), 72.. the bases of nt, r bit 2, r bit 3 and n col bit 0.
constexpr int kC64Off = 80;
__device__ __forceinline__ uint16_t c64_stage_offset(const StageDesc& S, int q) {
  auto sp = [&](int pos) { return pos >= 0 ? swz8(1u << pos) : 0u; };
  const uint32_t pc = kPerm24[S.c64_perm];
  const int X[4] = {S.thrpos[pc & 3], S.thrpos[(pc >> 2) & 3], S.thrpos[(pc >> 4) & 3], S.thrpos[(pc >> 6) & 3]};
  uint32_t v = 0;
  if (q < 8) {
    for (int b = 0; b < 3; ++b)
      if ((q >> b) & 1) v ^= sp(S.thrpos[4 + b]);
  } else if (q < 72) {
    const int l = (q - 8) & 31, g = l >> 2, t = l & 3;
    const bool load = q < 40;
    for (int b = 0; b < 3; ++b)
      if ((g >> b) & 1) v ^= load ? sp(X[b]) : sp(S.regpos[b]);
    for (int b = 0; b < 2; ++b)
      if ((t >> b) & 1) v ^= load ? sp(S.regpos[b]) : sp(X[b + 1]);
  } else if (q < 76) {
    const int which = q - 72;
    v = which == 0 ? sp(X[3]) : which == 1 ? sp(S.regpos[2]) : which == 2 ? sp(S.regpos[3]) : sp(X[0]);
  }
  return (uint16_t)v;
}

__device__ __forceinline__ void dense_stage_tf32(float2* tp, const StageDesc& S, const double2* __restrict__ gm2,
                                                 uint64_t base, int warp, int lane, bool split, const uint16_t* o8) {
  const int g = lane >> 2, t = lane & 3;
  uint32_t var = S.warp_var[warp];
  for (int b = 0; b < S.m_outer; ++b) var |= (uint32_t)((base >> S.var_outer[b]) & 1ull) << (S.m_tile + b);
  const double2* U = gm2 + S.dense_off + var * kDenseVar;
  // A entries U[o][i], o in {g, g+8} (a), i = 8 kh + t (+4) (c): complex -> split re / im
  uint32_t ur_h[2][2][2], ur_l[2][2][2], ui_h[2][2][2], ui_l[2][2][2];  // [kh][a][c]
#pragma unroll
  for (int kh = 0; kh < 2; ++kh)
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double2 u = __ldg(U + (g + 8 * a) * kDenseRow + 8 * kh + t + 4 * c);
        split_tf32((float)u.x, ur_h[kh][a][c], ur_l[kh][a][c]);
        split_tf32((float)u.y, ui_h[kh][a][c], ui_l[kh][a][c]);
      }
  // slot parts: the stage's table (k_pass_c64 setup, c64_stage_offsets)
  const uint32_t bB = (uint32_t)o8[warp] ^ o8[8 + lane], bD = (uint32_t)o8[warp] ^ o8[40 + lane];
  const uint32_t sN = o8[72], sR2 = o8[73], sR3 = o8[74], sC0 = o8[75];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    // B fragments: in amps r = t + 4 c + 8 kh of vector (8 nt + g): Re for K-steps 0-1, Im for 2-3
    uint32_t xr_h[2][2], xr_l[2][2], xi_h[2][2], xi_l[2][2];  // [kh][c]
#pragma unroll
    for (int kh = 0; kh < 2; ++kh)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float2 x = tp[bB ^ (nt ? sN : 0u) ^ (c ? sR2 : 0u) ^ (kh ? sR3 : 0u)];
        split_tf32(x.x, xr_h[kh][c], xr_l[kh][c]);
        split_tf32(x.y, xi_h[kh][c], xi_l[kh][c]);
      }
    float dre[4] = {0.f, 0.f, 0.f, 0.f}, dim[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kh = 0; kh < 2; ++kh) {
      // Re out += Ur Xr - Ui Xi ; Im out += Ui Xr + Ur Xi
      const uint32_t arh[4] = {ur_h[kh][0][0], ur_h[kh][1][0], ur_h[kh][0][1], ur_h[kh][1][1]};
      const uint32_t arl[4] = {ur_l[kh][0][0], ur_l[kh][1][0], ur_l[kh][0][1], ur_l[kh][1][1]};
      const uint32_t aih[4] = {ui_h[kh][0][0], ui_h[kh][1][0], ui_h[kh][0][1], ui_h[kh][1][1]};
      const uint32_t ail[4] = {ui_l[kh][0][0], ui_l[kh][1][0], ui_l[kh][0][1], ui_l[kh][1][1]};
      const uint32_t nih[4] = {aih[0] ^ 0x80000000u, aih[1] ^ 0x80000000u, aih[2] ^ 0x80000000u, aih[3] ^ 0x80000000u};
      const uint32_t nil[4] = {ail[0] ^ 0x80000000u, ail[1] ^ 0x80000000u, ail[2] ^ 0x80000000u, ail[3] ^ 0x80000000u};
      mma_tf32(dre, arh, xr_h[kh][0], xr_h[kh][1]);
      mma_tf32(dim, aih, xr_h[kh][0], xr_h[kh][1]);
      mma_tf32(dre, nih, xi_h[kh][0], xi_h[kh][1]);
      mma_tf32(dim, arh, xi_h[kh][0], xi_h[kh][1]);
      if (!split) continue;  // SV_OPT_C64_SPLIT = 1: one TF32 product (test of the tolerance's power)
      mma_tf32(dre, arh, xr_l[kh][0], xr_l[kh][1]);
      mma_tf32(dim, aih, xr_l[kh][0], xr_l[kh][1]);
      mma_tf32(dre, nih, xi_l[kh][0], xi_l[kh][1]);
      mma_tf32(dim, arh, xi_l[kh][0], xi_l[kh][1]);
      mma_tf32(dre, arl, xr_h[kh][0], xr_h[kh][1]);
      mma_tf32(dim, ail, xr_h[kh][0], xr_h[kh][1]);
      mma_tf32(dre, nil, xi_h[kh][0], xi_h[kh][1]);
      mma_tf32(dim, arl, xi_h[kh][0], xi_h[kh][1]);
    }
    // D: rows o = g (+8: d[2], d[3]), cols n = 8 nt + 2 t (+1: d[1], d[3])
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t ad = bD ^ (nt ? sN : 0u) ^ ((q & 1) ? sC0 : 0u) ^ ((q & 2) ? sR3 : 0u);
      tp[ad] = make_float2(dre[q], dim[q]);
    }
  }
}

__global__ void __launch_bounds__(256, SV_C64_CTAS) k_pass_c64(float2* __restrict__ psi, RegArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t N = 1u << a.k;
  const int nthr = blockDim.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float2* smem_tiles = reinterpret_cast<float2*>(smem_raw);  // two tiles
  RegOp* s_ops = reinterpret_cast<RegOp*>(smem_tiles + 2 * N);
  StageDesc* s_st = reinterpret_cast<StageDesc*>(s_ops + a.nops);
  double* s_mats = smem_align16<double>(smem_raw, s_st + a.nstages);
  uint64_t* s_ob = reinterpret_cast<uint64_t*>(s_mats + a.nmats);
  uint16_t* s_o8 = reinterpret_cast<uint16_t*>(s_ob + 4 * 64);  // [nstages][kC64Off] TF32 stage offsets
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.ops);
    uint4* dst = reinterpret_cast<uint4*>(s_ops);
    for (int i = tid; i < a.nops * 2; i += nthr) dst[i] = src[i];
    const uint64_t* ss = reinterpret_cast<const uint64_t*>(a.stages);
    uint64_t* sd = reinterpret_cast<uint64_t*>(s_st);
    for (int i = tid; i < a.nstages * (int)(sizeof(StageDesc) / 8); i += nthr) sd[i] = ss[i];
    for (int i = tid; i < a.nmats; i += nthr) s_mats[i] = a.mats[i];
    for (int h = tid; h < 4 * 64; h += nthr) {
      uint64_t off = 0;
      for (int b = 0; b < 6; ++b) {
        const int j = (h >> 6) * 6 + b;
        if (((h >> b) & 1) && j < a.n_outer) off |= 1ull << a.oq[j];
      }
      s_ob[h] = off;
    }
    for (int e = tid; e < a.nstages * kC64Off; e += nthr) {
      const StageDesc& S = *reinterpret_cast<const StageDesc*>(reinterpret_cast<const uint64_t*>(a.stages) +
                                                               (e / kC64Off) * (int)(sizeof(StageDesc) / 8));
      s_o8[e] = S.dense ? c64_stage_offset(S, e % kC64Off) : (uint16_t)0;
    }
  }
  __syncthreads();
  const int nthr_bits = a.k - 3;
  const double2* mats2 = reinterpret_cast<const double2*>(s_mats);
  const double2* gm2 = reinterpret_cast<const double2*>(a.mats);
  uint64_t dep_t = 0;
  for (int b = 0; b < nthr_bits; ++b)
    if ((tid >> b) & 1) dep_t |= 1ull << a.tq[b];
  const uint32_t swz_t = swz8((uint32_t)tid);
  auto tile_base = [&](int64_t tile) {
    uint64_t base = s_ob[tile & 63] | s_ob[64 + ((tile >> 6) & 63)] | s_ob[128 + ((tile >> 12) & 63)] |
                    s_ob[192 + ((tile >> 18) & 63)];
    for (int j = 24; j < a.n_outer; ++j)
      if ((tile >> j) & 1) base |= 1ull << a.oq[j];
    return base;
  };
  auto issue_load = [&](int64_t tile, int buf) {
    const uint64_t bt = tile_base(tile) | dep_t;
    float2* dp = smem_tiles + (size_t)buf * N;
#pragma unroll
    for (int i = 0; i < 8; ++i) cp_async8(dp + (swz_t ^ a.zsub[i]), psi + (bt | a.hsub[i]));
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if ((int64_t)blockIdx.x < a.ntiles) issue_load(blockIdx.x, 0);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++it) {
    const int cur = it & 1;
    const uint64_t base = tile_base(tile);
    const int64_t next = tile + gridDim.x;
    if (next < a.ntiles) {
      issue_load(next, cur ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    float2* tp = smem_tiles + (size_t)cur * N;
    for (int st = 0; st < a.nstages; ++st) {
      const StageDesc& S = s_st[st];
      if (S.dense) {
        dense_stage_tf32(tp, S, gm2, base, warp, lane, a.c64_terms != 1, s_o8 + st * kC64Off);
        __syncthreads();
        continue;
      }
      uint32_t tthr = 0;
      for (int b = 0; b < nthr_bits; ++b)
        if ((tid >> b) & 1) tthr |= 1u << S.thrpos[b];
      const uint32_t A = swz8(tthr);
      uint32_t SR[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) SR[r] = swz8(1u << S.regpos[r]);
      double2 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t ad = A;
#pragma unroll
        for (int r = 0; r < 3; ++r)
          if ((j >> r) & 1) ad ^= SR[r];
        v[j] = tile_ld(tp[ad]);
      }
      const int op_end = S.op_end;
      for (int i = S.op_begin; i < op_end; ++i) {
        const Op o = load_op(s_ops + i);
        const bool ok = ((base & o.couter) == o.couter) && ((tthr & o.cthr()) == o.cthr());
        if (!ok) continue;
        reg_apply<3>(v, o, mats2 + o.mat_off(), tthr, base);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t ad = A;
#pragma unroll
        for (int r = 0; r < 3; ++r)
          if ((j >> r) & 1) ad ^= SR[r];
        tile_st(tp[ad], v[j]);
      }
      __syncthreads();
    }
    {
      const uint64_t bt = base | dep_t;
#pragma unroll
      for (int i = 0; i < 8; ++i) psi[bt | a.hsub[i]] = tp[swz_t ^ a.zsub[i]];
    }
    // no barrier: every thread reloads (cp.async) exactly the slots it just stored from, and the
    // last stage ended with one
  }
}

size_t c64_pass_smem_bytes(int k, int nops, int nstages, int nmats) {
  return (size_t(8) << k) * 2 + (size_t)nops * sizeof(RegOp) + (size_t)nstages * sizeof(StageDesc) + 16 +
         (size_t)nmats * 8 + 4 * 64 * 8 + (size_t)nstages * kC64Off * 2;
}

__global__ void k_widen(const float2* __restrict__ a, double2* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = tile_ld(a[i]);
}
__global__ void k_narrow(const double2* __restrict__ a, float2* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    tile_st(b[i], a[i]);
}

size_t dense_pass_smem_bytes(int k, int nstages, bool c64) {
  return (size_t(c64 ? 8 : 16) << k) * SV_DENSE_NBUF + 16 + (size_t)nstages * sizeof(StageDesc) + 16 + 4 * 64 * 8 +
         (size_t)nstages * 256 * 4 + (size_t)nstages * (8 + 32 + 32 + 8) * 2;
}


size_t reg_smem_bytes(int k, int low, int nops, int nstages, int nmats, int ngrad, int nthr, bool dual, int n_da,
                      bool acc_thread, bool single_buf, bool r_global) {
  size_t b = (size_t(16) << k) * (dual ? 2 : 1) * ((dual && (n_da > 0 || single_buf)) ? 1 : 2);  // tile buffers
  b += (dual && !r_global) ? (size_t)n_da * (nthr / 32) * 512 * 8 : 0;
  b += (size_t)nops * sizeof(RegOp) + (size_t)nstages * sizeof(StageDesc) + 16;
  b += (size_t)nmats * 8 + 4 * 64 * 8;
  b += dual ? (size_t)ngrad * (acc_thread ? nthr : nthr / 32) * 8 : 0;
  return b;
}

}  // namespace

bool pass_no_dense(const Plan& plan, const PassDesc& pd) {
  if (plan.reverse || pd.R != 3) return false;
  for (int si = pd.stage_begin; si < pd.stage_end; ++si)
    if (plan.stages[si].dense) return false;
  return true;
}

bool pass_all_dense(const Plan& plan, const PassDesc& pd) {
  static const bool off = [] { const char* e = getenv("SV_DENSE_KERNEL"); return e && atoi(e) == 0; }();
  if (off || plan.reverse || pd.R != 3 || pd.stage_end <= pd.stage_begin) return false;
  for (int si = pd.stage_begin; si < pd.stage_end; ++si)
    if (plan.stages[si].dense != 1) return false;
  return true;
}

static cudaError_t set_reg_attrs() {
  static std::atomic<uint64_t> done{0};
  return once_per_device(done, [] {
    cudaError_t e = cudaFuncSetAttribute(k_pass_reg<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pass_reg<3, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pass_reg<3, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pass_reg<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pass_reg<3, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pass_dense<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_pass_dense<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    return e;
  });
}

// Resident CTAs per SM for the register passes of a plan: the largest pass' shared memory decides
// (one persistent grid serves every pass of the plan, so it must not exceed what is co-resident).
int reg_pass_ctas_per_sm(const Plan& plan, size_t i, bool dual, int n_local) {
  if (set_reg_attrs() != cudaSuccess) return 1;
  const PassDesc& pd = plan.passes[i];
  if (pd.R == 0) return 1;
  const int next_mat = (i + 1 < plan.passes.size()) ? plan.passes[i + 1].mat_begin : (int)plan.mats.size();
  const int nm = std::min(pd.seq_mats, next_mat - pd.mat_begin);
  int n_da = 0;
  for (int si = pd.stage_begin; si < pd.stage_end; ++si) n_da += plan.stages[si].dense == 2 ? (1 << plan.stages[si].m_outer) : 0;
  const int nthr = 1 << (pd.k - pd.R);
  // adjoint passes without adjoint dense stages: the single-buffered, 4-CTA instantiation; with
  // them, from 26 local qubits the instantiation with L2 R accumulators
  const bool single_buf = dual && n_da == 0 && n_local <= SV_DUAL_SINGLE_BUF_MAX_N;
  const bool r_global = dual && da_r_global(n_local);
  void (*dual_fn)(double2*, double2*, RegArgs) =
      single_buf ? k_pass_reg<3, true, true> : r_global ? k_pass_reg<3, true, false, true> : k_pass_reg<3, true>;
  // adjoint passes: per-thread overlap accumulators when they cost no resident CTA (queried on the
  // instantiation that will run)
  bool acc_thread = false;
  if (dual) {
    int b_warp = 0, b_thr = 0;
    const size_t sw = reg_smem_bytes(pd.k, pd.low, pd.op_end - pd.op_begin, pd.stage_end - pd.stage_begin, nm,
                                     pd.n_grad, nthr, dual, n_da, false, single_buf, r_global);
    const size_t st = reg_smem_bytes(pd.k, pd.low, pd.op_end - pd.op_begin, pd.stage_end - pd.stage_begin, nm,
                                     pd.n_grad, nthr, dual, n_da, true, single_buf, r_global);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b_warp, dual_fn, nthr, sw);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b_thr, dual_fn, nthr, st);
    acc_thread = b_thr >= b_warp && b_thr > 0 && pd.n_grad > 0;
    if (plan.pass_acc.size() != plan.passes.size()) plan.pass_acc.assign(plan.passes.size(), 0);
    plan.pass_acc[i] = acc_thread ? kPassAccThread : 0;
  }
  if (single_buf) plan.pass_acc[i] |= kPassSingleBuf;
  const size_t smem = reg_smem_bytes(pd.k, pd.low, pd.op_end - pd.op_begin, pd.stage_end - pd.stage_begin, nm,
                                     pd.n_grad, nthr, dual, n_da, acc_thread, single_buf, r_global);
  int blocks = 0;
  if (pass_all_dense(plan, pd)) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_pass_dense<double2>, nthr,
                                                                  dense_pass_smem_bytes(pd.k, pd.stage_end - pd.stage_begin, false));
    return (e == cudaSuccess && blocks > 0) ? blocks : 1;
  }
  cudaError_t e = dual ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, dual_fn, nthr, smem)
                       : (pass_no_dense(plan, pd) ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_pass_reg<3, false, true>, nthr, smem)
                                                  : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_pass_reg<3, false>, nthr, smem));
  return (e == cudaSuccess && blocks > 0) ? blocks : 1;
}

cudaError_t launch_pass_reg(double* psi, double* lam, const PassLaunch& L, cudaStream_t s) {
  const PassDesc& pd = *L.pd;
  RegArgs a;
  a.k = pd.k;
  a.low = pd.low;
  a.nops = pd.op_end - pd.op_begin;
  a.nstages = pd.stage_end - pd.stage_begin;
  a.nmats = pd.seq_mats < L.nmats ? pd.seq_mats : L.nmats;  // dense variants stay in global memory
  a.ngrad = pd.n_grad;
  a.grid = L.grid;
  for (int i = 0; i < kMaxTileQubits + 3; ++i) a.tq[i] = pd.tq[i];
  uint64_t tmask = 0;
  for (int p = 0; p < pd.k; ++p) tmask |= 1ull << pd.tq[p];
  a.n_outer = 0;
  for (int q = 0; q < L.n_local; ++q)
    if (!((tmask >> q) & 1ull)) a.oq[a.n_outer++] = (int8_t)q;
  a.ntiles = 1ll << (L.n_local - pd.k);
  {
    const int tb = pd.k - pd.R;
    for (int i = 0; i < 8; ++i) {
      a.hsub[i] = 0;
      for (int j = 0; j < 3; ++j)
        if ((i >> j) & 1) a.hsub[i] |= 1ull << pd.tq[tb + j];
      a.zsub[i] = swz((uint32_t)i << tb);
    }
  }
  a.ops = L.d_rops + pd.op_begin;
  a.mats = L.d_mats + pd.mat_begin;
  a.stages = L.d_stages + pd.stage_begin;
  a.partials = L.d_partials;
  const bool dual = lam != nullptr;
  const int nthr = 1 << (pd.k - pd.R);
  a.n_da = L.n_da;
  a.pstride = L.pstride > 0 ? L.pstride : L.grid;
  a.r_partials = L.r_partials;
  a.acc_thread = dual ? (L.acc_thread & kPassAccThread) : 0;
  a.single_buf = dual ? ((L.acc_thread & kPassSingleBuf) ? 1 : 0) : 0;
  const size_t smem = reg_smem_bytes(a.k, a.low, a.nops, a.nstages, a.nmats, a.ngrad, nthr, dual, a.n_da, a.acc_thread != 0,
                                     a.single_buf != 0, dual && da_r_global(L.n_local));
  {
    cudaError_t e = set_reg_attrs();
    if (e != cudaSuccess) return e;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (dual && nthr > 128) return cudaErrorInvalidValue;  // adjoint passes run 2^10-amplitude tiles
  if (dual) {
    if (pd.R != 3) return cudaErrorInvalidValue;
    if (a.single_buf && a.n_da == 0)
      k_pass_reg<3, true, true><<<L.grid, nthr, smem, s>>>(reinterpret_cast<double2*>(psi), reinterpret_cast<double2*>(lam), a);
    else if (da_r_global(L.n_local))
      k_pass_reg<3, true, false, true><<<L.grid, nthr, smem, s>>>(reinterpret_cast<double2*>(psi), reinterpret_cast<double2*>(lam), a);
    else
      k_pass_reg<3, true><<<L.grid, nthr, smem, s>>>(reinterpret_cast<double2*>(psi), reinterpret_cast<double2*>(lam), a);
  } else {
    if (pd.R != 3) return cudaErrorInvalidValue;
    if (L.all_dense) {
      k_pass_dense<double2><<<L.grid, nthr, dense_pass_smem_bytes(a.k, a.nstages, false), s>>>(reinterpret_cast<double2*>(psi), a);
    } else if (L.no_dense) {
      k_pass_reg<3, false, true><<<L.grid, nthr, smem, s>>>(reinterpret_cast<double2*>(psi), nullptr, a);
    } else {
      k_pass_reg<3, false><<<L.grid, nthr, smem, s>>>(reinterpret_cast<double2*>(psi), nullptr, a);
    }
  }
  return cudaGetLastError();
}


// complex64 forward pass (NEXT-3): register plans (2^8..2^11-amplitude tiles, 2^(k-3) threads);
// the caller (api.cpp) routes everything else through a complex128 scratch copy.
bool c64_pass_ok(const PassDesc& pd) { return pd.R == 3 && pd.k >= 8 && pd.k <= 11; }

cudaError_t launch_pass_c64(float* psi, const PassLaunch& L, cudaStream_t s) {
  const PassDesc& pd = *L.pd;
  if (!c64_pass_ok(pd)) return cudaErrorInvalidValue;
  RegArgs a;
  std::memset(&a, 0, sizeof(a));
  a.k = pd.k;
  a.low = pd.low;
  a.nops = pd.op_end - pd.op_begin;
  a.nstages = pd.stage_end - pd.stage_begin;
  a.nmats = pd.seq_mats < L.nmats ? pd.seq_mats : L.nmats;
  a.grid = L.grid;
  for (int i = 0; i < kMaxTileQubits + 3; ++i) a.tq[i] = pd.tq[i];
  uint64_t tmask = 0;
  for (int p = 0; p < pd.k; ++p) tmask |= 1ull << pd.tq[p];
  a.n_outer = 0;
  for (int q = 0; q < L.n_local; ++q)
    if (!((tmask >> q) & 1ull)) a.oq[a.n_outer++] = (int8_t)q;
  a.ntiles = 1ll << (L.n_local - pd.k);
  const int tb = pd.k - 3;  // thread bits: element e = tid + i 2^tb, i < 8
  for (int i = 0; i < 8; ++i) {
    a.hsub[i] = 0;
    for (int j = 0; j < 3; ++j)
      if ((i >> j) & 1) a.hsub[i] |= 1ull << pd.tq[tb + j];
    a.zsub[i] = swz8((uint32_t)i << tb);
  }
  a.ops = L.d_rops + pd.op_begin;
  a.mats = L.d_mats + pd.mat_begin;
  a.stages = L.d_stages + pd.stage_begin;
  a.c64_terms = L.c64_terms;
  const int nthr = 1 << tb;
  if (L.all_dense && L.c64_terms == 0) {
    // FP64 Gauss DMMA stages on the widened tile (SV_OPT_C64_SPLIT = 0)
    cudaError_t e = set_reg_attrs();
    if (e != cudaSuccess) return e;
    const size_t sm = dense_pass_smem_bytes(a.k, a.nstages, true);
    if (sm > 227 * 1024) return cudaErrorInvalidValue;
    int blocks = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_pass_dense<float2>, nthr, sm);
    if (e != cudaSuccess) return e;
    const int64_t grid = std::min<int64_t>(a.ntiles, (int64_t)device_sm_count() * std::max(1, blocks));
    a.grid = (int)grid;
    k_pass_dense<float2><<<(int)grid, nthr, sm, s>>>(reinterpret_cast<float2*>(psi), a);
    return cudaGetLastError();
  }
  const size_t smem = c64_pass_smem_bytes(a.k, a.nops, a.nstages, a.nmats);
  static std::atomic<uint64_t> attr{0};
  {
    cudaError_t e = once_per_device(
        attr, [] { return cudaFuncSetAttribute(k_pass_c64, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); });
    if (e != cudaSuccess) return e;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  k_pass_c64<<<L.grid, nthr, smem, s>>>(reinterpret_cast<float2*>(psi), a);
  return cudaGetLastError();
}

cudaError_t launch_widen(const float* a, double* b, int64_t n, cudaStream_t s) {
  k_widen<<<device_sm_count() * 4, 256, 0, s>>>(reinterpret_cast<const float2*>(a), reinterpret_cast<double2*>(b), n);
  return cudaGetLastError();
}
cudaError_t launch_narrow(const double* a, float* b, int64_t n, cudaStream_t s) {
  k_narrow<<<device_sm_count() * 4, 256, 0, s>>>(reinterpret_cast<const double2*>(a), reinterpret_cast<float2*>(b), n);
  return cudaGetLastError();
}

}  // namespace sv
