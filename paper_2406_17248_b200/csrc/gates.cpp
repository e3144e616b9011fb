// gates.cpp — host-side binding of one sv_gate to its class and matrix entries.
//
// Taxonomy (§3.1): X-like gates have only anti-diagonal entries [[0,a],[b,0]] (eq. at
// P:80-87, update new[i0] = a old[i1], new[i1] = b old[i0], reading c3); Z-like gates only
// diagonal entries [[a,0],[0,b]] (eq. at, "no pairing"); everything else is a general
// 2x2 or a two-qubit 4x4 group (P:579 gate list). Rotations R_P(t) = exp(-i t P/2) (reading c1).
// Adjoint generator D = (dU/dphi) U^dagger: -(i/2) P for R_P, i|1><1| for PS (reading c10).
#include <cmath>
#include <cstring>

#include "sv.h"
#include "sv_internal.h"

namespace sv {
namespace {

inline Cx cx(double re, double im = 0.0) { return Cx{re, im}; }
inline Cx cexpi(double t) { return Cx{std::cos(t), std::sin(t)}; }
inline Cx mul(Cx a, Cx b) { return Cx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

// Single-qubit Pauli matrices, row-major.
void pauli1(char p, Cx* m) {
  switch (p) {
    case 'X': m[0] = cx(0); m[1] = cx(1); m[2] = cx(1); m[3] = cx(0); break;
    case 'Y': m[0] = cx(0); m[1] = cx(0, -1); m[2] = cx(0, 1); m[3] = cx(0); break;
    default:  m[0] = cx(1); m[1] = cx(0); m[2] = cx(0); m[3] = cx(-1); break;
  }
}

// P (x) P on two targets with matrix index bit j <-> targets[j]: <r|PP|c> = p[r1][c1] p[r0][c0].
void pauli2(char p, Cx* m) {
  Cx a[4];
  pauli1(p, a);
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) m[r * 4 + c] = mul(a[((r >> 1) & 1) * 2 + ((c >> 1) & 1)], a[(r & 1) * 2 + (c & 1)]);
}

bool is_unitary(const Cx* m, int d) {
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c) {
      double re = 0, im = 0;
      for (int j = 0; j < d; ++j) {  // (U U^dagger)[r][c] = sum_j U[r][j] conj(U[c][j])
        const Cx a = m[r * d + j], b = m[c * d + j];
        re += a.re * b.re + a.im * b.im;
        im += a.im * b.re - a.re * b.im;
      }
      if (std::fabs(re - (r == c ? 1.0 : 0.0)) > 1e-10 || std::fabs(im) > 1e-10) return false;
    }
  return true;
}

bool kind_is_rotation(int kind) {
  return kind == SV_RX || kind == SV_RY || kind == SV_RZ || kind == SV_PS || kind == SV_RXX ||
         kind == SV_RYY || kind == SV_RZZ;
}

}  // namespace

int bind_gate(int n, const void* gp, const double* params, int32_t n_params, bool for_grad, BoundGate* out,
              std::string* err) {
  const sv_gate& g = *static_cast<const sv_gate*>(gp);
  BoundGate b;
  std::memset(&b, 0, sizeof(b));
  b.kind = g.kind;
  if (g.kind < 0 || g.kind >= SV_NUM_KINDS) { *err = "unknown gate kind"; return SV_E_ARG; }
  const bool two = g.kind >= SV_SWAP;
  b.t0 = g.targets[0];
  b.t1 = two ? g.targets[1] : -1;
  b.controls = g.controls;
  if (b.t0 < 0 || b.t0 >= n || (two && (b.t1 < 0 || b.t1 >= n))) { *err = "target qubit out of range"; return SV_E_QUBIT_RANGE; }
  if (n < 64 && (g.controls >> n) != 0) { *err = "control qubit out of range"; return SV_E_QUBIT_RANGE; }
  if (two && b.t0 == b.t1) { *err = "duplicate target"; return SV_E_DUPLICATE_TARGET; }
  uint64_t tmask = (1ull << b.t0) | (two ? (1ull << b.t1) : 0ull);
  if (g.controls & tmask) { *err = "control overlaps a target"; return SV_E_TARGET_CONTROL_OVERLAP; }
  if (g.param >= 0) {
    if (!kind_is_rotation(g.kind)) {
      *err = "parameter on a gate kind without a generator";
      return for_grad ? SV_E_NOT_DIFFERENTIABLE : SV_E_ARG;
    }
    if (g.param >= n_params || params == nullptr) { *err = "parameter index out of range"; return SV_E_PARAM_RANGE; }
  } else if (g.param < -1) {
    *err = "parameter index out of range";
    return SV_E_PARAM_RANGE;
  }
  const bool needs_mat = g.kind == SV_XLIKE || g.kind == SV_ZLIKE || g.kind == SV_MAT1 || g.kind == SV_MAT2;
  if (needs_mat && g.mat == nullptr) { *err = "matrix kind without mat"; return SV_E_ARG; }
  b.param = g.param;
  b.coeff = g.coeff;
  const double phi = (g.param >= 0 ? g.coeff * params[g.param] : 0.0) + g.offset;
  const double c = std::cos(phi / 2), s = std::sin(phi / 2);
  const double r = 0.7071067811865476;  // 1/sqrt(2), correctly rounded
  Cx* m = b.m;
  switch (g.kind) {
    case SV_X: b.cls = GC_XLIKE; m[0] = cx(1); m[1] = cx(1); break;
    case SV_Y: b.cls = GC_XLIKE; m[0] = cx(0, -1); m[1] = cx(0, 1); break;
    case SV_XLIKE: b.cls = GC_XLIKE; m[0] = cx(g.mat[0], g.mat[1]); m[1] = cx(g.mat[2], g.mat[3]); break;
    case SV_Z: b.cls = GC_ZLIKE; m[0] = cx(1); m[1] = cx(-1); break;
    case SV_S: b.cls = GC_ZLIKE; m[0] = cx(1); m[1] = cx(0, 1); break;
    case SV_SDG: b.cls = GC_ZLIKE; m[0] = cx(1); m[1] = cx(0, -1); break;
    case SV_T: b.cls = GC_ZLIKE; m[0] = cx(1); m[1] = cexpi(M_PI / 4); break;
    case SV_TDG: b.cls = GC_ZLIKE; m[0] = cx(1); m[1] = cexpi(-M_PI / 4); break;
    case SV_ZLIKE: b.cls = GC_ZLIKE; m[0] = cx(g.mat[0], g.mat[1]); m[1] = cx(g.mat[2], g.mat[3]); break;
    case SV_RZ: b.cls = GC_ZLIKE; m[0] = cexpi(-phi / 2); m[1] = cexpi(phi / 2); break;
    case SV_PS: b.cls = GC_ZLIKE; m[0] = cx(1); m[1] = cexpi(phi); break;
    case SV_H: b.cls = GC_GEN1; m[0] = cx(r); m[1] = cx(r); m[2] = cx(r); m[3] = cx(-r); break;
    case SV_RX: b.cls = GC_GEN1; m[0] = cx(c); m[1] = cx(0, -s); m[2] = cx(0, -s); m[3] = cx(c); break;
    case SV_RY: b.cls = GC_GEN1; m[0] = cx(c); m[1] = cx(-s); m[2] = cx(s); m[3] = cx(c); break;
    case SV_MAT1:
      b.cls = GC_GEN1;
      for (int e = 0; e < 4; ++e) m[e] = cx(g.mat[2 * e], g.mat[2 * e + 1]);
      break;
    case SV_SWAP: b.cls = GC_SWAP; break;
    case SV_RXX: case SV_RYY: {
      b.cls = GC_GEN2;
      Cx pp[16];
      pauli2(g.kind == SV_RXX ? 'X' : 'Y', pp);
      for (int e = 0; e < 16; ++e) m[e] = cx(((e % 5) == 0 ? c : 0.0) + s * pp[e].im, -s * pp[e].re);  // c I - i s PP
      break;
    }
    case SV_RZZ:
      // exp(-i phi Z(x)Z / 2): Z(x)Z = +1 on index 0 and 3, -1 on 1 and 2.
      b.cls = GC_DIAG2; m[0] = cexpi(-phi / 2); m[1] = cexpi(phi / 2); m[2] = cexpi(phi / 2); m[3] = cexpi(-phi / 2);
      break;
    case SV_MAT2:
      b.cls = GC_GEN2;
      for (int e = 0; e < 16; ++e) m[e] = cx(g.mat[2 * e], g.mat[2 * e + 1]);
      break;
  }
  if (for_grad) {
    // The reverse sweep un-applies U^dagger: user matrices must be unitary.
    Cx full[16];
    int d = 0;
    if (b.cls == GC_XLIKE) { d = 2; full[0] = cx(0); full[1] = m[0]; full[2] = m[1]; full[3] = cx(0); }
    else if (b.cls == GC_ZLIKE) { d = 2; full[0] = m[0]; full[1] = cx(0); full[2] = cx(0); full[3] = m[1]; }
    else if (b.cls == GC_GEN1) { d = 2; std::memcpy(full, m, sizeof(Cx) * 4); }
    else if (b.cls == GC_GEN2) { d = 4; std::memcpy(full, m, sizeof(Cx) * 16); }
    if (d && !is_unitary(full, d)) { *err = "user matrix is not unitary within 1e-10"; return SV_E_NOT_UNITARY; }
  }
  if (g.param >= 0) {
    // D = (dU/dphi) U^dagger on the target space: -(i/2) P for R_P, i|1><1| for PS.
    Cx p[16];
    if (g.kind == SV_PS) {
      b.gen_dim = 2;
      b.gen[0] = cx(0); b.gen[1] = cx(0); b.gen[2] = cx(0); b.gen[3] = cx(0, 1);
    } else {
      const bool pair = g.kind == SV_RXX || g.kind == SV_RYY || g.kind == SV_RZZ;
      const char axis = (g.kind == SV_RX || g.kind == SV_RXX) ? 'X' : (g.kind == SV_RY || g.kind == SV_RYY) ? 'Y' : 'Z';
      b.gen_dim = pair ? 4 : 2;
      if (pair) pauli2(axis, p); else pauli1(axis, p);
      for (int e = 0; e < b.gen_dim * b.gen_dim; ++e) b.gen[e] = cx(0.5 * p[e].im, -0.5 * p[e].re);  // -(i/2) p
    }
  }
  *out = b;
  return SV_OK;
}

// U^dagger of a bound gate (same class; generator unchanged: the sweep evaluates <lam|D|psi>
// before un-applying the gate).
BoundGate dagger(const BoundGate& g) {
  BoundGate d = g;
  auto cj = [](Cx a) { return Cx{a.re, -a.im}; };
  switch (g.cls) {
    case GC_XLIKE:  // [[0,a],[b,0]]^dagger = [[0, conj b], [conj a, 0]]
      d.m[0] = cj(g.m[1]); d.m[1] = cj(g.m[0]); break;
    case GC_ZLIKE: d.m[0] = cj(g.m[0]); d.m[1] = cj(g.m[1]); break;
    case GC_DIAG2: for (int j = 0; j < 4; ++j) d.m[j] = cj(g.m[j]); break;
    case GC_GEN1: for (int r = 0; r < 2; ++r) for (int c = 0; c < 2; ++c) d.m[c * 2 + r] = cj(g.m[r * 2 + c]); break;
    case GC_GEN2: for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) d.m[c * 4 + r] = cj(g.m[r * 4 + c]); break;
    case GC_SWAP: break;
  }
  return d;
}

}  // namespace sv
