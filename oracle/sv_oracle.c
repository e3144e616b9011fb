/*
 * oracle/sv_oracle.c — plain, slow, obviously-correct CPU oracle for the state-vector hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this file's library. The product path
 * (paper_2406_17248_b200/, include/sv.h) never includes, links or calls it, and this file
 * includes nothing from the product: its kind codes, matrix table, index helpers and
 * reductions are written out here independently.
 *
 * Precision: IEEE fp64 (complex128), as the paper fixes for its benchmarks ("double precision",
 * PAPER.md §7.1; "complex128 data type" §3.1). Built with -O2 -ffp-contract=off, no
 * -ffast-math, so every multiply and add rounds separately.
 *
 * What each function follows (P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * SURVEY.md §8(c) readings c2.k listed in DESIGN.md):
 *   or_gate_matrix      — gate matrices: X-like [[0,a],[b,0]] (§3.1 eq. P:80-87), Z-like
 *                         diag(a,b) (§3.1 eq. P:88-94), general / two-qubit kinds of the §7.1 gate
 *                         list; rotation convention R_P(t) = exp(-i t P / 2) (
 *                         reading c2.1); 4x4 basis bit j <-> targets[j] (reading c2.5).
 *   or_apply_matrix     — "interaction between quantum gate and quantum state" (§3.1): the
 *                         plain definition psi <- (Pi_C (x) M + (1 - Pi_C) (x) I) psi, qubit 0 =
 *                         least-significant index bit (Fig. 3; reading c2.2), arbitrary
 *                         control set ("Any control on any gate", Fig. 1).
 *   or_apply_circuit    — "Evolution of Circuit" (Fig. 1): gates in array order.
 *   or_expectation      — "Expectation of Observable" (Fig. 1), <psi|H|psi> for a Pauli sum
 *                         (pure-state form of <H> = tr(rho H), §3.2); each Pauli string
 *                         applied one qubit at a time through or_apply_matrix on a copy.
 *   or_adjoint_grad     — "Gradient calculation" (Fig. 1) by the adjoint method (§7.2 P:606;
 *                         the §4.1 body is absent, reading c2.8): forward pass, lambda = H psi,
 *                         reverse sweep un-applying U_k^dagger from psi and lambda, in that order.
 *   or_shift_grad       — exact parameter-shift rules per gate occurrence (2-term / 4-term,
 *                         reading c2.10), a second, independent gradient definition.
 *   or_sample           — "Sampling Measurement" (Fig. 1): inverse CDF of
 *                         |psi_i|^2 with SplitMix64 counter-based uniforms (sv.h contract).
 * Reductions: Neumaier compensated sums over fixed chunks combined in fixed order, so results do
 * not depend on the OpenMP thread count (reading c2.16).
 *
 * Parity pins for every function: tests/test_oracle.py (brute-force Kronecker products, closed
 * forms, SPEC worked values under tests/golden/).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

/* Oracle-private kind codes (the Python wrapper maps kind names to these). */
enum {
  OR_X = 0, OR_Y, OR_Z, OR_H, OR_S, OR_SDG, OR_T, OR_TDG,
  OR_RX, OR_RY, OR_RZ, OR_PS, OR_XLIKE, OR_ZLIKE, OR_MAT1,
  OR_SWAP, OR_RXX, OR_RYY, OR_RZZ, OR_MAT2, OR_NKINDS
};

int or_num_targets(int kind) {
  return (kind >= OR_SWAP && kind <= OR_MAT2) ? 2 : 1;
}

int or_is_parametrised(int kind) {
  return kind == OR_RX || kind == OR_RY || kind == OR_RZ || kind == OR_PS ||
         kind == OR_RXX || kind == OR_RYY || kind == OR_RZZ;
}

/* ---- gate matrices (row-major, dim x dim complex; dim = 2 or 4) ---- */

static void set2(cplx* m, cplx a, cplx b, cplx c, cplx d) { m[0] = a; m[1] = b; m[2] = c; m[3] = d; }

/* Builds the target-space matrix of `kind` at angle phi into m (dim*dim entries). `user` holds,
 * for XLIKE/ZLIKE: (a_re, a_im, b_re, b_im); MAT1: 4 complex row-major; MAT2: 16 complex.
 * Returns the dimension, or 0 for an unknown kind. */
int or_gate_matrix_c(int kind, double phi, const double* user, cplx* m) {
  const double c = cos(phi / 2.0), s = sin(phi / 2.0);
  const double r = 0.7071067811865476; /* M_SQRT1_2, correctly rounded (reading in DESIGN.md) */
  switch (kind) {
    case OR_X: set2(m, 0, 1, 1, 0); return 2;
    case OR_Y: set2(m, 0, -I, I, 0); return 2;
    case OR_Z: set2(m, 1, 0, 0, -1); return 2;
    case OR_H: set2(m, r, r, r, -r); return 2;
    case OR_S: set2(m, 1, 0, 0, I); return 2;
    case OR_SDG: set2(m, 1, 0, 0, -I); return 2;
    case OR_T: set2(m, 1, 0, 0, cexp(I * M_PI / 4.0)); return 2;
    case OR_TDG: set2(m, 1, 0, 0, cexp(-I * M_PI / 4.0)); return 2;
    case OR_RX: set2(m, c, -I * s, -I * s, c); return 2;                 /* exp(-i phi X/2) */
    case OR_RY: set2(m, c, -s, s, c); return 2;                          /* exp(-i phi Y/2) */
    case OR_RZ: set2(m, cexp(-I * phi / 2.0), 0, 0, cexp(I * phi / 2.0)); return 2;
    case OR_PS: set2(m, 1, 0, 0, cexp(I * phi)); return 2;
    case OR_XLIKE: set2(m, 0, user[0] + I * user[1], user[2] + I * user[3], 0); return 2;
    case OR_ZLIKE: set2(m, user[0] + I * user[1], 0, 0, user[2] + I * user[3]); return 2;
    case OR_MAT1:
      for (int e = 0; e < 4; ++e) m[e] = user[2 * e] + I * user[2 * e + 1];
      return 2;
    default: break;
  }
  for (int e = 0; e < 16; ++e) m[e] = 0;
  switch (kind) {
    case OR_SWAP: m[0] = 1; m[1 * 4 + 2] = 1; m[2 * 4 + 1] = 1; m[15] = 1; return 4;
    case OR_RXX: /* c I - i s X(x)X ; X(x)X maps basis j -> 3-j */
      for (int j = 0; j < 4; ++j) { m[j * 4 + j] = c; m[j * 4 + (3 - j)] = -I * s; }
      return 4;
    case OR_RYY: { /* c I - i s Y(x)Y ; Y(x)Y = [[0,0,0,-1],[0,0,1,0],[0,1,0,0],[-1,0,0,0]] */
      const double yy[4] = {-1, 1, 1, -1};
      for (int j = 0; j < 4; ++j) { m[j * 4 + j] = c; m[j * 4 + (3 - j)] = -I * s * yy[j]; }
      return 4;
    }
    case OR_RZZ: { /* exp(-i phi Z(x)Z / 2); Z(x)Z eigenvalue +1 on |00>,|11>, -1 on |01>,|10> */
      const double zz[4] = {1, -1, -1, 1};
      for (int j = 0; j < 4; ++j) m[j * 4 + j] = cexp(-I * phi * zz[j] / 2.0);
      return 4;
    }
    case OR_MAT2:
      for (int e = 0; e < 16; ++e) m[e] = user[2 * e] + I * user[2 * e + 1];
      return 4;
    default: return 0;
  }
}

/* Real-array export of the table for the tests: out = 2*dim*dim doubles. */
int or_gate_matrix(int kind, double phi, const double* user, double* out) {
  cplx m[16];
  int d = or_gate_matrix_c(kind, phi, user, m);
  for (int e = 0; e < d * d; ++e) { out[2 * e] = creal(m[e]); out[2 * e + 1] = cimag(m[e]); }
  return d;
}

/* Matrix of D = (dU/dphi) U^dagger restricted to the target space (reading c2.10):
 * R_P: -(i/2) P ; PS: i |1><1|. Returns dim, 0 if kind is not parametrised. */
static int or_generator_c(int kind, cplx* m) {
  cplx p[16];
  int d;
  switch (kind) {
    case OR_RX: d = or_gate_matrix_c(OR_X, 0, NULL, p); break;
    case OR_RY: d = or_gate_matrix_c(OR_Y, 0, NULL, p); break;
    case OR_RZ: d = or_gate_matrix_c(OR_Z, 0, NULL, p); break;
    case OR_PS: set2(m, 0, 0, 0, I); return 2;
    case OR_RXX: case OR_RYY: case OR_RZZ: {
      /* P = P1 (x) P1 built entrywise: <r|P(x)P|c> = P1[r1][c1] * P1[r0][c0], bit j <-> target j */
      cplx p1[4];
      or_gate_matrix_c(kind == OR_RXX ? OR_X : kind == OR_RYY ? OR_Y : OR_Z, 0, NULL, p1);
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c)
          p[r * 4 + c] = p1[((r >> 1) & 1) * 2 + ((c >> 1) & 1)] * p1[(r & 1) * 2 + (c & 1)];
      d = 4;
      break;
    }
    default: return 0;
  }
  for (int e = 0; e < d * d; ++e) m[e] = -0.5 * I * p[e];
  return d;
}

/* ---- the generic gate application (plain definition) ---- */

/* psi <- (Pi_C (x) M + (1 - Pi_C) (x) I) psi. k targets (1 or 2), M is 2^k x 2^k row-major with
 * matrix index bit b <-> targets[b]. Indices whose control bits are not all 1 are untouched. */
void or_apply_matrix_c(cplx* psi, int n, int k, const int* targets, uint64_t cmask, const cplx* M) {
  const int64_t N = (int64_t)1 << n;
  const int dim = 1 << k;
  uint64_t tmask = 0;
  for (int b = 0; b < k; ++b) tmask |= (uint64_t)1 << targets[b];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    if ((i & tmask) != 0 || (i & cmask) != cmask) continue;
    int64_t idx[4];
    cplx v[4], w[4];
    for (int j = 0; j < dim; ++j) {
      idx[j] = i;
      for (int b = 0; b < k; ++b)
        if ((j >> b) & 1) idx[j] |= (int64_t)1 << targets[b];
      v[j] = psi[idx[j]];
    }
    for (int r = 0; r < dim; ++r) {
      cplx acc = 0;
      for (int c = 0; c < dim; ++c) acc += M[r * dim + c] * v[c];
      w[r] = acc;
    }
    for (int j = 0; j < dim; ++j) psi[idx[j]] = w[j];
  }
}

void or_apply_matrix(double* psi, int n, int k, const int* targets, uint64_t cmask, const double* mat) {
  cplx M[16];
  for (int e = 0; e < (1 << k) * (1 << k); ++e) M[e] = mat[2 * e] + I * mat[2 * e + 1];
  or_apply_matrix_c((cplx*)psi, n, k, targets, cmask, M);
}

/* ---- circuits ---- */

/* Per-gate description: kind, targets[2], control mask, parameter index (-1 = fixed), angle =
 * coeff * params[param] + offset (or offset when param == -1), user matrix (32 doubles). */
typedef struct {
  const int32_t* kinds;
  const int32_t* targets;   /* 2 per gate */
  const uint64_t* cmasks;
  const int32_t* pidx;
  const double* coeff;
  const double* offset;
  const double* mats;       /* 32 per gate */
} or_circuit;

static double or_angle(const or_circuit* c, int64_t g, const double* params) {
  return (c->pidx[g] >= 0 ? c->coeff[g] * params[c->pidx[g]] : 0.0) + c->offset[g];
}

static void or_conj_transpose(int d, const cplx* m, cplx* out) {
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < d; ++c) out[c * d + r] = conj(m[r * d + c]);
}

/* Applies gate g (or its inverse when dagger != 0), with `extra` added to its angle. */
/* Instrumented gate-application counter (SPEC S:478, S:695 cost contract): every application of a
 * circuit gate (or its inverse) to a state vector through or_apply_gate increments it. */
static int64_t or_gate_applications = 0;
int64_t or_get_gate_applications(void) { return or_gate_applications; }
void or_reset_gate_applications(void) { or_gate_applications = 0; }

static void or_apply_gate(cplx* psi, int n, const or_circuit* c, int64_t g, const double* params,
                          double extra, int dagger) {
  cplx m[16], md[16];
  ++or_gate_applications;
  int d = or_gate_matrix_c(c->kinds[g], or_angle(c, g, params) + extra, c->mats + 32 * g, m);
  if (dagger) { or_conj_transpose(d, m, md); memcpy(m, md, sizeof(cplx) * d * d); }
  or_apply_matrix_c(psi, n, d == 4 ? 2 : 1, c->targets + 2 * g, c->cmasks[g], m);
}

/* psi <- U_N ... U_1 psi. shift_gate >= 0 adds `shift` to that one gate's angle (for shift rules). */
void or_apply_circuit(double* psi, int n, int64_t ngates, const int32_t* kinds, const int32_t* targets,
                      const uint64_t* cmasks, const int32_t* pidx, const double* coeff,
                      const double* offset, const double* mats, const double* params,
                      int64_t shift_gate, double shift) {
  or_circuit c = {kinds, targets, cmasks, pidx, coeff, offset, mats};
  for (int64_t g = 0; g < ngates; ++g)
    or_apply_gate((cplx*)psi, n, &c, g, params, g == shift_gate ? shift : 0.0, 0);
}

void or_apply_circuit_dagger(double* psi, int n, int64_t ngates, const int32_t* kinds,
                             const int32_t* targets, const uint64_t* cmasks, const int32_t* pidx,
                             const double* coeff, const double* offset, const double* mats,
                             const double* params) {
  or_circuit c = {kinds, targets, cmasks, pidx, coeff, offset, mats};
  for (int64_t g = ngates - 1; g >= 0; --g) or_apply_gate((cplx*)psi, n, &c, g, params, 0.0, 1);
}

/* ---- compensated reductions ---- */

typedef struct { double s, c; } neum;
static void neum_add(neum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x; else a->c += (x - t) + a->s;
  a->s = t;
}
static double neum_val(const neum* a) { return a->s + a->c; }

#define OR_CHUNK ((int64_t)1 << 16)

/* <a|b> = sum_i conj(a_i) b_i, Neumaier-summed per fixed chunk, chunks combined in order. */
static cplx or_inner(const cplx* a, const cplx* b, int64_t N) {
  int64_t nch = (N + OR_CHUNK - 1) / OR_CHUNK;
  double* part = (double*)malloc(sizeof(double) * 2 * nch);
#pragma omp parallel for schedule(static)
  for (int64_t ch = 0; ch < nch; ++ch) {
    neum re = {0, 0}, im = {0, 0};
    int64_t end = (ch + 1) * OR_CHUNK < N ? (ch + 1) * OR_CHUNK : N;
    for (int64_t i = ch * OR_CHUNK; i < end; ++i) {
      cplx p = conj(a[i]) * b[i];
      neum_add(&re, creal(p));
      neum_add(&im, cimag(p));
    }
    part[2 * ch] = neum_val(&re);
    part[2 * ch + 1] = neum_val(&im);
  }
  neum re = {0, 0}, im = {0, 0};
  for (int64_t ch = 0; ch < nch; ++ch) { neum_add(&re, part[2 * ch]); neum_add(&im, part[2 * ch + 1]); }
  free(part);
  return neum_val(&re) + I * neum_val(&im);
}

/* ---- Pauli sums ---- */

/* ops: nterms x n bytes, op[t*n + q] in {0:I, 1:X, 2:Y, 3:Z}. out <- P_t psi (out preallocated). */
static void or_apply_pauli_string(const cplx* psi, cplx* out, int n, const uint8_t* op) {
  const int64_t N = (int64_t)1 << n;
  memcpy(out, psi, sizeof(cplx) * N);
  static const int kind_of[4] = {-1, OR_X, OR_Y, OR_Z};
  for (int q = 0; q < n; ++q) {
    if (op[q] == 0) continue;
    cplx m[4];
    or_gate_matrix_c(kind_of[op[q]], 0, NULL, m);
    or_apply_matrix_c(out, n, 1, &q, 0, m);
  }
}

/* E = sum_t coeff_t <psi|P_t|psi>; returns the real part in *e_re and the (should-be-zero)
 * imaginary part in *e_im. Term contributions combined with Neumaier summation. */
void or_expectation(const double* psi_, int n, int64_t nterms, const uint8_t* ops, const double* coeffs,
                    double* e_re, double* e_im) {
  const cplx* psi = (const cplx*)psi_;
  const int64_t N = (int64_t)1 << n;
  cplx* tmp = (cplx*)malloc(sizeof(cplx) * N);
  neum re = {0, 0}, im = {0, 0};
  for (int64_t t = 0; t < nterms; ++t) {
    or_apply_pauli_string(psi, tmp, n, ops + t * n);
    cplx v = or_inner(psi, tmp, N);
    neum_add(&re, coeffs[t] * creal(v));
    neum_add(&im, coeffs[t] * cimag(v));
  }
  free(tmp);
  *e_re = neum_val(&re);
  *e_im = neum_val(&im);
}

/* lam <- H psi = sum_t coeff_t P_t psi (sum over terms in order). */
static void or_apply_hamiltonian(const cplx* psi, cplx* lam, int n, int64_t nterms, const uint8_t* ops,
                                 const double* coeffs) {
  const int64_t N = (int64_t)1 << n;
  cplx* tmp = (cplx*)malloc(sizeof(cplx) * N);
  memset(lam, 0, sizeof(cplx) * N);
  for (int64_t t = 0; t < nterms; ++t) {
    or_apply_pauli_string(psi, tmp, n, ops + t * n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) lam[i] += coeffs[t] * tmp[i];
  }
  free(tmp);
}

/* Re <lam| D |psi> with D = Pi_C (x) G on the gate's targets, G = or_generator_c(kind). */
static double or_generator_overlap(const cplx* lam, const cplx* psi, int n, int kind, const int* targets,
                                   uint64_t cmask) {
  const int64_t N = (int64_t)1 << n;
  cplx G[16];
  int d = or_generator_c(kind, G);
  int k = d == 4 ? 2 : 1;
  uint64_t tmask = 0;
  for (int b = 0; b < k; ++b) tmask |= (uint64_t)1 << targets[b];
  cplx* dpsi = (cplx*)calloc(N, sizeof(cplx));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    if ((i & tmask) != 0 || (i & cmask) != cmask) continue;
    int64_t idx[4];
    cplx v[4];
    for (int j = 0; j < d; ++j) {
      idx[j] = i;
      for (int b = 0; b < k; ++b)
        if ((j >> b) & 1) idx[j] |= (int64_t)1 << targets[b];
      v[j] = psi[idx[j]];
    }
    for (int r = 0; r < d; ++r) {
      cplx acc = 0;
      for (int c = 0; c < d; ++c) acc += G[r * d + c] * v[c];
      dpsi[idx[r]] = acc;
    }
  }
  cplx o = or_inner(lam, dpsi, N);
  free(dpsi);
  return creal(o);
}

/* Adjoint-method gradient, step by step:
 *   1. psi <- psi0; for k = 1..N: psi <- U_k psi
 *   2. lam <- H psi; E <- Re <psi|lam>
 *   3. for k = N..1: if gate k is parametrised: g[p(k)] += coeff_k * 2 Re <lam|D_k|psi>;
 *                    psi <- U_k^dagger psi; lam <- U_k^dagger lam
 * psi0 is not modified. Returns 0, or -1 if a parametrised occurrence has a non-differentiable kind. */
int or_adjoint_grad(const double* psi0, int n, int64_t ngates, const int32_t* kinds, const int32_t* targets,
                    const uint64_t* cmasks, const int32_t* pidx, const double* coeff, const double* offset,
                    const double* mats, const double* params, int32_t nparams, int64_t nterms,
                    const uint8_t* ops, const double* hcoeffs, double* out_e, double* out_grad) {
  const int64_t N = (int64_t)1 << n;
  or_circuit c = {kinds, targets, cmasks, pidx, coeff, offset, mats};
  for (int64_t g = 0; g < ngates; ++g)
    if (pidx[g] >= 0 && !or_is_parametrised(kinds[g])) return -1;
  cplx* psi = (cplx*)malloc(sizeof(cplx) * N);
  cplx* lam = (cplx*)malloc(sizeof(cplx) * N);
  memcpy(psi, psi0, sizeof(cplx) * N);
  for (int64_t g = 0; g < ngates; ++g) or_apply_gate(psi, n, &c, g, params, 0.0, 0);
  or_apply_hamiltonian(psi, lam, n, nterms, ops, hcoeffs);
  *out_e = creal(or_inner(psi, lam, N));
  neum* acc = (neum*)calloc(nparams > 0 ? nparams : 1, sizeof(neum));
  for (int64_t g = ngates - 1; g >= 0; --g) {
    if (pidx[g] >= 0) {
      double d = or_generator_overlap(lam, psi, n, kinds[g], targets + 2 * g, cmasks[g]);
      neum_add(&acc[pidx[g]], coeff[g] * 2.0 * d);
    }
    or_apply_gate(psi, n, &c, g, params, 0.0, 1);
    or_apply_gate(lam, n, &c, g, params, 0.0, 1);
  }
  for (int32_t p = 0; p < nparams; ++p) out_grad[p] = neum_val(&acc[p]);
  free(acc);
  free(psi);
  free(lam);
  return 0;
}

/* E(circuit with gate `shift_gate`'s angle shifted by `shift`) from psi0. */
static double or_shifted_energy(const double* psi0, int n, const or_circuit* c, int64_t ngates,
                                const double* params, int64_t shift_gate, double shift, int64_t nterms,
                                const uint8_t* ops, const double* hcoeffs, cplx* work) {
  const int64_t N = (int64_t)1 << n;
  memcpy(work, psi0, sizeof(cplx) * N);
  or_apply_circuit((double*)work, n, ngates, c->kinds, c->targets, c->cmasks, c->pidx, c->coeff, c->offset,
                   c->mats, params, shift_gate, shift);
  double re, im;
  or_expectation((const double*)work, n, nterms, ops, hcoeffs, &re, &im);
  return re;
}

/* Exact parameter-shift gradient, each occurrence shifted separately (reading c2.10):
 *   uncontrolled R_P, and PS with any controls: dE/dphi = [E(+pi/2) - E(-pi/2)] / 2 ... (for PS the
 *     generator |1><1| has spectrum {0,1}: dE/dphi = [E(+pi/2) - E(-pi/2)] / 2 as well)
 *   controlled R_P (generator spectrum {0, +-1/2}):
 *     dE/dphi = d+ [E(+pi/2) - E(-pi/2)] - d- [E(+3pi/2) - E(-3pi/2)], d+- = (sqrt2 +- 1)/(4 sqrt2).
 * g[p] = sum over occurrences of coeff_k * dE/dphi_k. Returns -1 on a non-differentiable kind. */
int or_shift_grad(const double* psi0, int n, int64_t ngates, const int32_t* kinds, const int32_t* targets,
                  const uint64_t* cmasks, const int32_t* pidx, const double* coeff, const double* offset,
                  const double* mats, const double* params, int32_t nparams, int64_t nterms,
                  const uint8_t* ops, const double* hcoeffs, double* out_grad) {
  const int64_t N = (int64_t)1 << n;
  or_circuit c = {kinds, targets, cmasks, pidx, coeff, offset, mats};
  cplx* work = (cplx*)malloc(sizeof(cplx) * N);
  for (int32_t p = 0; p < nparams; ++p) out_grad[p] = 0;
  const double dp = (sqrt(2.0) + 1.0) / (4.0 * sqrt(2.0)), dm = (sqrt(2.0) - 1.0) / (4.0 * sqrt(2.0));
  for (int64_t g = 0; g < ngates; ++g) {
    if (pidx[g] < 0) continue;
    if (!or_is_parametrised(kinds[g])) { free(work); return -1; }
    double ep = or_shifted_energy(psi0, n, &c, ngates, params, g, M_PI / 2, nterms, ops, hcoeffs, work);
    double em = or_shifted_energy(psi0, n, &c, ngates, params, g, -M_PI / 2, nterms, ops, hcoeffs, work);
    double deriv;
    if (kinds[g] == OR_PS || cmasks[g] == 0) {
      deriv = 0.5 * (ep - em);
    } else {
      double ep3 = or_shifted_energy(psi0, n, &c, ngates, params, g, 1.5 * M_PI, nterms, ops, hcoeffs, work);
      double em3 = or_shifted_energy(psi0, n, &c, ngates, params, g, -1.5 * M_PI, nterms, ops, hcoeffs, work);
      deriv = dp * (ep - em) - dm * (ep3 - em3);
    }
    out_grad[pidx[g]] += coeff[g] * deriv;
  }
  free(work);
  return 0;
}

/* psi <- |0...0>. */
void or_state_zero(double* psi, int n) {
  memset(psi, 0, sizeof(double) * 2 * ((size_t)1 << n));
  psi[0] = 1.0;
}

/* ---- sampling measurement ("Sampling Measurement", Fig. 1) ----
 * The plain inverse-CDF definition: with p_i = |psi_i|^2 and the running sums F_i = p_0 + ... + p_i
 * (left to right), shot s draws the basis index
 *     i_s = min { i : F_i >= u_s * F_{N-1} }   (N - 1 if no such i),
 * u_s = (splitmix64(seed + s) >> 11) * 2^-53 in [0, 1) — the counter-based uniform the library's
 * contract fixes (include/sv.h sv_sample), implemented here on its own: SplitMix64's published
 * output function (golden constant 0x9E3779B97F4A7C15, shifts 30/27/31, multipliers
 * 0xBF58476D1CE4E5B9 / 0x94D049BB133111EB). Marginals over measured qubits are read off i_s by the
 * caller. One binary search per shot over F (no sorting, no blocking). */
uint64_t or_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void or_sample(const double* psi_, int n, int64_t shots, uint64_t seed, int64_t* out_index) {
  const cplx* psi = (const cplx*)psi_;
  const int64_t N = (int64_t)1 << n;
  double* F = (double*)malloc(sizeof(double) * N);
  double run = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    double p = creal(psi[i]) * creal(psi[i]) + cimag(psi[i]) * cimag(psi[i]);
    run += p;
    F[i] = run;
  }
  const double total = F[N - 1];
  for (int64_t s = 0; s < shots; ++s) {
    const double u = (double)(or_splitmix64(seed + (uint64_t)s) >> 11) * (1.0 / 9007199254740992.0) * total;
    int64_t lo = 0, hi = N - 1; /* smallest i in [lo, hi] with F_i >= u (hi if none) */
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (F[mid] >= u) hi = mid; else lo = mid + 1;
    }
    out_index[s] = lo;
  }
  free(F);
}
