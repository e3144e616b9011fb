/*
 * sv.h — C ABI of the B200-native state-vector hot path (after MindSpore Quantum's "mqvector",
 * arXiv:2406.17248). Plain C types only: no torch, no CUDA types in any signature.
 *
 * Citations: P:n = PAPER.md line n (the paper text), S:n = SPEC.md line n, "reading cN" = the
 * DESIGN.md "Readings of the paper" entry N.
 *
 * What the library computes:
 *   a1  sv_create / sv_reset: the state psi = |0...0> of n qubits, 2^n complex128 amplitudes,
 *       interleaved (re, im), qubit 0 = least-significant index bit (Fig. 3, P:38-78, P:70-74;
 *       reading c2).
 *   a2  host side of every apply call: validate, bind angles (angle = coeff * params[param] +
 *       offset), classify by the paper's gate taxonomy — X-like anti-diagonal [[0,a],[b,0]]
 *       (§3.1 eq. P:80-87), Z-like diagonal [[a,0],[0,b]] (§3.1 eq. P:88-94), general 1-/2-qubit
 *       matrix gates (§7.1 gate list P:579) — with an arbitrary control set on any gate
 *       (Fig. 1 "Any control on any gate") — and plan fused passes.
 *   a3  sv_apply_gate / sv_apply_circuit: "Evolution of Circuit" (Fig. 1): psi <- U_N..U_1 psi.
 *   a4  sv_expectation: "Expectation of Observable" (Fig. 1): <psi|H|psi> for a real Pauli
 *       sum H (pure-state form of <H> = tr(rho H), §3.2).
 *   a5-a7 sv_expectation_with_grad: "Gradient calculation" (Fig. 1) by the adjoint method
 *       ("optimized adjoint method", §7.2; §4.1 body absent -> reading c8): E and dE/dtheta.
 *
 * Conventions: rotations R_P(t) = exp(-i t P / 2) for P in {X, Y, Z, XX, YY, ZZ} (reading
 * c1); PS(t) = diag(1, e^{i t}); H uses the correctly-rounded 1/sqrt(2) = 0.7071067811865476; a
 * two-qubit matrix's index bit j <-> targets[j] (reading c5).
 *
 * Errors: every entry point returns sv_status (0 = SV_OK). No exceptions cross the ABI. On error
 * nothing is applied (a circuit is validated as a whole before any device work) and
 * sv_last_error() returns a thread-local description. Asynchronous CUDA/NCCL failures surface at
 * the next synchronous call as SV_E_CUDA / SV_E_NCCL and poison the handle (SV_E_POISONED after).
 *
 * Ownership: the caller owns every array it passes; nothing is retained after a call returns.
 * A handle owns its device memory (cudaMalloc on the device current at creation); every entry point
 * makes that device current for the call and restores the caller's current device on return.
 * Handles are single-owner (not thread-safe); distinct handles, also on different devices, may be
 * used concurrently from different threads.
 *
 * Synchrony: sv_apply_* enqueue work on the handle's stream and return (asynchronous to the host,
 * stream-ordered). sv_expectation*, sv_get_state* synchronize the stream before returning.
 */
#ifndef SV_H_
#define SV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sv_state_s* sv_handle;
typedef int32_t sv_status;

enum {
  SV_OK = 0,
  SV_E_ARG = 1,                    /* null pointer, bad size, unknown kind, bad world size ...      */
  SV_E_QUBIT_RANGE = 2,            /* a target / control / Pauli index >= n                  */
  SV_E_TARGET_CONTROL_OVERLAP = 3, /* controls intersect targets                      */
  SV_E_DUPLICATE_TARGET = 4,       /* two-qubit gate with targets[0] == targets[1]           */
  SV_E_PARAM_RANGE = 5,            /* param index outside [0, n_params) (S:66 MissingParameter)      */
  SV_E_NOT_DIFFERENTIABLE = 6,     /* a param on a kind without a generator                  */
  SV_E_NOT_UNITARY = 7,            /* user matrix not unitary within 1e-10 in _with_grad     */
  SV_E_OOM = 8,                    /* device allocation failed (construction-time error)      */
  SV_E_CUDA = 9,
  SV_E_NCCL = 10,
  SV_E_POISONED = 11               /* a previous asynchronous failure poisoned this handle           */
};

/* Gate kinds, grouped by the paper's taxonomy (§3.1; reading c6). CNOT = SV_X with one
 * control, CZ = SV_Z with one control. */
enum sv_kind {
  /* X-like: anti-diagonal [[0,a],[b,0]] */
  SV_X = 0, SV_Y = 1, SV_XLIKE = 2,
  /* Z-like: diagonal [[a,0],[0,b]] */
  SV_Z = 3, SV_S = 4, SV_SDG = 5, SV_T = 6, SV_TDG = 7, SV_ZLIKE = 8, SV_RZ = 9, SV_PS = 10,
  /* general 2x2 */
  SV_H = 11, SV_RX = 12, SV_RY = 13, SV_MAT1 = 14,
  /* two-qubit (RZZ is diagonal) */
  SV_SWAP = 15, SV_RXX = 16, SV_RYY = 17, SV_RZZ = 18, SV_MAT2 = 19,
  SV_NUM_KINDS = 20
};

/* One gate. targets[1] is ignored for one-qubit kinds. controls: bit q set <=> qubit q is a
 * control (arbitrary set, disjoint from targets). param: index into params, or -1 for a
 * fixed gate; angle = coeff * params[param] + offset when param >= 0, else offset (rotation kinds
 * only; SV_E_ARG if a non-rotation kind carries param >= 0 outside _with_grad, where it is
 * SV_E_NOT_DIFFERENTIABLE). mat: XLIKE/ZLIKE -> (a_re, a_im, b_re, b_im); MAT1 -> 8 doubles
 * (2x2 row-major interleaved); MAT2 -> 32 doubles (4x4, index bit j <-> targets[j]); NULL for
 * other kinds. */
typedef struct {
  int32_t kind;
  int32_t targets[2];
  uint64_t controls;
  int32_t param;
  double coeff;
  double offset;
  const double* mat;
} sv_gate;

/* One Pauli term coeff * i^{popc(x&z)} X^x Z^z: qubit q carries X if x_q=1,z_q=0; Y if both;
 * Z if x_q=0,z_q=1. Real coeff => H Hermitian by construction; identity term allowed. */
typedef struct {
  uint64_t x_mask;
  uint64_t z_mask;
  double coeff;
} sv_pauli;

/* Counters since creation (or the last sv_reset_stats), for bench / roofline reporting. */
typedef struct {
  int64_t kernel_launches;       /* every kernel this library launched                           */
  int64_t gate_passes;           /* fused forward gate passes (one HBM read+write of the state)   */
  int64_t adjoint_passes;        /* fused reverse passes over (psi, lambda)                       */
  int64_t expectation_passes;    /* Pauli-group passes (expectation and lambda = H psi)           */
  int64_t exchanges;             /* sharded: global<->local qubit swaps                           */
  double algorithmic_bytes;      /* HBM bytes the executed plan must move   */
  int64_t gates_applied;         /* gates of the user's circuits applied (forward only)           */
  double exchange_bytes;         /* sharded: bytes this handle sent to peers in qubit swaps and
                                    cross-shard Pauli streams (each direction counted once)      */
  double exchange_ms;            /* sharded: device time of those exchanges (CUDA events around each
                                    exchange on the handle's stream; summed at sv_get_stats)      */
  int64_t gate_applications;     /* instrumented cost counter: gate-vector
                                    applications the executed plans performed — a forward plan of N
                                    gates adds N, an adjoint plan 2N (psi and lambda)             */
  int64_t plan_builds;           /* host plans built from scratch                                  */
  int64_t plan_refreshes;        /* host plans reused by structure with new matrix values (new
                                    angles of the same circuit: passes and stages kept)          */
} sv_stats;

/* Option keys for sv_set_option (A/B evidence; defaults are the tuned values). */
enum {
  SV_OPT_TILE_QUBITS = 1,        /* k: qubits per fused tile (0 = auto)                           */
  SV_OPT_FUSION = 2,             /* 1 (default) fuse gates into tile passes; 0 one pass per gate  */
  SV_OPT_LOW_QUBITS = 3,         /* qubits 0..L-1 always in a tile (coalescing granule), default 3 */
  SV_OPT_DENSE = 4,              /* 1 (default): fold register stages into dense FP64-MMA stages  */
  SV_OPT_KERNEL = 5,             /* 1 (default): register-blocked kernel; 0: shared-memory kernel */
  SV_OPT_ADJOINT_DENSE_COST = 6, /* reverse-sweep stages whose sequential cost (2 x FMA/amp + 8 per
                                   parametrised op) reaches this run as adjoint dense MMA stages;
                                   -1 (default): 96 for states of >= 24 local qubits, else 250
                                   (their fixed per-pass costs amortise over large states only);
                                   0: every eligible stage (incl. one outer variant bit at any
                                   size); 1 << 20: none */
  SV_OPT_C64_SPLIT = 7           /* complex64 dense stages: 3 (default) TF32 products of the hi/lo
                                   split (~2^-21 relative per product); 0: passes of dense stages
                                   only widen the tile to FP64 and run the Gauss DMMA stages of the
                                   complex128 kernel (FP32 rounding once per stage; slower than 3
                                   on B200); 1: the single hi x hi TF32 product (~2^-11) — kept
                                   only to show the tests' tolerance detects a precision loss */
};

/* a1: |0...0> on n_qubits (1 <= n <= 40 subject to memory), current CUDA device, new stream. */
sv_status sv_create(int32_t n_qubits, sv_handle* out);

/* Sharded state (SPMD, one process per GPU): the top log2(world) qubits are global; rank r holds
 * the 2^(n - log2 world) amplitudes whose global bits equal r. nccl_id points at the 128-byte
 * ncclUniqueId rank 0 created with sv_nccl_unique_id and broadcast (e.g. via torch.distributed).
 * world in {1, 2, 4, 8, ...} (power of two). Every rank must then make identical calls. */
sv_status sv_create_sharded(int32_t n_qubits, int32_t rank, int32_t world, const void* nccl_id, sv_handle* out);

/* Writes a fresh ncclUniqueId (128 bytes) into out (call on rank 0 only). */
sv_status sv_nccl_unique_id(void* out, int32_t out_bytes);

/* Loopback sharding on ONE GPU: `world` virtual shards, each its own device buffer, exchanges as
 * device-to-device copies. Same planner and exchange schedule as sv_create_sharded; used to test
 * the sharded path without several GPUs. */
sv_status sv_create_virtual_shards(int32_t n_qubits, int32_t world, sv_handle* out);

/* NEXT-4 density matrix ("mqmatrix", §3.2): rho of n qubits (initially
 * |0..0><0..0|) held as a 2n-qubit vector vec[r + 2^n c] = rho[r][c]. On such a handle
 * sv_apply_gate / sv_apply_circuit apply rho <- U rho U^dagger (eq. at: U on the row
 * qubits, U* on the column qubits, one fused pass plan over 2n qubits), sv_expectation returns
 * <H> = tr(rho H) (eq. at), sv_get_state / sv_set_state transfer rho row-major
 * (2 * 4^n doubles: rho[r][c] at 2 (r 2^n + c)), sv_reset restores |0><0|. Gradients, sampling,
 * batch mode and sharding are not available on density handles (SV_E_ARG). 1 <= n <= 17. */
sv_status sv_create_density(int32_t n_qubits, sv_handle* out);

/* NEXT-3 complex64 mode (the paper's "single-precision and double-precision simulation modes",
 * PAPER.md P:417): the state is held as 2^n complex64 amplitudes (8 bytes each: half the HBM of
 * sv_create). sv_apply_gate / sv_apply_circuit run complex64 fused passes (dense stages in FP32
 * on the CUDA cores, other ops evaluated in FP64 and rounded once per stage) and sv_expectation
 * reads the complex64 tiles (FP64 accumulation); results agree with the complex128 path to
 * ~1e-5 relative (float rounding), tolerance 1e-4. Host state transfer keeps the complex128
 * array format (values rounded on set); sv_set/get_state_device move 2*2^n floats. Gradients,
 * batch mode, sampling and circuits the complex64 kernel does not take (tiles without qubit 0 or
 * below 2^9 amplitudes, Pauli x-masks wider than a tile) run on a complex128 scratch copy
 * (widened, computed, and — for evolution — rounded back). Single GPU only. 1 <= n <= 40. */
sv_status sv_create_c64(int32_t n_qubits, sv_handle* out);

sv_status sv_destroy(sv_handle h);

/* Use this CUDA stream (a cudaStream_t passed as void*) for all subsequent work; NULL = the
 * handle's own stream. Work already queued on the previous stream is waited for first. The caller
 * keeps the stream alive while the handle uses it. */
sv_status sv_set_stream(sv_handle h, void* cuda_stream);

sv_status sv_set_option(sv_handle h, int32_t key, int64_t value);

sv_status sv_get_num_qubits(sv_handle h, int32_t* out);

/* psi <- |0...0>. Asynchronous. */
sv_status sv_reset(sv_handle h);

/* Full state in logical qubit order, 2*2^n doubles (re, im interleaved), from / to HOST memory.
 * For sharded handles every rank passes the full array (set) / receives it (get, gathered). */
sv_status sv_set_state(sv_handle h, const double* host_amps);
sv_status sv_get_state(sv_handle h, double* host_amps);

/* Sampled-amplitude readout (parity checks at sizes where the full state does not fit a host
 * buffer, e.g. 34 qubits sharded): out[2j], out[2j+1] = (re, im) of amplitude idx[j] (LOGICAL
 * index, qubit 0 = LSB; remaps of a sharded state are undone). count >= 0; idx[j] < 2^n
 * (SV_E_QUBIT_RANGE otherwise). Sharded handles: every rank passes the same indices and receives all
 * values (one all-reduce). complex64 states return their values widened. Synchronous. */
sv_status sv_get_amplitudes(sv_handle h, const uint64_t* idx, int64_t count, double* out);

/* Same, from / to DEVICE memory (device pointer on the handle's device), single-GPU handles
 * (complex64 handles: 2*2^n floats). */
sv_status sv_set_state_device(sv_handle h, const void* dev_amps);
sv_status sv_get_state_device(sv_handle h, void* dev_amps);

/* a3: apply one gate / a circuit (array order = evolution order) in place. */
sv_status sv_apply_gate(sv_handle h, const sv_gate* g, const double* params, int32_t n_params);
sv_status sv_apply_circuit(sv_handle h, const sv_gate* gates, int64_t n_gates, const double* params,
                           int32_t n_params);

/* a4: *out_value = <psi|H|psi>, H = sum_t terms[t]. Synchronous. Empty H -> 0. */
sv_status sv_expectation(sv_handle h, const sv_pauli* terms, int64_t n_terms, double* out_value);

/* a5-a7: evolves a COPY of the current state psi0 through the circuit, returns
 * E = <psi|H|psi> and out_grad[p] = dE/dparams[p] for p < n_params (chain rule over every
 * occurrence: sum_k coeff_k dE/dangle_k, reading c11). The handle's state is unchanged.
 * Needs two workspace vectors of 2^n amplitudes (allocated on first use, kept). Synchronous. */
sv_status sv_expectation_with_grad(sv_handle h, const sv_gate* gates, int64_t n_gates, const double* params,
                                   int32_t n_params, const sv_pauli* terms, int64_t n_terms,
                                   double* out_value, double* out_grad);

/* Batch mode (NEXT-1; "Gradient calculation in batch mode", Fig. 1): n_rows
 * parameter rows params[r * n_params + p]; out_values[r] = E(row r), out_grads[r * n_params + p] =
 * dE/dparams[p] at row r. Every row starts from the handle's current state, which is unchanged.
 * For states of <= 11 local qubits all rows run in ONE launch (one CTA per row, state and adjoint
 * vector in shared memory); larger states loop over rows with sv_expectation_with_grad.
 * Validation and errors as sv_expectation_with_grad. Synchronous. */
sv_status sv_expectation_with_grad_batch(sv_handle h, const sv_gate* gates, int64_t n_gates, const double* params,
                                         int32_t n_params, int32_t n_rows, const sv_pauli* terms, int64_t n_terms,
                                         double* out_values, double* out_grads);

/* Sampling measurement (NEXT-2; "Sampling Measurement", Fig. 1): draws `shots`
 * basis states from |psi_i|^2 by inverse CDF and writes, per shot, the measured bits of
 * qubits[0..n_measured) (bit j of out[s] = value of qubits[j]). Draw s uses the uniform
 * u_s = (splitmix64(seed + s) >> 11) * 2^-53 (counter-based, reproducible from (seed, s)); draws
 * are resolved in sorted order, results returned in shot order. The state is unchanged.
 * Single-GPU handles; synchronous. */
sv_status sv_sample(sv_handle h, const int32_t* qubits, int32_t n_measured, int64_t shots, uint64_t seed,
                    uint64_t* out);

sv_status sv_get_stats(sv_handle h, sv_stats* out);
sv_status sv_reset_stats(sv_handle h);

/* Thread-local text of the last non-OK status on this thread ("" if none). */
const char* sv_last_error(void);

/* Library version string. */
const char* sv_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SV_H_ */
