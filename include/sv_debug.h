/*
 * sv_debug.h — host-only introspection of the fused-pass planner (no GPU needed). Used by the CPU
 * test-suite to check planner invariants and by bench/profiling tools to report pass and stage
 * counts. Same conventions as sv.h.
 */
#ifndef SV_DEBUG_H_
#define SV_DEBUG_H_

#include <stdint.h>

#include "sv.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t k;            /* tile qubits of the pass                                             */
  int32_t low;          /* qubits 0..low-1 are tile positions 0..low-1 (contiguous chunk)       */
  int32_t R;            /* register qubits per thread (0 = shared-memory kernel)                 */
  int32_t n_ops;        /* ops (gates) applied by the pass                                       */
  int32_t n_stages;     /* register stages (R > 0)                                               */
  int32_t n_grad;       /* adjoint overlap slots in the pass                                     */
  uint64_t tile_mask;   /* physical qubits of the tile                                           */
  uint64_t nondiag_mask;/* qubits on which the pass' ops act non-diagonally (subset of tile_mask) */
  int32_t n_dense;      /* stages executed as dense FP64-MMA stages                              */
  int32_t mat_doubles;  /* matrix data of the pass (doubles)                                     */
  int32_t fma_per_amp;  /* FP64 fused multiply-adds per amplitude the pass executes (dense stages   */
                        /* 48 each: three real products per complex entry; sequential ops by class) */
  int32_t add_per_amp;  /* FP64 additions per amplitude besides them (dense stages: 3)             */
} sv_pass_info;

/* Plans `gates` for an n-qubit single-GPU state exactly as sv_apply_circuit (adjoint = 0) or the
 * reverse sweep of sv_expectation_with_grad (adjoint = 1) would, with tile_qubits (0 = auto) and
 * fusion (1 = on). Writes up to `cap` pass records to out and the pass count to *n_passes.
 * Errors as sv_apply_circuit's validation. Host only; no CUDA call. */
sv_status sv_plan_info(int32_t n_qubits, const sv_gate* gates, int64_t n_gates, const double* params,
                       int32_t n_params, int32_t adjoint, int32_t tile_qubits, int32_t fusion, sv_pass_info* out,
                       int64_t cap, int64_t* n_passes);

/* One step of a sharded schedule: kind 0 = segment of n_gates local gates (written to the
 * local_gates output in order), kind 1 = swap of physical qubit positions gpos (global, >= n_local)
 * and lpos (local): ranks r and r ^ 2^(gpos - n_local) exchange the halves of their shards whose
 * local bit lpos differs from their own bit (gpos - n_local). */
typedef struct {
  int32_t kind;
  int32_t gpos, lpos;
  int32_t n_gates;
} sv_shard_step;

/* Host-only: the schedule sv_apply_circuit would run on a `world`-way sharded state starting from
 * the identity layout, as seen by shard `rank`: segments of gates rewritten for that shard (global
 * controls resolved, diagonal factors on global qubits folded) with explicit matrices (MAT1 /
 * MAT2 kinds; mats: 32 doubles per gate, gate.mat points into local_mats), and swaps. final_perm
 * (n entries) receives the logical -> physical layout at the end. Used by the world-size-2 gloo
 * tests of the sharding logic on CPU. */
sv_status sv_shard_plan(int32_t n_qubits, int32_t world, int32_t rank, const sv_gate* gates, int64_t n_gates,
                        const double* params, int32_t n_params, sv_shard_step* steps, int64_t cap_steps,
                        int64_t* n_steps, sv_gate* local_gates, double* local_mats, int64_t cap_gates,
                        int64_t* n_local_gates, int32_t* final_perm);

#ifdef __cplusplus
}
#endif

#endif /* SV_DEBUG_H_ */
