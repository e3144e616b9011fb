// sv_internal.h — internal types shared by the host planner (plan.cpp, api.cpp) and the sm_100a
// kernels (kernels.cu). Not part of the ABI (include/sv.h is).
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <utility>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace sv {

// Per-device one-time setup (function attributes such as the dynamic shared-memory opt-in are per
// device): f() runs until it succeeds once on each device; a mask bit per device id, thread-safe
// (a race runs f twice, which is harmless for attribute setters).
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
template <class F>
cudaError_t once_per_device(std::atomic<uint64_t>& done, F&& f) {
  const uint64_t bit = 1ull << (current_device() & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = f();
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// Makes the handle's device current for the duration of an entry point (restores the caller's).
struct DeviceGuard {
  int prev = -1, want = -1;
  explicit DeviceGuard(int dev) : want(dev) {
    cudaGetDevice(&prev);
    if (prev != want) cudaSetDevice(want);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

struct Cx {
  double re, im;
};

// ---------------------------------------------------------------------------------------------
// Device-side op of a fused tile pass. A tile is the set of 2^k amplitudes whose indices agree on
// every qubit outside the tile's qubit list tq[0..k) (tq[p] = physical qubit of tile position p,
// tq[p] = p for p < L so the low L qubits form contiguous 16*2^L-byte chunks).
//
// Classes follow the paper's taxonomy (§3.1): X-like = anti-diagonal, Z-like = diagonal,
// general 2x2, and two-qubit groups.
enum OpType : int32_t {
  OP_M1 = 0,   // general 2x2 on tile position pa                 mat: 8 doubles (row-major)
  OP_AX1 = 1,  // X-like [[0,a],[b,0]] on tile position pa         mat: a, b (4 doubles)
  OP_D1 = 2,   // Z-like diag(a,b) on physical qubit qa (any)      mat: a, b (4 doubles)
  OP_M2 = 3,   // 4x4 on tile positions pa (index bit 0), pb (bit 1) mat: 32 doubles
  OP_D2 = 4,   // diagonal 4 entries on physical qubits qa (bit0), qb (bit1)  mat: 8 doubles
  OP_SWAP = 5, // SWAP of tile positions pa, pb                    mat: none
  // register-kernel op codes only (RegOp): rotations with real structure, no register controls
  // (mat: the 2x2 as for OP_M1; the kernel reads c = m00.re and s from m01): 4 FP64 per amplitude
  // instead of 8 for a general complex 2x2
  OP_RX = 6,   // [[c, -i s], [-i s, c]]
  OP_RY = 7,   // [[c, -s], [s, c]]
};

struct DevOp {
  int32_t type;
  int16_t pa, pb;      // tile positions of the targets (-1 when the target is outside the tile)
  int16_t qa, qb;      // physical qubits of the targets (local index space)
  int8_t ra, rb;       // register-kernel: register index of pa / pb in the op's stage (-1: thread bit / outer)
  uint8_t cj;          // register-kernel: control mask over register indices of the op's stage
  uint8_t pad0;
  int32_t mat_off;     // offset (doubles) of the op's matrix in the pass' matrix block
  int32_t grad_slot;   // >= 0: adjoint overlap slot (global across the reverse plan); -1 none
  int32_t gen_off;     // offset of the generator matrix G (2x2 or 4x4 complex) for grad ops
  int16_t gen_dim;     // 2 or 4 (generator acts on the targets) or 0
  int16_t gen_diag;    // 1: generator diagonal (entries gen_off[0..gen_dim)), evaluated per element
  int16_t stage;       // register-kernel: stage index within the pass
  int16_t grad_local;  // index among the pass' grad ops (-1 none)
  int32_t src;         // index of the bound gate the op applies (plan refresh with new angles)
  uint64_t ctile;      // control bits in tile-position space
  uint64_t cthr;       // register-kernel: control bits on the thread-bit positions of the op's stage
  uint64_t couter;     // control bits in local physical index space, outside the tile
};
static_assert(sizeof(DevOp) == 64, "DevOp layout");

// Register-kernel stage: which tile positions the 2^R amplitudes a thread holds in registers span
// (regpos), and the order of the remaining positions over thread-index bits (thrpos; bits 0..4 =
// lane). Ops of a stage whose non-diagonal targets are all register positions run from registers.
//
// Dense stages (forward passes): all ops of the stage are folded on the host into one 16x16
// complex matrix per "variant" — the assignment of the thread / outer bits the ops read through
// controls or diagonal factors — and applied as a real 32x32 GEMM over the tile's 2^(k-4)
// vectors with FP64 tensor-core MMAs (mma.sync m8n8k4 f64). For dense stages thrpos holds
// [c0 c1 c2 | n0 | w0 w1 ...]: column-in-MMA bits, N-tile bit, warp bits; the m_tile variant
// positions are the first warp bits; swz_reg[0..8) are the swizzled offsets of the B-fragment
// loads (n, kq), swz_reg[8..16) those of the D-fragment stores (n, mh, v). Variant matrices are
// row-major 16 x 16 complex with a row stride of 20 entries (bank-conflict-free A fragments).
struct StageDesc {
  int8_t regpos[4];
  int8_t thrpos[12];
  int32_t op_begin, op_end;  // range in the pass' op list (pass-relative); dense: op_begin = matrix offset
  uint16_t swz_reg[16];      // swizzled smem offset contribution of register index j (XOR-linear)
  uint8_t dense;             // 1: dense MMA stage
  uint8_t m_tile;            // variant bits on warp positions (thrpos[4 .. 4+m_tile))
  uint8_t m_outer;           // variant bits on outer qubits (var_outer[0 .. m_outer))
  uint8_t next_dense;        // distance to the pass' next dense stage (0: none; L1 prefetch)
  int8_t var_outer[8];
  uint32_t dense_off;        // dense: first variant matrix (double2 units in the pass' matrix block)
  uint16_t warp_swz[8];      // dense: swz(tile-position bits of warp w)
  uint8_t warp_var[8];       // dense: tile-variant index of warp w
  uint16_t lane_b[32];       // dense: swz(lane part of the B-fragment load address)
  uint16_t lane_d[32];       // dense: swz(lane part of the D-fragment store address)
  // adjoint dense stages (dense == 2): R = sum_v psi_v lambda_v^H over the warp's vectors, loaded
  // with amp = 8 mt + lane/4, vector = 4 kt + lane%4
  uint16_t lane_r[32];       // swz(lane part of the R-fragment load address)
  uint16_t off_r[8];         // swz(uniform part) for (mt, kt), index mt * 4 + kt
  int32_t da_index;          // first R accumulator slot of this adjoint dense stage in its pass (+ outer variant)
  int32_t c64_perm;          // complex64 dense stage: permutation (0..23) of thrpos[0..3] for the
                             // TF32 fragment lanes, chosen on the host for few bank conflicts
};
static_assert(sizeof(StageDesc) == 312, "StageDesc layout");
constexpr uint8_t kPassAccThread = 1, kPassSingleBuf = 2;  // Plan::pass_acc flags
// adjoint dense stages accumulate R in global (L2-resident, per CTA) instead of shared memory from
// this many local qubits (C4g 2.45 -> 2.57 grad evals/s: a third CTA per SM; C2 at 20q loses 2%)
#ifndef SV_DA_R_GLOBAL_MIN_N
#define SV_DA_R_GLOBAL_MIN_N 26
#endif
constexpr int kDARGlobalMinN = SV_DA_R_GLOBAL_MIN_N;
inline bool da_r_global(int n_local) { return n_local >= kDARGlobalMinN; }


// Compact op of the register kernel (32 bytes: two 16-byte shared loads per op).
//   code bits [0,4) type, [4,8) ra (15 = not a register bit), [8,12) rb, [12,16) cj,
//             [16,21) pa (31 = outside the tile), [21,26) pb, [26,28) generator (0 none, 1 2x2, 2 4x4),
//             [28] generator diagonal, [29,32) D1 flags (bit0: a == 1, bit1: a == 1 and b == -1)
struct RegOp {
  uint32_t code;
  uint16_t mat_off;    // double2 units, relative to the pass' matrix block
  uint16_t gen_off;    // double2 units
  uint16_t cthr;       // control bits on thread positions (tile-position space)
  int16_t grad_local;  // index among the pass' grad ops, -1 none
  uint8_t qa, qb;      // physical qubits (outer target bits of diagonal ops)
  uint16_t pad;        // bits 0-11: adjoint passes, length of the diagonal run this op starts (0:
                       // none); bit 15 (kRopHasCtrl): the op has outer or thread-position controls
  uint64_t couter;     // control bits outside the tile (local physical index space)
  int32_t grad_slot;   // global adjoint slot (-1 none)
  uint32_t pad2;
};
static_assert(sizeof(RegOp) == 32, "RegOp layout");
constexpr uint16_t kRopRunMask = 0x0fff;
constexpr uint16_t kRopHasCtrl = 0x8000;

constexpr int kMaxTileQubits = 13;
constexpr int kMaxOpsPerPass = 256;
constexpr int kMaxMatDoublesPerPass = 2048;      // sequential ops' matrices per pass
constexpr int kMaxDenseMatDoublesPerPass = 8192; // dense-stage variant matrices per pass (64 KiB)

struct PassDesc {
  int32_t k;                // tile qubits
  int32_t low;              // L: tq[p] = p for p < low
  int8_t tq[kMaxTileQubits + 3];  // physical qubit of each tile position
  int32_t op_begin, op_end; // range in the plan's op array
  int32_t mat_begin;        // base offset of this pass' matrices in the plan's matrix array
  int32_t n_grad;           // grad ops in this pass (adjoint)
  int32_t R;                // register qubits per thread (0: shared-memory kernel)
  int32_t seq_mats;         // matrix doubles the kernel stages in shared memory (ops' matrices);
                            // dense-stage variant matrices follow in global memory (read via L1/L2)
  int32_t stage_begin, stage_end;  // range in the plan's stage array
};

// A compiled plan: passes over one vector (forward) or two (adjoint).
// Allocator whose value-construction leaves doubles uninitialised: resizing the plan's matrix
// array does not zero (and page-fault) megabytes serially before the parallel fill writes them.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind { using other = NoInitAlloc<U>; };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept { ::new (static_cast<void*>(p)) U; }
  template <class U, class... A>
  void construct(U* p, A&&... a) { ::new (static_cast<void*>(p)) U(std::forward<A>(a)...); }
};

struct PlanJobs;  // plan.cpp: the deferred dense-stage fills, kept for refresh_plan
struct Plan {
  std::vector<PassDesc> passes;
  std::vector<DevOp> ops;
  std::vector<RegOp> rops;  // compact copy of ops for register passes (same indexing)
  std::vector<double, NoInitAlloc<double>> mats;  // op matrices, generators, dense variants (per pass)
  std::vector<StageDesc> stages;
  int n_grad_slots = 0;
  std::vector<int32_t> slot_param;   // slot -> parameter index
  std::vector<double> slot_coeff;    // slot -> chain-rule coefficient (coeff of the occurrence)
  // Adjoint dense stages (host side): the overlaps of their parametrised ops come from the
  // per-variant correlation matrices R_var = sum psi lambda^H at the stage start (accumulated on the
  // device) as d_j = sum_var tr(B_{j,var} R_var), B_{j,var} = V_{j-1}^dagger (Pi_C G_j) V_{j-1}.
  struct DAStage {
    int pass = 0, da_index = 0, m_tile = 0, m_outer = 0;
    int global_slot = 0;                 // first R slot (plan order); one slot per outer variant
    std::vector<int> slots;              // grad slots of the stage's parametrised ops (stage order)
    std::vector<std::vector<Cx>> B;      // [grad op][var * 256 + a * 16 + b]
  };
  std::vector<DAStage> da;
  int max_da_per_pass = 0;  // R accumulator slots (2^m_outer per adjoint dense stage) of the largest pass
  int da_slots_total = 0;
  bool reverse = false;  // adjoint plan: passes run on (psi, lambda) with the DUAL kernel
  int64_t n_src_gates = 0;  // bound gates the plan applies (cost counter: x1 forward, x2 adjoint)
  mutable int grid_cache = 0, grid_cache_n = -1;  // plan_grid memo (occupancy query once per plan)
  mutable std::vector<int> pass_grid;             // per-pass CTAs (register passes: occupancy of that pass)
  mutable std::vector<uint8_t> pass_acc;          // adjoint passes: bit 0 (kPassAccThread) per-thread overlap
                                                  // accumulators, bit 1 (kPassSingleBuf) single-buffered tile
  std::shared_ptr<PlanJobs> jobs;                 // dense-variant / adjoint-B fills (re-run on refresh)
};
constexpr int kMaxDAPerPass = 4;  // adjoint dense stages per pass (16 KiB of R accumulators each at 2^10 tiles; measured best, profiles/r01_da_per_pass_sweep.txt)

// ---------------------------------------------------------------------------------------------
// Host-side gate after binding: class + entries, logical qubits.
enum GateClass : int32_t { GC_XLIKE = 0, GC_ZLIKE = 1, GC_GEN1 = 2, GC_GEN2 = 3, GC_DIAG2 = 4, GC_SWAP = 5 };

struct BoundGate {
  int32_t cls;
  int32_t kind;
  int32_t t0, t1;        // logical targets (t1 = -1 for one-qubit)
  uint64_t controls;     // logical control mask
  Cx m[16];              // XLIKE/ZLIKE: m[0]=a, m[1]=b; GEN1: 2x2; GEN2: 4x4; DIAG2: m[0..3]
  int32_t param;         // -1 fixed
  double coeff;          // chain-rule coefficient
  int32_t gen_dim;       // generator dimension for parametrised gates (2 / 4), else 0
  Cx gen[16];            // D = (dU/dphi) U^dagger on the target space (2x2 or 4x4)
};

// Binding (gates.cpp). Returns SV status code; fills `out`. `err` receives a message.
int bind_gate(int n, const void* sv_gate_ptr, const double* params, int32_t n_params, bool for_grad,
              BoundGate* out, std::string* err);
BoundGate dagger(const BoundGate& g);

// Planner (plan.cpp). perm: logical qubit -> physical (local) qubit; n_local: local qubits.
struct PlanOptions {
  int tile_qubits = 0;   // 0 = auto
  int low_qubits = 3;
  bool fusion = true;
  int kernel = 1;        // 1: register-blocked stage kernel where possible, 0: shared-memory kernel
  int dense = 1;         // 1: dense FP64-MMA stages in forward passes where cheaper, 0: never
  int da_cost = -1;  // adjoint dense stage cost threshold (SV_OPT_ADJOINT_DENSE_COST; -1 auto by size)
};
int choose_tile_qubits(int n_local, const PlanOptions& o, bool dual);
// f(0 .. n-1) on the library's persistent host worker pool (plan.cpp)
void host_parallel_for(int n, const std::function<void(int)>& f);
void build_plan(const std::vector<BoundGate>& gates, int n_local, const PlanOptions& o, bool reverse_for_adjoint,
                Plan* plan);
// Structural reuse: `plan` was built by build_plan for gates of the same structure (kinds, qubits,
// controls, parameter slots) — only matrix VALUES differ (new angles, new user matrices). Rewrites
// every op's matrix from `gates`, re-fills the dense-stage variants and adjoint B matrices, and
// re-derives the value-dependent op codes (fast diagonal flags, RX / RY forms, diagonal runs).
// The pass / stage / layout decisions are kept (they stay correct for any values).
void refresh_plan(const std::vector<BoundGate>& gates, Plan* plan);
// FP64 FMAs per amplitude of pass i of a plan (dense stages 64, sequential ops by class).
int pass_fma_per_amp(const Plan& plan, size_t i);
int pass_add_per_amp(const Plan& plan, size_t i);  // FP64 additions per amplitude (Gauss sums)

// ---------------------------------------------------------------------------------------------
// Kernel launchers (kernels.cu).
struct PassLaunch {
  const PassDesc* pd;
  const DevOp* d_ops;      // device pointer to the plan's ops
  const double* d_mats;    // device pointer to the plan's matrices
  const StageDesc* d_stages;  // device pointer to the plan's stages
  const RegOp* d_rops;        // device pointer to the plan's compact ops
  double* d_partials;      // [n_slots][grid] adjoint overlap partials (or null)
  int nmats;               // matrix doubles of this pass
  int n_da = 0;            // adjoint dense stages of this pass
  double* r_partials = nullptr;  // their R accumulators: [da][warp][512][grid]
  int grid;                // CTAs
  int pstride = 0;         // stride of d_partials' slot rows (>= grid; 0: grid)
  bool all_dense = false;  // forward register pass of dense stages only (k_pass_dense)
  bool no_dense = false;   // forward register pass without dense stages (k_pass_reg<3, false, true>)
  int c64_terms = 3;       // complex64 dense stages: TF32 split products (3) or one product (1)
  int acc_thread = 0;      // adjoint: overlaps accumulate per thread in shared memory (no per-op shuffles)
  int n_local;
  uint64_t rank_bits;      // (sharded) global index bits of this shard, for controls/diagonals on
                           // global qubits folded by the planner (0 single-GPU)
};
cudaError_t launch_pass(double* psi, double* lam, const PassLaunch& L, cudaStream_t s);
cudaError_t launch_pass_reg(double* psi, double* lam, const PassLaunch& L, cudaStream_t s);
// complex64 state (NEXT-3)
bool c64_pass_ok(const PassDesc& pd);
int device_sm_count();  // SMs of the current device (cached)
cudaError_t launch_pass_c64(float* psi, const PassLaunch& L, cudaStream_t s);
cudaError_t launch_widen(const float* a, double* b, int64_t n, cudaStream_t s);
cudaError_t launch_narrow(const double* a, float* b, int64_t n, cudaStream_t s);
int pass_grid(int n_local, int k, bool dual);
int plan_grid(const Plan& plan, int n_local);
int reg_pass_ctas_per_sm(const Plan& plan, size_t pass, bool dual, int n_local);
bool pass_no_dense(const Plan& plan, const PassDesc& pd);   // forward register pass without dense stages
bool pass_all_dense(const Plan& plan, const PassDesc& pd);  // k_pass_dense eligible  // resident CTAs/SM of a register pass

cudaError_t launch_init_zero(double* psi, int64_t n_amps, bool one_at_zero, cudaStream_t s);
// out[j] = psi[idx[j]] (complex128 out; idx[j] == ~0 -> 0); psi complex128, or complex64 if c64
cudaError_t launch_gather(const void* psi, bool c64, const uint64_t* idx, int64_t count, double* out, cudaStream_t s);
// Sharding: swap halves of two virtual shards (a[y0|2^l] <-> b[y0]); pack / unpack the half of a
// shard with local bit l == h (elements off .. off+count of that half) to / from a buffer.
cudaError_t launch_swap_halves(double* a, double* b, int nl, int l, cudaStream_t s);
cudaError_t launch_pack_half(double* shard, double* buf, int l, int h, int64_t off, int64_t count, bool pack,
                             cudaStream_t s);

// Pauli groups (kernels.cu): terms sharing one x-mask.
struct PauliGroupDev {
  uint64_t x;
  int32_t term_begin, term_end;   // range in the z / coeff arrays
};
cudaError_t launch_pauli_group(const double* psi, double* lam, bool lam_accumulate, int n_local, uint64_t x,
                               const uint64_t* d_z, const double* d_c /* complex coeff pairs */, int nterms,
                               double* d_partials, int grid, cudaStream_t s);
int pauli_grid(int n_local);
// A tiled multi-group Pauli pass: tile positions tq (physical qubits), groups with x-masks inside
// the tile; term arrays (z, complex c) of its groups are contiguous from term_base.
struct PauliPassDesc {
  int32_t k, low, ngroups, nterms, term_base;
  int8_t tq[16];
  uint64_t xphys[32];
  uint32_t xtile[32];
  int32_t tbeg[32], tend[32];  // relative to term_base
  uint8_t gkind[32];           // bits 0-2: representative rule (PR_*); bits 3-4: PG_* type; bits 5-7: warp bit - 5
  int32_t diag_rb[17];         // E only: diagonal entry terms with register-part z mask h: [rb[h], rb[h+1])
  int32_t diag_g;              // E only: index of the diagonal entry, -1 none
  int32_t cls_beg[11];         // E only: off-diagonal entries sorted by class rule * 2 + (c' imaginary)
  uint32_t zt_reg[32];         // register-part (tile positions >= kPauliTileTidBits) z mask of entry g's first term
};
// Pauli pass entry types ((PauliPassDesc::gkind >> 2) & 3): one term with c' = c i^{popc(x&z)} real /
// imaginary, several terms sharing x (lambda modes), the diagonal group (x = 0)
enum { PG_SINGLE_RE = 0, PG_SINGLE_IM = 1, PG_MULTI = 2, PG_DIAG = 3 };
// Representative rule of an E-only off-diagonal entry (gkind & 7), tile geometry of k_pauli_tile:
// element e = tid + 512 j (tid = tile positions 0..8: lanes 0..4, warps 5..8; j = positions 9..11).
// Rules 0..3: register bit JB of x; PR_WARP: a warp bit of x; PR_ALL: x inside the lane bits.
enum { PR_WARP = 4, PR_ALL = 5 };
constexpr int kPauliTileTidBits = 9;  // k_pauli_tile's E-only entry classes assume 3 register bits
int pauli_tile_grid(int n_local, int k);
cudaError_t launch_pauli_tile(const double* psi, double* lam, int mode, int n_local, const PauliPassDesc& pp,
                              const uint64_t* d_z, const double* d_c, double* d_partials, int grid, cudaStream_t s);
cudaError_t launch_pauli_tile_c64(const float* psi, int n_local, const PauliPassDesc& pp, const uint64_t* d_z,
                                  const double* d_c, double* d_partials, int grid, cudaStream_t s);
// One streamed chunk (partner amplitudes [off, off + cnt), cnt a power of two, off a multiple of
// cnt) of a cross-shard Pauli group; partials accumulate over chunks (first: overwrite).
cudaError_t launch_pauli_cross(const double* psi, const double* partner, double* lam, int64_t off, int64_t cnt,
                               uint64_t xl, const uint64_t* d_z, const double* d_c, int nterms, double* d_partials,
                               int grid, bool first, cudaStream_t s);
cudaError_t launch_reduce_slots(const double* d_partials, int n_slots, int per_slot, double* d_out,
                                cudaStream_t s);
// out[i] = sum over g < n_cta of partials[g * per + i] (per-CTA contiguous partials, fixed order)
cudaError_t launch_reduce_strided(const double* d_partials, int64_t per, int n_cta, double* d_out, cudaStream_t s);
// Re<x|y> per-CTA partials (grid of them)
cudaError_t launch_redot(const double* x, const double* y, int64_t n, double* d_partials, int grid, cudaStream_t s);

// Batch mode (kernels_batch.cu): one CTA per parameter row, whole state in shared memory.
struct BatchOp {
  int32_t dim;        // 2 (one target) or 4 (two targets, matrix index bit j <-> t_j)
  int32_t t0, t1;
  int32_t param;      // -1: no gradient slot
  double coeff;       // chain-rule coefficient
  uint64_t cmask;     // controls
  int32_t mat_off;    // double2 offset of the full matrix in the row's block
  int32_t gen_off;    // double2 offset of the generator D (row-independent)
};
struct BatchArgs {
  const BatchOp* ops;
  int32_t nops, nterms, nparams, pad;
  const double* mats;   // [rows][row_stride double2]
  int64_t row_stride;   // double2 per row
  const double* gens;
  const uint64_t* x;
  const uint64_t* z;
  const double* c;      // complex coefficients incl. i^{popc(x&z)}
  double* out_e;        // [rows]
  double* out_g;        // [rows][nparams]
};
constexpr int kBatchMaxQubits = 11;
// Density matrix: tr(rho P) over one x-group of Pauli terms (rho as a 2n-qubit vector).
cudaError_t launch_dm_trace(const double* vec, int n, uint64_t x, const uint64_t* d_z, const double* d_c, int nterms,
                            double* d_partials, int grid, cudaStream_t s);
// Sampling (kernels.cu): block masses, then per-block inverse-CDF resolution of sorted draws.
cudaError_t launch_block_prob(const double* psi, int n_local, int bl, double* out, cudaStream_t s);
cudaError_t launch_sample_blocks(const double* psi, int bl, int nblk, const int64_t* blk, const int64_t* beg,
                                 const double* target, int64_t* out, cudaStream_t s);
cudaError_t launch_batch_grad(const double* psi0, int n, const BatchArgs& a, int rows, cudaStream_t s);

}  // namespace sv
