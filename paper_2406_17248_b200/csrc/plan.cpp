// plan.cpp — host planner: groups consecutive gates into fused tile passes.
//
// The paper applies one gate per sweep of the state (§3.1). On a B200 one
// sweep of a 30-qubit complex128 state moves 34 GB through HBM, so gates are fused: a pass picks
// a set T of k "tile" qubits (always including the low qubits 0..L-1, so each tile is made of
// contiguous 16*2^L-byte chunks), and every gate whose non-diagonal targets lie in T and which
// may legally move ahead of the gates left for later passes is applied to the tile while it sits
// on chip. Diagonal (Z-like) gates and controls never constrain T: each element knows its own
// index, so they are evaluated on any qubit.
//
// Legality: a gate g may move ahead of a skipped gate s iff they commute; sufficient condition
// used here: the qubits on which either acts non-diagonally are disjoint from all qubits of the
// other (operators block-diagonal on shared qubits commute). Controls act diagonally.
#include <algorithm>
#include <mutex>
#include <functional>
#include <condition_variable>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "sv.h"
#include "sv_internal.h"

namespace sv {

void emit_rops(Plan* plan);  // below (compact register-kernel op codes)

namespace {

inline int popc(uint64_t x) { return __builtin_popcountll(x); }

bool is_diag_class(int cls) { return cls == GC_ZLIKE || cls == GC_DIAG2; }

uint64_t target_mask(const BoundGate& g) {
  return (1ull << g.t0) | (g.t1 >= 0 ? (1ull << g.t1) : 0ull);
}

// Ops/matrix doubles an op contributes (to respect per-pass capacities).
int mat_doubles(const BoundGate& g) {
  int m = 0;
  switch (g.cls) {
    case GC_GEN1: m = 8; break;
    case GC_XLIKE: case GC_ZLIKE: m = 4; break;
    case GC_GEN2: m = 32; break;
    case GC_DIAG2: m = 8; break;
    default: m = 0;
  }
  if (g.param >= 0) m += 2 * g.gen_dim * g.gen_dim;
  return m;
}

struct PassGroup {
  uint64_t tmask;
  std::vector<int> gates;
};


// Swizzled 16-byte slot of tile index t (bank-conflict-free for 8 lanes spanning three tile
// positions with distinct residues mod 3). XOR-linear: sw(a ^ b) = sw(a) ^ sw(b).
uint32_t swz(uint32_t t) { return t ^ ((t >> 3 ^ t >> 6 ^ t >> 9 ^ t >> 12) & 7u); }

// Runs f(0 .. n-1) on host threads (n independent work items; small n runs inline).
// Persistent host worker pool for independent planning work items (dense variant matrices):
// workers sleep on a condition variable; a job hands out indices through an atomic counter and the
// calling thread participates. Spawning threads per call cost more than the work it split.
class PlanPool {
 public:
  static PlanPool& get() {
    static PlanPool pool;
    return pool;
  }
  int size() const { return (int)workers_.size() + 1; }
  void run(int n, const std::function<void(int)>& f) {
    // one job at a time: a second thread planning concurrently (distinct handles may be driven
    // from different threads, sv.h) runs its items inline instead of sharing the counter
    std::unique_lock<std::mutex> job_lock(run_m_, std::try_to_lock);
    if (workers_.empty() || n < 8 || !job_lock.owns_lock()) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    std::unique_lock<std::mutex> lk(m_);
    job_ = &f;
    n_ = n;
    next_.store(0);
    active_ = (int)workers_.size();
    ++gen_;
    lk.unlock();
    cv_.notify_all();
    for (int i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) f(i);
    lk.lock();
    done_cv_.wait(lk, [&] { return active_ == 0; });
    job_ = nullptr;
  }

 private:
  PlanPool() {
    static const bool serial = std::getenv("SV_PLAN_SERIAL") != nullptr;
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int nw = serial ? 0 : std::min(hw, 16) - 1;
    for (int t = 0; t < nw; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~PlanPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (std::thread& t : workers_) t.join();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      const std::function<void(int)>* f = job_;
      const int n = n_;
      lk.unlock();
      if (f)
        for (int i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) (*f)(i);
      lk.lock();
      if (--active_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_m_;  // held for a whole job
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  std::atomic<int> next_{0};
};

template <class F>
void parallel_for(int n, F f) {
  const std::function<void(int)> fn(f);
  PlanPool::get().run(n, fn);
}

bool op_is_diag(const DevOp& o) { return o.type == OP_D1 || o.type == OP_D2; }

// ---------------------------------------------------------------- register stages

struct StagePlan {
  StageDesc sd;
  std::vector<DevOp> ops;  // in execution order, ra/rb/cj/cthr relative to this stage
  uint32_t regset = 0;     // register positions
};

// Commutation masks of an op in physical qubits: N = non-diagonal targets, A = all qubits.
void phys_masks(const DevOp& o, const PassDesc& pd, uint64_t* N, uint64_t* A) {
  uint64_t t = (1ull << o.qa) | (o.qb >= 0 ? (1ull << o.qb) : 0ull);
  uint64_t c = o.couter;
  for (int p = 0; p < pd.k; ++p)
    if ((o.ctile >> p) & 1ull) c |= 1ull << pd.tq[p];
  *N = op_is_diag(o) ? 0ull : t;
  *A = t | c;
}

uint32_t pos_mask(const DevOp& o) {
  if (op_is_diag(o)) return 0u;
  return (1u << o.pa) | (o.pb >= 0 ? (1u << o.pb) : 0u);
}

// Sets the register-relative fields of the stage's ops (ra, rb, cj, cthr) for register positions
// regpos[0..R) and canonicalises two-qubit non-diagonal ops to ra < rb (swapping matrix bits).
void bind_stage_ops(StagePlan* sp, const int* regpos, int R, int stage_idx, Plan* plan, const PassDesc& pd) {
  int reg_of[32];
  for (int p = 0; p < 32; ++p) reg_of[p] = -1;
  for (int r = 0; r < R; ++r) reg_of[regpos[r]] = r;
  auto perm = [](int i) { return ((i & 1) << 1) | ((i >> 1) & 1); };
  auto swap_bits = [&](double* m) {
    double t[32];
    for (int r = 0; r < 4; ++r)
      for (int c = 0; c < 4; ++c) {
        t[2 * (perm(r) * 4 + perm(c))] = m[2 * (r * 4 + c)];
        t[2 * (perm(r) * 4 + perm(c)) + 1] = m[2 * (r * 4 + c) + 1];
      }
    std::memcpy(m, t, sizeof(t));
  };
  for (DevOp& o : sp->ops) {
    o.stage = (int16_t)stage_idx;
    o.ra = (int8_t)(o.pa >= 0 ? reg_of[o.pa] : -1);
    o.rb = (int8_t)(o.pb >= 0 ? reg_of[o.pb] : -1);
    o.cj = 0;
    o.cthr = 0;
    for (int p = 0; p < pd.k; ++p)
      if ((o.ctile >> p) & 1ull) {
        if (reg_of[p] >= 0) o.cj |= (uint8_t)(1u << reg_of[p]);
        else o.cthr |= 1ull << p;
      }
    if ((o.type == OP_M2 || o.type == OP_SWAP) && o.ra > o.rb) {
      std::swap(o.ra, o.rb);
      std::swap(o.pa, o.pb);
      std::swap(o.qa, o.qb);
      if (o.type == OP_M2) swap_bits(plan->mats.data() + pd.mat_begin + o.mat_off);
      if (o.grad_slot >= 0 && !o.gen_diag && o.gen_dim == 4) swap_bits(plan->mats.data() + pd.mat_begin + o.gen_off);
    }
  }
}

// Greedy split of `ops` (pass order) into register stages of <= R register positions. An op joins
// the current stage if it may legally move ahead of the ops left for later stages (same
// commutation rule as the pass planner) and its non-diagonal target positions fit the register
// set; with max_var_total >= 0 it must also keep the stage's variant bits (thread / outer bits
// read by controls or diagonal factors, see StageDesc) within the limits.
std::vector<StagePlan> split_stages(const std::vector<DevOp>& ops, const PassDesc& pd, int R, int max_var_tile,
                                    int max_var_total) {
  std::vector<StagePlan> out;
  std::vector<int> pending(ops.size());
  for (size_t i = 0; i < ops.size(); ++i) pending[i] = (int)i;
  while (!pending.empty()) {
    uint32_t regset = 0, vt = 0;
    uint64_t bN = 0, bA = 0, vo = 0;
    std::vector<int> taken, skipped;
    for (int i : pending) {
      const DevOp& op = ops[i];
      uint64_t N, A;
      phys_masks(op, pd, &N, &A);
      bool ok = !(N & bA) && !(A & bN);
      const uint32_t pm = pos_mask(op);
      uint32_t nreg = regset;
      if (ok && (pm & ~regset)) {
        if (__builtin_popcount(regset | pm) <= R) nreg = regset | pm;
        else ok = false;
      }
      uint32_t nvt = vt;
      uint64_t nvo = vo;
      if (ok && max_var_total >= 0) {
        nvt |= (uint32_t)op.ctile;
        nvo |= op.couter;
        if (op_is_diag(op)) {
          for (int t = 0; t < (op.type == OP_D2 ? 2 : 1); ++t) {
            const int pos = t ? op.pb : op.pa;
            if (pos >= 0) nvt |= 1u << pos;
            else nvo |= 1ull << (t ? op.qb : op.qa);
          }
        }
        nvt &= ~nreg;
        if (__builtin_popcount(nvt) > max_var_tile || __builtin_popcount(nvt) + __builtin_popcountll(nvo) > max_var_total)
          ok = false;
      }
      if (ok) { taken.push_back(i); regset = nreg; vt = nvt; vo = nvo; }
      else { skipped.push_back(i); bN |= N; bA |= A; }
    }
    if (taken.empty()) {  // the variant limit admits nothing: the first pending op goes alone
      taken.push_back(skipped.front());
      skipped.erase(skipped.begin());
      regset = pos_mask(ops[taken[0]]);
    }
    StagePlan sp;
    std::memset(&sp.sd, 0, sizeof(sp.sd));
    sp.regset = regset;
    for (int i : taken) sp.ops.push_back(ops[i]);
    out.push_back(std::move(sp));
    pending.swap(skipped);
  }
  return out;
}

// Layout of a sequential stage: lanes 0..2 on thread positions with distinct residues mod 3
// (conflict-free 16-byte shared phases), register set filled to R from the highest free
// positions, then the remaining thread positions.
void layout_sequential(StagePlan* sp, const PassDesc& pd, int R) {
  const int k = pd.k;
  uint32_t regset = sp->regset;
  std::vector<int> free_pos;
  for (int p = 0; p < k; ++p)
    if (!((regset >> p) & 1u)) free_pos.push_back(p);
  std::vector<int> lanes;
  for (int res = 0; res < 3; ++res)
    for (size_t f = 0; f < free_pos.size(); ++f)
      if (free_pos[f] % 3 == res && (int)free_pos.size() - 1 >= R - __builtin_popcount(regset)) {
        lanes.push_back(free_pos[f]);
        free_pos.erase(free_pos.begin() + f);
        break;
      }
  while (__builtin_popcount(regset) < R && !free_pos.empty()) {
    regset |= 1u << free_pos.back();
    free_pos.pop_back();
  }
  sp->regset = regset;
  std::vector<int> thr = lanes;
  thr.insert(thr.end(), free_pos.begin(), free_pos.end());
  StageDesc& sd = sp->sd;
  int rp[4] = {-1, -1, -1, -1}, nr = 0;
  for (int p = 0; p < k; ++p)
    if ((regset >> p) & 1u) rp[nr++] = p;
  for (int r = 0; r < 4; ++r) sd.regpos[r] = (int8_t)rp[r];
  for (int b = 0; b < 12; ++b) sd.thrpos[b] = (int8_t)(b < (int)thr.size() ? thr[b] : -1);
  for (int j = 0; j < (1 << R); ++j) {
    uint32_t dep = 0;
    for (int r = 0; r < R; ++r)
      if ((j >> r) & 1) dep |= 1u << rp[r];
    sd.swz_reg[j] = (uint16_t)swz(dep);
  }
}

// ---------------------------------------------------------------- dense (FP64-MMA) stages

constexpr int kDenseStride = 16;  // complex entries per row of a stored variant matrix (kernels_reg.cu kDenseRow)
// Dense-stage policy (tunable by environment for A/B runs): minimum sequential FP64 cost
// (FMA/amp) worth a 64 FMA/amp dense stage, and the maximum number of variant bits.
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
const int g_dense_min_cost = env_int("SV_DENSE_MIN_COST", 20);
// variant bits (tile + outer) of a forward dense stage: 8 from 28 local qubits (C4 at 30q: 141 instead
// of 144 stages, circuit 628 -> 616 ms), 6 below (C3 at 24q: 46.6 vs 44.8 grad evals/s with 8)
const int g_dense_max_var_env = env_int("SV_DENSE_MAX_VAR", -1);
int dense_max_var_for(int n_local) { return g_dense_max_var_env >= 0 ? g_dense_max_var_env : (n_local >= 28 ? 8 : 6); }
const int g_da_min_cost = env_int("SV_DA_MIN_COST", -1);   // adjoint dense stages: cost threshold override
// Default threshold by state size: the per-pass fixed costs of adjoint dense stages (R partials
// written and reduced per CTA, host contraction) amortise over large states only. Measured
// (profiles/r01_da_sweep.txt, r01_c2_da_sweep.txt): C4g 30q best at 96-150 (1.60 grad evals/s vs
// 1.46 at 200), C2 20q best at 200-300 (303 vs 263 at 96).
int da_min_cost_for(int n_local, int opt) {
  if (g_da_min_cost >= 0) return g_da_min_cost;
  if (opt >= 0) return opt;
  return n_local >= 24 ? 96 : 250;
}
const int g_da_enable = env_int("SV_DA", 1);
// shortest run of diagonal ops the DUAL kernel evaluates as one (its fixed cost: conj(lambda) psi,
// parking psi / lambda, the phase tables' product and one application)
const int g_diag_run_min = env_int("SV_DIAG_RUN_MIN", 4);
const int g_da_max_per_pass = env_int("SV_DA_MAX_PER_PASS", kMaxDAPerPass);

const int g_da_max_tile = env_int("SV_DA_MAX_TILE", 2);
// outer variant bits of an adjoint dense stage: 1 for large states (C4g 1.90 -> 1.97 grad evals/s),
// 0 below 26 local qubits (C3 28.2 -> 28.7); profiles/r01_da_outer_sweep.txt. Env overrides.
const int g_da_max_outer_env = env_int("SV_DA_MAX_OUTER", -1);
int da_max_outer_for(int n_local) { return g_da_max_outer_env >= 0 ? g_da_max_outer_env : (n_local >= 26 ? 1 : 0); }

// FP64 pipe cost per amplitude of an op applied sequentially (DFMA path), for the dense choice.
int seq_cost(const DevOp& o, const double* m) {
  switch (o.type) {
    case OP_M1: return 8;
    case OP_AX1: return 4;
    case OP_M2: return 32;
    case OP_SWAP: return 0;
    case OP_D2: return 4;
    case OP_D1:
      if (m[0] == 1.0 && m[1] == 0.0) return (m[2] == -1.0 && m[3] == 0.0) ? 0 : 2;
      return 4;
  }
  return 0;
}

// Applies one op to the 16-dim register-space vector u, given the values of the variant bits it
// reads (tile positions in tbits, outer qubits in obits). reg_new[p]: dense register index of
// tile position p (-1 if p is not a register position).
void dense_apply(Cx* u, const DevOp& o, const double* m, const int* reg_new, uint32_t tbits, uint64_t obits) {
  uint32_t cj = 0, cthr = 0;
  for (int p = 0; p < 32; ++p)
    if ((o.ctile >> p) & 1ull) {
      if (reg_new[p] >= 0) cj |= 1u << reg_new[p];
      else cthr |= 1u << p;
    }
  if ((cthr & tbits) != cthr) return;
  if ((o.couter & obits) != o.couter) return;
  auto bit_of = [&](int pos, int q, int j) -> uint32_t {
    if (pos >= 0 && reg_new[pos] >= 0) return ((uint32_t)j >> reg_new[pos]) & 1u;
    if (pos >= 0) return (tbits >> pos) & 1u;
    return (uint32_t)((obits >> q) & 1ull);
  };
  auto cm = [](Cx a, Cx b) { return Cx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; };
  auto ca = [](Cx a, Cx b) { return Cx{a.re + b.re, a.im + b.im}; };
  const Cx* M = reinterpret_cast<const Cx*>(m);
  switch (o.type) {
    case OP_M1: case OP_AX1: {
      const int r = reg_new[o.pa];
      Cx mm[4];
      if (o.type == OP_M1) { mm[0] = M[0]; mm[1] = M[1]; mm[2] = M[2]; mm[3] = M[3]; }
      else { mm[0] = Cx{0, 0}; mm[1] = M[0]; mm[2] = M[1]; mm[3] = Cx{0, 0}; }
      for (int j = 0; j < 16; ++j) {
        if ((j >> r) & 1) continue;
        if (((uint32_t)j & cj) != cj) continue;
        const int j1 = j | (1 << r);
        const Cx a = u[j], b = u[j1];
        u[j] = ca(cm(mm[0], a), cm(mm[1], b));
        u[j1] = ca(cm(mm[2], a), cm(mm[3], b));
      }
      break;
    }
    case OP_M2: case OP_SWAP: {
      const int ra = reg_new[o.pa], rb = reg_new[o.pb];
      for (int j = 0; j < 16; ++j) {
        if (((j >> ra) & 1) || ((j >> rb) & 1)) continue;
        if (((uint32_t)j & cj) != cj) continue;
        const int idx[4] = {j, j | (1 << ra), j | (1 << rb), j | (1 << ra) | (1 << rb)};
        Cx x[4], y[4];
        for (int c = 0; c < 4; ++c) x[c] = u[idx[c]];
        if (o.type == OP_SWAP) { y[0] = x[0]; y[1] = x[2]; y[2] = x[1]; y[3] = x[3]; }
        else
          for (int rr = 0; rr < 4; ++rr) {
            Cx acc{0, 0};
            for (int c = 0; c < 4; ++c) acc = ca(acc, cm(M[rr * 4 + c], x[c]));
            y[rr] = acc;
          }
        for (int c = 0; c < 4; ++c) u[idx[c]] = y[c];
      }
      break;
    }
    case OP_D1:
      for (int j = 0; j < 16; ++j) {
        if (((uint32_t)j & cj) != cj) continue;
        u[j] = cm(M[bit_of(o.pa, o.qa, j)], u[j]);
      }
      break;
    case OP_D2:
      for (int j = 0; j < 16; ++j) {
        if (((uint32_t)j & cj) != cj) continue;
        u[j] = cm(M[bit_of(o.pa, o.qa, j) | (bit_of(o.pb, o.qb, j) << 1)], u[j]);
      }
      break;
  }
}


// U <- op U for a whole 16 x 16 register-space matrix (row-major U[j * 16 + c]): the same
// arithmetic as dense_apply column by column, with the control / variant decode done once.
void dense_apply_cols(Cx* U, const DevOp& o, const double* m, const int* reg_new, uint32_t tbits, uint64_t obits) {
  uint32_t cj = 0, cthr = 0;
  for (int p = 0; p < 32; ++p)
    if ((o.ctile >> p) & 1ull) {
      if (reg_new[p] >= 0) cj |= 1u << reg_new[p];
      else cthr |= 1u << p;
    }
  if ((cthr & tbits) != cthr) return;
  if ((o.couter & obits) != o.couter) return;
  auto bit_of = [&](int pos, int q, int j) -> uint32_t {
    if (pos >= 0 && reg_new[pos] >= 0) return ((uint32_t)j >> reg_new[pos]) & 1u;
    if (pos >= 0) return (tbits >> pos) & 1u;
    return (uint32_t)((obits >> q) & 1ull);
  };
  auto cm = [](Cx a, Cx b) { return Cx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; };
  auto ca = [](Cx a, Cx b) { return Cx{a.re + b.re, a.im + b.im}; };
  const Cx* M = reinterpret_cast<const Cx*>(m);
  switch (o.type) {
    case OP_M1: case OP_AX1: {
      const int r = reg_new[o.pa];
      Cx mm[4];
      if (o.type == OP_M1) { mm[0] = M[0]; mm[1] = M[1]; mm[2] = M[2]; mm[3] = M[3]; }
      else { mm[0] = Cx{0, 0}; mm[1] = M[0]; mm[2] = M[1]; mm[3] = Cx{0, 0}; }
      for (int j = 0; j < 16; ++j) {
        if ((j >> r) & 1) continue;
        if (((uint32_t)j & cj) != cj) continue;
        Cx* a = U + j * 16;
        Cx* b = U + (j | (1 << r)) * 16;
        for (int c = 0; c < 16; ++c) {
          const Cx x = a[c], y = b[c];
          a[c] = ca(cm(mm[0], x), cm(mm[1], y));
          b[c] = ca(cm(mm[2], x), cm(mm[3], y));
        }
      }
      break;
    }
    case OP_M2: case OP_SWAP: {
      const int ra = reg_new[o.pa], rb = reg_new[o.pb];
      for (int j = 0; j < 16; ++j) {
        if (((j >> ra) & 1) || ((j >> rb) & 1)) continue;
        if (((uint32_t)j & cj) != cj) continue;
        Cx* row[4] = {U + j * 16, U + (j | (1 << ra)) * 16, U + (j | (1 << rb)) * 16,
                      U + (j | (1 << ra) | (1 << rb)) * 16};
        for (int c = 0; c < 16; ++c) {
          Cx x[4], y[4];
          for (int k = 0; k < 4; ++k) x[k] = row[k][c];
          if (o.type == OP_SWAP) { y[0] = x[0]; y[1] = x[2]; y[2] = x[1]; y[3] = x[3]; }
          else
            for (int rr = 0; rr < 4; ++rr) {
              Cx acc{0, 0};
              for (int k = 0; k < 4; ++k) acc = ca(acc, cm(M[rr * 4 + k], x[k]));
              y[rr] = acc;
            }
          for (int k = 0; k < 4; ++k) row[k][c] = y[k];
        }
      }
      break;
    }
    case OP_D1:
      for (int j = 0; j < 16; ++j) {
        if (((uint32_t)j & cj) != cj) continue;
        const Cx f = M[bit_of(o.pa, o.qa, j)];
        for (int c = 0; c < 16; ++c) U[j * 16 + c] = cm(f, U[j * 16 + c]);
      }
      break;
    case OP_D2:
      for (int j = 0; j < 16; ++j) {
        if (((uint32_t)j & cj) != cj) continue;
        const Cx f = M[bit_of(o.pa, o.qa, j) | (bit_of(o.pb, o.qb, j) << 1)];
        for (int c = 0; c < 16; ++c) U[j * 16 + c] = cm(f, U[j * 16 + c]);
      }
      break;
  }
}

// u <- (Pi_C (x) G) u in register space: the generator of a parametrised op restricted to the
// control-satisfied subspace (zero elsewhere). G: op's generator (diagonal entries if gen_diag).
void dense_gen_apply(Cx* u, const DevOp& o, const double* gm, const int* reg_new, uint32_t tbits, uint64_t obits) {
  uint32_t cj = 0, cthr = 0;
  for (int p = 0; p < 32; ++p)
    if ((o.ctile >> p) & 1ull) {
      if (reg_new[p] >= 0) cj |= 1u << reg_new[p];
      else cthr |= 1u << p;
    }
  const bool var_ok = ((cthr & tbits) == cthr) && ((o.couter & obits) == o.couter);
  auto bit_of = [&](int pos, int q, int j) -> uint32_t {
    if (pos >= 0 && reg_new[pos] >= 0) return ((uint32_t)j >> reg_new[pos]) & 1u;
    if (pos >= 0) return (tbits >> pos) & 1u;
    return (uint32_t)((obits >> q) & 1ull);
  };
  auto cm = [](Cx a, Cx b) { return Cx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; };
  auto ca = [](Cx a, Cx b) { return Cx{a.re + b.re, a.im + b.im}; };
  const Cx* G = reinterpret_cast<const Cx*>(gm);
  Cx out[16];
  for (int j = 0; j < 16; ++j) out[j] = Cx{0, 0};
  if (var_ok) {
    if (o.gen_diag) {
      for (int j = 0; j < 16; ++j) {
        if (((uint32_t)j & cj) != cj) continue;
        uint32_t idx = bit_of(o.pa, o.qa, j);
        if (o.gen_dim == 4) idx |= bit_of(o.pb, o.qb, j) << 1;
        out[j] = cm(G[idx], u[j]);
      }
    } else if (o.gen_dim == 2) {
      const int r = reg_new[o.pa];
      for (int j = 0; j < 16; ++j) {
        if ((j >> r) & 1) continue;
        if (((uint32_t)j & cj) != cj) continue;
        const int j1 = j | (1 << r);
        out[j] = ca(cm(G[0], u[j]), cm(G[1], u[j1]));
        out[j1] = ca(cm(G[2], u[j]), cm(G[3], u[j1]));
      }
    } else {
      const int ra = reg_new[o.pa], rb = reg_new[o.pb];
      for (int j = 0; j < 16; ++j) {
        if (((j >> ra) & 1) || ((j >> rb) & 1)) continue;
        if (((uint32_t)j & cj) != cj) continue;
        const int idx[4] = {j, j | (1 << ra), j | (1 << rb), j | (1 << ra) | (1 << rb)};
        for (int rr = 0; rr < 4; ++rr) {
          Cx acc{0, 0};
          for (int c = 0; c < 4; ++c) acc = ca(acc, cm(G[rr * 4 + c], u[idx[c]]));
          out[idx[rr]] = acc;
        }
      }
    }
  }
  for (int j = 0; j < 16; ++j) u[j] = out[j];
}

// One dense stage's variant matrices, deferred: U_v = G_n ... G_1 in register space for every
// variant v (tile variant bits vlist, outer bits olist), written to plan->mats at dst (row stride
// kDenseStride). The op matrices are read at opm + op.mat_off (pass-relative offsets).
struct DenseJob {
  std::vector<DevOp> ops;
  size_t opm = 0, dst = 0;
  int reg_new[32];
  std::vector<int> vlist, olist;
  int m_tile = 0, m_outer = 0;
  int da = -1;  // adjoint dense stage: index in plan->da whose B matrices this job also fills
};

}  // namespace
struct PlanJobs {
  std::vector<DenseJob> jobs;
};
namespace {

// B_{j,v} = V^dagger (Pi_C G_j) V for variant v of an adjoint dense stage (V: product of the
// stage's ops before its j-th parametrised op, register space).
void fill_da_variant(const DenseJob& J, Plan::DAStage* ds, int v, uint32_t tbits, uint64_t obits, const double* opm) {
  auto cm = [](Cx a, Cx b) { return Cx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; };
  Cx V[256];  // columns c: V[j * 16 + c]
  for (int j = 0; j < 16; ++j)
    for (int c = 0; c < 16; ++c) V[j * 16 + c] = Cx{j == c ? 1.0 : 0.0, 0.0};
  int gj = 0;
  for (const DevOp& o : J.ops) {
    if (o.grad_slot >= 0) {
      Cx GV[256];
      for (int c = 0; c < 16; ++c) {
        Cx u[16];
        for (int j = 0; j < 16; ++j) u[j] = V[j * 16 + c];
        dense_gen_apply(u, o, opm + o.gen_off, J.reg_new, tbits, obits);
        for (int j = 0; j < 16; ++j) GV[j * 16 + c] = u[j];
      }
      Cx* Bd = ds->B[(size_t)gj].data() + (size_t)v * 256;
      for (int a = 0; a < 16; ++a)
        for (int b = 0; b < 16; ++b) {
          Cx acc{0, 0};
          for (int j = 0; j < 16; ++j) {
            const Cx vc = Cx{V[j * 16 + a].re, -V[j * 16 + a].im};
            const Cx t = cm(vc, GV[j * 16 + b]);
            acc.re += t.re;
            acc.im += t.im;
          }
          Bd[a * 16 + b] = acc;
        }
      ++gj;
    }
    for (int c = 0; c < 16; ++c) {
      Cx u[16];
      for (int j = 0; j < 16; ++j) u[j] = V[j * 16 + c];
      dense_apply(u, o, opm + o.mat_off, J.reg_new, tbits, obits);
      for (int j = 0; j < 16; ++j) V[j * 16 + c] = u[j];
    }
  }
}

void fill_dense_variants(Plan* plan, const std::vector<DenseJob>& jobs) {
  std::vector<int> first(jobs.size() + 1, 0);
  for (size_t j = 0; j < jobs.size(); ++j) first[j + 1] = first[j] + (1 << (jobs[j].m_tile + jobs[j].m_outer));
  const size_t vdoubles = 2 * 16 * (size_t)kDenseStride;
  parallel_for(first.back(), [&](int item) {
    const size_t j = (size_t)(std::upper_bound(first.begin(), first.end(), item) - first.begin()) - 1;
    const DenseJob& J = jobs[j];
    const int v = item - first[j];
    uint32_t tbits = 0;
    for (int b = 0; b < J.m_tile; ++b)
      if ((v >> b) & 1) tbits |= 1u << J.vlist[b];
    uint64_t obits = 0;
    for (int b = 0; b < J.m_outer; ++b)
      if ((v >> (J.m_tile + b)) & 1) obits |= 1ull << J.olist[b];
    const double* opm = plan->mats.data() + J.opm;
    Cx U[256];
    for (int r = 0; r < 16; ++r)
      for (int c = 0; c < 16; ++c) U[r * 16 + c] = Cx{r == c ? 1.0 : 0.0, 0.0};
    // runs of diagonal ops (QAOA phase layers) are collected into one diagonal and applied to the
    // rows of U once, before the next non-diagonal op
    Cx dg[16];
    bool dg_pending = false;
    auto flush = [&] {
      if (!dg_pending) return;
      for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 16; ++c) {
          const Cx a = U[r * 16 + c];
          U[r * 16 + c] = Cx{dg[r].re * a.re - dg[r].im * a.im, dg[r].re * a.im + dg[r].im * a.re};
        }
      dg_pending = false;
    };
    for (const DevOp& o : J.ops) {
      if (op_is_diag(o)) {
        if (!dg_pending) {
          for (int r = 0; r < 16; ++r) dg[r] = Cx{1.0, 0.0};
          dg_pending = true;
        }
        dense_apply(dg, o, opm + o.mat_off, J.reg_new, tbits, obits);
      } else {
        flush();
        dense_apply_cols(U, o, opm + o.mat_off, J.reg_new, tbits, obits);
      }
    }
    flush();
    if (J.da >= 0) fill_da_variant(J, &plan->da[(size_t)J.da], v, tbits, obits, opm);
    double* d = plan->mats.data() + J.dst + (size_t)v * vdoubles;
    for (int r = 0; r < 16; ++r)
      for (int c = 0; c < kDenseStride; ++c) {
        const Cx e = c < 16 ? U[r * 16 + c] : Cx{0, 0};
        *d++ = e.re;
        *d++ = e.im;
      }
  });
}

// Folds a 4-register stage into dense variant matrices (appended to plan->mats) when cheaper than
// the sequential path and feasible: variant bits <= 3 in total, tile variant bits on warp
// positions. Returns false (stage untouched) otherwise.
bool make_dense(StagePlan* sp, const PassDesc& pd, Plan* plan, size_t mat_budget_doubles, std::vector<DenseJob>* jobs,
                bool adjoint = false, int pass_index = 0, int da_index = 0, int da_slots_left = 0, int da_min_cost = 96,
                int da_max_outer = 1, int max_var = 6) {
  const int k = pd.k;
  const int nw_bits = k - 8;  // 2^(k-3) threads: 16 vectors of 16 amplitudes per warp
  if (nw_bits < 1 || __builtin_popcount(sp->regset) > 4) return false;
  uint32_t regmask = sp->regset;
  int cost = 0;
  uint32_t vt = 0;
  uint64_t vo = 0;
  for (const DevOp& o : sp->ops) {
    cost += seq_cost(o, plan->mats.data() + pd.mat_begin + o.mat_off);
    vt |= (uint32_t)o.ctile & ~regmask;
    vo |= o.couter;
    if (op_is_diag(o))
      for (int t = 0; t < (o.type == OP_D2 ? 2 : 1); ++t) {
        const int pos = t ? o.pb : o.pa;
        if (pos >= 0 && !((regmask >> pos) & 1u)) vt |= 1u << pos;
        if (pos < 0) vo |= 1ull << (t ? o.qb : o.qa);
      }
  }
  // pad the register set to 4 positions with non-variant positions (identity on them)
  for (int p = k - 1; p >= 0 && __builtin_popcount(regmask) < 4; --p)
    if (!((regmask >> p) & 1u) && !((vt >> p) & 1u)) regmask |= 1u << p;
  if (__builtin_popcount(regmask) != 4) return false;
  const int m_tile = __builtin_popcount(vt), m_outer = __builtin_popcountll(vo);
  static const bool plan_debug = std::getenv("SV_PLAN_DEBUG") != nullptr;
  if (plan_debug)
    std::fprintf(stderr, "stage: ops %d cost %d m_tile %d m_outer %d\n", (int)sp->ops.size(), cost, m_tile, m_outer);
  if (adjoint) {
    // adjoint dense stage: per-warp R accumulators need warp-uniform variants (no outer bits);
    // worth it once the sequential dual cost (psi + lambda + overlaps) passes the dense cost
    int ngrad = 0;
    for (const DevOp& o : sp->ops) ngrad += o.grad_slot >= 0 ? 1 : 0;
    if (2 * cost + 8 * ngrad < da_min_cost || m_outer > da_max_outer || m_tile > std::min(g_da_max_tile, nw_bits) ||
        (1 << m_outer) > da_slots_left)
      return false;
  } else if (cost < g_dense_min_cost || m_tile > nw_bits || m_outer > 8 || m_tile + m_outer > max_var) {
    return false;
  }
  const int nvar = 1 << (m_tile + m_outer);
  const size_t per = 2 * 16 * kDenseStride;
  const size_t used = plan->mats.size() - pd.mat_begin;
  if (used + (size_t)nvar * per > mat_budget_doubles) return false;
  // layout: R0, R1 and column bits c0, c1, c2 such that {R0, R1, c0} and {R0, c1, c2} have
  // distinct residues mod 3 (conflict-free B loads and D stores)
  int regs[4], nr = 0;
  for (int p = 0; p < k; ++p)
    if ((regmask >> p) & 1u) regs[nr++] = p;
  std::vector<int> free_pos;
  for (int p = 0; p < k; ++p)
    if (!((regmask >> p) & 1u) && !((vt >> p) & 1u)) free_pos.push_back(p);
  if (free_pos.size() < 4) return false;
  auto d3 = [](int a, int b, int c) { return (a % 3) != (b % 3) && (a % 3) != (c % 3) && (b % 3) != (c % 3); };
  int best[5] = {0, 1, 0, 1, 2}, best_score = -1;
  for (int r0 = 0; r0 < 4 && best_score < 3; ++r0)
    for (int r1 = 0; r1 < 4 && best_score < 3; ++r1) {
      if (r1 == r0) continue;
      for (size_t a = 0; a < free_pos.size() && best_score < 3; ++a)
        for (size_t b = 0; b < free_pos.size() && best_score < 3; ++b)
          for (size_t c = 0; c < free_pos.size() && best_score < 3; ++c) {
            if (a == b || a == c || b == c) continue;
            const int sc = (d3(regs[r0], regs[r1], free_pos[a]) ? 1 : 0) + (d3(regs[r0], free_pos[b], free_pos[c]) ? 1 : 0) +
                           (adjoint && d3(free_pos[a], free_pos[b], regs[r0]) ? 1 : 0) + (adjoint ? 0 : 1);
            if (sc > best_score) { best_score = sc; best[0] = r0; best[1] = r1; best[2] = (int)a; best[3] = (int)b; best[4] = (int)c; }
          }
    }
  int newreg[4] = {regs[best[0]], regs[best[1]], -1, -1};
  for (int r = 0, w = 2; r < 4; ++r)
    if (r != best[0] && r != best[1]) newreg[w++] = regs[r];
  const int c0 = free_pos[best[2]], c1 = free_pos[best[3]], c2 = free_pos[best[4]];
  std::vector<int> rest;
  for (int p : free_pos)
    if (p != c0 && p != c1 && p != c2) rest.push_back(p);
  std::vector<int> vlist;
  for (int p = 0; p < k; ++p)
    if ((vt >> p) & 1u) vlist.push_back(p);
  // thrpos: c0 c1 c2 | n0 | warp bits (variant positions first)
  std::vector<int> order = {c0, c1, c2, rest[0]};
  std::vector<int> wl = vlist;
  for (size_t i = 1; i < rest.size(); ++i) wl.push_back(rest[i]);
  if ((int)wl.size() != nw_bits) return false;
  order.insert(order.end(), wl.begin(), wl.end());
  int reg_new[32];
  for (int p = 0; p < 32; ++p) reg_new[p] = -1;
  for (int r = 0; r < 4; ++r) reg_new[newreg[r]] = r;
  std::vector<int> olist;
  for (int q = 0; q < 64; ++q)
    if ((vo >> q) & 1ull) olist.push_back(q);
  // variant matrices U_v = G_n ... G_1 (register space), row stride kDenseStride: reserved here,
  // computed by fill_dense_variants() for every stage of the plan at once (independent work items
  // on the host pool; QAOA-like plans carry thousands of variants)
  const size_t off = plan->mats.size() - pd.mat_begin;
  const size_t vdoubles = 2 * 16 * (size_t)kDenseStride;
  plan->mats.resize(plan->mats.size() + (size_t)nvar * vdoubles);
  {
    DenseJob J;
    J.ops = sp->ops;
    J.opm = (size_t)pd.mat_begin;
    J.dst = (size_t)pd.mat_begin + off;
    std::memcpy(J.reg_new, reg_new, sizeof(reg_new));
    J.vlist = vlist;
    J.olist = olist;
    J.m_tile = m_tile;
    J.m_outer = m_outer;
    jobs->push_back(std::move(J));
  }
  StageDesc& S = sp->sd;
  std::memset(&S, 0, sizeof(S));
  S.dense = 1;
  S.m_tile = (uint8_t)m_tile;
  S.m_outer = (uint8_t)m_outer;
  for (int b = 0; b < 8; ++b) S.var_outer[b] = (int8_t)(b < m_outer ? olist[b] : -1);
  for (int r = 0; r < 4; ++r) S.regpos[r] = (int8_t)newreg[r];
  for (int b = 0; b < 12; ++b) S.thrpos[b] = (int8_t)(b < (int)order.size() ? order[b] : -1);
  S.dense_off = (uint32_t)(off / 2);
  const uint32_t p2 = 1u << newreg[2], p3 = 1u << newreg[3], n0 = 1u << order[3], bc0 = 1u << c0;
  const uint32_t p0 = 1u << newreg[0], p1 = 1u << newreg[1], bc1 = 1u << c1, bc2 = 1u << c2;
  for (int w = 0; w < 8; ++w) {
    uint32_t tw = 0;
    for (int b = 0; b < nw_bits; ++b)
      if ((w >> b) & 1) tw |= 1u << order[4 + b];
    S.warp_swz[w] = (uint16_t)swz(tw);
    S.warp_var[w] = (uint8_t)(w & ((1 << m_tile) - 1));
  }
  for (int l = 0; l < 32; ++l) {
    const uint32_t lb = (uint32_t)l;
    S.lane_b[l] = (uint16_t)swz(((lb >> 2) & 1u ? bc0 : 0u) | ((lb >> 3) & 1u ? bc1 : 0u) | ((lb >> 4) & 1u ? bc2 : 0u) |
                                ((lb & 1u) ? p0 : 0u) | ((lb & 2u) ? p1 : 0u));
    S.lane_d[l] = (uint16_t)swz(((lb >> 2) & 1u ? p0 : 0u) | ((lb >> 3) & 1u ? p1 : 0u) | ((lb >> 4) & 1u ? p2 : 0u) |
                                ((lb & 1u) ? bc1 : 0u) | ((lb & 2u) ? bc2 : 0u));
    // R layout: amp a = lane/4 (bits R0 R1 R2) + 8 mt (R3); vector v = lane%4 (c0 c1) + 4 kt (c2, n0)
    S.lane_r[l] = (uint16_t)swz(((lb >> 2) & 1u ? p0 : 0u) | ((lb >> 3) & 1u ? p1 : 0u) | ((lb >> 4) & 1u ? p2 : 0u) |
                                ((lb & 1u) ? bc0 : 0u) | ((lb & 2u) ? bc1 : 0u));
  }
  for (int mt = 0; mt < 2; ++mt)
    for (int kt = 0; kt < 4; ++kt)
      S.off_r[mt * 4 + kt] = (uint16_t)swz((mt ? p3 : 0u) | ((kt & 1) ? bc2 : 0u) | ((kt & 2) ? n0 : 0u));
  S.da_index = da_index;
  {
    // complex64 tiles (8-byte slots, 4-bit XOR fold: position p lands in bank class bit p mod 4):
    // pick the order of the warp's four vector positions whose TF32 fragment lanes (B: three
    // vector bits + register bits 0, 1; D: register bits 0..2 + vector bits 1, 2) spread over
    // the most bank classes
    static const int perms[24][4] = {{0,1,2,3},{0,1,3,2},{0,2,1,3},{0,2,3,1},{0,3,1,2},{0,3,2,1},
                                     {1,0,2,3},{1,0,3,2},{1,2,0,3},{1,2,3,0},{1,3,0,2},{1,3,2,0},
                                     {2,0,1,3},{2,0,3,1},{2,1,0,3},{2,1,3,0},{2,3,0,1},{2,3,1,0},
                                     {3,0,1,2},{3,0,2,1},{3,1,0,2},{3,1,2,0},{3,2,0,1},{3,2,1,0}};
    auto classes = [](std::initializer_list<int> pos) {
      int m = 0;
      for (int p : pos) m |= 1 << (p & 3);
      return __builtin_popcount(m);
    };
    int best = 0, best_score = -1;
    for (int pi = 0; pi < 24; ++pi) {
      int X[4];
      for (int b = 0; b < 4; ++b) X[b] = order[perms[pi][b]];
      const int sc = classes({X[0], X[1], X[2], newreg[0], newreg[1]}) + classes({newreg[0], newreg[1], newreg[2], X[1], X[2]});
      if (sc > best_score) { best_score = sc; best = pi; }
    }
    S.c64_perm = best;
  }
  if (adjoint) {
    S.dense = 2;
    Plan::DAStage ds;
    ds.pass = pass_index;
    ds.da_index = da_index;
    ds.m_tile = m_tile;
    ds.m_outer = m_outer;
    ds.global_slot = plan->da_slots_total + da_index;
    // B_{j,var} = V^dagger (Pi_C G_j) V with V the product of the stage's ops before j, filled
    // per variant with the variant matrices (fill_dense_variants)
    for (size_t i = 0; i < sp->ops.size(); ++i)
      if (sp->ops[i].grad_slot >= 0) {
        ds.slots.push_back(sp->ops[i].grad_slot);
        ds.B.emplace_back((size_t)nvar * 256);
      }
    jobs->back().da = (int)plan->da.size();
    plan->da.push_back(std::move(ds));
  }
  for (int nt = 0; nt < 2; ++nt)
    for (int kq = 0; kq < 4; ++kq)
      S.swz_reg[nt * 4 + kq] = (uint16_t)swz((nt ? n0 : 0u) | ((kq & 1) ? p2 : 0u) | ((kq & 2) ? p3 : 0u));
  for (int nt = 0; nt < 2; ++nt)
    for (int mh = 0; mh < 2; ++mh)
      for (int v = 0; v < 2; ++v)
        S.swz_reg[8 + nt * 4 + mh * 2 + v] = (uint16_t)swz((nt ? n0 : 0u) | (mh ? p3 : 0u) | (v ? bc0 : 0u));
  return true;
}

// Plans the register stages of pass `pd` (ops already emitted in pass order) and rewrites the
// pass' op range in stage order.
// Adjoint stages: diagonal ops the DUAL kernel can evaluate as one run (no register controls,
// purely imaginary diagonal generator) are moved back to join the previous run of the stage when
// they commute with every op in between (disjoint non-diagonal supports, the planner's rule; the
// overlap <lam|D|psi> is unchanged by moving D past a commuting unitary N: <N^+ lam|D|N^+ psi> =
// <lam|N D N^+|psi> = <lam|D|psi>). Longer runs: one conj(lam) psi, one phase application each.
bool diag_run_eligible(const DevOp& o, const PassDesc& pd, const Plan* plan) {
  if ((o.type != OP_D1 && o.type != OP_D2) || o.cj != 0) return false;
  if (o.grad_slot < 0) return true;
  if (!o.gen_diag) return false;
  const double* gm = plan->mats.data() + pd.mat_begin + o.gen_off;
  for (int e = 0; e < o.gen_dim; ++e)
    if (gm[2 * e] != 0.0) return false;
  return true;
}

void group_diag_runs(StagePlan* sp, const PassDesc& pd, const Plan* plan) {
  std::vector<DevOp> out;
  out.reserve(sp->ops.size());
  std::vector<char> elig;
  for (const DevOp& o : sp->ops) {
    const bool e = diag_run_eligible(o, pd, plan);
    size_t pos = out.size();
    if (e) {
      uint64_t N, A;
      phys_masks(o, pd, &N, &A);
      long j = (long)out.size() - 1;
      for (; j >= 0 && !elig[(size_t)j]; --j) {
        uint64_t Nj, Aj;
        phys_masks(out[(size_t)j], pd, &Nj, &Aj);
        if ((N & Aj) || (Nj & A)) break;  // does not commute: stay after it
      }
      if (j >= 0 && elig[(size_t)j]) pos = (size_t)j + 1;
    }
    out.insert(out.begin() + (long)pos, o);
    elig.insert(elig.begin() + (long)pos, e ? 1 : 0);
  }
  sp->ops.swap(out);
}

void plan_pass_stages(Plan* plan, PassDesc* pd, bool forward, bool dense, int n_local, int da_cost,
                      std::vector<DenseJob>* jobs) {
  const int k = pd->k;
  std::vector<DevOp> pops(plan->ops.begin() + pd->op_begin, plan->ops.begin() + pd->op_end);
  std::vector<StagePlan> final_stages;
  auto add_sequential = [&](std::vector<StagePlan> sub) {
    for (StagePlan& sp : sub) {
      layout_sequential(&sp, *pd, pd->R);
      final_stages.push_back(std::move(sp));
    }
  };
  pd->seq_mats = (int32_t)(plan->mats.size() - pd->mat_begin);
  if (forward && dense && k >= 9) {
    const size_t budget = size_t(1) << 22;  // variant matrices live in global memory (L2-resident)
    const int max_var = dense_max_var_for(n_local);
    std::vector<StagePlan> st4 = split_stages(pops, *pd, 4, std::min(3, k - 8), max_var);
    std::vector<DevOp> seq;  // consecutive non-dense candidates are re-staged together
    for (StagePlan& sp : st4) {
      if (make_dense(&sp, *pd, plan, budget, jobs, false, 0, 0, 0, 96, 1, max_var)) {
        if (!seq.empty()) { add_sequential(split_stages(seq, *pd, pd->R, -1, -1)); seq.clear(); }
        final_stages.push_back(std::move(sp));
      } else {
        seq.insert(seq.end(), sp.ops.begin(), sp.ops.end());
      }
    }
    if (!seq.empty()) add_sequential(split_stages(seq, *pd, pd->R, -1, -1));
  } else if (!forward && dense && k >= 9 && g_da_enable) {
    const int da_min = da_min_cost_for(n_local, da_cost);
    // da_cost 0 ("every eligible stage") also admits one outer variant bit at any size
    const int da_outer = da_cost == 0 ? std::max(1, da_max_outer_for(n_local)) : da_max_outer_for(n_local);
    std::vector<StagePlan> st4 = split_stages(pops, *pd, 4, std::min(g_da_max_tile, k - 8), g_da_max_tile + da_outer);
    int nda = 0;  // R accumulator slots of this pass (2^m_outer per adjoint dense stage)
    std::vector<DevOp> seq;
    for (StagePlan& sp : st4) {
      if (nda < g_da_max_per_pass &&
          make_dense(&sp, *pd, plan, size_t(1) << 22, jobs, true, (int)plan->passes.size(), nda, g_da_max_per_pass - nda,
                     da_min, da_outer)) {
        nda += 1 << sp.sd.m_outer;
        if (!seq.empty()) { add_sequential(split_stages(seq, *pd, pd->R, -1, -1)); seq.clear(); }
        final_stages.push_back(std::move(sp));
      } else {
        seq.insert(seq.end(), sp.ops.begin(), sp.ops.end());
      }
    }
    if (!seq.empty()) add_sequential(split_stages(seq, *pd, pd->R, -1, -1));
    plan->max_da_per_pass = std::max(plan->max_da_per_pass, nda);
    plan->da_slots_total += nda;
  } else {
    add_sequential(split_stages(pops, *pd, pd->R, -1, -1));
  }
  // write back in stage order
  pd->stage_begin = (int)plan->stages.size();
  int pos = 0;
  for (size_t si = 0; si < final_stages.size(); ++si) {
    StagePlan& sp = final_stages[si];
    if (!sp.sd.dense) {
      int rp[4];
      for (int r = 0; r < 4; ++r) rp[r] = sp.sd.regpos[r];
      bind_stage_ops(&sp, rp, pd->R, (int)si, plan, *pd);
      if (!forward) group_diag_runs(&sp, *pd, plan);
    } else {
      for (DevOp& o : sp.ops) o.stage = (int16_t)si;
    }
    sp.sd.op_begin = pos;
    for (const DevOp& o : sp.ops) plan->ops[pd->op_begin + pos++] = o;
    sp.sd.op_end = pos;
    plan->stages.push_back(sp.sd);
  }
  pd->stage_end = (int)plan->stages.size();
  for (int i = pd->stage_begin; i < pd->stage_end; ++i) {
    plan->stages[i].next_dense = 0;
    for (int j = i + 1; j < pd->stage_end && j - i < 256; ++j)
      if (plan->stages[j].dense) { plan->stages[i].next_dense = (uint8_t)(j - i); break; }
  }
  int gl = 0;
  for (int i = pd->op_begin; i < pd->op_end; ++i)
    plan->ops[i].grad_local = (int16_t)(plan->ops[i].grad_slot >= 0 ? gl++ : -1);
}

}  // namespace

void host_parallel_for(int n, const std::function<void(int)>& f) { PlanPool::get().run(n, f); }

int choose_tile_qubits(int n_local, const PlanOptions& o, bool dual) {
  // forward passes: 2^11-amplitude tiles (256 threads, three double-buffered CTAs per SM);
  // adjoint (psi + lambda) passes: 2^10 (128 threads, two register-heavy CTAs per SM — measured
  // 8-10% faster than one 2^11 CTA per SM on C2/C3/C4g, profiles/r01_dual_tile_sweep.txt)
  int kmax = dual ? 10 : 11;
  {
    static const int dk = [] { const char* e = getenv("SV_DUAL_K"); return e ? atoi(e) : 0; }();
    static const int fk = [] { const char* e = getenv("SV_FWD_K"); return e ? atoi(e) : 0; }();
    if (dual && dk > 0) kmax = dk;
    if (!dual && fk > 0) kmax = fk;
  }
  if (o.tile_qubits > 0) kmax = std::min(o.tile_qubits, kMaxTileQubits);
  if (dual) kmax = std::min(kmax, 10);  // the DUAL register kernel runs 128-thread CTAs
  kmax = std::max(kmax, std::min(n_local, 2));  // a two-qubit gate must fit a tile
  if (n_local <= kmax) return n_local;
  // keep at least ~2^9 tiles in flight for small states (L2-resident, latency-bound).
  int k = std::max(std::min(kmax, n_local - 9), std::min(kmax, 6));
  return std::min(k, n_local);
}

void build_plan(const std::vector<BoundGate>& gates, int n_local, const PlanOptions& o, bool reverse, Plan* plan) {
  static const bool tmg = std::getenv("SV_PLAN_TIMING") != nullptr;
  const auto tb0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (tmg) std::fprintf(stderr, "build_plan %s at %.3f ms\n", what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb0).count());
  };
  const int k = choose_tile_qubits(n_local, o, reverse);
  const int L = std::min(o.low_qubits, k);
  const uint64_t lowmask = (L >= 64) ? ~0ull : ((1ull << L) - 1);
  const uint64_t allq = (n_local >= 64) ? ~0ull : ((1ull << n_local) - 1);

  // ---- 1. group gates into passes (greedy, order-legal) ----
  std::vector<PassGroup> groups;
  std::vector<int> pending(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) pending[i] = (int)i;
  while (!pending.empty()) {
    PassGroup pg;
    pg.tmask = lowmask;
    uint64_t blockN = 0, blockAll = 0;
    int n_ops = 0, n_mat = 0;
    std::vector<int> skipped;
    for (size_t idx = 0; idx < pending.size(); ++idx) {
      const int gi = pending[idx];
      const BoundGate& g = gates[gi];
      const uint64_t N = is_diag_class(g.cls) ? 0ull : target_mask(g);
      const uint64_t A = target_mask(g) | g.controls;
      bool take = !(N & blockAll) && !(A & blockN);
      if (take && (N & ~pg.tmask)) {
        if (popc(pg.tmask | N) <= k && (o.fusion || pg.gates.empty())) {
          pg.tmask |= N;
        } else if (pg.gates.empty() && popc(N) <= k) {
          // the low-qubit granule must yield (tiny tiles): T = N plus as many low qubits as fit
          uint64_t t = N;
          for (int q = 0; q < L && popc(t) < k; ++q) t |= 1ull << q;
          pg.tmask = t;
        } else {
          take = false;
        }
      }
      if (take && !o.fusion && !pg.gates.empty()) take = false;
      const int md = mat_doubles(g);
      if (take && (n_ops + 1 > kMaxOpsPerPass || n_mat + md > kMaxMatDoublesPerPass)) take = false;
      if (take) {
        pg.gates.push_back(gi);
        n_ops += 1;
        n_mat += md;
      } else {
        skipped.push_back(gi);
        blockN |= N;
        blockAll |= A;
        if ((blockN & allq) == allq) {
          // every qubit carries a skipped non-diagonal gate: nothing further can move ahead
          for (size_t r = idx + 1; r < pending.size(); ++r) skipped.push_back(pending[r]);
          break;
        }
      }
    }
    if (pg.gates.empty()) {  // cannot happen (the first pending gate always fits); guard anyway
      pg.gates.push_back(skipped.front());
      pg.tmask |= target_mask(gates[skipped.front()]);
      skipped.erase(skipped.begin());
    }
    groups.push_back(std::move(pg));
    pending.swap(skipped);
  }

  lap("grouped");
  // ---- 2. emit passes (forward order, or reversed with daggered ops for the adjoint sweep) ----
  plan->passes.clear();
  plan->reverse = reverse;
  plan->n_src_gates = (int64_t)gates.size();
  plan->grid_cache = 0;
  plan->grid_cache_n = -1;  // the plan_grid memo belongs to the plan being replaced
  plan->pass_grid.clear();
  plan->ops.clear();
  plan->mats.clear();
  plan->stages.clear();
  plan->da.clear();
  plan->max_da_per_pass = 0;
  plan->da_slots_total = 0;
  plan->slot_param.clear();
  plan->slot_coeff.clear();
  plan->n_grad_slots = 0;
  std::vector<DenseJob> jobs;  // dense-stage variant matrices, filled once every pass is planned
  std::vector<int> order(groups.size());
  for (size_t i = 0; i < groups.size(); ++i) order[i] = reverse ? (int)(groups.size() - 1 - i) : (int)i;
  for (int gidx : order) {
    PassGroup& pg = groups[gidx];
    // pad T to k qubits, lowest qubits first (extends the contiguous low run when possible)
    uint64_t T = pg.tmask;
    for (int q = 0; q < n_local && popc(T) < k; ++q) T |= 1ull << q;
    PassDesc pd;
    std::memset(&pd, 0, sizeof(pd));
    pd.k = k;
    int low = 0;
    while (low < k && (T >> low) & 1ull) ++low;
    pd.low = low;
    int pos_of[64];
    for (int q = 0; q < 64; ++q) pos_of[q] = -1;
    int p = 0;
    for (int q = 0; q < n_local; ++q)
      if ((T >> q) & 1ull) { pd.tq[p] = (int8_t)q; pos_of[q] = p; ++p; }
    pd.op_begin = (int)plan->ops.size();
    pd.mat_begin = (int)plan->mats.size();
    std::vector<int> gl = pg.gates;
    if (reverse) std::reverse(gl.begin(), gl.end());
    for (int gi : gl) {
      const BoundGate g = reverse ? dagger(gates[gi]) : gates[gi];
      DevOp op;
      std::memset(&op, 0, sizeof(op));
      op.grad_slot = -1;
      op.grad_local = -1;
      op.ra = op.rb = -1;
      op.qa = (int16_t)g.t0;
      op.qb = (int16_t)g.t1;
      op.pa = (int16_t)pos_of[g.t0];
      op.pb = (int16_t)(g.t1 >= 0 ? pos_of[g.t1] : -1);
      for (int q = 0; q < n_local; ++q)
        if ((g.controls >> q) & 1ull) {
          if (pos_of[q] >= 0) op.ctile |= 1ull << pos_of[q];
          else op.couter |= 1ull << q;
        }
      op.mat_off = (int)plan->mats.size() - pd.mat_begin;
      auto push = [&](Cx c) { plan->mats.push_back(c.re); plan->mats.push_back(c.im); };
      switch (g.cls) {
        case GC_GEN1: op.type = OP_M1; for (int e = 0; e < 4; ++e) push(g.m[e]); break;
        case GC_XLIKE: op.type = OP_AX1; push(g.m[0]); push(g.m[1]); break;
        case GC_ZLIKE: op.type = OP_D1; push(g.m[0]); push(g.m[1]); break;
        case GC_GEN2: op.type = OP_M2; for (int e = 0; e < 16; ++e) push(g.m[e]); break;
        case GC_DIAG2: op.type = OP_D2; for (int e = 0; e < 4; ++e) push(g.m[e]); break;
        case GC_SWAP: op.type = OP_SWAP; break;
      }
      if (reverse && g.param >= 0) {
        op.grad_slot = plan->n_grad_slots++;
        plan->slot_param.push_back(g.param);
        plan->slot_coeff.push_back(g.coeff);
        op.gen_off = (int)plan->mats.size() - pd.mat_begin;
        op.gen_dim = (int16_t)g.gen_dim;
        const bool diag = (g.kind == SV_RZ || g.kind == SV_PS || g.kind == SV_RZZ);
        op.gen_diag = diag ? 1 : 0;
        if (diag) {
          for (int j = 0; j < g.gen_dim; ++j) push(g.gen[j * g.gen_dim + j]);
        } else {
          for (int e = 0; e < g.gen_dim * g.gen_dim; ++e) push(g.gen[e]);
        }
        pd.n_grad++;
      }
      op.src = gi;
      plan->ops.push_back(op);
    }
    pd.op_end = (int)plan->ops.size();
    if (o.kernel == 1 && k - 3 >= 5) {
      pd.R = 3;
      {
        static const bool tm = std::getenv("SV_PLAN_TIMING") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        plan_pass_stages(plan, &pd, !reverse, o.dense != 0, n_local, o.da_cost, &jobs);
        if (tm)
          std::fprintf(stderr, "pass %zu stages %.3f ms\n", plan->passes.size(),
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      }
    } else {
      pd.R = 0;
      pd.seq_mats = (int32_t)(plan->mats.size() - pd.mat_begin);
      pd.stage_begin = pd.stage_end = (int)plan->stages.size();
      int gl = 0;
      for (int i = pd.op_begin; i < pd.op_end; ++i)
        plan->ops[i].grad_local = (int16_t)(plan->ops[i].grad_slot >= 0 ? gl++ : -1);
    }
    plan->passes.push_back(pd);
  }
  lap("emitted");
  fill_dense_variants(plan, jobs);
  lap("dense variants");
  emit_rops(plan);
  plan->jobs = std::make_shared<PlanJobs>();
  plan->jobs->jobs = std::move(jobs);
}

// (matrix entries of one op, in the emission layout of build_plan)
static void write_op_mats(double* dst, const BoundGate& g) {
  auto put = [&](int& k, Cx c) { dst[k++] = c.re; dst[k++] = c.im; };
  int k = 0;
  switch (g.cls) {
    case GC_GEN1: for (int e = 0; e < 4; ++e) put(k, g.m[e]); break;
    case GC_XLIKE: put(k, g.m[0]); put(k, g.m[1]); break;
    case GC_ZLIKE: put(k, g.m[0]); put(k, g.m[1]); break;
    case GC_GEN2: for (int e = 0; e < 16; ++e) put(k, g.m[e]); break;
    case GC_DIAG2: for (int e = 0; e < 4; ++e) put(k, g.m[e]); break;
    default: break;
  }
}

void refresh_plan(const std::vector<BoundGate>& gates, Plan* plan) {
  for (const PassDesc& pd : plan->passes)
    for (int i = pd.op_begin; i < pd.op_end; ++i) {
      const DevOp& o = plan->ops[i];
      const BoundGate g = plan->reverse ? dagger(gates[(size_t)o.src]) : gates[(size_t)o.src];
      write_op_mats(plan->mats.data() + pd.mat_begin + o.mat_off, g);
      if (o.grad_slot >= 0) {  // generators can carry values too (sharded shards fold rank-bit signs)
        double* gm = plan->mats.data() + pd.mat_begin + o.gen_off;
        int k = 0;
        if (o.gen_diag)
          for (int j = 0; j < g.gen_dim; ++j) { gm[k++] = g.gen[j * g.gen_dim + j].re; gm[k++] = g.gen[j * g.gen_dim + j].im; }
        else
          for (int e = 0; e < g.gen_dim * g.gen_dim; ++e) { gm[k++] = g.gen[e].re; gm[k++] = g.gen[e].im; }
      }
    }
  if (plan->jobs) {
    // the jobs hold copies of their ops; their matrices are read from plan->mats
    fill_dense_variants(plan, plan->jobs->jobs);
  }
  emit_rops(plan);
}

// compact register-kernel ops (value-dependent codes: fast diagonal flags, RX / RY, diagonal runs)
void emit_rops(Plan* plan) {
  plan->rops.assign(plan->ops.size(), RegOp{});
  for (const PassDesc& pd : plan->passes) {
    if (pd.R == 0) continue;
    for (int i = pd.op_begin; i < pd.op_end; ++i) {
      const DevOp& o = plan->ops[i];
      RegOp r;
      std::memset(&r, 0, sizeof(r));
      const uint32_t ra = o.ra >= 0 ? (uint32_t)o.ra : 15u, rb = o.rb >= 0 ? (uint32_t)o.rb : 15u;
      const uint32_t pa = o.pa >= 0 ? (uint32_t)o.pa : 31u, pb = o.pb >= 0 ? (uint32_t)o.pb : 31u;
      const uint32_t gen = o.grad_slot >= 0 ? (o.gen_dim == 4 ? 2u : 1u) : 0u;
      uint32_t dfl = 0;
      uint32_t type = (uint32_t)o.type;
      if (o.type == OP_M1 && o.cj == 0 && o.ra >= 0) {
        // real-structured rotations (RX / RY and their daggers) run as OP_RX / OP_RY: exact for any
        // matrix of that form; a generator must be the rotation's own (-i/2 X or -i/2 Y)
        const double* m = plan->mats.data() + pd.mat_begin + o.mat_off;  // m00 m01 m10 m11 (re, im)
        const bool rx = m[1] == 0.0 && m[2] == 0.0 && m[7] == 0.0 && m[6] == m[0] && m[4] == 0.0 && m[5] == m[3];
        const bool ry = m[1] == 0.0 && m[3] == 0.0 && m[5] == 0.0 && m[7] == 0.0 && m[6] == m[0] && m[4] == -m[2];
        bool gen_ok = true;
        if (o.grad_slot >= 0) {
          const double* gm = plan->mats.data() + pd.mat_begin + o.gen_off;
          const double gx[8] = {0, 0, 0, -0.5, 0, -0.5, 0, 0}, gy[8] = {0, 0, -0.5, 0, 0.5, 0, 0, 0};
          const double* want = rx ? gx : gy;
          gen_ok = o.gen_dim == 2 && !o.gen_diag;
          for (int e = 0; e < 8 && gen_ok; ++e) gen_ok = gm[e] == want[e];
        }
        if ((rx || ry) && gen_ok) type = rx ? OP_RX : OP_RY;
      }
      if (o.type == OP_D1) {
        const double* m = plan->mats.data() + pd.mat_begin + o.mat_off;
        if (m[0] == 1.0 && m[1] == 0.0) {
          dfl |= 1u;
          if (m[2] == -1.0 && m[3] == 0.0) dfl |= 2u;
        }
      }
      r.code = type | (ra << 4) | (rb << 8) | ((uint32_t)o.cj << 12) | (pa << 16) | (pb << 21) |
               (gen << 26) | ((o.gen_diag ? 1u : 0u) << 28) | (dfl << 29);
      r.mat_off = (uint16_t)(o.mat_off / 2);
      r.gen_off = (uint16_t)(o.gen_off / 2);
      r.cthr = (uint16_t)o.cthr;
      r.grad_local = o.grad_local;
      r.qa = (uint8_t)(o.qa >= 0 ? o.qa : 0);
      r.qb = (uint8_t)(o.qb >= 0 ? o.qb : 0);
      r.couter = o.couter;
      r.grad_slot = o.grad_slot;
      r.pad = (o.couter != 0 || o.cthr != 0) ? kRopHasCtrl : 0;  // kernels skip the control test otherwise
      plan->rops[i] = r;
    }
    // adjoint passes: runs of >= 2 consecutive diagonal ops of a sequential stage without register
    // controls (their generators purely imaginary diagonals: RZ, RZZ, PS) are evaluated together by
    // the DUAL kernel (conj(lambda) psi is invariant under diagonal un-applies, so every overlap of
    // the run uses it; the run's phases are multiplied into per-thread factor tables and applied
    // once). The first op of a run carries the run length.
    if (!plan->reverse) continue;
    for (int si = pd.stage_begin; si < pd.stage_end; ++si) {
      const StageDesc& S = plan->stages[si];
      if (S.dense) continue;
      auto eligible = [&](int i) { return diag_run_eligible(plan->ops[i], pd, plan); };
      const int b = pd.op_begin + S.op_begin, e = pd.op_begin + S.op_end;
      for (int i = b; i < e;) {
        int j = i;
        while (j < e && eligible(j)) ++j;
        if (j - i >= g_diag_run_min) {
          plan->rops[i].pad = (uint16_t)((plan->rops[i].pad & kRopHasCtrl) | std::min(j - i, (int)kRopRunMask));
          static const bool dbg = std::getenv("SV_PLAN_DEBUG") != nullptr;
          if (dbg) std::fprintf(stderr, "diag run: pass %d stage %d ops %d\n", (int)(&pd - plan->passes.data()), si, j - i);
          i = std::min(j, i + (int)kRopRunMask);
        } else {
          i = j + 1;
        }
      }
    }
  }
}

// FP64 additions per amplitude outside the FMAs: the Gauss form's sums (one per input element and
// two per A entry amortised over the warp's 16 vectors: 24 DADDs per 256 amplitudes = 3 per amp)
int pass_add_per_amp(const Plan& plan, size_t i) {
  const PassDesc& pd = plan.passes[i];
  int f = 0;
  if (pd.R > 0)
    for (int si = pd.stage_begin; si < pd.stage_end; ++si) {
      const StageDesc& S = plan.stages[si];
      if (S.dense) f += S.dense == 2 ? 3 * 3 : 3;
    }
  return f;
}

int pass_fma_per_amp(const Plan& plan, size_t i) {
  const PassDesc& pd = plan.passes[i];
  int f = 0;
  if (pd.R > 0) {
    for (int si = pd.stage_begin; si < pd.stage_end; ++si) {
      const StageDesc& S = plan.stages[si];
      // Gauss form (kernels_reg.cu dense_apply): 48 DMMA FMAs per amplitude; adjoint dense
      // stages apply it to psi and lambda and accumulate R (48 more)
      if (S.dense) { f += S.dense == 2 ? 3 * 48 : 48; continue; }
      for (int j = pd.op_begin + S.op_begin; j < pd.op_begin + S.op_end; ++j)
        f += seq_cost(plan.ops[j], plan.mats.data() + pd.mat_begin + plan.ops[j].mat_off);
    }
  } else {
    for (int j = pd.op_begin; j < pd.op_end; ++j) f += seq_cost(plan.ops[j], plan.mats.data() + pd.mat_begin + plan.ops[j].mat_off);
  }
  return f;
}

}  // namespace sv
