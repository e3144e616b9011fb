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
#include <cstring>

#include "sv.h"
#include "sv_internal.h"

namespace sv {
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

bool op_is_diag(const DevOp& o) { return o.type == OP_D1 || o.type == OP_D2; }

// Splits the ops of one pass into register stages (see StageDesc) and reorders them stage by
// stage. An op joins the current stage if it may legally move ahead of the ops left for later
// stages (same commutation rule as the pass planner) and its non-diagonal target positions fit
// the stage's R register positions.
void plan_stages(Plan* plan, PassDesc* pd, int R) {
  const int k = pd->k;
  std::vector<DevOp> ops(plan->ops.begin() + pd->op_begin, plan->ops.begin() + pd->op_end);
  auto phys_masks = [&](const DevOp& o, uint64_t* N, uint64_t* A) {
    uint64_t t = (1ull << o.qa) | (o.qb >= 0 ? (1ull << o.qb) : 0ull);
    uint64_t c = o.couter;
    for (int p = 0; p < k; ++p)
      if ((o.ctile >> p) & 1ull) c |= 1ull << pd->tq[p];
    *N = op_is_diag(o) ? 0ull : t;
    *A = t | c;
  };
  auto pos_mask = [&](const DevOp& o) -> uint32_t {
    if (op_is_diag(o)) return 0u;
    return (1u << o.pa) | (o.pb >= 0 ? (1u << o.pb) : 0u);
  };
  std::vector<int> pending(ops.size());
  for (size_t i = 0; i < ops.size(); ++i) pending[i] = (int)i;
  std::vector<DevOp> out;
  pd->stage_begin = (int)plan->stages.size();
  int stage_idx = 0;
  while (!pending.empty()) {
    uint32_t regset = 0;
    uint64_t bN = 0, bA = 0;
    std::vector<int> taken, skipped;
    for (int i : pending) {
      uint64_t N, A;
      phys_masks(ops[i], &N, &A);
      bool ok = !(N & bA) && !(A & bN);
      const uint32_t pm = pos_mask(ops[i]);
      if (ok && (pm & ~regset)) {
        if (__builtin_popcount(regset | pm) <= R) regset |= pm;
        else ok = false;
      }
      if (ok) taken.push_back(i);
      else { skipped.push_back(i); bN |= N; bA |= A; }
    }
    // layout: lanes 0..2 on thread positions with distinct residues mod 3 (conflict-free 16-byte
    // shared-memory phases), then fill the register set, then the remaining thread positions.
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
    // fill registers from the highest free positions
    while (__builtin_popcount(regset) < R && !free_pos.empty()) {
      regset |= 1u << free_pos.back();
      free_pos.pop_back();
    }
    std::vector<int> thr = lanes;
    thr.insert(thr.end(), free_pos.begin(), free_pos.end());
    StageDesc sd;
    std::memset(&sd, 0, sizeof(sd));
    int rp[4] = {-1, -1, -1, -1}, nr = 0;
    int reg_of[32];
    for (int p = 0; p < 32; ++p) reg_of[p] = -1;
    for (int p = 0; p < k; ++p)
      if ((regset >> p) & 1u) { rp[nr] = p; reg_of[p] = nr; ++nr; }
    for (int r = 0; r < 4; ++r) sd.regpos[r] = (int8_t)rp[r];
    for (int b = 0; b < 12; ++b) sd.thrpos[b] = (int8_t)(b < (int)thr.size() ? thr[b] : -1);
    for (int j = 0; j < (1 << R); ++j) {
      uint32_t dep = 0;
      for (int r = 0; r < R; ++r)
        if ((j >> r) & 1) dep |= 1u << rp[r];
      sd.swz_reg[j] = (uint16_t)swz(dep);
    }
    sd.op_begin = (int)out.size();
    for (int i : taken) {
      DevOp o = ops[i];
      o.stage = (int16_t)stage_idx;
      o.ra = (int8_t)(o.pa >= 0 ? reg_of[o.pa] : -1);
      o.rb = (int8_t)(o.pb >= 0 ? reg_of[o.pb] : -1);
      o.cj = 0;
      o.cthr = 0;
      for (int p = 0; p < k; ++p)
        if ((o.ctile >> p) & 1ull) {
          if (reg_of[p] >= 0) o.cj |= (uint8_t)(1u << reg_of[p]);
          else o.cthr |= 1ull << p;
        }
      // two-qubit non-diagonal ops: canonical register order ra < rb (swap matrix index bits)
      if ((o.type == OP_M2 || o.type == OP_SWAP) && o.ra > o.rb) {
        std::swap(o.ra, o.rb);
        std::swap(o.pa, o.pb);
        std::swap(o.qa, o.qb);
        auto perm = [](int i) { return ((i & 1) << 1) | ((i >> 1) & 1); };
        if (o.type == OP_M2) {
          double* m = plan->mats.data() + pd->mat_begin + o.mat_off;
          double t[32];
          for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
              t[2 * (perm(r) * 4 + perm(c))] = m[2 * (r * 4 + c)];
              t[2 * (perm(r) * 4 + perm(c)) + 1] = m[2 * (r * 4 + c) + 1];
            }
          std::memcpy(m, t, sizeof(t));
        }
        if (o.grad_slot >= 0 && !o.gen_diag && o.gen_dim == 4) {
          double* g = plan->mats.data() + pd->mat_begin + o.gen_off;
          double t[32];
          for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
              t[2 * (perm(r) * 4 + perm(c))] = g[2 * (r * 4 + c)];
              t[2 * (perm(r) * 4 + perm(c)) + 1] = g[2 * (r * 4 + c) + 1];
            }
          std::memcpy(g, t, sizeof(t));
        }
      }
      out.push_back(o);
    }
    sd.op_end = (int)out.size();
    plan->stages.push_back(sd);
    ++stage_idx;
    pending.swap(skipped);
  }
  std::copy(out.begin(), out.end(), plan->ops.begin() + pd->op_begin);
  pd->stage_end = (int)plan->stages.size();
  // local grad indices
  int gl = 0;
  for (int i = pd->op_begin; i < pd->op_end; ++i) plan->ops[i].grad_local = (int16_t)(plan->ops[i].grad_slot >= 0 ? gl++ : -1);
}

}  // namespace

int choose_tile_qubits(int n_local, const PlanOptions& o, bool dual) {
  int kmax = dual ? 11 : 12;
  if (o.tile_qubits > 0) kmax = std::min(o.tile_qubits, kMaxTileQubits);
  kmax = std::max(kmax, std::min(n_local, 2));  // a two-qubit gate must fit a tile
  if (n_local <= kmax) return n_local;
  // keep at least ~2^9 tiles in flight for small states (L2-resident, latency-bound).
  int k = std::max(std::min(kmax, n_local - 9), std::min(kmax, 6));
  return std::min(k, n_local);
}

void build_plan(const std::vector<BoundGate>& gates, int n_local, const PlanOptions& o, bool reverse, Plan* plan) {
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

  // ---- 2. emit passes (forward order, or reversed with daggered ops for the adjoint sweep) ----
  plan->passes.clear();
  plan->ops.clear();
  plan->mats.clear();
  plan->stages.clear();
  plan->slot_param.clear();
  plan->slot_coeff.clear();
  plan->n_grad_slots = 0;
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
      plan->ops.push_back(op);
    }
    pd.op_end = (int)plan->ops.size();
    const int R = reverse ? 3 : 4;
    if (o.kernel == 1 && k - R >= 5) {
      pd.R = R;
      plan_stages(plan, &pd, R);
    } else {
      pd.R = 0;
      pd.stage_begin = pd.stage_end = (int)plan->stages.size();
      int gl = 0;
      for (int i = pd.op_begin; i < pd.op_end; ++i)
        plan->ops[i].grad_local = (int16_t)(plan->ops[i].grad_slot >= 0 ? gl++ : -1);
    }
    plan->passes.push_back(pd);
  }
}

}  // namespace sv
