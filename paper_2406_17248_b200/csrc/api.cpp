// api.cpp — the C ABI (include/sv.h): handles, validation, orchestration of plans and kernels.
//
// Every numerical step runs in kernels.cu; this file only validates, binds (gates.cpp), plans
// (plan.cpp), uploads plan data and launches. Sharding (sv_create_sharded / virtual shards) lives
// in shard.cpp.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <thread>
#include <string>
#include <vector>

#include "sv.h"
#include "sv_internal.h"
#include "sv_handle.h"

namespace sv {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(sv_state_s* h, cudaError_t e, const char* where) {
  if (h) h->poisoned = true;
  return fail(SV_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool DevBuf::ensure(size_t bytes) {
  if (bytes <= cap) return true;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  size_t want = bytes < 4096 ? 4096 : bytes;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return false;
  }
  cap = want;
  return true;
}
bool PinnedBuf::ensure(size_t bytes) {
  if (bytes <= cap) return true;
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
  const size_t want = bytes < 65536 ? 65536 : bytes + bytes / 4;
  if (cudaMallocHost(&p, want) != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return false;
  }
  cap = want;
  return true;
}
void PinnedBuf::release() {
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
}

bool DevBuf::ensure_async(size_t bytes, cudaStream_t s) {
  if (bytes <= cap) return true;
  if (p) {
    if (async) cudaFreeAsync(p, s);
    else cudaFree(p);
  }
  p = nullptr;
  cap = 0;
  const size_t want = bytes < 65536 ? 65536 : bytes + bytes / 2;
  if (cudaMallocAsync(&p, want, s) != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return false;
  }
  async = true;
  cap = want;
  return true;
}

void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  async = false;
}

int check_handle(sv_state_s* h) {
  if (!h) return fail(SV_E_ARG, "null handle");
  if (h->poisoned) return fail(SV_E_POISONED, "handle poisoned by an earlier CUDA/NCCL failure");
  return SV_OK;
}

// Validates and binds a whole circuit (all-or-nothing).
int bind_circuit(sv_state_s* h, const sv_gate* gates, int64_t n_gates, const double* params, int32_t n_params,
                 bool for_grad, std::vector<BoundGate>* out) {
  if (n_gates < 0 || (n_gates > 0 && !gates)) return fail(SV_E_ARG, "bad gate array");
  if (n_params < 0) return fail(SV_E_ARG, "negative n_params");
  out->resize((size_t)n_gates);
  std::string err;
  for (int64_t i = 0; i < n_gates; ++i) {
    int rc = bind_gate(h->n, &gates[i], params, n_params, for_grad, &(*out)[(size_t)i], &err);
    if (rc != SV_OK) return fail(rc, "gate " + std::to_string(i) + ": " + err);
  }
  return SV_OK;
}

// 64-bit key of a byte range, eight bytes per step (a 600-gate bound circuit is ~330 KB: a
// byte-at-a-time hash cost ~0.4 ms per plan lookup). Multiply-rotate rounds with a final avalanche.
static uint64_t hash_bytes(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  auto round = [](uint64_t acc, uint64_t w) {
    acc ^= w * 0x9E3779B97F4A7C15ull;
    acc = (acc << 31) | (acc >> 33);
    return acc * 0xC2B2AE3D27D4EB4Full;
  };
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, p + i, 8);
    h = round(h, w);
  }
  uint64_t t = 0;
  std::memcpy(&t, p + i, n - i);
  h = round(h, t ^ ((uint64_t)n << 56));
  h ^= h >> 33;
  h *= 0xFF51AFD7ED558CCDull;
  h ^= h >> 33;
  return h;
}

void release_plan_cache(sv_state_s* h) {
  for (CachedPlan* c : h->plan_cache) {
    c->buf.release();
    if (c->used_ev) cudaEventDestroy(c->used_ev);
    if (c->ready_ev) cudaEventDestroy(c->ready_ev);
    delete c;
  }
  h->plan_cache.clear();
}

// Records the plan's last use on the handle's stream (see CachedPlan::used_ev).
static void mark_plan_used(sv_state_s* h, const CachedPlan& cp) {
  CachedPlan& c = const_cast<CachedPlan&>(cp);
  if (!c.used_ev && cudaEventCreateWithFlags(&c.used_ev, cudaEventDisableTiming) != cudaSuccess) {
    c.used_ev = nullptr;
    c.used_rec = false;
    cudaGetLastError();
    return;
  }
  c.used_rec = cudaEventRecord(c.used_ev, h->stream) == cudaSuccess;
  if (!c.used_rec) cudaGetLastError();
}

struct PlanMeta {
  int v[9];
};
static PlanMeta plan_meta(const sv_state_s* h, const std::vector<BoundGate>& gates, bool reverse) {
  return PlanMeta{{h->n_local, reverse ? 1 : 0, h->opts.tile_qubits, h->opts.low_qubits, h->opts.fusion ? 1 : 0,
                   h->opts.kernel, h->opts.dense, h->opts.da_cost, (int)gates.size()}};
}

static uint64_t plan_key(const std::vector<BoundGate>& gates, const PlanMeta& meta) {
  uint64_t key = 1469598103934665603ull;
  key = hash_bytes(gates.data(), gates.size() * sizeof(BoundGate), key);
  return hash_bytes(&meta, sizeof(meta), key);
}

static bool plan_ident_equal(const CachedPlan& c, const std::vector<BoundGate>& gates, const PlanMeta& meta) {
  const size_t gb = gates.size() * sizeof(BoundGate);
  return c.ident.size() == gb + sizeof(meta) && std::memcmp(c.ident.data(), gates.data(), gb) == 0 &&
         std::memcmp(c.ident.data() + gb, &meta, sizeof(meta)) == 0;
}

static constexpr int kCacheEntries = 8;

// A cache slot for a new plan: a fresh entry, or the least recently used one.
static CachedPlan* plan_slot(sv_state_s* h) {
  CachedPlan* c = nullptr;
  if ((int)h->plan_cache.size() < kCacheEntries) {
    c = new CachedPlan();
    h->plan_cache.push_back(c);
    return c;
  }
  for (CachedPlan* x : h->plan_cache)
    if (!c || x->stamp < c->stamp) c = x;
  return c;
}

static int upload_plan(sv_state_s* h, CachedPlan* c, uint64_t key, const CachedPlan** out);

// The structure of a circuit: everything planning decisions depend on except matrix values (the
// angles of an optimiser step, user matrices): class, kind, qubits, controls, parameter slot,
// chain-rule coefficient, generator size.
static std::vector<int64_t> struct_ident(const std::vector<BoundGate>& gates, const PlanMeta& meta) {
  std::vector<int64_t> v;
  v.reserve(gates.size() * 7 + 10);
  for (const BoundGate& g : gates) {
    int64_t cb;
    std::memcpy(&cb, &g.coeff, 8);
    v.push_back(((int64_t)g.cls << 32) | (uint32_t)g.kind);
    v.push_back(((int64_t)g.t0 << 32) | (uint32_t)g.t1);
    v.push_back((int64_t)g.controls);
    v.push_back(((int64_t)g.param << 32) | (uint32_t)g.gen_dim);
    v.push_back(cb);
  }
  for (int m : meta.v) v.push_back(m);
  return v;
}

int get_plan(sv_state_s* h, const std::vector<BoundGate>& gates, bool reverse, const CachedPlan** out) {
  const PlanMeta meta = plan_meta(h, gates, reverse);
  const uint64_t key = plan_key(gates, meta);
  for (CachedPlan* c : h->plan_cache)
    if (c->key == key && plan_ident_equal(*c, gates, meta)) {
      c->stamp = ++h->plan_clock;
      *out = c;
      return SV_OK;
    }
  auto set_ident = [&](CachedPlan* c) {
    const size_t gb = gates.size() * sizeof(BoundGate);
    c->ident.resize(gb + sizeof(meta));
    std::memcpy(c->ident.data(), gates.data(), gb);
    std::memcpy(c->ident.data() + gb, &meta, sizeof(meta));
  };
  // same structure, new values (an optimiser step): refresh that plan's matrices in place
  std::vector<int64_t> sid = struct_ident(gates, meta);
  const uint64_t skey = hash_bytes(sid.data(), sid.size() * 8, 0x5bd1e995ull);
  static const bool no_refresh = std::getenv("SV_PLAN_REFRESH") && std::atoi(std::getenv("SV_PLAN_REFRESH")) == 0;
  if (!no_refresh)
    for (CachedPlan* c : h->plan_cache)
      if (c->key != 0 && c->skey == skey && c->sident == sid) {
        c->key = 0;
        set_ident(c);
        refresh_plan(gates, &c->plan);
        h->stats.plan_refreshes += 1;
        return upload_plan(h, c, key, out);
      }
  CachedPlan* c = plan_slot(h);
  c->key = 0;
  set_ident(c);
  c->skey = skey;
  c->sident.swap(sid);
  build_plan(gates, h->n_local, h->opts, reverse, &c->plan);
  h->stats.plan_builds += 1;
  return upload_plan(h, c, key, out);
}

static int upload_plan(sv_state_s* h, CachedPlan* c, uint64_t key, const CachedPlan** out) {
  // one buffer: [ops | stages | mats | rops], each section 64-byte aligned; one H2D copy
  const Plan& plan = c->plan;
  auto al = [](size_t x) { return (x + 63) & ~size_t(63); };
  const size_t ob = plan.ops.size() * sizeof(DevOp), sb = plan.stages.size() * sizeof(StageDesc),
               mb = plan.mats.size() * sizeof(double), rb = plan.rops.size() * sizeof(RegOp);
  const size_t so = al(ob), mo = so + al(sb), ro = mo + al(mb), total = ro + al(rb);
  const void* old_p = c->buf.p;
  const size_t old_cap = c->buf.cap;
  if (!c->buf.ensure_async(total + 64, h->stream)) return fail(SV_E_OOM, "plan buffers");
  // an existing buffer whose last use is recorded is refilled on the upload stream (after that use)
  // and the handle's stream waits for the copy: the copy overlaps the kernels queued before it; a
  // (re)allocated buffer is stream-ordered on the handle's stream and is filled there
  bool side = old_p != nullptr && c->buf.p == old_p && c->buf.cap == old_cap && c->used_rec;
  if (side && !h->upload_stream &&
      cudaStreamCreateWithFlags(&h->upload_stream, cudaStreamNonBlocking) != cudaSuccess) {
    h->upload_stream = nullptr;
    cudaGetLastError();
  }
  if (side && !c->ready_ev && cudaEventCreateWithFlags(&c->ready_ev, cudaEventDisableTiming) != cudaSuccess) {
    c->ready_ev = nullptr;
    cudaGetLastError();
  }
  side = side && h->upload_stream && c->ready_ev;
  // page-locked staging: the copy is truly asynchronous (a pageable source would hold the host
  // until the stream reaches it); the previous upload from the same buffer must have completed
  cudaError_t e = cudaSuccess;
  if (h->plan_upload_done) {
    e = cudaEventSynchronize(h->plan_upload_done);
    if (e != cudaSuccess) return cuda_fail(h, e, "plan upload");
  } else {
    e = cudaEventCreateWithFlags(&h->plan_upload_done, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(h, e, "plan upload event");
  }
  if (!h->pin_plan.ensure(total + 64)) return fail(SV_E_OOM, "plan staging");
  char* hs = static_cast<char*>(h->pin_plan.p);
  std::memcpy(hs, plan.ops.data(), ob);
  std::memcpy(hs + so, plan.stages.data(), sb);
  {
    // the variant matrices dominate (16 MB for C3): copied in parallel chunks on the host pool
    constexpr size_t kChunk = size_t(1) << 20;
    const int nch = (int)((mb + kChunk - 1) / kChunk);
    const char* src = reinterpret_cast<const char*>(plan.mats.data());
    host_parallel_for(nch, [&](int i) {
      const size_t b = (size_t)i * kChunk;
      std::memcpy(hs + mo + b, src + b, std::min(kChunk, mb - b));
    });
  }
  std::memcpy(hs + ro, plan.rops.data(), rb);
  c->so = so;
  c->mo = mo;
  c->ro = ro;
  if (side) {
    e = cudaStreamWaitEvent(h->upload_stream, c->used_ev, 0);
    if (e == cudaSuccess && total) e = cudaMemcpyAsync(c->buf.p, hs, total, cudaMemcpyHostToDevice, h->upload_stream);
    if (e == cudaSuccess) e = cudaEventRecord(h->plan_upload_done, h->upload_stream);
    if (e == cudaSuccess) e = cudaEventRecord(c->ready_ev, h->upload_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, c->ready_ev, 0);
  } else {
    if (total) e = cudaMemcpyAsync(c->buf.p, hs, total, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaEventRecord(h->plan_upload_done, h->stream);
  }
  if (e != cudaSuccess) return cuda_fail(h, e, "plan upload");
  c->key = key;
  c->stamp = ++h->plan_clock;
  *out = c;
  return SV_OK;
}

// Runs all passes of a plan on psi (and lam for the adjoint plan).
int run_plan(sv_state_s* h, const CachedPlan& cp, double* psi, double* lam, double* d_partials, int grid,
             double* r_partials, double* r_sum) {
  const Plan& plan = cp.plan;
  const char* base = static_cast<const char*>(cp.buf.p);
  const_cast<CachedPlan&>(cp).used_rec = false;  // (until all passes are enqueued: mark_plan_used)
  size_t da_done = 0;
  for (size_t i = 0; i < plan.passes.size(); ++i) {
    const PassDesc& pd = plan.passes[i];
    int n_da = 0;  // R accumulator slots
    for (int si = pd.stage_begin; si < pd.stage_end; ++si) n_da += plan.stages[si].dense == 2 ? (1 << plan.stages[si].m_outer) : 0;
    const int next_mat = (i + 1 < plan.passes.size()) ? plan.passes[i + 1].mat_begin : (int)plan.mats.size();
    PassLaunch L;
    L.pd = &pd;
    L.d_ops = reinterpret_cast<const DevOp*>(base);
    L.d_stages = reinterpret_cast<const StageDesc*>(base + cp.so);
    L.d_mats = reinterpret_cast<const double*>(base + cp.mo);
    L.d_rops = reinterpret_cast<const RegOp*>(base + cp.ro);
    L.d_partials = d_partials;
    L.nmats = next_mat - pd.mat_begin;
    const int pg = plan_grid(plan, h->n_local);  // fills plan.pass_grid
    L.pstride = grid > 0 ? grid : pg;
    L.grid = i < plan.pass_grid.size() ? std::min(plan.pass_grid[i], L.pstride) : L.pstride;
    L.n_local = h->n_local;
    L.rank_bits = 0;
    L.n_da = n_da;
    L.all_dense = !lam && pass_all_dense(plan, pd);
    L.no_dense = !lam && pass_no_dense(plan, pd);
    L.acc_thread = (lam && i < plan.pass_acc.size()) ? plan.pass_acc[i] : 0;
    L.r_partials = r_partials;
    if (n_da && (!r_partials || !r_sum)) return fail(SV_E_ARG, "internal: adjoint dense stage without R buffers");
    cudaError_t e = launch_pass(psi, lam, L, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "pass launch");
    h->stats.kernel_launches += 1;
    if (n_da) {
      const int nw = (1 << (pd.k - pd.R)) / 32;
      // R partials: per-CTA contiguous when accumulated in global memory, slot-major otherwise
      e = da_r_global(h->n_local)
              ? launch_reduce_strided(r_partials, (int64_t)n_da * nw * 512, L.grid, r_sum + da_done * (size_t)nw * 512,
                                      h->stream)
              : launch_reduce_slots(r_partials, n_da * nw * 512, L.grid, r_sum + da_done * (size_t)nw * 512, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "R reduction");
      h->stats.kernel_launches += 1;
      da_done += (size_t)n_da;
    }
    const double amps = (double)(1ull << h->n_local);
    if (i == 0) h->stats.gate_applications += plan.n_src_gates * (lam ? 2 : 1);
    if (lam) {
      h->stats.adjoint_passes += 1;
      h->stats.algorithmic_bytes += 64.0 * amps;
    } else {
      h->stats.gate_passes += 1;
      h->stats.algorithmic_bytes += 32.0 * amps;
    }
  }
  mark_plan_used(h, cp);
  return SV_OK;
}

int c64_promote(sv_state_s* h) {
  const int64_t N = int64_t(1) << h->n_local;
  if (!h->promo.ensure(size_t(16) << h->n_local)) return fail(SV_E_OOM, "complex128 scratch of a complex64 state");
  h->psi = static_cast<double*>(h->promo.p);
  cudaError_t e = launch_widen(h->psi32, h->psi, N, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "widen");
  h->stats.kernel_launches += 1;
  h->stats.algorithmic_bytes += 24.0 * (double)N;
  return SV_OK;
}

static int c64_demote(sv_state_s* h) {
  const int64_t N = int64_t(1) << h->n_local;
  cudaError_t e = launch_narrow(h->psi, h->psi32, N, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "narrow");
  h->stats.kernel_launches += 1;
  h->stats.algorithmic_bytes += 24.0 * (double)N;
  return SV_OK;
}

// complex64 forward passes: every pass must be a register pass the complex64 kernel takes (tile
// position 0 = qubit 0, 2^9..2^11-amplitude tiles); otherwise the circuit runs on a complex128
// scratch copy (widen, complex128 passes, narrow).
static int run_plan_c64(sv_state_s* h, const CachedPlan& cp) {
  const_cast<CachedPlan&>(cp).used_rec = false;
  const Plan& plan = cp.plan;
  bool native = true;
  for (const PassDesc& pd : plan.passes) native &= c64_pass_ok(pd);
  if (!native) {
    int rc = c64_promote(h);
    if (rc) return rc;
    rc = run_plan(h, cp, h->psi, nullptr, nullptr, 0, nullptr, nullptr);
    if (rc) return rc;
    return c64_demote(h);
  }
  const char* base = static_cast<const char*>(cp.buf.p);
  for (size_t i = 0; i < plan.passes.size(); ++i) {
    const PassDesc& pd = plan.passes[i];
    const int next_mat = (i + 1 < plan.passes.size()) ? plan.passes[i + 1].mat_begin : (int)plan.mats.size();
    PassLaunch L;
    L.pd = &pd;
    L.d_ops = reinterpret_cast<const DevOp*>(base);
    L.d_stages = reinterpret_cast<const StageDesc*>(base + cp.so);
    L.d_mats = reinterpret_cast<const double*>(base + cp.mo);
    L.d_rops = reinterpret_cast<const RegOp*>(base + cp.ro);
    L.d_partials = nullptr;
    L.nmats = next_mat - pd.mat_begin;
    const int64_t ntiles = int64_t(1) << (h->n_local - pd.k);
    L.grid = (int)std::min<int64_t>(ntiles, (int64_t)device_sm_count() * 3);
    L.n_local = h->n_local;
    L.rank_bits = 0;
    L.c64_terms = h->c64_split;
    L.all_dense = pass_all_dense(plan, pd);
    cudaError_t e = launch_pass_c64(h->psi32, L, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "complex64 pass launch");
    h->stats.kernel_launches += 1;
    h->stats.gate_passes += 1;
    h->stats.algorithmic_bytes += 16.0 * (double)(int64_t(1) << h->n_local);
  }
  mark_plan_used(h, cp);
  return SV_OK;
}

int apply_bound(sv_state_s* h, const std::vector<BoundGate>& bg) {
  if (bg.empty()) return SV_OK;
  const CachedPlan* cp = nullptr;
  int rc = get_plan(h, bg, false, &cp);
  if (rc != SV_OK) return rc;
  if (h->c64) {
    rc = run_plan_c64(h, *cp);
    if (rc != SV_OK) return rc;
    h->stats.gates_applied += (int64_t)bg.size();
    return SV_OK;
  }
  rc = run_plan(h, *cp, h->psi, nullptr, nullptr, 0, nullptr, nullptr);
  if (rc != SV_OK) return rc;
  h->stats.gates_applied += (int64_t)bg.size();
  return SV_OK;
}

// ---- Pauli sums ----



int group_terms(sv_state_s* h, const sv_pauli* terms, int64_t n_terms, PauliGroups* g) {
  if (n_terms < 0 || (n_terms > 0 && !terms)) return fail(SV_E_ARG, "bad term array");
  const uint64_t lim = h->n >= 64 ? ~0ull : ((1ull << h->n) - 1);
  std::map<uint64_t, std::vector<int64_t>> by_x;
  for (int64_t t = 0; t < n_terms; ++t) {
    if ((terms[t].x_mask & ~lim) || (terms[t].z_mask & ~lim)) return fail(SV_E_QUBIT_RANGE, "Pauli term on a qubit >= n");
    by_x[terms[t].x_mask].push_back(t);
  }
  for (auto& kv : by_x) {
    // chunks of <= 256 terms per launch
    for (size_t off = 0; off < kv.second.size(); off += 256) {
      g->xs.push_back(kv.first);
      g->begin.push_back((int)g->z.size());
      for (size_t j = off; j < kv.second.size() && j < off + 256; ++j) {
        const sv_pauli& p = terms[kv.second[j]];
        g->z.push_back(p.z_mask);
        // i^{popc(x & z)}: Y = i X Z on each qubit with both bits set
        const int ph = __builtin_popcountll(p.x_mask & p.z_mask) & 3;
        const double re[4] = {1, 0, -1, 0}, im[4] = {0, 1, 0, -1};
        g->c.push_back(p.coeff * re[ph]);
        g->c.push_back(p.coeff * im[ph]);
      }
      g->end.push_back((int)g->z.size());
    }
  }
  return SV_OK;
}

// Launches one Pauli-group pass per group over psi; lam (optional) receives H psi.
// Writes per-CTA partials of group g to d_partials[g * grid ...].
int pauli_k(int n_local) { return std::min(n_local, 12); }

// True when every x-group fits one Pauli tile with the low qubits (no pair-kernel fallback).
bool pauli_groups_all_tiled(const sv_state_s* h, const PauliGroups& G) {
  const int k = pauli_k(h->n_local);
  const uint64_t lowmask = (1ull << std::min(3, k)) - 1;
  for (uint64_t x : G.xs)
    if (__builtin_popcountll(lowmask | x) > k) return false;
  return true;
}

// Tiled evaluation of all Pauli groups: groups whose x-masks fit together in one 2^k tile (low
// qubits + the x bits) share one pass (k_pauli_tile). Writes one partial slot (grid doubles) per
// pass; *nslots receives the pass count. lam (optional) receives H psi.
// Plans the tiled Pauli passes of a Hamiltonian (k_pauli_tile): groups whose x-masks fit one 2^k tile
// together (with the low qubits) share a pass. E only (lam == nullptr) emits one entry per
// off-diagonal term and one diagonal entry; lambda passes one entry per x-group. Passes are first
// minimised in number (greedy, widest x-masks first), then rebalanced by evaluation cost at that
// pass count. The tile's register positions (9..11) get the three qubits that hit most off-diagonal
// entries' x-masks (their pair-symmetric representatives then vary in registers, not threads).
static void plan_pauli_passes(const PauliGroups& G, int nl, bool e_only, std::vector<PauliPassDesc>* passes,
                              std::vector<uint64_t>* z_all, std::vector<double>* c_all, std::vector<int>* wide) {
  const int k = pauli_k(nl);
  const int L = std::min(3, k);
  const uint64_t lowmask = (1ull << L) - 1;
  std::vector<int> order(G.xs.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    return __builtin_popcountll(G.xs[x]) > __builtin_popcountll(G.xs[y]);
  });
  std::vector<int> fit;  // groups that fit a tile
  for (int gi : order) {
    if (__builtin_popcountll(lowmask | G.xs[gi]) <= k) fit.push_back(gi);
    else wide->push_back(gi);
  }
  auto entries = [&](int gi) { return (e_only && G.xs[gi] != 0) ? G.end[gi] - G.begin[gi] : 1; };
  // evaluation cost per element (units ~ one pair-symmetric off-diagonal term in E-only mode)
  auto cost = [&](int gi) {
    const int nt = G.end[gi] - G.begin[gi];
    if (G.xs[gi] == 0) return 1.0 + 0.28 * nt;  // measured: the 20-term diagonal group ~ 6.5 off-diagonal terms
    return e_only ? (double)nt : 1.0 + 0.25 * (nt - 1);
  };
  auto partition = [&](double cap) {
    std::vector<std::vector<int>> out;
    std::vector<int> remaining = fit;
    while (!remaining.empty()) {
      uint64_t T = lowmask;
      std::vector<int> taken, rest;
      int ne = 0, nterms = 0;
      double c = 0.0;
      for (int gi : remaining) {
        const int nt = G.end[gi] - G.begin[gi];
        const bool first = taken.empty();
        if (ne + entries(gi) <= 32 && __builtin_popcountll(T | G.xs[gi]) <= k && nterms + nt <= 1024 &&
            (first || c + cost(gi) <= cap)) {
          T |= G.xs[gi];
          taken.push_back(gi);
          ne += entries(gi);
          nterms += nt;
          c += cost(gi);
        } else {
          rest.push_back(gi);
        }
      }
      out.push_back(taken);
      remaining.swap(rest);
    }
    return out;
  };
  std::vector<std::vector<int>> parts = partition(1e300);
  if (parts.size() > 1) {
    double total = 0.0, mx = 0.0;
    for (int gi : fit) { total += cost(gi); mx = std::max(mx, cost(gi)); }
    const size_t P0 = parts.size();
    for (double cap = std::max(mx, total / (double)P0); cap < total; cap *= 1.1) {
      std::vector<std::vector<int>> q = partition(cap);
      if (q.size() <= P0) { parts.swap(q); break; }
    }
  }
  for (const std::vector<int>& taken : parts) {
    PauliPassDesc pp;
    std::memset(&pp, 0, sizeof(pp));
    uint64_t T = lowmask;
    for (int gi : taken) T |= G.xs[gi];
    for (int q = 0; q < nl && __builtin_popcountll(T) < k; ++q) T |= 1ull << q;
    pp.k = k;
    // tile position order (k = 12, k_pauli_tile geometry): low qubits 0..2, two more lane qubits,
    // the warp-bit qubits, the register qubits J (positions TB..11). An off-diagonal entry evaluates
    // only one element of each pair (e, e^x) when x has a register or warp bit: J is the set hitting
    // most entries, the lane qubits the pair leaving fewest entries with x inside the lanes.
    constexpr int TB = kPauliTileTidBits;
    constexpr int NJ = 12 - TB;
    std::vector<int> others;
    for (int q = L; q < nl; ++q)
      if ((T >> q) & 1ull) others.push_back(q);
    uint64_t J = 0, lanes = 0;
    if (k == 12 && others.size() == 9) {
      std::vector<uint64_t> xs;
      std::vector<int> wt;
      for (int gi : taken)
        if (G.xs[gi] != 0) { xs.push_back(G.xs[gi] & ~lowmask); wt.push_back(entries(gi)); }
      int best = -1;
      for (uint32_t sub = 0; sub < (1u << 9); ++sub) {
        if (__builtin_popcount(sub) != NJ) continue;
        uint64_t cand = 0;
        for (int i = 0; i < 9; ++i)
          if ((sub >> i) & 1u) cand |= 1ull << others[i];
        int hit = 0;
        for (size_t e = 0; e < xs.size(); ++e)
          if (xs[e] & cand) hit += wt[e];
        if (hit > best) { best = hit; J = cand; }
      }
      int worst = 1 << 30;
      for (size_t i0 = 0; i0 < 9; ++i0)
        for (size_t i1 = i0 + 1; i1 < 9; ++i1) {
          const uint64_t cand = (1ull << others[i0]) | (1ull << others[i1]);
          if (cand & J) continue;
          int slow = 0;
          for (size_t e = 0; e < xs.size(); ++e)
            if ((xs[e] & ~cand) == 0) slow += wt[e];
          if (slow < worst) { worst = slow; lanes = cand; }
        }
    }
    int p = 0;
    for (int q = 0; q < L; ++q) pp.tq[p++] = (int8_t)q;
    for (int q : others)
      if ((lanes >> q) & 1ull) pp.tq[p++] = (int8_t)q;
    for (int q : others)
      if (!((J >> q) & 1ull) && !((lanes >> q) & 1ull)) pp.tq[p++] = (int8_t)q;
    for (int q : others)
      if ((J >> q) & 1ull) pp.tq[p++] = (int8_t)q;
    int pos_of[64];
    for (int i = 0; i < k; ++i) pos_of[(int)pp.tq[i]] = i;
    int low = 0;
    while (low < k && pp.tq[low] == low) ++low;
    pp.low = low;
    pp.diag_g = -1;
    pp.term_base = (int)z_all->size();
    auto tile_mask = [&](uint64_t m) {
      uint32_t t = 0;
      for (int q = 0; q < nl; ++q)
        if (((m >> q) & 1ull) && ((T >> q) & 1ull)) t |= 1u << pos_of[q];
      return t;
    };
    auto rule_of = [&](uint32_t xt) {
      int rule = PR_ALL, wb = 5;
      if (k == 12) {
        for (int bb = NJ - 1; bb >= 0; --bb)
          if ((xt >> (TB + bb)) & 1u) rule = bb;
        if (rule == PR_ALL)
          for (int bb = 5; bb < TB; ++bb)
            if ((xt >> bb) & 1u) { rule = PR_WARP; wb = bb; break; }
      }
      return std::make_pair(rule, wb);
    };
    auto emit = [&](uint64_t x, const std::vector<int>& ts, int type) {
      const int g = pp.ngroups++;
      pp.xphys[g] = x;
      const uint32_t xt = tile_mask(x);
      pp.xtile[g] = xt;
      const auto rw = rule_of(xt);
      pp.gkind[g] = (uint8_t)(rw.first | (type << 3) | ((rw.second - 5) << 5));
      pp.zt_reg[g] = ts.empty() ? 0u : tile_mask(G.z[ts[0]]) >> TB;
      pp.tbeg[g] = (int)z_all->size() - pp.term_base;
      for (int t : ts) {
        z_all->push_back(G.z[t]);
        c_all->push_back(G.c[2 * t]);
        c_all->push_back(G.c[2 * t + 1]);
      }
      pp.tend[g] = (int)z_all->size() - pp.term_base;
    };
    auto single_type = [&](int t) { return G.c[2 * t + 1] != 0.0 ? PG_SINGLE_IM : PG_SINGLE_RE; };
    auto sorted_terms = [&](int gi) {
      // terms ordered by the tile-position Z bits above the kernel's thread bits (k_pauli_tile sums
      // runs of equal element-part masks once)
      std::vector<int> ts;
      for (int t = G.begin[gi]; t < G.end[gi]; ++t) ts.push_back(t);
      std::stable_sort(ts.begin(), ts.end(), [&](int x, int y) { return (tile_mask(G.z[x]) >> TB) < (tile_mask(G.z[y]) >> TB); });
      return ts;
    };
    if (e_only) {
      // off-diagonal terms first, one entry each, sorted by class (representative rule, c' type):
      // entry g is term g of the pass; the diagonal entry last
      std::vector<std::pair<int, int>> ents;  // (class, term)
      int diag_gi = -1;
      for (int gi : taken) {
        if (G.xs[gi] == 0) { diag_gi = gi; continue; }
        const int r = rule_of(tile_mask(G.xs[gi])).first;
        const int ci = (r < NJ ? r : (r == PR_WARP ? 3 : 4)) * 2;
        for (int t : sorted_terms(gi)) ents.push_back({ci + (single_type(t) == PG_SINGLE_IM ? 1 : 0), t});
      }
      std::stable_sort(ents.begin(), ents.end(), [](const std::pair<int, int>& u, const std::pair<int, int>& v) { return u.first < v.first; });
      for (int c = 0; c <= 10; ++c) {
        int cnt = 0;
        for (const auto& e : ents) cnt += e.first < c ? 1 : 0;
        pp.cls_beg[c] = cnt;
      }
      for (const auto& e : ents) {
        int gi = 0;
        while (!(e.second >= G.begin[gi] && e.second < G.end[gi])) ++gi;
        emit(G.xs[gi], {e.second}, single_type(e.second));
        if (e.first < 8) {  // pair-symmetric rule: each representative stands for its pair (factor 2)
          (*c_all)[c_all->size() - 2] *= 2.0;
          (*c_all)[c_all->size() - 1] *= 2.0;
        }
      }
      if (diag_gi >= 0) {
        const std::vector<int> ts = sorted_terms(diag_gi);
        emit(0, ts, PG_DIAG);
        pp.diag_g = pp.ngroups - 1;
        // the kernel walks the diagonal terms by their register-part z mask h (sorted)
        const int rel0 = pp.tbeg[pp.ngroups - 1];
        for (int hh = 0; hh <= 16; ++hh) {
          int r = rel0;
          for (int t : ts)
            if ((int)(tile_mask(G.z[t]) >> TB) < hh) ++r;
          pp.diag_rb[hh] = r;
        }
      }
    } else {
      for (int gi : taken) {
        const std::vector<int> ts = sorted_terms(gi);
        const uint64_t x = G.xs[gi];
        if (x == 0) emit(x, ts, PG_DIAG);
        else if (ts.size() == 1) emit(x, ts, single_type(ts[0]));
        else emit(x, ts, PG_MULTI);
      }
    }
    pp.nterms = (int)z_all->size() - pp.term_base;
    passes->push_back(pp);
  }
}

int run_groups(sv_state_s* h, const PauliGroups& G, const double* psi, double* lam, double* d_partials, int grid,
               int* nslots, const float* psi32, bool lam_accumulate) {
  const int nl = h->n_local;
  std::vector<PauliPassDesc> passes;
  std::vector<uint64_t> z_all;
  std::vector<double> c_all;
  std::vector<int> wide;  // wide: x-mask does not fit a tile -> per-group pair kernel
  plan_pauli_passes(G, nl, lam == nullptr, &passes, &z_all, &c_all, &wide);
  // wide groups' terms follow the passes' terms
  std::vector<int> wide_base;
  for (int gi : wide) {
    wide_base.push_back((int)z_all.size());
    for (int t = G.begin[gi]; t < G.end[gi]; ++t) {
      z_all.push_back(G.z[t]);
      c_all.push_back(G.c[2 * t]);
      c_all.push_back(G.c[2 * t + 1]);
    }
  }
  const size_t zb = (z_all.size() * 8 + 15) & ~size_t(15), cb = c_all.size() * 8;
  if (!h->d_terms.ensure(zb + cb + 16)) return fail(SV_E_OOM, "term buffers");
  // page-locked staging: the upload does not hold the host until the stream drains (the gradient
  // plans its reverse sweep meanwhile); the previous upload from this buffer must be complete
  cudaError_t e = cudaSuccess;
  if (h->terms_upload_done) {
    e = cudaEventSynchronize(h->terms_upload_done);
  } else {
    e = cudaEventCreateWithFlags(&h->terms_upload_done, cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(h, e, "term upload");
  if (!h->pin_terms.ensure(zb + cb + 16)) return fail(SV_E_OOM, "term staging");
  char* hs = static_cast<char*>(h->pin_terms.p);
  std::memcpy(hs, z_all.data(), z_all.size() * 8);
  std::memcpy(hs + zb, c_all.data(), cb);
  e = cudaMemcpyAsync(h->d_terms.p, hs, zb + cb, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaEventRecord(h->terms_upload_done, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "term upload");
  const uint64_t* dz = static_cast<const uint64_t*>(h->d_terms.p);
  const double* dc = reinterpret_cast<const double*>(static_cast<const char*>(h->d_terms.p) + zb);
  const double amps = (double)(1ull << nl);
  int slot = 0;
  for (size_t p = 0; p < passes.size(); ++p, ++slot) {
    // lambda passes: the first writes (and gives its E), later ones accumulate; the last tiled
    // pass reports E = Re<psi|lambda> over all tiled groups (earlier accumulating passes report 0)
    const int mode = lam == nullptr ? 0 : lam_accumulate ? 2 : (slot == 0 ? 1 : (p + 1 == passes.size() ? 3 : 2));
    if (mode == 3) {  // its partial supersedes the first pass' one
      e = cudaMemsetAsync(d_partials, 0, (size_t)grid * 8, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "partials");
    }
    e = psi32 ? launch_pauli_tile_c64(psi32, nl, passes[p], dz, dc, d_partials + (size_t)slot * grid, grid, h->stream)
              : launch_pauli_tile(psi, lam, mode, nl, passes[p], dz, dc, d_partials + (size_t)slot * grid, grid, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "pauli pass launch");
    h->stats.kernel_launches += 1;
    h->stats.expectation_passes += 1;
    h->stats.algorithmic_bytes += (mode == 0 ? 16.0 : (mode == 1 ? 32.0 : 48.0)) * amps;
  }
  if (psi32 && !wide.empty()) return fail(SV_E_ARG, "internal: wide Pauli groups on a complex64 state");
  for (size_t w = 0; w < wide.size(); ++w, ++slot) {
    const int gi = wide[w];
    const int nt = G.end[gi] - G.begin[gi];
    // the pair kernel writes lambda when it is the first launch, else accumulates
    e = launch_pauli_group(psi, lam, lam_accumulate || slot > 0, nl, G.xs[gi], dz + wide_base[w], dc + 2 * wide_base[w], nt,
                           d_partials + (size_t)slot * grid, std::min(grid, pauli_grid(nl)), h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "pauli group launch");
    if (pauli_grid(nl) < grid) {  // zero the unused tail of this slot (fixed-width reduction)
      e = cudaMemsetAsync(d_partials + (size_t)slot * grid + pauli_grid(nl), 0, (size_t)(grid - pauli_grid(nl)) * 8,
                          h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "partials");
    }
    h->stats.kernel_launches += 1;
    h->stats.expectation_passes += 1;
    h->stats.algorithmic_bytes += (lam == nullptr ? 16.0 : (slot == 0 ? 32.0 : 48.0)) * amps;
  }
  *nslots = slot;
  return SV_OK;
}

// Density matrix: rho <- U rho U^dagger is U on the row qubits and U* on the column qubits of the
// 2n-qubit vector vec[r + 2^n c] (§3.2 eq. at).
std::vector<BoundGate> density_expand(const std::vector<BoundGate>& bg, int n) {
  std::vector<BoundGate> out;
  out.reserve(2 * bg.size());
  for (const BoundGate& g : bg) {
    out.push_back(g);
    BoundGate c = g;
    c.t0 = g.t0 + n;
    c.t1 = g.t1 >= 0 ? g.t1 + n : -1;
    c.controls = g.controls << n;
    for (int e = 0; e < 16; ++e) c.m[e].im = -c.m[e].im;
    c.param = -1;
    out.push_back(c);
  }
  return out;
}

}  // namespace sv

using namespace sv;

extern "C" {

const char* sv_last_error(void) { return g_last_error.c_str(); }
const char* sv_version(void) { return "paper_2406_17248_b200 sv 0.1 (sm_100a)"; }

sv_status sv_create(int32_t n_qubits, sv_handle* out) {
  if (!out) return fail(SV_E_ARG, "null out");
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > 40) return fail(SV_E_ARG, "n_qubits must be in [1, 40]");
  sv_state_s* h = new sv_state_s();
  h->n = n_qubits;
  h->n_local = n_qubits;
  cudaGetDevice(&h->device);
  cudaError_t e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete h; return fail(SV_E_CUDA, std::string("stream: ") + cudaGetErrorString(e)); }
  h->stream = h->own_stream;
  const size_t bytes = (size_t(16) << n_qubits);
  if (!h->state.ensure(bytes)) {
    cudaStreamDestroy(h->own_stream);
    delete h;
    return fail(SV_E_OOM, "cannot allocate the state vector (" + std::to_string(bytes) + " bytes)");
  }
  h->psi = static_cast<double*>(h->state.p);
  e = launch_init_zero(h->psi, int64_t(1) << n_qubits, true, h->stream);
  if (e != cudaSuccess) { sv_destroy(h); return fail(SV_E_CUDA, cudaGetErrorString(e)); }
  h->stats.kernel_launches += 1;
  *out = h;
  return SV_OK;
}

sv_status sv_create_density(int32_t n_qubits, sv_handle* out) {
  if (n_qubits < 1 || n_qubits > 17) {
    if (out) *out = nullptr;
    return fail(SV_E_ARG, "density matrices: n_qubits must be in [1, 17]");
  }
  int rc = sv_create(2 * n_qubits, out);
  if (rc) return rc;
  (*out)->n = n_qubits;
  (*out)->density = true;
  return SV_OK;
}

static cudaError_t init_c64(sv_state_s* h) {
  cudaError_t e = cudaMemsetAsync(h->psi32, 0, size_t(8) << h->n_local, h->stream);
  static const float one[2] = {1.0f, 0.0f};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->psi32, one, sizeof(one), cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // `one` is pageable
  return e;
}

sv_status sv_create_c64(int32_t n_qubits, sv_handle* out) {
  if (!out) return fail(SV_E_ARG, "null out");
  *out = nullptr;
  if (n_qubits < 1 || n_qubits > 40) return fail(SV_E_ARG, "n_qubits must be in [1, 40]");
  sv_state_s* h = new sv_state_s();
  h->n = n_qubits;
  h->n_local = n_qubits;
  h->c64 = true;
  cudaGetDevice(&h->device);
  cudaError_t e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) { delete h; return fail(SV_E_CUDA, std::string("stream: ") + cudaGetErrorString(e)); }
  h->stream = h->own_stream;
  const size_t bytes = (size_t(8) << n_qubits);
  if (!h->state.ensure(bytes)) {
    cudaStreamDestroy(h->own_stream);
    delete h;
    return fail(SV_E_OOM, "cannot allocate the complex64 state vector (" + std::to_string(bytes) + " bytes)");
  }
  h->psi32 = static_cast<float*>(h->state.p);
  e = init_c64(h);
  if (e != cudaSuccess) { sv_destroy(h); return fail(SV_E_CUDA, cudaGetErrorString(e)); }
  *out = h;
  return SV_OK;
}

sv_status sv_destroy(sv_handle h) {
  if (!h) return SV_OK;
  DeviceGuard dev_guard(h->device);
  cudaStreamSynchronize(h->stream);
  h->state.release();
  h->promo.release();
  h->pin_in.release();
  h->pin_out.release();
  h->pin_plan.release();
  h->pin_terms.release();
  h->pin_e.release();
  if (h->plan_upload_done) cudaEventDestroy(h->plan_upload_done);
  if (h->upload_stream) {
    cudaStreamSynchronize(h->upload_stream);
    cudaStreamDestroy(h->upload_stream);
  }
  if (h->terms_upload_done) cudaEventDestroy(h->terms_upload_done);
  h->work_psi.release();
  h->work_lam.release();
  h->work_r.release();
  release_plan_cache(h);
  for (auto& pr : h->xev) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  h->xev.clear();
  h->d_ops.release();
  h->d_mats.release();
  h->d_terms.release();
  h->d_partials.release();
  h->d_out.release();
  destroy_sharding(h);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
  return SV_OK;
}

sv_status sv_set_stream(sv_handle h, void* stream) {
  if (!h) return fail(SV_E_ARG, "null handle");
  // work already queued on the previous stream must finish before buffers it uses can be replaced
  // stream-ordered on the new one
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
  return SV_OK;
}

sv_status sv_set_option(sv_handle h, int32_t key, int64_t value) {
  if (!h) return fail(SV_E_ARG, "null handle");
  switch (key) {
    case SV_OPT_TILE_QUBITS:
      if (value < 0 || value > kMaxTileQubits) return fail(SV_E_ARG, "tile qubits out of range");
      h->opts.tile_qubits = (int)value;
      return SV_OK;
    case SV_OPT_FUSION: h->opts.fusion = value != 0; return SV_OK;
    case SV_OPT_LOW_QUBITS:
      if (value < 0 || value > 8) return fail(SV_E_ARG, "low qubits out of range");
      h->opts.low_qubits = (int)value;
      return SV_OK;
    case SV_OPT_DENSE: h->opts.dense = value != 0 ? 1 : 0; return SV_OK;
    case SV_OPT_KERNEL: h->opts.kernel = value != 0 ? 1 : 0; return SV_OK;
    case SV_OPT_ADJOINT_DENSE_COST:
      if (value < -1 || value > (1 << 20)) return fail(SV_E_ARG, "adjoint dense cost threshold out of range");
      h->opts.da_cost = (int)value;
      return SV_OK;
    case SV_OPT_C64_SPLIT:
      if (value != 0 && value != 1 && value != 3) return fail(SV_E_ARG, "complex64 split must be 0, 1 or 3");
      h->c64_split = (int)value;
      return SV_OK;
    default: return fail(SV_E_ARG, "unknown option");
  }
}

sv_status sv_get_num_qubits(sv_handle h, int32_t* out) {
  if (!h || !out) return fail(SV_E_ARG, "null argument");
  *out = h->n;
  return SV_OK;
}

sv_status sv_reset(sv_handle h) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (h->world > 1) return shard_reset(h);
  if (h->c64) {
    cudaError_t e = init_c64(h);
    if (e != cudaSuccess) return cuda_fail(h, e, "reset");
    return SV_OK;
  }
  cudaError_t e = launch_init_zero(h->psi, int64_t(1) << h->n_local, true, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "reset");
  h->stats.kernel_launches += 1;
  return SV_OK;
}

sv_status sv_set_state(sv_handle h, const double* host) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (!host) return fail(SV_E_ARG, "null host buffer");
  if (h->world > 1) return shard_set_state(h, host);
  if (h->c64) {  // complex128 host values rounded to complex64
    std::vector<float> v(size_t(2) << h->n);
    for (size_t i = 0; i < v.size(); ++i) v[i] = (float)host[i];
    cudaError_t e = cudaMemcpyAsync(h->psi32, v.data(), v.size() * 4, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "set_state");
    return SV_OK;
  }
  if (h->density) {  // row-major rho[r][c] -> vec[r + 2^n c]
    const uint64_t D = 1ull << h->n;
    std::vector<double> v(2 * D * D);
    for (uint64_t r = 0; r < D; ++r)
      for (uint64_t c = 0; c < D; ++c) {
        v[2 * (r + D * c)] = host[2 * (r * D + c)];
        v[2 * (r + D * c) + 1] = host[2 * (r * D + c) + 1];
      }
    cudaError_t e = cudaMemcpyAsync(h->psi, v.data(), v.size() * 8, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "set_state");
    return SV_OK;
  }
  cudaError_t e = cudaMemcpyAsync(h->psi, host, size_t(16) << h->n, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "set_state");
  return SV_OK;
}

sv_status sv_get_state(sv_handle h, double* host) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (!host) return fail(SV_E_ARG, "null host buffer");
  if (h->world > 1) return shard_get_state(h, host);
  if (h->c64) {
    std::vector<float> v(size_t(2) << h->n);
    cudaError_t e = cudaMemcpyAsync(v.data(), h->psi32, v.size() * 4, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "get_state");
    for (size_t i = 0; i < v.size(); ++i) host[i] = (double)v[i];
    return SV_OK;
  }
  if (h->density) {
    const uint64_t D = 1ull << h->n;
    std::vector<double> v(2 * D * D);
    cudaError_t e = cudaMemcpyAsync(v.data(), h->psi, v.size() * 8, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "get_state");
    for (uint64_t r = 0; r < D; ++r)
      for (uint64_t c = 0; c < D; ++c) {
        host[2 * (r * D + c)] = v[2 * (r + D * c)];
        host[2 * (r * D + c) + 1] = v[2 * (r + D * c) + 1];
      }
    return SV_OK;
  }
  cudaError_t e = cudaMemcpyAsync(host, h->psi, size_t(16) << h->n, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "get_state");
  return SV_OK;
}

}  // extern "C"

int sv::gather_amplitudes(sv_state_s* h, const void* psi, bool c64, const std::vector<uint64_t>& idx, double* out,
                          bool accumulate) {
  const size_t cnt = idx.size();
  if (!cnt) return SV_OK;
  const size_t ib = (cnt * 8 + 63) & ~size_t(63);
  if (!h->d_terms.ensure(ib + cnt * 16 + 64)) return fail(SV_E_OOM, "amplitude readout buffers");
  char* db = static_cast<char*>(h->d_terms.p);
  std::vector<double> tmp(2 * cnt);
  cudaError_t e = cudaMemcpyAsync(db, idx.data(), cnt * 8, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess)
    e = launch_gather(psi, c64, reinterpret_cast<const uint64_t*>(db), (int64_t)cnt, reinterpret_cast<double*>(db + ib),
                      h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(tmp.data(), db + ib, cnt * 16, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "amplitude readout");
  h->stats.kernel_launches += 1;
  for (size_t j = 0; j < 2 * cnt; ++j) out[j] = accumulate ? out[j] + tmp[j] : tmp[j];
  return SV_OK;
}

extern "C" {

sv_status sv_get_amplitudes(sv_handle h, const uint64_t* idx, int64_t count, double* out) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (count < 0 || (count > 0 && (!idx || !out))) return fail(SV_E_ARG, "bad amplitude readout arguments");
  if (h->density) return fail(SV_E_ARG, "amplitude readout is for state vectors (use sv_get_state)");
  const uint64_t lim = h->n >= 64 ? ~0ull : (1ull << h->n);
  for (int64_t j = 0; j < count; ++j)
    if (idx[j] >= lim) return fail(SV_E_QUBIT_RANGE, "amplitude index >= 2^n");
  if (count == 0) return SV_OK;
  if (h->world > 1) return shard_get_amplitudes(h, idx, count, out);
  std::vector<uint64_t> v(idx, idx + count);
  return gather_amplitudes(h, h->c64 ? static_cast<const void*>(h->psi32) : static_cast<const void*>(h->psi), h->c64, v,
                           out, false);
}

sv_status sv_set_state_device(sv_handle h, const void* dev) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (!dev) return fail(SV_E_ARG, "null device buffer");
  if (h->world > 1) return fail(SV_E_ARG, "device-pointer state transfer is single-GPU only");
  cudaError_t e = h->c64 ? cudaMemcpyAsync(h->psi32, dev, size_t(8) << h->n_local, cudaMemcpyDeviceToDevice, h->stream)
                         : cudaMemcpyAsync(h->psi, dev, size_t(16) << h->n_local, cudaMemcpyDeviceToDevice, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "set_state_device");
  return SV_OK;
}

sv_status sv_get_state_device(sv_handle h, void* dev) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (!dev) return fail(SV_E_ARG, "null device buffer");
  if (h->world > 1) return fail(SV_E_ARG, "device-pointer state transfer is single-GPU only");
  cudaError_t e = h->c64 ? cudaMemcpyAsync(dev, h->psi32, size_t(8) << h->n_local, cudaMemcpyDeviceToDevice, h->stream)
                         : cudaMemcpyAsync(dev, h->psi, size_t(16) << h->n_local, cudaMemcpyDeviceToDevice, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "get_state_device");
  return SV_OK;
}

sv_status sv_apply_gate(sv_handle h, const sv_gate* g, const double* params, int32_t n_params) {
  return sv_apply_circuit(h, g, 1, params, n_params);
}

sv_status sv_apply_circuit(sv_handle h, const sv_gate* gates, int64_t n_gates, const double* params, int32_t n_params) {
  NvtxRange nvtx("sv_apply_circuit");
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  std::vector<BoundGate> bg;
  rc = bind_circuit(h, gates, n_gates, params, n_params, false, &bg);
  if (rc) return rc;
  if (h->world > 1) return shard_apply(h, bg);
  if (h->density) return apply_bound(h, density_expand(bg, h->n));
  return apply_bound(h, bg);
}

sv_status sv_expectation(sv_handle h, const sv_pauli* terms, int64_t n_terms, double* out_value) {
  NvtxRange nvtx("sv_expectation");
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (!out_value) return fail(SV_E_ARG, "null out_value");
  PauliGroups G;
  rc = group_terms(h, terms, n_terms, &G);
  if (rc) return rc;
  if (h->world > 1) return shard_expectation(h, G, out_value);
  *out_value = 0.0;
  if (G.xs.empty()) return SV_OK;
  if (h->density) {
    // tr(rho H): one diagonal-gather pass over 2^n elements per x-group
    const int n = h->n;
    int64_t gsz = ((int64_t(1) << n) + 255) / 256;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(gsz, 592));
    const size_t ng = G.xs.size();
    const size_t zb = (G.z.size() * 8 + 15) & ~size_t(15), cb = G.c.size() * 8;
    if (!h->d_terms.ensure(zb + cb + 16) || !h->d_partials.ensure(ng * grid * 8 + 8) || !h->d_out.ensure(ng * 8 + 8))
      return fail(SV_E_OOM, "density expectation buffers");
    h->h_stage.assign(zb + cb + 16, 0);
    std::memcpy(h->h_stage.data(), G.z.data(), G.z.size() * 8);
    std::memcpy(h->h_stage.data() + zb, G.c.data(), cb);
    cudaError_t e = cudaMemcpyAsync(h->d_terms.p, h->h_stage.data(), zb + cb, cudaMemcpyHostToDevice, h->stream);
    const uint64_t* dz = static_cast<const uint64_t*>(h->d_terms.p);
    const double* dc = reinterpret_cast<const double*>(static_cast<const char*>(h->d_terms.p) + zb);
    double* dp = static_cast<double*>(h->d_partials.p);
    for (size_t gi = 0; gi < ng && e == cudaSuccess; ++gi)
      e = launch_dm_trace(h->psi, n, G.xs[gi], dz + G.begin[gi], dc + 2 * G.begin[gi], G.end[gi] - G.begin[gi],
                          dp + gi * (size_t)grid, grid, h->stream);
    if (e == cudaSuccess) e = launch_reduce_slots(dp, (int)ng, grid, static_cast<double*>(h->d_out.p), h->stream);
    std::vector<double> gv(ng);
    if (e == cudaSuccess) e = cudaMemcpyAsync(gv.data(), h->d_out.p, ng * 8, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "density expectation");
    h->stats.kernel_launches += (int64_t)ng + 1;
    double E = 0.0;
    for (double v : gv) E += v;
    *out_value = E;
    return SV_OK;
  }
  const int grid = pauli_tile_grid(h->n_local, pauli_k(h->n_local));
  const size_t ng = G.xs.size();
  if (!h->d_partials.ensure(ng * grid * 8) || !h->d_out.ensure(ng * 8)) return fail(SV_E_OOM, "partials");
  double* dp = static_cast<double*>(h->d_partials.p);
  int nslots = 0;
  const bool c64_native = h->c64 && pauli_groups_all_tiled(h, G);
  if (h->c64 && !c64_native) {
    rc = c64_promote(h);
    if (rc) return rc;
  }
  rc = c64_native ? run_groups(h, G, nullptr, nullptr, dp, grid, &nslots, h->psi32)
                  : run_groups(h, G, h->psi, nullptr, dp, grid, &nslots);
  if (rc) return rc;
  const size_t ns_e = (size_t)nslots;
  cudaError_t e = launch_reduce_slots(dp, (int)ns_e, grid, static_cast<double*>(h->d_out.p), h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "reduce");
  h->stats.kernel_launches += 1;
  std::vector<double> gv(ns_e);
  e = cudaMemcpyAsync(gv.data(), h->d_out.p, ns_e * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "expectation");
  double E = 0.0;
  for (double v : gv) E += v;
  *out_value = E;
  return SV_OK;
}

sv_status sv_expectation_with_grad(sv_handle h, const sv_gate* gates, int64_t n_gates, const double* params,
                                   int32_t n_params, const sv_pauli* terms, int64_t n_terms, double* out_value,
                                   double* out_grad) {
  NvtxRange nvtx("sv_expectation_with_grad");
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (!out_value || (n_params > 0 && !out_grad)) return fail(SV_E_ARG, "null output");
  if (h->density) return fail(SV_E_ARG, "gradients are not available on density-matrix handles");
  if (h->c64) {  // complex64 state: this operation reads a complex128 copy (the state is unchanged)
    const int prc = c64_promote(h);
    if (prc) return prc;
  }
  std::vector<BoundGate> bg;
  rc = bind_circuit(h, gates, n_gates, params, n_params, true, &bg);
  if (rc) return rc;
  PauliGroups G;
  rc = group_terms(h, terms, n_terms, &G);
  if (rc) return rc;
  if (h->world > 1) return shard_expectation_with_grad(h, bg, n_params, G, out_value, out_grad);
  const size_t bytes = size_t(16) << h->n_local;
  if (!h->work_psi.ensure(bytes) || !h->work_lam.ensure(bytes)) return fail(SV_E_OOM, "gradient workspaces");
  double* psi = static_cast<double*>(h->work_psi.p);
  double* lam = static_cast<double*>(h->work_lam.p);
  cudaError_t e = cudaMemcpyAsync(psi, h->psi, bytes, cudaMemcpyDeviceToDevice, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "copy psi0");
  h->stats.algorithmic_bytes += 2.0 * (double)bytes;
  // 1. forward
  static const bool tmg = std::getenv("SV_PLAN_TIMING") != nullptr;
  const auto tg0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (tmg) std::fprintf(stderr, "grad %s at %.3f ms\n", what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg0).count());
  };
  const CachedPlan* fwdp = nullptr;
  rc = get_plan(h, bg, false, &fwdp);
  if (rc) return rc;
  lap("fwd plan");
  {
    NvtxRange r("forward");
    rc = run_plan(h, *fwdp, psi, nullptr, nullptr, 0, nullptr, nullptr);
  }
  if (rc) return rc;
  lap("fwd launched");
  h->stats.gates_applied += (int64_t)bg.size();
  // 2. lambda = H psi, E
  double E = 0.0;
  if (G.xs.empty()) {
    e = cudaMemsetAsync(lam, 0, bytes, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "zero lambda");
  } else {
    const int pgrid = pauli_tile_grid(h->n_local, pauli_k(h->n_local));
    const size_t ng = G.xs.size();
    if (!h->d_partials.ensure(ng * pgrid * 8 + 8) || !h->d_out.ensure(ng * 8 + 8)) return fail(SV_E_OOM, "partials");
    int nslots = 0;
    {
      NvtxRange r("lambda = H psi");
      rc = run_groups(h, G, psi, lam, static_cast<double*>(h->d_partials.p), pgrid, &nslots);
    }
    if (rc) return rc;
    e = launch_reduce_slots(static_cast<double*>(h->d_partials.p), nslots, pgrid, static_cast<double*>(h->d_out.p),
                            h->stream);
    // page-locked destination: the copy stays asynchronous (a pageable one would hold the host
    // until the forward passes finish, serialising the reverse plan behind them)
    if (!h->pin_e.ensure((size_t)nslots * 8 + 8)) return fail(SV_E_OOM, "energy staging");
    const double* ev = static_cast<const double*>(h->pin_e.p);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h->pin_e.p, h->d_out.p, (size_t)nslots * 8, cudaMemcpyDeviceToHost, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "energy");
    h->stats.kernel_launches += 1;
    // (the copy completes at the synchronisation inside run_reverse)
    std::vector<double> d;
    const CachedPlan* revp = nullptr;
    lap("lambda launched");
    rc = get_plan(h, bg, true, &revp);
    if (rc) return rc;
    lap("rev plan");
    {
      NvtxRange r("adjoint sweep");
      rc = run_reverse(h, *revp, psi, lam, &d);
    }
    if (rc) return rc;
    lap("reverse done");
    e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "energy");
    for (int i = 0; i < nslots; ++i) E += ev[i];
    *out_value = E;
    for (int32_t p = 0; p < n_params; ++p) out_grad[p] = 0.0;
    for (size_t sl = 0; sl < d.size(); ++sl) out_grad[revp->plan.slot_param[sl]] += revp->plan.slot_coeff[sl] * 2.0 * d[sl];
    return SV_OK;
  }
  // empty H: E = 0, gradient 0 (the sweep would only produce zeros)
  e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "sync");
  *out_value = 0.0;
  for (int32_t p = 0; p < n_params; ++p) out_grad[p] = 0.0;
  return SV_OK;
}

}  // extern "C"

// Runs a reverse (adjoint) plan on (psi, lambda) and returns the per-slot overlaps
// d_s = Re<lambda|D_s|psi> in slot order: sequential stages through per-CTA partials, adjoint dense
// stages through their correlation matrices R (host contraction with B_{j,var}). Synchronous.
int sv::run_reverse(sv_state_s* h, const CachedPlan& cp, double* psi, double* lam, std::vector<double>* d_out) {
  const Plan& rev = cp.plan;
  const size_t ns = (size_t)rev.n_grad_slots;
  d_out->assign(ns, 0.0);
  if (rev.passes.empty()) return SV_OK;
  const int agrid = plan_grid(rev, h->n_local);
  const size_t nda = rev.da.size();
  const size_t nslots_r = (size_t)rev.da_slots_total;
  const int nw = (1 << (rev.passes[0].k - rev.passes[0].R)) / 32;
  const size_t part_slots = ns * (size_t)agrid;
  const size_t r_part = nda ? (size_t)rev.max_da_per_pass * nw * 512 * agrid : 0, r_sum = nslots_r * (size_t)nw * 512;
  if (!h->work_r.ensure((part_slots + ns + r_part + r_sum) * 8 + 64)) return fail(SV_E_OOM, "adjoint buffers");
  double* dp = static_cast<double*>(h->work_r.p);
  double* dout = dp + part_slots;
  double* rp = dout + ns;
  double* rsum = rp + r_part;
  // passes may run fewer CTAs than the plan grid: unwritten partial columns must read as zero
  if (ns) {
    cudaError_t ze = cudaMemsetAsync(dp, 0, part_slots * 8, h->stream);
    if (ze != cudaSuccess) return cuda_fail(h, ze, "partials clear");
  }
  int rc = run_plan(h, cp, psi, lam, dp, agrid, nda ? rp : nullptr, nda ? rsum : nullptr);
  if (rc) return rc;
  cudaError_t e = cudaSuccess;
  if (ns) e = launch_reduce_slots(dp, (int)ns, agrid, dout, h->stream);
  std::vector<double> rs(r_sum);
  if (e == cudaSuccess && ns) e = cudaMemcpyAsync(d_out->data(), dout, ns * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess && nda) e = cudaMemcpyAsync(rs.data(), rsum, r_sum * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "gradient readback");
  h->stats.kernel_launches += ns ? 1 : 0;
  for (size_t di = 0; di < nda; ++di) {
    const Plan::DAStage& ds = rev.da[di];
    const int ntv = 1 << ds.m_tile, nvar = 1 << (ds.m_tile + ds.m_outer);
    std::vector<Cx> R((size_t)nvar * 256, Cx{0, 0});
    for (int ov = 0; ov < (1 << ds.m_outer); ++ov)
    for (int w = 0; w < nw; ++w) {
      const int var = (w & (ntv - 1)) | (ov << ds.m_tile);
      const double* f = rs.data() + ((size_t)(ds.global_slot + ov) * nw + (size_t)w) * 512;
      for (int mt = 0; mt < 2; ++mt)
        for (int nt = 0; nt < 2; ++nt)
          for (int v = 0; v < 2; ++v)
            for (int l = 0; l < 32; ++l) {
              const int a = 8 * mt + (l >> 2), b = 8 * nt + 2 * (l & 3) + v;
              Cx& r = R[(size_t)var * 256 + (size_t)a * 16 + b];
              r.re += f[((((mt * 2 + nt) * 2 + 0) * 2 + v) << 5) + l];
              r.im += f[((((mt * 2 + nt) * 2 + 1) * 2 + v) << 5) + l];
            }
    }
    for (size_t j = 0; j < ds.slots.size(); ++j) {
      double d = 0.0;  // Re tr(B R) = sum_{a,b} Re(B[a][b] R[b][a])
      for (int var = 0; var < nvar; ++var) {
        const Cx* Bm = ds.B[j].data() + (size_t)var * 256;
        const Cx* Rm = R.data() + (size_t)var * 256;
        for (int a = 0; a < 16; ++a)
          for (int b = 0; b < 16; ++b) d += Bm[a * 16 + b].re * Rm[b * 16 + a].re - Bm[a * 16 + b].im * Rm[b * 16 + a].im;
      }
      (*d_out)[(size_t)ds.slots[j]] = d;
    }
  }
  return SV_OK;
}

extern "C" {

sv_status sv_get_stats(sv_handle h, sv_stats* out) {
  if (!h || !out) return fail(SV_E_ARG, "null argument");
  DeviceGuard dev_guard(h->device);
  for (auto& pr : h->xev) {  // exchange device time: events recorded around each exchange
    float ms = 0.0f;
    if (cudaEventSynchronize(pr.second) == cudaSuccess && cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess)
      h->stats.exchange_ms += (double)ms;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  h->xev.clear();
  *out = h->stats;
  return SV_OK;
}

sv_status sv_reset_stats(sv_handle h) {
  if (!h) return fail(SV_E_ARG, "null argument");
  DeviceGuard dev_guard(h->device);
  for (auto& pr : h->xev) {
    cudaEventSynchronize(pr.second);
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  h->xev.clear();
  std::memset(&h->stats, 0, sizeof(h->stats));
  return SV_OK;
}

}  // extern "C"

#include "sv_debug.h"

extern "C" sv_status sv_plan_info(int32_t n_qubits, const sv_gate* gates, int64_t n_gates, const double* params,
                                  int32_t n_params, int32_t adjoint, int32_t tile_qubits, int32_t fusion,
                                  sv_pass_info* out, int64_t cap, int64_t* n_passes) {
  if (n_qubits < 1 || n_qubits > 40 || !n_passes) return fail(SV_E_ARG, "bad arguments");
  sv_state_s tmp;
  tmp.n = tmp.n_local = n_qubits;
  std::vector<BoundGate> bg;
  int rc = bind_circuit(&tmp, gates, n_gates, params, n_params, adjoint != 0, &bg);
  if (rc) return rc;
  PlanOptions o;
  o.tile_qubits = tile_qubits;
  o.fusion = fusion != 0;
  Plan plan;
  build_plan(bg, n_qubits, o, adjoint != 0, &plan);
  *n_passes = (int64_t)plan.passes.size();
  for (size_t i = 0; i < plan.passes.size() && (int64_t)i < cap; ++i) {
    const PassDesc& pd = plan.passes[i];
    sv_pass_info& r = out[i];
    r.k = pd.k;
    r.low = pd.low;
    r.R = pd.R;
    r.n_ops = pd.op_end - pd.op_begin;
    r.n_stages = pd.stage_end - pd.stage_begin;
    r.n_grad = pd.n_grad;
    r.tile_mask = 0;
    for (int p = 0; p < pd.k; ++p) r.tile_mask |= 1ull << pd.tq[p];
    r.n_dense = 0;
    for (int si = pd.stage_begin; si < pd.stage_end; ++si) r.n_dense += plan.stages[si].dense ? 1 : 0;
    r.mat_doubles = (int32_t)(((i + 1 < plan.passes.size()) ? plan.passes[i + 1].mat_begin : (int)plan.mats.size()) - pd.mat_begin);
    r.fma_per_amp = pass_fma_per_amp(plan, i);
    r.add_per_amp = pass_add_per_amp(plan, i);
    r.nondiag_mask = 0;
    for (int j = pd.op_begin; j < pd.op_end; ++j) {
      const DevOp& op = plan.ops[j];
      if (op.type == OP_D1 || op.type == OP_D2) continue;
      r.nondiag_mask |= 1ull << op.qa;
      if (op.qb >= 0) r.nondiag_mask |= 1ull << op.qb;
    }
  }
  return SV_OK;
}

extern "C" sv_status sv_expectation_with_grad_batch(sv_handle h, const sv_gate* gates, int64_t n_gates,
                                                    const double* params, int32_t n_params, int32_t n_rows,
                                                    const sv_pauli* terms, int64_t n_terms, double* out_values,
                                                    double* out_grads) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (n_rows < 0 || !out_values || (n_rows > 0 && n_params > 0 && (!params || !out_grads)))
    return fail(SV_E_ARG, "bad batch arguments");
  if (n_rows == 0) return SV_OK;
  if (h->density) return fail(SV_E_ARG, "batch mode is not available on density-matrix handles");
  if (h->c64) {  // complex64 state: this operation reads a complex128 copy (the state is unchanged)
    const int prc = c64_promote(h);
    if (prc) return prc;
  }
  if (h->world > 1 || h->n_local > kBatchMaxQubits) {
    for (int32_t r = 0; r < n_rows; ++r) {
      rc = sv_expectation_with_grad(h, gates, n_gates, params ? params + (size_t)r * n_params : nullptr, n_params, terms,
                                    n_terms, out_values + r, out_grads ? out_grads + (size_t)r * n_params : nullptr);
      if (rc) return rc;
    }
    return SV_OK;
  }
  // row 0 is bound (and validated) through the normal path; the other rows only re-bind their
  // parametrised gates (below, on host threads, straight into the matrix block)
  std::vector<std::vector<BoundGate>> rows(1);
  rc = bind_circuit(h, gates, n_gates, params, n_params, true, &rows[0]);
  if (rc) return fail(rc, std::string("row 0: ") + g_last_error);
  PauliGroups G;
  rc = group_terms(h, terms, n_terms, &G);
  if (rc) return rc;
  // ops, full matrices per row, generators
  const std::vector<BoundGate>& g0 = rows[0];
  std::vector<BatchOp> ops(g0.size());
  std::vector<Cx> gens;
  int mo = 0;
  auto full = [](const BoundGate& b, Cx* m) -> int {
    const Cx z{0, 0}, one{1, 0};
    switch (b.cls) {
      case GC_XLIKE: m[0] = z; m[1] = b.m[0]; m[2] = b.m[1]; m[3] = z; return 2;
      case GC_ZLIKE: m[0] = b.m[0]; m[1] = z; m[2] = z; m[3] = b.m[1]; return 2;
      case GC_GEN1: for (int e = 0; e < 4; ++e) m[e] = b.m[e]; return 2;
      case GC_GEN2: for (int e = 0; e < 16; ++e) m[e] = b.m[e]; return 4;
      case GC_DIAG2: for (int e = 0; e < 16; ++e) m[e] = z; for (int j = 0; j < 4; ++j) m[j * 5] = b.m[j]; return 4;
      case GC_SWAP: for (int e = 0; e < 16; ++e) m[e] = z; m[0] = one; m[6] = one; m[9] = one; m[15] = one; return 4;
    }
    return 0;
  };
  for (size_t k = 0; k < g0.size(); ++k) {
    const BoundGate& b = g0[k];
    BatchOp& o = ops[k];
    std::memset(&o, 0, sizeof(o));
    Cx m[16];
    o.dim = full(b, m);
    o.t0 = b.t0;
    o.t1 = b.t1 >= 0 ? b.t1 : 0;
    o.cmask = b.controls;
    o.param = b.param;
    o.coeff = b.coeff;
    o.mat_off = mo;
    mo += o.dim * o.dim;
    o.gen_off = (int)gens.size();
    if (b.param >= 0) {
      // full generator matrix of the gate's dimension (diagonal gens expanded)
      if (b.gen_dim == o.dim) for (int e = 0; e < o.dim * o.dim; ++e) gens.push_back(b.gen[e]);
      else return fail(SV_E_ARG, "generator dimension mismatch");
    }
  }
  const int64_t stride = mo;
  std::vector<uint64_t> xs, zs;
  std::vector<double> cs;
  for (size_t gi = 0; gi < G.xs.size(); ++gi)
    for (int t = G.begin[gi]; t < G.end[gi]; ++t) {
      xs.push_back(G.xs[gi]);
      zs.push_back(G.z[t]);
      cs.push_back(G.c[2 * t]);
      cs.push_back(G.c[2 * t + 1]);
    }
  // one upload from page-locked staging: [ops | gens | mats | x | z | c]; the per-row matrices are
  // written straight into it
  auto al = [](size_t v) { return (v + 63) & ~size_t(63); };
  const size_t b_ops = ops.size() * sizeof(BatchOp), b_gen = gens.size() * 16,
               b_mat = (size_t)stride * (size_t)n_rows * 16, b_x = xs.size() * 8, b_c = cs.size() * 8;
  const size_t o_gen = al(b_ops), o_mat = o_gen + al(b_gen), o_x = o_mat + al(b_mat), o_z = o_x + al(b_x),
               o_c = o_z + al(b_x), total = o_c + al(b_c) + 64;
  if (!h->d_terms.ensure(total)) return fail(SV_E_OOM, "batch buffers");
  const size_t nout = (size_t)n_rows * (1 + (size_t)std::max(n_params, 0));
  if (!h->d_out.ensure(nout * 8 + 8)) return fail(SV_E_OOM, "batch outputs");
  if (!h->pin_in.ensure(total) || !h->pin_out.ensure(nout * 8 + 8)) return fail(SV_E_OOM, "batch host staging");
  char* hs = static_cast<char*>(h->pin_in.p);
  Cx* mats = reinterpret_cast<Cx*>(hs + o_mat);
  for (size_t k = 0; k < g0.size(); ++k) full(g0[k], mats + ops[k].mat_off);
  std::vector<int64_t> pgates;  // the row-dependent (parametrised) gates
  for (size_t k = 0; k < g0.size(); ++k)
    if (g0[k].param >= 0) pgates.push_back((int64_t)k);
  {
    std::vector<int> row_rc((size_t)n_rows, SV_OK);
    std::vector<std::string> row_err((size_t)n_rows);
    // row chunks on the persistent host pool (no thread spawn per call)
    const int nt = std::max(1, std::min(64, (n_rows - 1 + 63) / 64));
    auto work = [&](int t) {
      BoundGate b;
      std::string err;
      for (int32_t r = 1 + t; r < n_rows; r += nt) {
        Cx* mr = mats + (size_t)r * stride;
        std::memcpy(mr, mats, (size_t)stride * sizeof(Cx));  // row-independent gates
        const double* pr = params ? params + (size_t)r * n_params : nullptr;
        for (int64_t k : pgates) {
          const int grc = bind_gate(h->n, &gates[k], pr, n_params, true, &b, &err);
          if (grc != SV_OK) {
            row_rc[(size_t)r] = grc;
            row_err[(size_t)r] = "gate " + std::to_string(k) + ": " + err;
            break;
          }
          full(b, mr + ops[(size_t)k].mat_off);
        }
      }
    };
    host_parallel_for(nt, work);
    for (int32_t r = 1; r < n_rows; ++r)
      if (row_rc[(size_t)r] != SV_OK)
        return fail(row_rc[(size_t)r], std::string("row ") + std::to_string(r) + ": " + row_err[(size_t)r]);
  }
  std::memcpy(hs, ops.data(), b_ops);
  std::memcpy(hs + o_gen, gens.data(), b_gen);
  std::memcpy(hs + o_x, xs.data(), b_x);
  std::memcpy(hs + o_z, zs.data(), b_x);
  std::memcpy(hs + o_c, cs.data(), b_c);
  cudaError_t e = cudaMemcpyAsync(h->d_terms.p, hs, total, cudaMemcpyHostToDevice, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "batch upload");
  const char* db = static_cast<const char*>(h->d_terms.p);
  double* dout = static_cast<double*>(h->d_out.p);
  BatchArgs a;
  std::memset(&a, 0, sizeof(a));
  a.ops = reinterpret_cast<const BatchOp*>(db);
  a.nops = (int)ops.size();
  a.nterms = (int)xs.size();
  a.nparams = std::max(n_params, 0);
  a.gens = reinterpret_cast<const double*>(db + o_gen);
  a.mats = reinterpret_cast<const double*>(db + o_mat);
  a.row_stride = stride;
  a.x = reinterpret_cast<const uint64_t*>(db + o_x);
  a.z = reinterpret_cast<const uint64_t*>(db + o_z);
  a.c = reinterpret_cast<const double*>(db + o_c);
  a.out_e = dout;
  a.out_g = dout + n_rows;
  e = launch_batch_grad(h->psi, h->n_local, a, n_rows, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "batch launch");
  h->stats.kernel_launches += 1;
  const double* hv = static_cast<const double*>(h->pin_out.p);
  e = cudaMemcpyAsync(h->pin_out.p, dout, nout * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "batch readback");
  for (int32_t r = 0; r < n_rows; ++r) out_values[r] = hv[(size_t)r];
  if (n_params > 0)
    for (size_t i = 0; i < (size_t)n_rows * n_params; ++i) out_grads[i] = hv[(size_t)n_rows + i];
  h->stats.gates_applied += (int64_t)n_rows * n_gates;
  return SV_OK;
}

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

extern "C" sv_status sv_sample(sv_handle h, const int32_t* qubits, int32_t n_measured, int64_t shots, uint64_t seed,
                               uint64_t* out) {
  int rc = check_handle(h);
  if (rc) return rc;
  DeviceGuard dev_guard(h->device);
  if (shots < 0 || n_measured < 0 || n_measured > 64 || (shots > 0 && !out) || (n_measured > 0 && !qubits))
    return fail(SV_E_ARG, "bad sampling arguments");
  if (h->world > 1) return fail(SV_E_ARG, "sampling is single-GPU in this version");
  if (h->density) return fail(SV_E_ARG, "sampling is not available on density-matrix handles");
  if (h->c64) {  // complex64 state: this operation reads a complex128 copy (the state is unchanged)
    const int prc = c64_promote(h);
    if (prc) return prc;
  }
  for (int j = 0; j < n_measured; ++j)
    if (qubits[j] < 0 || qubits[j] >= h->n) return fail(SV_E_QUBIT_RANGE, "measured qubit out of range");
  if (shots == 0) return SV_OK;
  const int n = h->n_local;
  const int bl = std::min(n, 16);
  const int64_t nb = int64_t(1) << (n - bl);
  if (!h->d_partials.ensure((size_t)nb * 8 + 8)) return fail(SV_E_OOM, "block masses");
  cudaError_t e = launch_block_prob(h->psi, n, bl, static_cast<double*>(h->d_partials.p), h->stream);
  std::vector<double> mass((size_t)nb);
  if (e == cudaSuccess) e = cudaMemcpyAsync(mass.data(), h->d_partials.p, nb * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "block masses");
  h->stats.kernel_launches += 1;
  std::vector<double> pref((size_t)nb + 1, 0.0);
  for (int64_t b = 0; b < nb; ++b) pref[(size_t)b + 1] = pref[(size_t)b] + mass[(size_t)b];
  const double total = pref[(size_t)nb];
  // sorted draws (target mass = u * total), shot order remembered
  std::vector<std::pair<double, int64_t>> draws((size_t)shots);
  for (int64_t s = 0; s < shots; ++s)
    draws[(size_t)s] = {(double)(splitmix64(seed + (uint64_t)s) >> 11) * 0x1.0p-53 * total, s};
  std::sort(draws.begin(), draws.end());
  std::vector<int64_t> blk, beg;
  std::vector<double> target((size_t)shots);
  int64_t b = 0;
  for (int64_t i = 0; i < shots; ++i) {
    const double u = draws[(size_t)i].first;
    while (b < nb - 1 && pref[(size_t)b + 1] < u) ++b;
    if (blk.empty() || blk.back() != b) { blk.push_back(b); beg.push_back(i); }
    target[(size_t)i] = u - pref[(size_t)b];
  }
  beg.push_back(shots);
  const size_t nblk = blk.size();
  auto al = [](size_t v) { return (v + 63) & ~size_t(63); };
  const size_t o_beg = al(nblk * 8), o_t = o_beg + al((nblk + 1) * 8), o_out = o_t + al((size_t)shots * 8),
               total_b = o_out + (size_t)shots * 8 + 64;
  if (!h->d_terms.ensure(total_b)) return fail(SV_E_OOM, "sampling buffers");
  h->h_stage.assign(o_out, 0);
  std::memcpy(h->h_stage.data(), blk.data(), nblk * 8);
  std::memcpy(h->h_stage.data() + o_beg, beg.data(), (nblk + 1) * 8);
  std::memcpy(h->h_stage.data() + o_t, target.data(), (size_t)shots * 8);
  char* db = static_cast<char*>(h->d_terms.p);
  e = cudaMemcpyAsync(db, h->h_stage.data(), o_out, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess)
    e = launch_sample_blocks(h->psi, bl, (int)nblk, reinterpret_cast<const int64_t*>(db),
                             reinterpret_cast<const int64_t*>(db + o_beg), reinterpret_cast<const double*>(db + o_t),
                             reinterpret_cast<int64_t*>(db + o_out), h->stream);
  std::vector<int64_t> idx((size_t)shots);
  if (e == cudaSuccess) e = cudaMemcpyAsync(idx.data(), db + o_out, (size_t)shots * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "sampling");
  h->stats.kernel_launches += 1;
  for (int64_t i = 0; i < shots; ++i) {
    const uint64_t x = (uint64_t)idx[(size_t)i];
    uint64_t o = 0;
    for (int j = 0; j < n_measured; ++j) o |= ((x >> qubits[j]) & 1ull) << j;
    out[draws[(size_t)i].second] = o;
  }
  return SV_OK;
}
