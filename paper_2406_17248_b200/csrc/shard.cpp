// shard.cpp — state vectors sharded across GPUs by their top qubits.
//
// Layout: with P = 2^g shards, physical qubit positions 0 .. nl-1 (nl = n - g) are the local index
// bits of a shard and positions nl .. n-1 are its rank bits. A logical -> physical permutation is
// kept per state (lazy remapping); sv_get_state un-permutes.
//
//   * gates whose non-diagonal targets are local run as ordinary fused passes on every shard;
//   * controls and diagonal factors on global qubits need no communication: each shard knows its
//     rank bits, so a global control either drops the gate on that shard or disappears, and a
//     diagonal factor on a global qubit becomes a per-shard scalar / local diagonal;
//   * a non-diagonal target on a global qubit first swaps that qubit with a local one: rank r and
//     r ^ 2^j exchange the halves of their shards selected by the local bit (NCCL grouped
//     send/recv, chunked through bounce buffers; virtual shards: one swap kernel);
//   * expectation groups whose x-mask touches a global qubit swap it in the same way; partials of
//     all shards are summed in fixed order and all-reduced across ranks;
//   * the adjoint sweep replays the forward schedule backwards on psi and lambda together (every
//     swap is its own inverse) and all-reduces (E, gradient) once at the end.
//
// Two transports share all of the above: NCCL (one process per GPU, sv_create_sharded) and virtual
// shards (all P shards on one GPU, sv_create_virtual_shards) used to test the sharded executor on
// one device.
#include <nccl.h>
#include <cstdlib>

#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include "sv_debug.h"
#include "sv_handle.h"

namespace sv {

struct ShardState {
  int g = 0;                    // global qubits (log2 of the shard count)
  bool virt = false;            // virtual shards on one device
  std::vector<int> ranks;       // shard ids held by this handle (virtual: 0..P-1, NCCL: {rank})
  std::vector<DevBuf> bufs;     // state shards
  std::vector<DevBuf> wpsi, wlam;  // gradient workspaces per held shard
  std::vector<int> perm;        // logical qubit -> physical position (the state's layout)
  ncclComm_t comm = nullptr;
  DevBuf sendb, recvb, scalar;  // NCCL bounce buffers, all-reduce scratch
};

namespace {

constexpr int64_t kChunkAmps = int64_t(1) << 26;  // 1 GiB of complex128 per exchange chunk

int nccl_fail(sv_state_s* h, ncclResult_t r, const char* where) {
  h->poisoned = true;
  return fail(SV_E_NCCL, std::string(where) + ": " + ncclGetErrorString(r));
}

struct Step {
  int kind = 0;                      // 0: segment of gates, 1: swap of physical positions (G, L)
  std::vector<BoundGate> gates;      // physical positions
  int gpos = 0, lpos = 0;
};

BoundGate to_physical(const BoundGate& g, const std::vector<int>& perm) {
  BoundGate p = g;
  p.t0 = perm[g.t0];
  p.t1 = g.t1 >= 0 ? perm[g.t1] : -1;
  p.controls = 0;
  for (size_t q = 0; q < perm.size(); ++q)
    if ((g.controls >> q) & 1ull) p.controls |= 1ull << perm[q];
  return p;
}

bool nondiag(const BoundGate& g) { return !(g.cls == GC_ZLIKE || g.cls == GC_DIAG2); }

void do_swap_perm(std::vector<int>& perm, int G, int L) {
  for (int& p : perm) {
    if (p == G) p = L;
    else if (p == L) p = G;
  }
}

// Splits a circuit into local segments and global<->local swaps, updating perm. Each segment takes
// every pending gate that is local (non-diagonal targets on local positions) and may legally move
// ahead of the gates left behind (same commutation rule as the pass planner), so a swap is only
// issued when nothing else can run; the swapped-out local qubit is the one whose next
// non-diagonal use lies furthest ahead (Belady).
std::vector<Step> schedule(const std::vector<BoundGate>& gates, std::vector<int>& perm, int nl) {
  std::vector<Step> steps;
  std::vector<int> pending(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) pending[i] = (int)i;
  auto tmask = [](const BoundGate& g) { return (1ull << g.t0) | (g.t1 >= 0 ? (1ull << g.t1) : 0ull); };
  while (!pending.empty()) {
    Step seg;
    std::vector<int> skipped;
    uint64_t bN = 0, bA = 0;  // logical qubits
    for (int gi : pending) {
      const BoundGate& g = gates[(size_t)gi];
      const uint64_t N = nondiag(g) ? tmask(g) : 0ull;
      const uint64_t A = tmask(g) | g.controls;
      bool ok = !(N & bA) && !(A & bN);
      if (ok && N) {
        const BoundGate p = to_physical(g, perm);
        ok = p.t0 < nl && (p.t1 < 0 || p.t1 < nl);
      }
      if (ok) seg.gates.push_back(to_physical(g, perm));
      else { skipped.push_back(gi); bN |= N; bA |= A; }
    }
    if (!seg.gates.empty()) steps.push_back(std::move(seg));
    pending.swap(skipped);
    if (pending.empty()) break;
    // the first pending gate is blocked only by global non-diagonal targets: swap them in
    const BoundGate& g = gates[(size_t)pending[0]];
    for (int t = 0; t < 2; ++t) {
      const int q = t == 0 ? g.t0 : g.t1;
      if (q < 0 || perm[(size_t)q] < nl) continue;
      const int G = perm[(size_t)q];
      int L = -1, best = -1;
      for (int c = nl - 1; c >= 0; --c) {
        const BoundGate p = to_physical(g, perm);
        if (c == p.t0 || c == p.t1) continue;
        int lq = -1;
        for (size_t x = 0; x < perm.size(); ++x)
          if (perm[x] == c) lq = (int)x;
        int next = (int)pending.size();  // first pending gate using lq non-diagonally
        for (size_t k = 0; k < pending.size(); ++k) {
          const BoundGate& h = gates[(size_t)pending[k]];
          if (nondiag(h) && ((tmask(h) >> lq) & 1ull)) { next = (int)k; break; }
        }
        if (next > best) { best = next; L = c; }
      }
      Step sw;
      sw.kind = 1;
      sw.gpos = G;
      sw.lpos = L;
      steps.push_back(sw);
      do_swap_perm(perm, G, L);
    }
  }
  return steps;
}

// Rewrites physical gates for the shard with rank bits r: global controls resolve, diagonal
// factors on global qubits become local diagonals / scalars. Non-diagonal targets are local.
std::vector<BoundGate> localize(const std::vector<BoundGate>& phys, int nl, uint64_t r) {
  const uint64_t lmask = nl >= 64 ? ~0ull : ((1ull << nl) - 1);
  std::vector<BoundGate> out;
  out.reserve(phys.size());
  for (const BoundGate& g0 : phys) {
    const uint64_t cg = g0.controls >> nl;
    if ((r & cg) != cg) continue;  // a global control is 0 on this shard: identity here
    BoundGate g = g0;
    g.controls &= lmask;
    const bool t0g = g.t0 >= nl, t1g = g.t1 >= nl;
    if (!t0g && !t1g) { out.push_back(g); continue; }
    // diagonal with global target(s)
    Cx e0, e1;             // local diagonal entries (scalar if no local target remains)
    int tl = -1;           // remaining local target, -1: scalar
    double gsign = 0.0;    // generator structure, see below
    if (g.cls == GC_ZLIKE) {
      const uint32_t b = (uint32_t)((r >> (g.t0 - nl)) & 1ull);
      e0 = e1 = g.m[b];
      if (g.param >= 0) gsign = (g.kind == SV_PS) ? (double)b : (b ? -1.0 : 1.0);
    } else {  // GC_DIAG2: entries m[b0 | b1 << 1]
      if (t0g && t1g) {
        const uint32_t b0 = (uint32_t)((r >> (g.t0 - nl)) & 1ull), b1 = (uint32_t)((r >> (g.t1 - nl)) & 1ull);
        e0 = e1 = g.m[b0 | (b1 << 1)];
        gsign = ((b0 ^ b1) ? -1.0 : 1.0);
      } else if (t0g) {
        const uint32_t b0 = (uint32_t)((r >> (g.t0 - nl)) & 1ull);
        tl = g.t1;
        e0 = g.m[b0];
        e1 = g.m[b0 | 2u];
        gsign = b0 ? -1.0 : 1.0;
      } else {
        const uint32_t b1 = (uint32_t)((r >> (g.t1 - nl)) & 1ull);
        tl = g.t0;
        e0 = g.m[b1 << 1];
        e1 = g.m[1u | (b1 << 1)];
        gsign = b1 ? -1.0 : 1.0;
      }
    }
    // generator of the rewritten op (diagonal): RZ / RZZ: -(i/2) s Z_local or -(i/2) s (scalar);
    // PS: i b (scalar on the global |1>)
    BoundGate o = g;
    o.cls = GC_ZLIKE;
    o.t1 = -1;
    const bool ps = (g.kind == SV_PS);
    Cx ga{0, 0}, gb{0, 0};
    if (tl >= 0) {
      o.t0 = tl;
      o.m[0] = e0;
      o.m[1] = e1;
      ga = Cx{0, -0.5 * gsign};
      gb = Cx{0, 0.5 * gsign};
    } else {
      const Cx gs = ps ? Cx{0, gsign} : Cx{0, -0.5 * gsign};
      if (g.controls) {
        // scalar on the control-satisfied subspace: diag(1, f) on one control, others stay
        int c = __builtin_ctzll(g.controls);
        o.t0 = c;
        o.controls = g.controls & ~(1ull << c);
        o.m[0] = Cx{1, 0};
        o.m[1] = e1;
        ga = Cx{0, 0};
        gb = gs;
      } else {
        o.t0 = 0;
        o.m[0] = e0;
        o.m[1] = e1;
        ga = gb = gs;
      }
    }
    if (g.param >= 0) {
      o.kind = SV_RZ;  // diagonal generator (plan emission keys on RZ / PS / RZZ)
      o.gen_dim = 2;
      o.gen[0] = ga;
      o.gen[1] = Cx{0, 0};
      o.gen[2] = Cx{0, 0};
      o.gen[3] = gb;
    } else {
      o.kind = SV_ZLIKE;
    }
    out.push_back(o);
  }
  return out;
}

uint64_t permute_mask(uint64_t m, const std::vector<int>& perm) {
  uint64_t o = 0;
  for (size_t q = 0; q < perm.size(); ++q)
    if ((m >> q) & 1ull) o |= 1ull << perm[q];
  return o;
}

// ---- transports ----

// Swap physical positions G (global) and L (local) of the vectors `vecs` (per held shard).
int swap_qubits(sv_state_s* h, const std::vector<std::vector<double*>>& vecs, int G, int L) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  const int j = G - nl;
  h->stats.exchanges += 1;
  // SV_VIRTUAL_BOUNCE=<chunk amplitudes>: virtual shards exchange through the NCCL path's
  // pack / bounce-buffer / unpack sequence (device copies instead of ncclSend/ncclRecv), chunked,
  // so the tests exercise that code on one GPU.
  const char* bounce_env = std::getenv("SV_VIRTUAL_BOUNCE");
  const int64_t bounce_chunk = bounce_env ? std::max<int64_t>(1, std::atoll(bounce_env)) : 0;
  if (S.virt && bounce_chunk > 0) {
    const int64_t half = int64_t(1) << (nl - 1);
    const int64_t chunk = std::min(half, bounce_chunk);
    if (!S.sendb.ensure((size_t)chunk * 16) || !S.recvb.ensure((size_t)chunk * 16)) return fail(SV_E_OOM, "bounce buffers");
    for (const auto& v : vecs) {
      for (size_t a = 0; a < S.ranks.size(); ++a) {
        const int r = S.ranks[a];
        if ((r >> j) & 1) continue;
        const size_t p = (size_t)(r | (1 << j));
        for (int64_t off = 0; off < half; off += chunk) {
          const int64_t cnt = std::min(chunk, half - off);
          // r packs its half with bit L = 1, p its half with bit L = 0; each unpacks the other's
          cudaError_t e = launch_pack_half(v[a], static_cast<double*>(S.sendb.p), L, 1, off, cnt, true, h->stream);
          if (e == cudaSuccess) e = launch_pack_half(v[p], static_cast<double*>(S.recvb.p), L, 0, off, cnt, true, h->stream);
          if (e == cudaSuccess) e = launch_pack_half(v[a], static_cast<double*>(S.recvb.p), L, 1, off, cnt, false, h->stream);
          if (e == cudaSuccess) e = launch_pack_half(v[p], static_cast<double*>(S.sendb.p), L, 0, off, cnt, false, h->stream);
          if (e != cudaSuccess) return cuda_fail(h, e, "bounce exchange");
          h->stats.kernel_launches += 4;
        }
      }
    }
    h->stats.algorithmic_bytes += 32.0 * (double)(1ull << nl) * (double)S.ranks.size() * vecs.size() / 2.0;
    return SV_OK;
  }
  if (S.virt) {
    for (const auto& v : vecs) {
      for (size_t a = 0; a < S.ranks.size(); ++a) {
        const int r = S.ranks[a];
        if ((r >> j) & 1) continue;
        const int p = r | (1 << j);
        // shard r (bit j = 0) sends its half with bit L = 1; partner p sends its half with bit L = 0
        cudaError_t e = launch_swap_halves(v[a], v[(size_t)p], nl, L, h->stream);
        if (e != cudaSuccess) return cuda_fail(h, e, "swap kernel");
        h->stats.kernel_launches += 1;
      }
    }
    h->stats.algorithmic_bytes += 32.0 * (double)(1ull << nl) * (double)S.ranks.size() * vecs.size() / 2.0;
    return SV_OK;
  }
  // NCCL: one held shard
  const int r = S.ranks[0];
  const int peer = r ^ (1 << j);
  const int h_send = ((r >> j) & 1) ? 0 : 1;  // send the half whose bit L differs from our bit j
  const int64_t half = int64_t(1) << (nl - 1);
  const int64_t chunk = std::min(half, kChunkAmps);
  if (!S.sendb.ensure((size_t)chunk * 16) || !S.recvb.ensure((size_t)chunk * 16)) return fail(SV_E_OOM, "bounce buffers");
  for (const auto& v : vecs) {
    double* shard = v[0];
    for (int64_t off = 0; off < half; off += chunk) {
      const int64_t cnt = std::min(chunk, half - off);
      cudaError_t e = launch_pack_half(shard, static_cast<double*>(S.sendb.p), L, h_send, off, cnt, true, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "pack");
      ncclResult_t nr = ncclGroupStart();
      if (nr == ncclSuccess) nr = ncclSend(S.sendb.p, (size_t)cnt * 2, ncclDouble, peer, S.comm, h->stream);
      if (nr == ncclSuccess) nr = ncclRecv(S.recvb.p, (size_t)cnt * 2, ncclDouble, peer, S.comm, h->stream);
      ncclResult_t ne = ncclGroupEnd();
      if (nr != ncclSuccess) return nccl_fail(h, nr, "exchange");
      if (ne != ncclSuccess) return nccl_fail(h, ne, "exchange");
      e = launch_pack_half(shard, static_cast<double*>(S.recvb.p), L, h_send, off, cnt, false, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "unpack");
      h->stats.kernel_launches += 2;
    }
  }
  h->stats.algorithmic_bytes += 32.0 * (double)half * vecs.size();
  return SV_OK;
}

int allreduce_host(sv_state_s* h, double* vals, size_t n) {
  ShardState& S = *h->shard;
  if (S.virt || n == 0) return SV_OK;
  if (!S.scalar.ensure(n * 8)) return fail(SV_E_OOM, "allreduce scratch");
  cudaError_t e = cudaMemcpyAsync(S.scalar.p, vals, n * 8, cudaMemcpyHostToDevice, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "allreduce upload");
  ncclResult_t r = ncclAllReduce(S.scalar.p, S.scalar.p, n, ncclDouble, ncclSum, S.comm, h->stream);
  if (r != ncclSuccess) return nccl_fail(h, r, "allreduce");
  e = cudaMemcpyAsync(vals, S.scalar.p, n * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "allreduce download");
  return SV_OK;
}

// Runs one segment (physical gates) on every held shard of `vecs` (forward).
int run_segment(sv_state_s* h, const std::vector<BoundGate>& phys, const std::vector<double*>& vec) {
  ShardState& S = *h->shard;
  for (size_t a = 0; a < S.ranks.size(); ++a) {
    std::vector<BoundGate> loc = localize(phys, h->n_local, (uint64_t)S.ranks[a]);
    if (loc.empty()) continue;
    const CachedPlan* cp = nullptr;
    int rc = get_plan(h, loc, false, &cp);
    if (rc) return rc;
    rc = run_plan(h, *cp, vec[a], nullptr, nullptr, 0, nullptr, nullptr);
    if (rc) return rc;
  }
  return SV_OK;
}

int init_shards(sv_state_s* h, const std::vector<double*>& vec) {
  ShardState& S = *h->shard;
  for (size_t a = 0; a < S.ranks.size(); ++a) {
    cudaError_t e = launch_init_zero(vec[a], int64_t(1) << h->n_local, S.ranks[a] == 0, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "init");
    h->stats.kernel_launches += 1;
  }
  for (size_t q = 0; q < S.perm.size(); ++q) S.perm[q] = (int)q;
  return SV_OK;
}

std::vector<double*> state_ptrs(ShardState& S) {
  std::vector<double*> v;
  for (auto& b : S.bufs) v.push_back(static_cast<double*>(b.p));
  return v;
}

sv_status create_common(int32_t n, int32_t world, bool virt, int32_t rank, sv_handle* out) {
  if (!out) return fail(SV_E_ARG, "null out");
  *out = nullptr;
  if (world < 1 || (world & (world - 1))) return fail(SV_E_ARG, "world must be a power of two");
  const int g = __builtin_ctz((unsigned)world);
  if (n < 1 || n > 44 || n - g < 1) return fail(SV_E_ARG, "n_qubits out of range for this world size");
  if (!virt && (rank < 0 || rank >= world)) return fail(SV_E_ARG, "rank out of range");
  sv_state_s* h = new sv_state_s();
  h->n = n;
  h->n_local = n - g;
  h->world = world;
  h->rank = virt ? 0 : rank;
  cudaGetDevice(&h->device);
  if (cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return fail(SV_E_CUDA, "stream");
  }
  h->stream = h->own_stream;
  h->shard = new ShardState();
  ShardState& S = *h->shard;
  S.g = g;
  S.virt = virt;
  S.perm.resize((size_t)n);
  if (virt)
    for (int r = 0; r < world; ++r) S.ranks.push_back(r);
  else
    S.ranks.push_back(rank);
  S.bufs.resize(S.ranks.size());
  for (auto& b : S.bufs)
    if (!b.ensure(size_t(16) << h->n_local)) {
      sv_destroy(h);
      return fail(SV_E_OOM, "cannot allocate the state shard");
    }
  h->psi = static_cast<double*>(S.bufs[0].p);
  *out = h;
  return SV_OK;
}

}  // namespace

void destroy_sharding(sv_state_s* h) {
  if (!h->shard) return;
  ShardState& S = *h->shard;
  for (auto& b : S.bufs) b.release();
  for (auto& b : S.wpsi) b.release();
  for (auto& b : S.wlam) b.release();
  S.sendb.release();
  S.recvb.release();
  S.scalar.release();
  if (S.comm) ncclCommDestroy(S.comm);
  delete h->shard;
  h->shard = nullptr;
}

int shard_reset(sv_state_s* h) { return init_shards(h, state_ptrs(*h->shard)); }

// Logical amplitude index i -> (shard, local index) under perm.
static inline void locate(uint64_t i, const std::vector<int>& perm, int nl, uint64_t* shard, uint64_t* local) {
  uint64_t x = 0;
  for (size_t q = 0; q < perm.size(); ++q)
    if ((i >> q) & 1ull) x |= 1ull << perm[q];
  *shard = x >> nl;
  *local = x & ((1ull << nl) - 1);
}

int shard_set_state(sv_state_s* h, const double* host) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  const uint64_t N = 1ull << h->n, NL = 1ull << nl;
  for (size_t q = 0; q < S.perm.size(); ++q) S.perm[q] = (int)q;  // identity layout: contiguous shards
  for (size_t a = 0; a < S.ranks.size(); ++a) {
    const double* src = host + 2 * NL * (uint64_t)S.ranks[a];
    cudaError_t e = cudaMemcpyAsync(S.bufs[a].p, src, NL * 16, cudaMemcpyHostToDevice, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "set_state");
  }
  (void)N;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "set_state");
  return SV_OK;
}

int shard_get_state(sv_state_s* h, double* host) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  const uint64_t N = 1ull << h->n, NL = 1ull << nl;
  // all shards in physical order on the host
  std::vector<double> phys(2 * N);
  if (S.virt) {
    for (size_t a = 0; a < S.ranks.size(); ++a) {
      cudaError_t e = cudaMemcpyAsync(phys.data() + 2 * NL * (uint64_t)S.ranks[a], S.bufs[a].p, NL * 16,
                                      cudaMemcpyDeviceToHost, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "get_state");
    }
  } else {
    DevBuf all;
    if (!all.ensure(N * 16)) return fail(SV_E_OOM, "gather buffer");
    ncclResult_t r = ncclAllGather(S.bufs[0].p, all.p, NL * 2, ncclDouble, S.comm, h->stream);
    if (r != ncclSuccess) { all.release(); return nccl_fail(h, r, "allgather"); }
    cudaError_t e = cudaMemcpyAsync(phys.data(), all.p, N * 16, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    all.release();
    if (e != cudaSuccess) return cuda_fail(h, e, "get_state");
  }
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "get_state");
  for (uint64_t i = 0; i < N; ++i) {
    uint64_t sh, lo;
    locate(i, S.perm, nl, &sh, &lo);
    const uint64_t x = (sh << nl) | lo;
    host[2 * i] = phys[2 * x];
    host[2 * i + 1] = phys[2 * x + 1];
  }
  return SV_OK;
}

// Sampled amplitudes in logical order: every held shard gathers the indices it owns (others read
// as 0), the NCCL transport sums the per-rank vectors with one all-reduce (x + 0 = x: exact).
int shard_get_amplitudes(sv_state_s* h, const uint64_t* idx, int64_t count, double* out) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  std::fill(out, out + 2 * count, 0.0);
  for (size_t a = 0; a < S.ranks.size(); ++a) {
    std::vector<uint64_t> loc((size_t)count);
    for (int64_t j = 0; j < count; ++j) {
      uint64_t sh, lo;
      locate(idx[j], S.perm, nl, &sh, &lo);
      loc[(size_t)j] = sh == (uint64_t)S.ranks[a] ? lo : ~0ull;
    }
    int rc = gather_amplitudes(h, S.bufs[a].p, false, loc, out, true);
    if (rc) return rc;
  }
  return allreduce_host(h, out, (size_t)(2 * count));
}

int shard_apply(sv_state_s* h, const std::vector<BoundGate>& bg) {
  ShardState& S = *h->shard;
  std::vector<Step> steps = schedule(bg, S.perm, h->n_local);
  std::vector<double*> st = state_ptrs(S);
  for (const Step& s : steps) {
    int rc = s.kind == 0 ? run_segment(h, s.gates, st) : swap_qubits(h, {st}, s.gpos, s.lpos);
    if (rc) return rc;
  }
  h->stats.gates_applied += (int64_t)bg.size();
  return SV_OK;
}

// Swaps global positions of the x-masks in `groups` to local ones (state perm updated), one group
// at a time, then evaluates the group on every held shard. Returns the per-handle partial sum
// (not yet all-reduced). lam (optional, per shard) receives H psi.
static int sharded_groups(sv_state_s* h, const PauliGroups& G, std::vector<int>& perm,
                          const std::vector<std::vector<double*>>& swap_vecs, const std::vector<double*>& psi,
                          const std::vector<double*>& lam, double* out_e, std::vector<std::pair<int, int>>* swaps) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  const uint64_t lmask = (1ull << nl) - 1;
  const int grid = pauli_grid(nl);
  double E = 0.0;
  if (!h->d_partials.ensure((size_t)grid * 8 + 8) || !h->d_out.ensure(64)) return fail(SV_E_OOM, "partials");
  std::vector<bool> lam_started(psi.size(), false);
  if (!lam.empty())
    for (size_t a = 0; a < lam.size(); ++a) {
      cudaError_t e = cudaMemsetAsync(lam[a], 0, size_t(16) << nl, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "zero lambda");
    }
  for (size_t gi = 0; gi < G.xs.size(); ++gi) {
    uint64_t xp = permute_mask(G.xs[gi], perm);
    while (xp >> nl) {
      const int Gpos = 63 - __builtin_clzll(xp);
      int L = -1;
      for (int c = nl - 1; c >= 0; --c)
        if (!((xp >> c) & 1ull)) { L = c; break; }
      if (L < 0) break;  // X/Y support wider than a shard: cross-shard evaluation below
      int rc = swap_qubits(h, swap_vecs, Gpos, L);
      if (rc) return rc;
      do_swap_perm(perm, Gpos, L);
      if (swaps) swaps->push_back({Gpos, L});
      xp = permute_mask(G.xs[gi], perm);
    }
    const uint64_t xg = xp >> nl;
    for (size_t a = 0; a < S.ranks.size(); ++a) {
      const uint64_t r = (uint64_t)S.ranks[a];
      std::vector<uint64_t> z;
      std::vector<double> c;
      const uint64_t rsig = xg ? (r ^ xg) : r;  // cross-shard: signs of the partner's rank bits
      for (int t = G.begin[gi]; t < G.end[gi]; ++t) {
        const uint64_t zp = permute_mask(G.z[t], perm);
        const double sgn = (__builtin_popcountll((zp >> nl) & rsig) & 1) ? -1.0 : 1.0;
        z.push_back(zp & lmask);
        c.push_back(sgn * G.c[2 * t]);
        c.push_back(sgn * G.c[2 * t + 1]);
      }
      const size_t zb = (z.size() * 8 + 15) & ~size_t(15);
      if (!h->d_terms.ensure(zb + c.size() * 8 + 16)) return fail(SV_E_OOM, "terms");
      h->h_stage.assign(zb + c.size() * 8, 0);
      std::memcpy(h->h_stage.data(), z.data(), z.size() * 8);
      std::memcpy(h->h_stage.data() + zb, c.data(), c.size() * 8);
      cudaError_t e = cudaMemcpyAsync(h->d_terms.p, h->h_stage.data(), h->h_stage.size(), cudaMemcpyHostToDevice, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "terms");
      double* dp = static_cast<double*>(h->d_partials.p);
      const uint64_t* dz = static_cast<const uint64_t*>(h->d_terms.p);
      const double* dc = reinterpret_cast<const double*>(static_cast<const char*>(h->d_terms.p) + zb);
      if (xg == 0) {
        e = launch_pauli_group(psi[a], lam.empty() ? nullptr : lam[a], true, nl, xp, dz, dc, (int)z.size(), dp, grid,
                               h->stream);
      } else {
        // partner shard r ^ xg: another virtual shard, or a full copy fetched over NCCL
        const double* partner = nullptr;
        if (S.virt) {
          partner = psi[(size_t)(r ^ xg)];
        } else {
          const int peer = (int)(r ^ xg);
          if (!S.recvb.ensure(size_t(16) << nl)) return fail(SV_E_OOM, "partner shard buffer");
          ncclResult_t nr = ncclGroupStart();
          if (nr == ncclSuccess) nr = ncclSend(psi[a], (size_t(2) << nl), ncclDouble, peer, S.comm, h->stream);
          if (nr == ncclSuccess) nr = ncclRecv(S.recvb.p, (size_t(2) << nl), ncclDouble, peer, S.comm, h->stream);
          ncclResult_t ne = ncclGroupEnd();
          if (nr != ncclSuccess) return nccl_fail(h, nr, "partner exchange");
          if (ne != ncclSuccess) return nccl_fail(h, ne, "partner exchange");
          partner = static_cast<const double*>(S.recvb.p);
        }
        e = launch_pauli_cross(psi[a], partner, lam.empty() ? nullptr : lam[a], nl, xp & lmask, dz, dc, (int)z.size(), dp,
                               grid, h->stream);
      }
      if (e == cudaSuccess) e = launch_reduce_slots(dp, 1, grid, static_cast<double*>(h->d_out.p), h->stream);
      double v = 0;
      if (e == cudaSuccess) e = cudaMemcpyAsync(&v, h->d_out.p, 8, cudaMemcpyDeviceToHost, h->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "sharded expectation");
      h->stats.kernel_launches += 2;
      h->stats.expectation_passes += 1;
      E += v;
    }
  }
  *out_e = E;
  return SV_OK;
}

int shard_expectation(sv_state_s* h, const PauliGroups& G, double* out) {
  ShardState& S = *h->shard;
  std::vector<double*> st = state_ptrs(S);
  double E = 0.0;
  int rc = sharded_groups(h, G, S.perm, {st}, st, {}, &E, nullptr);
  if (rc) return rc;
  rc = allreduce_host(h, &E, 1);
  if (rc) return rc;
  *out = E;
  return SV_OK;
}

int shard_expectation_with_grad(sv_state_s* h, const std::vector<BoundGate>& bg, int32_t n_params,
                                const PauliGroups& G, double* out_value, double* out_grad) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  const size_t bytes = size_t(16) << nl;
  S.wpsi.resize(S.ranks.size());
  S.wlam.resize(S.ranks.size());
  std::vector<double*> psi, lam;
  for (size_t a = 0; a < S.ranks.size(); ++a) {
    if (!S.wpsi[a].ensure(bytes) || !S.wlam[a].ensure(bytes)) return fail(SV_E_OOM, "gradient workspaces");
    psi.push_back(static_cast<double*>(S.wpsi[a].p));
    lam.push_back(static_cast<double*>(S.wlam[a].p));
    cudaError_t e = cudaMemcpyAsync(psi[a], S.bufs[a].p, bytes, cudaMemcpyDeviceToDevice, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "copy psi0");
  }
  // 1. forward (on the copy; its layout evolves from the state's)
  std::vector<int> perm = S.perm;
  std::vector<Step> steps = schedule(bg, perm, nl);
  for (const Step& s : steps) {
    int rc = s.kind == 0 ? run_segment(h, s.gates, psi) : swap_qubits(h, {psi}, s.gpos, s.lpos);
    if (rc) return rc;
  }
  // 2. lambda = H psi, E (x-masks swapped local on psi first)
  double E = 0.0;
  std::vector<std::pair<int, int>> hswaps;
  int rc = sharded_groups(h, G, perm, {psi, lam}, psi, lam, &E, &hswaps);  // lambda follows every swap
  if (rc) return rc;
  // 3. undo the Hamiltonian swaps on (psi, lambda), then the forward schedule backwards
  for (auto it = hswaps.rbegin(); it != hswaps.rend(); ++it) {
    rc = swap_qubits(h, {psi, lam}, it->first, it->second);
    if (rc) return rc;
  }
  std::vector<double> grad((size_t)std::max(n_params, 1), 0.0);
  for (auto it = steps.rbegin(); it != steps.rend(); ++it) {
    if (it->kind == 1) {
      rc = swap_qubits(h, {psi, lam}, it->gpos, it->lpos);
      if (rc) return rc;
      continue;
    }
    for (size_t a = 0; a < S.ranks.size(); ++a) {
      std::vector<BoundGate> loc = localize(it->gates, nl, (uint64_t)S.ranks[a]);
      if (loc.empty()) continue;
      const CachedPlan* revp = nullptr;
      rc = get_plan(h, loc, true, &revp);
      if (rc) return rc;
      std::vector<double> d;
      rc = run_reverse(h, *revp, psi[a], lam[a], &d);
      if (rc) return rc;
      for (size_t sl = 0; sl < d.size(); ++sl)
        grad[(size_t)revp->plan.slot_param[sl]] += revp->plan.slot_coeff[sl] * 2.0 * d[sl];
    }
  }
  // 4. one all-reduce of (E, gradient)
  std::vector<double> red;
  red.push_back(E);
  for (int32_t p = 0; p < n_params; ++p) red.push_back(grad[(size_t)p]);
  rc = allreduce_host(h, red.data(), red.size());
  if (rc) return rc;
  *out_value = red[0];
  for (int32_t p = 0; p < n_params; ++p) out_grad[p] = red[1 + (size_t)p];
  h->stats.gates_applied += (int64_t)bg.size();
  return SV_OK;
}

}  // namespace sv

extern "C" {

sv_status sv_nccl_unique_id(void* out, int32_t out_bytes) {
  if (!out || out_bytes < (int32_t)sizeof(ncclUniqueId)) return sv::fail(SV_E_ARG, "buffer too small for ncclUniqueId");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return sv::fail(SV_E_NCCL, ncclGetErrorString(r));
  std::memcpy(out, &id, sizeof(id));
  return SV_OK;
}

sv_status sv_shard_plan(int32_t n_qubits, int32_t world, int32_t rank, const sv_gate* gates, int64_t n_gates,
                        const double* params, int32_t n_params, sv_shard_step* steps, int64_t cap_steps,
                        int64_t* n_steps, sv_gate* local_gates, double* local_mats, int64_t cap_gates,
                        int64_t* n_local_gates, int32_t* final_perm) {
  using namespace sv;
  if (world < 1 || (world & (world - 1)) || !n_steps || !n_local_gates) return fail(SV_E_ARG, "bad arguments");
  const int g = __builtin_ctz((unsigned)world);
  if (n_qubits - g < 1 || rank < 0 || rank >= world) return fail(SV_E_ARG, "bad sizes");
  sv_state_s tmp;
  tmp.n = tmp.n_local = n_qubits;
  std::vector<BoundGate> bg;
  std::string err;
  bg.resize((size_t)n_gates);
  for (int64_t i = 0; i < n_gates; ++i) {
    int rc = bind_gate(n_qubits, &gates[i], params, n_params, false, &bg[(size_t)i], &err);
    if (rc) return fail(rc, "gate " + std::to_string(i) + ": " + err);
  }
  const int nl = n_qubits - g;
  std::vector<int> perm((size_t)n_qubits);
  for (int q = 0; q < n_qubits; ++q) perm[(size_t)q] = q;
  std::vector<Step> st = schedule(bg, perm, nl);
  *n_steps = (int64_t)st.size();
  int64_t ng = 0;
  for (size_t i = 0; i < st.size(); ++i) {
    std::vector<BoundGate> loc;
    if (st[i].kind == 0) loc = localize(st[i].gates, nl, (uint64_t)rank);
    if ((int64_t)i < cap_steps) {
      steps[i].kind = st[i].kind;
      steps[i].gpos = st[i].gpos;
      steps[i].lpos = st[i].lpos;
      steps[i].n_gates = (int32_t)loc.size();
    }
    for (const BoundGate& b : loc) {
      if (ng < cap_gates) {
        sv_gate& o = local_gates[ng];
        double* m = local_mats + 32 * ng;
        std::memset(m, 0, 32 * sizeof(double));
        o.controls = b.controls;
        o.param = -1;
        o.coeff = 1.0;
        o.offset = 0.0;
        o.mat = m;
        o.targets[0] = b.t0;
        o.targets[1] = b.t1;
        auto put = [&](int e, Cx c) { m[2 * e] = c.re; m[2 * e + 1] = c.im; };
        switch (b.cls) {
          case GC_XLIKE: o.kind = SV_MAT1; put(1, b.m[0]); put(2, b.m[1]); break;
          case GC_ZLIKE: o.kind = SV_MAT1; put(0, b.m[0]); put(3, b.m[1]); break;
          case GC_GEN1: o.kind = SV_MAT1; for (int e = 0; e < 4; ++e) put(e, b.m[e]); break;
          case GC_GEN2: o.kind = SV_MAT2; for (int e = 0; e < 16; ++e) put(e, b.m[e]); break;
          case GC_DIAG2: o.kind = SV_MAT2; for (int j = 0; j < 4; ++j) put(j * 5, b.m[j]); break;
          case GC_SWAP: o.kind = SV_MAT2; put(0, Cx{1, 0}); put(6, Cx{1, 0}); put(9, Cx{1, 0}); put(15, Cx{1, 0}); break;
        }
      }
      ++ng;
    }
  }
  *n_local_gates = ng;
  if (final_perm)
    for (int q = 0; q < n_qubits; ++q) final_perm[q] = perm[(size_t)q];
  return SV_OK;
}

sv_status sv_create_virtual_shards(int32_t n_qubits, int32_t world, sv_handle* out) {
  int rc = sv::create_common(n_qubits, world, true, 0, out);
  if (rc) return rc;
  rc = sv::shard_reset(*out);
  if (rc) { sv_destroy(*out); *out = nullptr; }
  return rc;
}

sv_status sv_create_sharded(int32_t n_qubits, int32_t rank, int32_t world, const void* nccl_id, sv_handle* out) {
  if (!nccl_id) return sv::fail(SV_E_ARG, "null nccl id");
  if (world == 1) {
    int rc = sv_create(n_qubits, out);
    return rc;
  }
  int rc = sv::create_common(n_qubits, world, false, rank, out);
  if (rc) return rc;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&(*out)->shard->comm, world, id, rank);
  if (r != ncclSuccess) {
    sv_destroy(*out);
    *out = nullptr;
    return sv::fail(SV_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  rc = sv::shard_reset(*out);
  if (rc) { sv_destroy(*out); *out = nullptr; }
  return rc;
}

}  // extern "C"
