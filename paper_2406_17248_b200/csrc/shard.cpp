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
  DevBuf scalar;                // all-reduce scratch
  // pipelined exchanges: two bounce buffers per direction (this side; the partner side only for the
  // virtual-shard emulation of the NCCL transport), a transfer stream, per-buffer events
  DevBuf sendb[2], recvb[2], psend[2], precv[2];
  cudaStream_t xstream = nullptr;
  cudaEvent_t ev_pack[2] = {nullptr, nullptr}, ev_comm[2] = {nullptr, nullptr}, ev_unpack[2] = {nullptr, nullptr};
  DevBuf eacc;                  // sharded expectation: one device double per evaluation unit
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

// Exchange timing: events around each exchange on the handle's stream (summed at sv_get_stats).
struct XTimer {
  sv_state_s* h;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  explicit XTimer(sv_state_s* hh) : h(hh) {
    if (cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess) cudaEventRecord(e0, h->stream);
    else { if (e0) cudaEventDestroy(e0); e0 = e1 = nullptr; }
  }
  ~XTimer() {
    if (!e0) return;
    cudaEventRecord(e1, h->stream);
    h->xev.push_back({e0, e1});
  }
};

int ensure_xstream(sv_state_s* h) {
  ShardState& S = *h->shard;
  if (S.xstream) return SV_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&S.xstream, cudaStreamNonBlocking);
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = cudaEventCreateWithFlags(&S.ev_pack[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&S.ev_comm[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&S.ev_unpack[b], cudaEventDisableTiming);
  }
  return e == cudaSuccess ? SV_OK : cuda_fail(h, e, "exchange stream");
}

// One side of a pairwise half-shard exchange: the shard, the half it sends (local bit L == hsend;
// the received half lands in the same positions) and its two send / receive bounce buffers.
struct XSide {
  double* shard;
  int hsend;
  double* sendb[2];
  double* recvb[2];
};

// Pipelined chunked exchange (SURVEY §8(e) "pairwise half-shard exchange ... chunked through a
// bounce buffer"): chunk i is packed on the handle's stream, moved by `comm(b, cnt)` on the transfer
// stream (NCCL grouped send/recv, or device copies between virtual shards), and unpacked on the
// handle's stream; with two buffers per direction pack(i+1) and unpack(i-1) run while chunk i is in
// flight. Events order buffer reuse: comm(i) waits pack(i) and unpack(i-2); unpack(i) waits comm(i).
template <class Comm>
int exchange_pipelined(sv_state_s* h, XSide* sides, int nsides, int L, int64_t half, int64_t chunk, Comm comm) {
  ShardState& S = *h->shard;
  int rc = ensure_xstream(h);
  if (rc) return rc;
  const int64_t nch = (half + chunk - 1) / chunk;
  cudaError_t e = cudaSuccess;
  for (int64_t i = 0; i <= nch && e == cudaSuccess; ++i) {
    if (i < nch) {
      const int b = (int)(i & 1);
      const int64_t off = i * chunk, cnt = std::min(chunk, half - off);
      // pack(i) reuses sendb[b] after comm(i-2): ordered, unpack(i-2) (earlier on this stream) waited for it
      for (int sd = 0; sd < nsides && e == cudaSuccess; ++sd)
        e = launch_pack_half(sides[sd].shard, sides[sd].sendb[b], L, sides[sd].hsend, off, cnt, true, h->stream);
      if (e == cudaSuccess) e = cudaEventRecord(S.ev_pack[b], h->stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(S.xstream, S.ev_pack[b], 0);
      if (e == cudaSuccess && i >= 2) e = cudaStreamWaitEvent(S.xstream, S.ev_unpack[b], 0);  // recvb[b] free
      if (e == cudaSuccess) {
        const int crc = comm(b, cnt);
        if (crc) return crc;
      }
      if (e == cudaSuccess) e = cudaEventRecord(S.ev_comm[b], S.xstream);
      h->stats.kernel_launches += nsides;
    }
    if (i >= 1 && e == cudaSuccess) {
      const int64_t j = i - 1;
      const int b = (int)(j & 1);
      const int64_t off = j * chunk, cnt = std::min(chunk, half - off);
      e = cudaStreamWaitEvent(h->stream, S.ev_comm[b], 0);
      for (int sd = 0; sd < nsides && e == cudaSuccess; ++sd)
        e = launch_pack_half(sides[sd].shard, sides[sd].recvb[b], L, sides[sd].hsend, off, cnt, false, h->stream);
      if (e == cudaSuccess) e = cudaEventRecord(S.ev_unpack[b], h->stream);
      h->stats.kernel_launches += nsides;
    }
  }
  if (e != cudaSuccess) return cuda_fail(h, e, "pipelined exchange");
  return SV_OK;
}

// Swap physical positions G (global) and L (local) of the vectors `vecs` (per held shard).
int swap_qubits(sv_state_s* h, const std::vector<std::vector<double*>>& vecs, int G, int L) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  const int j = G - nl;
  h->stats.exchanges += 1;
  NvtxRange nvtx("qubit swap exchange");
  XTimer timer(h);
  const int64_t half = int64_t(1) << (nl - 1);
  // SV_VIRTUAL_BOUNCE=<chunk amplitudes>: virtual shards exchange through the NCCL transport's
  // pipelined pack / bounce-buffer / unpack sequence, with device copies on the transfer stream in
  // place of ncclSend / ncclRecv, so the tests exercise that code (and its event ordering) on one GPU.
  const char* bounce_env = std::getenv("SV_VIRTUAL_BOUNCE");
  const int64_t bounce_chunk = bounce_env ? std::max<int64_t>(1, std::atoll(bounce_env)) : 0;
  if (S.virt && bounce_chunk > 0) {
    const int64_t chunk = std::min(half, bounce_chunk);
    for (int b = 0; b < 2; ++b)
      if (!S.sendb[b].ensure((size_t)chunk * 16) || !S.recvb[b].ensure((size_t)chunk * 16) ||
          !S.psend[b].ensure((size_t)chunk * 16) || !S.precv[b].ensure((size_t)chunk * 16))
        return fail(SV_E_OOM, "bounce buffers");
    for (const auto& v : vecs) {
      for (size_t a = 0; a < S.ranks.size(); ++a) {
        const int r = S.ranks[a];
        if ((r >> j) & 1) continue;
        const size_t p = (size_t)(r | (1 << j));
        // r sends its half with bit L = 1, the partner p its half with bit L = 0
        XSide sides[2] = {{v[a], 1, {}, {}}, {v[p], 0, {}, {}}};
        for (int b = 0; b < 2; ++b) {
          sides[0].sendb[b] = static_cast<double*>(S.sendb[b].p);
          sides[0].recvb[b] = static_cast<double*>(S.recvb[b].p);
          sides[1].sendb[b] = static_cast<double*>(S.psend[b].p);
          sides[1].recvb[b] = static_cast<double*>(S.precv[b].p);
        }
        int rc = exchange_pipelined(h, sides, 2, L, half, chunk, [&](int b, int64_t cnt) {
          cudaError_t e = cudaMemcpyAsync(sides[1].recvb[b], sides[0].sendb[b], (size_t)cnt * 16, cudaMemcpyDeviceToDevice,
                                          S.xstream);
          if (e == cudaSuccess)
            e = cudaMemcpyAsync(sides[0].recvb[b], sides[1].sendb[b], (size_t)cnt * 16, cudaMemcpyDeviceToDevice, S.xstream);
          return e == cudaSuccess ? (int)SV_OK : cuda_fail(h, e, "bounce copy");
        });
        if (rc) return rc;
      }
    }
    h->stats.algorithmic_bytes += 32.0 * (double)(1ull << nl) * (double)S.ranks.size() * vecs.size() / 2.0;
    h->stats.exchange_bytes += 16.0 * (double)half * (double)S.ranks.size() * vecs.size();
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
    h->stats.exchange_bytes += 16.0 * (double)half * (double)S.ranks.size() * vecs.size();
    return SV_OK;
  }
  // NCCL: one held shard
  const int r = S.ranks[0];
  const int peer = r ^ (1 << j);
  const int h_send = ((r >> j) & 1) ? 0 : 1;  // send the half whose bit L differs from our bit j
  const int64_t chunk = std::min(half, kChunkAmps);
  for (int b = 0; b < 2; ++b)
    if (!S.sendb[b].ensure((size_t)chunk * 16) || !S.recvb[b].ensure((size_t)chunk * 16))
      return fail(SV_E_OOM, "bounce buffers");
  for (const auto& v : vecs) {
    XSide side{v[0], h_send, {static_cast<double*>(S.sendb[0].p), static_cast<double*>(S.sendb[1].p)},
               {static_cast<double*>(S.recvb[0].p), static_cast<double*>(S.recvb[1].p)}};
    int rc = exchange_pipelined(h, &side, 1, L, half, chunk, [&](int b, int64_t cnt) {
      ncclResult_t nr = ncclGroupStart();
      if (nr == ncclSuccess) nr = ncclSend(side.sendb[b], (size_t)cnt * 2, ncclDouble, peer, S.comm, S.xstream);
      if (nr == ncclSuccess) nr = ncclRecv(side.recvb[b], (size_t)cnt * 2, ncclDouble, peer, S.comm, S.xstream);
      ncclResult_t ne = ncclGroupEnd();
      if (nr != ncclSuccess) return nccl_fail(h, nr, "exchange");
      if (ne != ncclSuccess) return nccl_fail(h, ne, "exchange");
      return (int)SV_OK;
    });
    if (rc) return rc;
  }
  h->stats.algorithmic_bytes += 32.0 * (double)half * vecs.size();
  h->stats.exchange_bytes += 16.0 * (double)half * vecs.size();
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
  for (int b = 0; b < 2; ++b) {
    S.sendb[b].release();
    S.recvb[b].release();
    S.psend[b].release();
    S.precv[b].release();
    if (S.ev_pack[b]) cudaEventDestroy(S.ev_pack[b]);
    if (S.ev_comm[b]) cudaEventDestroy(S.ev_comm[b]);
    if (S.ev_unpack[b]) cudaEventDestroy(S.ev_unpack[b]);
  }
  if (S.xstream) cudaStreamDestroy(S.xstream);
  S.eacc.release();
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
    // chunked all-gather: a (P x chunk) device buffer instead of the whole 2^n state on every GPU
    // (256 GiB at 34 qubits); rank r's chunk lands at its shard's offset in physical order
    const uint64_t P = (uint64_t)h->world;
    const uint64_t CH = std::min<uint64_t>(NL, uint64_t(1) << 24);  // amplitudes per rank and chunk
    DevBuf all;
    if (!all.ensure(P * CH * 16)) return fail(SV_E_OOM, "gather buffer");
    for (uint64_t c0 = 0; c0 < NL; c0 += CH) {
      const uint64_t cn = std::min(CH, NL - c0);
      ncclResult_t r = ncclAllGather(static_cast<const double*>(S.bufs[0].p) + 2 * c0, all.p, cn * 2, ncclDouble,
                                     S.comm, h->stream);
      if (r != ncclSuccess) { all.release(); return nccl_fail(h, r, "allgather"); }
      for (uint64_t rk = 0; rk < P; ++rk) {
        cudaError_t e = cudaMemcpyAsync(phys.data() + 2 * (NL * rk + c0), static_cast<const double*>(all.p) + 2 * cn * rk,
                                        cn * 16, cudaMemcpyDeviceToHost, h->stream);
        if (e != cudaSuccess) { all.release(); return cuda_fail(h, e, "get_state"); }
      }
      // the next chunk's all-gather reuses the buffer: wait for the copies out of it
      cudaError_t e = cudaStreamSynchronize(h->stream);
      if (e != cudaSuccess) { all.release(); return cuda_fail(h, e, "get_state"); }
    }
    all.release();
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

// The listed logical groups in one shard's physical layout: x / z masks permuted to physical local
// positions, the rank-bit part of every Z factor folded into the coefficient (rsig: the rank bits the
// sign is read from — this shard's, or the partner's for a cross-shard group).
static PauliGroups shard_groups(const PauliGroups& G, const std::vector<int>& sel, const std::vector<int>& perm, int nl,
                                uint64_t rsig) {
  PauliGroups out;
  const uint64_t lmask = (1ull << nl) - 1;
  for (int gi : sel) {
    out.xs.push_back(permute_mask(G.xs[(size_t)gi], perm) & lmask);
    out.begin.push_back((int)out.z.size());
    for (int t = G.begin[(size_t)gi]; t < G.end[(size_t)gi]; ++t) {
      const uint64_t zp = permute_mask(G.z[(size_t)t], perm);
      const double sgn = (__builtin_popcountll((zp >> nl) & rsig) & 1) ? -1.0 : 1.0;
      out.z.push_back(zp & lmask);
      out.c.push_back(sgn * G.c[2 * (size_t)t]);
      out.c.push_back(sgn * G.c[2 * (size_t)t + 1]);
    }
    out.end.push_back((int)out.z.size());
  }
  return out;
}

// Sharded <H> (and lambda = H psi): groups whose x-mask is local in the current layout are evaluated
// together by the tiled multi-group passes on every held shard; a group with global x bits first
// swaps them with local qubits (the state's layout perm is updated; `swaps` records them); a group
// whose x-mask is wider than a shard streams the partner shard r ^ x_g in chunks (NCCL: 1 GiB
// chunks through a bounce buffer; virtual shards: read in place) — no whole-shard copy, so a
// 34-qubit state fits on 2 GPUs. Partials stay on the device until one read-back at the end.
// Returns the per-handle E (not yet all-reduced). lam (optional, per shard) receives H psi and E is
// then Re<psi|lam>.
static int sharded_groups(sv_state_s* h, const PauliGroups& G, std::vector<int>& perm,
                          const std::vector<std::vector<double*>>& swap_vecs, const std::vector<double*>& psi,
                          const std::vector<double*>& lam, double* out_e, std::vector<std::pair<int, int>>* swaps) {
  ShardState& S = *h->shard;
  const int nl = h->n_local;
  const uint64_t lmask = (1ull << nl) - 1;
  const bool grad = !lam.empty();
  const int grid_t = pauli_tile_grid(nl, pauli_k(nl)), grid_x = pauli_grid(nl);
  const int grid_max = std::max(grid_t, grid_x);
  const size_t max_units = (G.xs.size() + 2) * S.ranks.size() * 2 + 8;
  if (!h->d_partials.ensure((G.xs.size() + 2) * (size_t)grid_max * 8 + 64) || !S.eacc.ensure(max_units * 8))
    return fail(SV_E_OOM, "partials");
  double* dp = static_cast<double*>(h->d_partials.p);
  double* eacc = static_cast<double*>(S.eacc.p);
  size_t units = 0;
  cudaError_t e = cudaSuccess;
  if (grad)
    for (size_t a = 0; a < lam.size() && e == cudaSuccess; ++a) e = cudaMemsetAsync(lam[a], 0, size_t(16) << nl, h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "zero lambda");
  auto eval_local = [&](const std::vector<int>& sel) -> int {
    for (size_t a = 0; a < S.ranks.size(); ++a) {
      const PauliGroups Gs = shard_groups(G, sel, perm, nl, (uint64_t)S.ranks[a]);
      int ns = 0;
      int rc = run_groups(h, Gs, psi[a], grad ? lam[a] : nullptr, dp, grid_t, &ns, nullptr, true);
      if (rc) return rc;
      if (!grad && ns > 0) {
        if (units + (size_t)ns > max_units) return fail(SV_E_ARG, "internal: expectation units");
        cudaError_t er = launch_reduce_slots(dp, ns, grid_t, eacc + units, h->stream);
        if (er != cudaSuccess) return cuda_fail(h, er, "reduce");
        units += (size_t)ns;
        h->stats.kernel_launches += 1;
      }
    }
    return SV_OK;
  };
  // 1. every group that is local in the current layout: one tiled evaluation per shard
  std::vector<int> now, later;
  for (size_t gi = 0; gi < G.xs.size(); ++gi) ((permute_mask(G.xs[gi], perm) >> nl) ? later : now).push_back((int)gi);
  if (!now.empty()) {
    int rc = eval_local(now);
    if (rc) return rc;
  }
  // 2. groups with global x bits: swap them local where possible, else stream the partner shard
  for (int gi : later) {
    uint64_t xp = permute_mask(G.xs[(size_t)gi], perm);
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
      xp = permute_mask(G.xs[(size_t)gi], perm);
    }
    const uint64_t xg = xp >> nl;
    if (xg == 0) {
      int rc = eval_local({gi});
      if (rc) return rc;
      continue;
    }
    const uint64_t xl = xp & lmask;
    const int64_t NL = int64_t(1) << nl, chunk = std::min<int64_t>(NL, kChunkAmps);
    for (size_t a = 0; a < S.ranks.size(); ++a) {
      const uint64_t r = (uint64_t)S.ranks[a];
      const PauliGroups Gs = shard_groups(G, {gi}, perm, nl, r ^ xg);  // signs of the partner's rank bits
      const int nt = (int)Gs.z.size();
      const size_t zb = ((size_t)nt * 8 + 15) & ~size_t(15);
      if (!h->d_terms.ensure(zb + (size_t)nt * 16 + 16)) return fail(SV_E_OOM, "terms");
      if (h->terms_upload_done) {
        e = cudaEventSynchronize(h->terms_upload_done);  // the term buffer is free again
        if (e != cudaSuccess) return cuda_fail(h, e, "terms");
      }
      h->h_stage.assign(zb + (size_t)nt * 16, 0);
      std::memcpy(h->h_stage.data(), Gs.z.data(), (size_t)nt * 8);
      std::memcpy(h->h_stage.data() + zb, Gs.c.data(), (size_t)nt * 16);
      e = cudaMemcpyAsync(h->d_terms.p, h->h_stage.data(), h->h_stage.size(), cudaMemcpyHostToDevice, h->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // pageable staging
      if (e != cudaSuccess) return cuda_fail(h, e, "terms");
      const uint64_t* dz = static_cast<const uint64_t*>(h->d_terms.p);
      const double* dc = reinterpret_cast<const double*>(static_cast<const char*>(h->d_terms.p) + zb);
      if (!S.virt && (!S.recvb[0].ensure((size_t)chunk * 16))) return fail(SV_E_OOM, "partner chunk buffer");
      const int peer = (int)(r ^ xg);
      XTimer timer(h);
      for (int64_t off = 0; off < NL; off += chunk) {
        const double* partner = nullptr;
        if (S.virt) {
          partner = psi[(size_t)peer] + 2 * off;
        } else {
          // both ranks of the pair stream the same chunk index to each other (no pack: contiguous)
          ncclResult_t nr = ncclGroupStart();
          if (nr == ncclSuccess) nr = ncclSend(psi[a] + 2 * off, (size_t)chunk * 2, ncclDouble, peer, S.comm, h->stream);
          if (nr == ncclSuccess) nr = ncclRecv(S.recvb[0].p, (size_t)chunk * 2, ncclDouble, peer, S.comm, h->stream);
          ncclResult_t ne = ncclGroupEnd();
          if (nr != ncclSuccess) return nccl_fail(h, nr, "partner stream");
          if (ne != ncclSuccess) return nccl_fail(h, ne, "partner stream");
          partner = static_cast<const double*>(S.recvb[0].p);
          h->stats.exchange_bytes += 16.0 * (double)chunk;
        }
        e = launch_pauli_cross(psi[a], partner, grad ? lam[a] : nullptr, off, chunk, xl, dz, dc, nt, dp, grid_x,
                               off == 0, h->stream);
        if (e != cudaSuccess) return cuda_fail(h, e, "cross-shard Pauli chunk");
        h->stats.kernel_launches += 1;
      }
      h->stats.expectation_passes += 1;
      if (!grad) {
        e = launch_reduce_slots(dp, 1, grid_x, eacc + units, h->stream);
        if (e != cudaSuccess) return cuda_fail(h, e, "reduce");
        ++units;
        h->stats.kernel_launches += 1;
      }
    }
  }
  // 3. lambda mode: E = Re<psi|lambda> per shard (lambda holds every group's H psi)
  if (grad)
    for (size_t a = 0; a < S.ranks.size(); ++a) {
      e = launch_redot(psi[a], lam[a], int64_t(1) << nl, dp, grid_x, h->stream);
      if (e == cudaSuccess) e = launch_reduce_slots(dp, 1, grid_x, eacc + units, h->stream);
      if (e != cudaSuccess) return cuda_fail(h, e, "Re<psi|lambda>");
      ++units;
      h->stats.kernel_launches += 2;
    }
  // one read-back; fixed-order sum
  std::vector<double> ev(units);
  if (units) e = cudaMemcpyAsync(ev.data(), eacc, units * 8, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(h, e, "sharded expectation");
  double E = 0.0;
  for (double v : ev) E += v;
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
