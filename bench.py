"""bench.py — throughput of the B200 state-vector hot path (driver contract).

Default (N=1): BASELINE.json configs[3] "C4", the config the metric is quoted on: a 30-qubit
random circuit (depth 40: Haar 1q matrix on every qubit + CZ bricks, 1780 gates, seed 3040) on a
complex128 state (16 GiB), plus the 50-term JW-shaped Hamiltonian (seed 3030).
  step  = sv_reset + sv_apply_circuit(C4) + sv_expectation(H)   (all inputs resident; 16 GiB > L2,
          so no L2 flush is needed between steps)
  value = C4 gates / step time  (gates/s, higher is better)
Extra keys: effective state-vector GB/s, achieved HBM GB/s of the plan and its fraction of the
measured peak, the adjoint-gradient throughput at 30q (C4g: 30q HEA, 2 layers, 120 params),
roofline of the dominant kernel (the fused forward pass), the CPU oracle baseline, e2e through the
C-ABI with host buffers, clocks during the timed region.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed on the host cores on a
bounded sample of the same workload (the tier's reference arm).

Multi-GPU (N>1): BASELINE.json configs[4] "C5", a 34-qubit random circuit (depth 40, seed 3440)
+ 50-term JW <H>, sharded over the N GPUs by its top log2(N) qubits (pipelined NCCL half-shard
exchanges over NVLink, chunked cross-shard Pauli streams, one all-reduce). The total problem is
fixed (strong scaling); value = 30q-equivalent gates/s (gates x 2^(n-30) / s, equal to gates/s at
30 qubits) so the per-GPU rate compares with N=1's C4. `python bench.py --gpus N` without a torchrun
environment re-launches itself under torch.distributed.run with N ranks and fails loudly when the
box has fewer than N GPUs. `--virtual-shards P` runs the sharded executor with P shards on one GPU
(weak scaling, 30 + log2 P qubits). See DESIGN.md §7.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_PATH = os.path.join(ROOT, "profiles", "fp64_peak.json")  # tools/measure_fp64_peak.py (committed)
NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md; 900 GB/s nominal)
TF32_SPLIT_PEAK_TFLOPS = 277.3 / 3  # measured mma.sync TF32 peak / 3 products (complex64 dense stages)
# dram__bytes_read.sum + dram__bytes_write.sum per forward-pass launch from the committed ncu
# --set full capture (profiles/r02_ncu_pass30_full.txt); None until captured.
TRAFFIC_PER_LAUNCH = {"C4": (17.184045 + 17.121930) * 1e9}  # profiles/r02_ncu_pass30_full.txt (k_pass_dense)
TRAFFIC_PER_LAUNCH_C64 = (8.608543 + 8.541884) * 1e9  # profiles/r02_ncu_c64_pass30_full.txt (k_pass_c64)
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback (used only without MEASURED_PEAKS.json)


def _fp64_peak():
    """The measured FP64 peak (DMMA / DFMA / mixed, best) with its clock record."""
    with open(FP64_PEAK_PATH) as f:
        d = json.load(f)
    return float(d["peak_tflops"]), (f"measured {d['when']} on this pool's B200 at {d['sm_mhz_median_under_load']:.0f} MHz "
                                     f"({d['source']}: DMMA {d['dmma_tflops']}, DFMA {d['dfma_tflops']}, mixed "
                                     f"{d['mixed_tflops']} TF); profiles/fp64_peak.json")


def _peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML from a thread (first sample
    at entry, then every 20 ms, and one more at exit, so even a millisecond region has a reading);
    `nvidia-smi -lms` as the fallback when pynvml is missing."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.rows = []
        self.out = ""

    def _bus_id(self):
        """PCI bus id of CUDA device `index` (NVML enumerates every GPU of the host, whatever
        CUDA_VISIBLE_DEVICES selects)."""
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            return f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        except Exception:
            return None

    def _nvml_sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.rows.append((float(sm), float(mx), r))

    def __enter__(self):
        import threading
        self.rows = []
        self.nvml = False
        try:
            import pynvml
            pynvml.nvmlInit()
            bus = self._bus_id()
            self.h = (pynvml.nvmlDeviceGetHandleByPciBusId(bus) if bus else
                      pynvml.nvmlDeviceGetHandleByIndex(self.index))
            self._nvml_sample()  # the first reading, taken as the region starts
            self.nvml = True
            self.stop = threading.Event()

            def loop():
                while not self.stop.wait(0.02):
                    try:
                        self._nvml_sample()
                    except Exception:
                        return
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = False
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self._bus_id() or str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.nvml:
            try:
                self._nvml_sample()  # and one as it ends (before the caller's next work)
            except Exception:
                pass
            self.stop.set()
            self.thread.join(timeout=1)
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.rows:
            reasons = sorted({name for (_, _, r) in self.rows for name, bit in self.REASONS if r & bit})
            return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                    "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons, "samples": len(self.rows),
                    "source": "nvml"}
        rows = []
        for line in (self.out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[4], parts[5], parts[6], parts[7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[2 + j].lower().startswith("active")})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


def _ham_terms(ham):
    return len(ham)


def cpu_oracle_sample(config: str, seconds_target: float = 20.0):
    """The oracle as it stands, timed on the host cores on a bounded sample of the workload:
    the first G gates of the config's circuit at full width (n=30 for C4), G chosen to take about
    `seconds_target` seconds. Returns (gates/s, cores, sample description)."""
    import oracle
    w = W.config(config)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    psi = oracle.zero_state(w.n)
    # the first gate touches the pages (untimed); then gates one by one until ~seconds_target
    psi = oracle.apply_circuit(w.n, w.gates[:1], w.params, psi)
    G = 0
    t0 = time.perf_counter()
    while G < len(w.gates) - 1 and time.perf_counter() - t0 < seconds_target:
        psi = oracle.apply_circuit(w.n, w.gates[1 + G:2 + G], w.params, psi)
        G += 1
    dt = time.perf_counter() - t0
    return G / dt, cores, f"oracle.apply_circuit on gates 1..{G} of {config} at n={w.n} ({dt:.1f} s)"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    w = W.config(args.config)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    # each step: a bounded sample (the first G gates of the circuit at full width)
    psi = oracle.zero_state(w.n)
    t0 = time.perf_counter()
    psi = oracle.apply_circuit(w.n, w.gates[:1], w.params, psi)
    t1 = time.perf_counter() - t0
    G = int(max(1, min(len(w.gates), 20.0 / max(1, args.steps + args.warmup) / max(t1, 1e-3))))
    for _ in range(args.warmup):
        oracle.apply_circuit(w.n, w.gates[:G], w.params, psi)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.apply_circuit(w.n, w.gates[:G], w.params, psi)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = G / (ms / 1e3)
    sample = f"first {G} gates of {args.config} at n={w.n} per step (no <H>)"
    # a sampled workload, not the full C4 step: its own metric string (the units agree, so the ratio
    # of the two arms is gates/s over gates/s, but it is not a same-config comparison)
    metric = f"gates/sec (oracle sample of the {args.config} circuit evolution; first {G} gates per step, no <H>)"
    line = {"metric": metric, "value": value, "unit": "gates/s", "impl": "reference", "same_config": False,
            "sample": sample,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic", "config": {"workload": args.config, "n_qubits": w.n, "gates": len(w.gates),
                                            "sample_gates": G},
            "cpu_baseline": {"value": value, "unit": "gates/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# the headline metric string (BASELINE.json)
C4_METRIC = "gates/sec (30q random circuit C4 evolution + 50-term <H>), SV GB/s, grad evals/sec"

GRAD_CONFIGS = ("C1", "C2", "C3", "C3dc", "C4g")


def cpu_grad_sample(config: str, threads: int, budget_s: float = 8.0):
    """The oracle's adjoint gradient (or_adjoint_grad, as it stands) timed on the host cores with
    `threads` OpenMP threads, in a subprocess (the thread count is fixed per process), on a bounded
    sample: the full task when it fits the budget, else the first G gates of the circuit with the
    first T Hamiltonian terms (G doubled until one evaluation takes about budget_s / 4; T = all terms
    up to 20 qubits, else the single lightest term — the oracle applies every Pauli string qubit by
    qubit, which alone is minutes per term at 30 qubits). Returns a cpu_baseline dict (value = evaluations per second of
    the sample, which is named)."""
    code = f"""
import json, sys, time
sys.path.insert(0, {ROOT!r})
import oracle, workloads as W
w = W.config({config!r})
if w.n > 20:  # one lightest term (fewest non-identity qubits: fewest oracle passes)
    w.ham = sorted(w.ham, key=lambda t: len(t[1]))[:1]
T = len(w.ham)
G = len(w.gates) if w.n <= 16 else (8 if w.n <= 24 else 2)
while True:
    t0 = time.perf_counter(); oracle.adjoint_grad(w.n, w.gates[:G], w.params, w.ham[:T]); dt = time.perf_counter() - t0
    if G >= len(w.gates) or dt > {budget_s} / 4: break
    G = min(len(w.gates), 2 * G)
reps = max(1, int({budget_s} / max(dt, 1e-6) / 2))
t0 = time.perf_counter()
for _ in range(reps): oracle.adjoint_grad(w.n, w.gates[:G], w.params, w.ham[:T])
dt = (time.perf_counter() - t0) / reps
print(json.dumps({{"G": G, "total": len(w.gates), "T": T, "terms": len(W.config({config!r}).ham), "n": w.n, "s": dt}}))
"""
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
        full = d["G"] == d["total"] and d["T"] == d["terms"]
        return {"value": 1.0 / d["s"], "unit": "grad evals/s" + ("" if full else " (sample)"), "cores": threads,
                "kind": "oracle", "sample": (f"oracle.adjoint_grad on the full {config} task" if full else
                                             f"oracle.adjoint_grad on the first {d['G']} of {d['total']} gates and "
                                             f"{d['T']} of {d['terms']} terms of {config} (n={d['n']}), "
                                             f"{d['s']:.2f} s per evaluation")}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "grad evals/s", "cores": threads, "kind": "oracle", "sample": f"failed: {e}"}


def run_grad_config(args, P, torch):
    """Gradient-evaluation throughput of BASELINE configs C1-C3 (and C4g): value = expectation +
    full adjoint gradient evaluations per second through the C ABI (host call included). C1 runs in
    batch mode (one launch of 4096 parameter rows: NEXT-1)."""
    w = W.config(args.config)
    ga, pa = P.GateArray(w.gates), P.PauliArray(w.ham)
    sv = P.StateVector(w.n)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    P.sv_set_stream(sv.h, stream.cuda_stream)
    rows = None
    if args.config == "C1":
        rows = np.random.default_rng(1).uniform(-np.pi, np.pi, (4096, len(w.params)))

    # an optimiser loop: the parameters change every step (as in VQE / QAOA training), so every
    # evaluation binds and plans its circuit afresh (no plan-cache hits); C1's rows are new too
    prng = np.random.default_rng(7)

    def step(i, moving=True):
        if rows is not None:
            r = rows + (1e-3 * i if moving else 0.0)
            return P.sv_expectation_with_grad_batch(sv.h, ga, r, pa)
        p = w.params + (1e-3 * prng.standard_normal(len(w.params)) if moving else 0.0)
        return P.sv_expectation_with_grad(sv.h, ga, p, pa)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    P.sv_reset_stats(sv.h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        t0 = time.perf_counter()
        e0.record(stream)
        for i in range(args.steps):
            out = step(args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize()
        dt_wall = (time.perf_counter() - t0) / args.steps
    # value: device time on the handle's stream (CUDA events); e2e: host wall clock around the same
    # public calls (each one uploads its parameters and reads E and the gradient back, synchronously)
    dt = e0.elapsed_time(e1) / 1e3 / args.steps
    st = P.sv_get_stats(sv.h)  # the timed (moving-parameter) steps only
    # the same evaluation with unchanged parameters (plans reused from the handle's cache)
    step(0, moving=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step(0, moving=False)
    torch.cuda.synchronize()
    dt_fixed = (time.perf_counter() - t0) / args.steps
    evals = rows.shape[0] if rows is not None else 1
    line = {"metric": "expectation + adjoint-gradient evaluations per second", "value": evals / dt,
            "unit": "grad evals/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic", "config": {"workload": args.config, "n_qubits": w.n, "gates": len(w.gates),
                                            "params": len(w.params), "ham_terms": len(w.ham),
                                            "rows_per_step": evals,
                                            "param_updates": "parameters changed every step (optimiser loop)"},
            "fixed_params_value": evals / dt_fixed,
            "launches_per_eval": int(st["kernel_launches"]) / max(1, args.steps),
            "gpu_launches": int(st["kernel_launches"]), "clocks": clk.summary(),
            "e2e": {"value": evals / dt_wall, "unit": "grad evals/s",
                    "h2d_bytes_per_step": int(ga.nbytes + pa.nbytes + (rows.nbytes if rows is not None else w.params.nbytes)),
                    "d2h_bytes_per_step": int(8 * evals * (1 + len(w.params)))}}
    if not args.no_cpu_baseline:
        nproc = os.cpu_count() or 1
        line["cpu_baseline"] = cpu_grad_sample(args.config, nproc)
        line["cpu_baseline_1thread"] = cpu_grad_sample(args.config, 1)
    print(json.dumps(line), flush=True)
    sv.close()


def run_density_config(args, P, torch):
    """NEXT-4 density matrix: gates/s of rho <- U rho U^dagger for C4's generator at n = DM<n>
    qubits (a 2n-qubit vector), plus tr(rho H) with a 50-term JW H."""
    n = int(args.config[2:] or 14)
    w = W.random_circuit(n, 40, seed=3040)
    ham = W.jw_hamiltonian(n, 50, 3030)
    ga, pa = P.GateArray(w.gates), P.PauliArray(ham)
    dm = P.DensityMatrix(n)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    P.sv_set_stream(dm.h, stream.cuda_stream)

    def step():
        dm.reset()
        P.sv_apply_circuit(dm.h, ga, w.params)
        return P.sv_expectation(dm.h, pa)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    P.sv_reset_stats(dm.h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            E = step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_wall = 1e3 * (time.perf_counter() - t0) / args.steps
    ms = e0.elapsed_time(e1) / args.steps
    st = P.sv_get_stats(dm.h)
    line = {"metric": "density-matrix gates/sec (rho <- U rho U^dagger) + tr(rho H)", "value": len(w.gates) / (ms / 1e3),
            "unit": "gates/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic", "config": {"workload": f"DM{n}: {n}-qubit density matrix (a {2 * n}-qubit vector), "
                                                      "C4 generator depth 40, 50-term JW H", "n_qubits": n,
                                            "gates": len(w.gates)},
            "E": E, "gpu_launches": int(st["kernel_launches"]), "clocks": clk.summary(),
            "e2e": {"value": len(w.gates) / (ms_wall / 1e3), "unit": "gates/s", "h2d_bytes_per_step": int(ga.nbytes + pa.nbytes),
                    "d2h_bytes_per_step": 8}}
    print(json.dumps(line), flush=True)
    dm.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--virtual-shards", type=int, default=0,
                    help="run the sharded path with P virtual shards on one GPU (tests the N>1 executor)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-grad", action="store_true")
    ap.add_argument("--precision", default="c128", choices=["c128", "c64"],
                    help="c64: NEXT-3 complex64 state (single GPU; the gradient leg stays complex128)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:
        # one process per GPU: re-launch under torch.distributed.run with --gpus ranks
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py --gpus {args.gpus}: this box exposes {have} GPU(s); refusing to report a "
                  f"{have}-GPU number as {args.gpus}", file=sys.stderr, flush=True)
            sys.exit(2)
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world_env is not None and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}")

    import torch
    import paper_2406_17248_b200 as P
    import paper_2406_17248_b200.dist as PD

    if args.config in GRAD_CONFIGS:
        return run_grad_config(args, P, torch)
    if args.config.startswith("DM"):
        return run_density_config(args, P, torch)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    shards = world if world > 1 else max(1, args.virtual_shards)
    if world > 1 or args.config == "C5":
        # BASELINE configs[4]: 34 qubits, 256 GiB total (128 / 64 / 32 GiB per GPU at N = 2 / 4 / 8)
        w = W.config("C5")
        n = w.n
        workload = f"C5: {n}q random circuit depth 40 (Haar 1q + CZ bricks, seed 3440) + 50-term JW H, sharded over {shards} GPUs"
    elif shards > 1:
        # virtual shards on one GPU (weak scaling): C4's generator at n = 30 + log2(P) qubits
        g = shards.bit_length() - 1
        n = 30 + g
        w = W.random_circuit(n, 40, seed=3440)
        w.ham = W.jw_hamiltonian(n, 50, 3440)
        workload = f"C5w: {n}q random circuit depth 40 (Haar 1q + CZ bricks) + 50-term JW H, {shards} virtual shards on 1 GPU"
    else:
        w = W.config(args.config)
        n = w.n
        workload = args.config
    ga = P.GateArray(w.gates)
    pa = P.PauliArray(w.ham)
    if world > 1:
        sv = PD.create_sharded(n)
    elif shards > 1:
        sv = P.StateVector(n, handle=P.sv_create_virtual_shards(n, shards))
    elif args.precision == "c64":
        sv = P.StateVectorC64(n)
    else:
        sv = P.StateVector(n)
    stream = torch.cuda.Stream()  # a real stream object: its handle is passed to the library
    torch.cuda.set_stream(stream)
    P.sv_set_stream(sv.h, stream.cuda_stream)

    def step():
        sv.reset()
        P.sv_apply_circuit(sv.h, ga, w.params)
        return P.sv_expectation(sv.h, pa)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    P.sv_reset_stats(sv.h)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evc0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    evc1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        E = None
        for i in range(args.steps):
            sv.reset()
            evc0[i].record(stream)
            P.sv_apply_circuit(sv.h, ga, w.params)
            evc1[i].record(stream)
            E = P.sv_expectation(sv.h, pa)
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    circ_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(evc0, evc1)]))
    st = P.sv_get_stats(sv.h)
    if dist:
        t = torch.tensor([ms_total, circ_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, circ_ms = float(t[0].item()), float(t[1].item())
    ms_step = ms_total / args.steps
    n_gates = len(w.gates)
    amps_total = float(1 << n)
    # 30q-equivalent gates/s: gates x (state size / 2^30) per second (= plain gates/s at N = 1)
    value = n_gates * (amps_total / float(1 << 30)) / (ms_step / 1e3)
    hbm_peak, peak_src = _peaks()
    fp64_peak, fp64_src = _fp64_peak()
    amps = amps_total / shards  # per shard
    passes_total = st["gate_passes"] / args.steps  # every shard this handle holds
    passes = passes_total / (1 if world > 1 else shards)  # per shard
    x_ms = st["exchange_ms"] / args.steps  # exchange device time inside the timed steps
    x_bytes = st["exchange_bytes"] / args.steps
    pass_ms = (circ_ms - (x_ms if shards > 1 else 0.0)) / max(passes_total, 1)  # one shard's pass on this GPU
    pass_bytes = (16.0 if args.precision == "c64" else 32.0) * amps
    achieved = pass_bytes / (pass_ms / 1e3) / 1e9
    plan_bytes = st["algorithmic_bytes"] / args.steps / (1 if world > 1 else shards)
    eff_bytes = sum((16.0 if args.precision == "c64" else 32.0) * amps_total / (1 << len(g.controls)) for g in w.gates)
    roof = None
    if shards == 1:
        plan = P.sv_plan_info(n, ga, w.params)
        # FP64 work of the executed plan: 2 flops per FMA (dense stages: 48 per amplitude, three
        # real products per complex entry) + the Gauss sums (3 DADDs per amplitude and dense stage)
        c64 = args.precision == "c64"
        # (complex64: the TF32 dense stages run the four-product form, 64 FMAs per amplitude)
        pass_flops = [(2.0 * (p["fma_per_amp"] + 16 * p["n_dense"]) if c64 else
                       2.0 * p["fma_per_amp"] + p["add_per_amp"]) * amps for p in plan]
        fp64_flops = sum(pass_flops)
        # complex64: the dense stages run TF32 MMAs with a 3-term split, so the peak for the
        # algorithmic (complex matrix-vector) flops is the measured TF32 mma.sync rate / 3
        peak = TF32_SPLIT_PEAK_TFLOPS if c64 else fp64_peak
        # t_roof = sum over passes of max(bytes / BW, FP64 flops / rate)
        bw = hbm_peak * 1e9
        t_roof = sum(max(pass_bytes / bw, f / (peak * 1e12)) for f in pass_flops)
        roof = {
            "bound": "tensor",
            "kernel": ("k_pass_c64 (complex64 tiles; dense stages on TF32 tensor cores, 3-term split; register stages)"
                       if c64 else
                       "k_pass_dense / k_pass_reg<3,false> (fused forward tile passes: FP64 DMMA dense stages + register stages)"),
            "achieved": fp64_flops / passes / (pass_ms / 1e3) / 1e12, "peak": peak,
            "peak_source": ("measured legacy mma.sync TF32 277 TF (tools/microbench/mma_legacy.cu, "
                            "profiles/r01_mma_legacy_microbench.jsonl) / 3 for the 3-term split" if c64 else fp64_src),
            "unit": "TFLOP/s", "frac": fp64_flops / passes / (pass_ms / 1e3) / 1e12 / peak,
            "traffic": TRAFFIC_PER_LAUNCH.get(args.config) if args.precision == "c128" else TRAFFIC_PER_LAUNCH_C64,
            "algorithmic_flops_per_launch": fp64_flops / passes, "avg_launch_ms": pass_ms,
            "t_roof_ms": 1e3 * t_roof, "t_roof_frac": 1e3 * t_roof / circ_ms,
            "hbm": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "peak_source": peak_src,
                    "unit": "GB/s", "frac": achieved / hbm_peak, "algorithmic_bytes_per_launch": pass_bytes}}
    else:
        roof = {"bound": "hbm", "kernel": "k_pass_dense / k_pass_reg<3,false> (forward passes on each shard)",
                "achieved": achieved, "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": None, "algorithmic_bytes_per_launch": pass_bytes,
                "avg_launch_ms": pass_ms, "passes_per_shard": passes,
                "exchange": {"swaps_per_step": st["exchanges"] / args.steps, "bytes_per_step": x_bytes,
                             "ms_per_step": x_ms, "achieved_gbs": (x_bytes / (x_ms / 1e3) / 1e9) if x_ms > 0 else None,
                             "peak_gbs": NVLINK_PEER_GBS if world > 1 else None,
                             "peak_source": ("measured peer copy per direction (B200_PROFILING.md; 900 nominal)"
                                             if world > 1 else "virtual shards: device copies on one GPU (no NVLink)"),
                             "frac": ((x_bytes / (x_ms / 1e3) / 1e9) / NVLINK_PEER_GBS) if (world > 1 and x_ms > 0) else None}}
    clocks = clk.summary()

    # e2e: the same step through the public C ABI with host inputs (gate / term arrays marshalled
    # from host memory every step; plan upload H2D and the expectation D2H inside the timed region)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ga_h = P.GateArray(w.gates)
        pa_h = P.PauliArray(w.ham)
        sv.reset()
        P.sv_apply_circuit(sv.h, ga_h, w.params)
        P.sv_expectation(sv.h, pa_h)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = ga.nbytes + pa.nbytes + w.params.nbytes
    e2e = {"value": n_gates * (amps_total / float(1 << 30)) / e2e_s,
           "unit": "gates/s" if n == 30 else "gates/s (30q-equivalent)",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8}

    grad = None
    if not args.no_grad and args.config == "C4" and shards == 1:
        wg = W.config("C4g")
        gag, pag = P.GateArray(wg.gates), P.PauliArray(wg.ham)
        sv.reset()
        P.sv_expectation_with_grad(sv.h, gag, wg.params, pag)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 2
        prng = np.random.default_rng(11)
        for _ in range(reps):  # parameters change every evaluation (optimiser loop)
            Eg, gg = P.sv_expectation_with_grad(sv.h, gag, wg.params + 1e-3 * prng.standard_normal(len(wg.params)), pag)
        dtg = (time.perf_counter() - t0) / reps
        grad = {"workload": "C4g: 30q HEA 2 layers RY/RZ + CNOT ladder, 120 params, 50-term JW H",
                "grad_evals_per_s": 1.0 / dtg, "ms_per_eval": 1e3 * dtg, "E": Eg,
                "param_updates": "parameters changed every evaluation"}

    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1 and shards == 1:
        try:
            v, cores, sample = cpu_oracle_sample(args.config)
            cpu = {"value": v, "unit": "gates/s", "cores": cores, "kind": "oracle", "sample": sample}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "gates/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": C4_METRIC,
            "value": value, "unit": "gates/s" if n == 30 else "gates/s (30q-equivalent: gates x 2^(n-30))",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if (world > 1 or args.config == "C5") else "weak", "vs_baseline": None,
            "dtype": "c64 (f32 dense stages, f64 register ops)" if args.precision == "c64" else "c128 (f64)",
            "data": "synthetic",
            "config": {"workload": workload, "n_qubits": n, "gates": n_gates, "ham_terms": len(w.ham),
                       "state_bytes": int((8 if args.precision == "c64" else 16) * amps_total), "shards": shards,
                       "l2": f"inputs ({int((8 if args.precision == 'c64' else 16) * amps) >> 30} GiB per shard) larger than L2; no flush",
                       "parallelism": (f"state sharded over {world} GPUs (NCCL)" if world > 1 else
                                       f"{shards} virtual shards on 1 GPU" if shards > 1 else "1 GPU")},
            "circuit_ms": circ_ms, "passes_per_circuit": passes, "E": E,
            "sv_effective_gbs": eff_bytes / (circ_ms / 1e3) / 1e9,
            "plan_hbm_gbs": plan_bytes / (ms_step / 1e3) / 1e9,
            "plan_hbm_frac": plan_bytes / (ms_step / 1e3) / 1e9 / hbm_peak,
            "roofline": roof,
            "grad": grad,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(st["kernel_launches"]),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    sv.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
