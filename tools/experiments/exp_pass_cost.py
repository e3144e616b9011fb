"""Per-pass cost vs content at 30 qubits: a single pass (all gates on tile qubits 0..10) with
0..8 dense stages, one light op, and a torch copy of the state for the HBM floor."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = int(os.environ.get("EXP_N", "30"))
sv = P.StateVectorC64(n) if os.environ.get("EXP_C64") else P.StateVector(n)
stream = torch.cuda.Stream()
P.sv_set_stream(sv.h, stream.cuda_stream)
G = W.Gate


def t(gates, reps=5):
    ga = P.GateArray(gates)
    for _ in range(2):
        P.sv_apply_circuit(sv.h, ga, None)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        P.sv_apply_circuit(sv.h, ga, None)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


if os.environ.get("EXP_SKIP_FLOOR"):
    pass
x = torch.empty(2 << n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(2):
    y.copy_(x)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    y.copy_(x)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"torch copy 16 GiB: {ms:.2f} ms {2 * 16 * 2**n / ms / 1e6:.0f} GB/s", flush=True)
del x, y
rng = np.random.default_rng(1)
for name, gates in (("Z q0", [G("Z", (0,))]), ("X q0", [G("X", (0,))]), ("H q(n-1)", [G("H", (n - 1,))])):
    ms = t(gates)
    print(f"{name}: {ms:.2f} ms {2 * 16 * 2**n / ms / 1e6:.0f} GB/s", flush=True)
width = int(os.environ.get("EXP_WIDTH", "11"))
depths = [int(x) for x in os.environ.get("EXP_DEPTHS", "1,2,3,4,6,8,12").split(",")]
for depth in depths:
    w = W.random_circuit(width, depth, seed=5)
    pl = P.sv_plan_info(n, w.gates)
    ms = t(w.gates)
    print(f"rand{width} depth {depth}: passes {len(pl)} stages {sum(p['n_stages'] for p in pl)} dense "
          f"{sum(p['n_dense'] for p in pl)}: {ms:.2f} ms", flush=True)
