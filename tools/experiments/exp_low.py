"""Light-pass HBM efficiency vs the number of contiguous low qubits per tile (SV_OPT_LOW_QUBITS)
and the tile's high-qubit placement: times sv_apply_circuit of single light passes at 30 qubits."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_17248_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

n = 30
sv = P.StateVector(n)
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


for lowq in (3, 4, 5, 6, 7):
    sv.set_option(P.SV_OPT_LOW_QUBITS, lowq)
    for name, qs in (("hi13-20", list(range(13, 21))), ("hi22-29", list(range(22, 30))), ("lo3-10", list(range(3, 11)))):
        gates = [G("X", (q + 1,), controls=(q,)) for q in qs[:-1]]
        ms = t(gates)
        plan = P.sv_plan_info(n, gates, tile_qubits=0)
        print(f"low={lowq} {name}: {ms:.2f} ms  {2 * 16 * 2**n / ms / 1e6:.0f} GB/s  passes={len(plan)}", flush=True)
