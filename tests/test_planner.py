"""Host-side planner invariants (no GPU): every gate lands in exactly one pass, non-diagonal
targets lie in the pass' tile, tiles keep the low-qubit granule when they can, the register stages
cover all ops, dense stages only where the register kernel runs, and planning terminates for every
shape and option (sv_plan_info, include/sv_debug.h)."""
import numpy as np
import pytest

import workloads as W

P = pytest.importorskip("paper_2406_17248_b200")

CIRCUITS = [
    ("CP", n) for n in (1, 2, 3, 5, 8, 9, 10, 12, 13, 14, 17, 20, 24)
]


def _circ(n, seed=0):
    return W.random_complex(n, 8, seed=seed + n, n_params=4,
                            extra_kinds=("MAT1", "MAT2", "XLIKE", "ZLIKE", "PS", "SDG", "TDG"))


@pytest.mark.timeout(120)
@pytest.mark.parametrize("n", [c[1] for c in CIRCUITS])
@pytest.mark.parametrize("adjoint", [0, 1])
def test_plan_invariants(n, adjoint):
    w = _circ(n)
    for tq in (0, 2, 4, 7, 9, 10, 11, 12, 13):
        for fusion in (1, 0):
            plan = P.sv_plan_info(n, w.gates, w.params, adjoint=adjoint, tile_qubits=tq, fusion=fusion)
            assert sum(p["n_ops"] for p in plan) == len(w.gates)
            for p in plan:
                assert p["nondiag_mask"] & ~p["tile_mask"] == 0
                assert bin(p["tile_mask"]).count("1") == p["k"] <= 13
                if not fusion:
                    assert p["n_ops"] == 1
                if p["R"] == 0:
                    assert p["n_stages"] == 0 and p["n_dense"] == 0
                else:
                    assert p["n_stages"] >= 1 and p["k"] - p["R"] >= 5
                if adjoint:
                    assert p["n_dense"] <= 4  # adjoint dense stages (R accumulators) per reverse pass


def test_fusion_reduces_passes_for_c4():
    w = W.config("C4")
    fused = P.sv_plan_info(w.n, w.gates)
    assert len(fused) <= 70, len(fused)          # 1780 gates in a few dozen HBM passes
    assert all(p["k"] == 11 and p["low"] >= 3 for p in fused)
    assert sum(p["n_dense"] for p in fused) > 0.5 * sum(p["n_stages"] for p in fused)


def test_dense_stage_work_accounting():
    """The roofline's FP64 work per pass (bench.py): a forward dense stage executes 48 DMMA FMAs
    and 3 additions per amplitude (three-product form: 3 x 16 complex-entry fragments per 16
    amplitudes, one sum per input element and two per A entry over the warp's 16 vectors); an
    adjoint dense stage three times that (R, U^+ psi, U^+ lambda). Sequential ops add FMAs only."""
    w = W.config("C4")
    for p in P.sv_plan_info(w.n, w.gates):
        assert p["add_per_amp"] == 3 * p["n_dense"]
        assert p["fma_per_amp"] >= 48 * p["n_dense"]
        if p["n_dense"] == p["n_stages"]:
            assert p["fma_per_amp"] == 48 * p["n_dense"]
    g = W.config("C4g")
    rev = P.sv_plan_info(g.n, g.gates, g.params, adjoint=1)
    assert any(p["n_dense"] for p in rev)  # adjoint dense stages at 30 qubits
    for p in rev:
        assert p["add_per_amp"] == 9 * p["n_dense"]
        assert p["fma_per_amp"] >= 144 * p["n_dense"]


def test_forward_variant_bits_by_size():
    """Forward dense stages take up to 8 variant bits from 28 local qubits (plan.cpp
    dense_max_var_for): C4 at 30 qubits plans fewer stages than the same generator would with 6."""
    w = W.config("C4")
    plan = P.sv_plan_info(w.n, w.gates)
    assert sum(p["n_stages"] for p in plan) <= 141


def test_adjoint_slots_match_parametrised_gates():
    w = W.config("C2")
    plan = P.sv_plan_info(w.n, w.gates, w.params, adjoint=1)
    assert sum(p["n_grad"] for p in plan) == sum(1 for g in w.gates if g.param >= 0)


def test_validation_without_gpu():
    with pytest.raises(P.SvError) as e:
        P.sv_plan_info(3, [W.Gate("X", (3,))])
    assert e.value.status == "SV_E_QUBIT_RANGE"
    with pytest.raises(P.SvError) as e:
        P.sv_plan_info(3, [W.Gate("MAT1", (0,), param=0, mat=np.eye(2))], [0.1], adjoint=1)
    assert e.value.status == "SV_E_NOT_DIFFERENTIABLE"
