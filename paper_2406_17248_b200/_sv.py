"""ctypes binding of libsv.so (include/sv.h). Argument marshalling only: every step of the hot
path runs in the library's sm_100a kernels. There is no fallback: if the library is missing or
fails to load, import raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsv.so")

# enum sv_kind (include/sv.h)
KIND = {"X": 0, "Y": 1, "XLIKE": 2, "Z": 3, "S": 4, "SDG": 5, "T": 6, "TDG": 7, "ZLIKE": 8, "RZ": 9, "PS": 10,
        "H": 11, "RX": 12, "RY": 13, "MAT1": 14, "SWAP": 15, "RXX": 16, "RYY": 17, "RZZ": 18, "MAT2": 19}
STATUS = {0: "SV_OK", 1: "SV_E_ARG", 2: "SV_E_QUBIT_RANGE", 3: "SV_E_TARGET_CONTROL_OVERLAP",
          4: "SV_E_DUPLICATE_TARGET", 5: "SV_E_PARAM_RANGE", 6: "SV_E_NOT_DIFFERENTIABLE", 7: "SV_E_NOT_UNITARY",
          8: "SV_E_OOM", 9: "SV_E_CUDA", 10: "SV_E_NCCL", 11: "SV_E_POISONED"}
SV_OPT_TILE_QUBITS, SV_OPT_FUSION, SV_OPT_LOW_QUBITS, SV_OPT_DENSE, SV_OPT_KERNEL = 1, 2, 3, 4, 5
SV_OPT_ADJOINT_DENSE_COST = 6
SV_OPT_C64_SPLIT = 7


class SvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class sv_gate(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("targets", ctypes.c_int32 * 2), ("controls", ctypes.c_uint64),
                ("param", ctypes.c_int32), ("coeff", ctypes.c_double), ("offset", ctypes.c_double),
                ("mat", ctypes.POINTER(ctypes.c_double))]


class sv_pauli(ctypes.Structure):
    _fields_ = [("x_mask", ctypes.c_uint64), ("z_mask", ctypes.c_uint64), ("coeff", ctypes.c_double)]


class sv_stats(ctypes.Structure):  # include/sv.h
    _fields_ = [("kernel_launches", ctypes.c_int64), ("gate_passes", ctypes.c_int64),
                ("adjoint_passes", ctypes.c_int64), ("expectation_passes", ctypes.c_int64),
                ("exchanges", ctypes.c_int64), ("algorithmic_bytes", ctypes.c_double),
                ("gates_applied", ctypes.c_int64), ("exchange_bytes", ctypes.c_double),
                ("exchange_ms", ctypes.c_double), ("gate_applications", ctypes.c_int64),
                ("plan_builds", ctypes.c_int64), ("plan_refreshes", ctypes.c_int64)]


class sv_pass_info(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("low", ctypes.c_int32), ("R", ctypes.c_int32), ("n_ops", ctypes.c_int32),
                ("n_stages", ctypes.c_int32), ("n_grad", ctypes.c_int32), ("tile_mask", ctypes.c_uint64),
                ("nondiag_mask", ctypes.c_uint64), ("n_dense", ctypes.c_int32), ("mat_doubles", ctypes.c_int32),
                ("fma_per_amp", ctypes.c_int32), ("add_per_amp", ctypes.c_int32)]


class sv_shard_step(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("gpos", ctypes.c_int32), ("lpos", ctypes.c_int32),
                ("n_gates", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python build.py` (or __graft_entry__.build()); "
                          "there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, H = ctypes.c_void_p, ctypes.c_void_p
    i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sigs = {
        "sv_create": [i32, ctypes.POINTER(H)],
        "sv_create_sharded": [i32, i32, i32, P, ctypes.POINTER(H)],
        "sv_nccl_unique_id": [P, i32],
        "sv_create_virtual_shards": [i32, i32, ctypes.POINTER(H)],
        "sv_create_density": [i32, ctypes.POINTER(H)],
        "sv_create_c64": [i32, ctypes.POINTER(H)],
        "sv_destroy": [H],
        "sv_set_stream": [H, P],
        "sv_set_option": [H, i32, i64],
        "sv_get_num_qubits": [H, ctypes.POINTER(i32)],
        "sv_reset": [H],
        "sv_set_state": [H, P],
        "sv_get_state": [H, P],
        "sv_get_amplitudes": [H, P, i64, P],
        "sv_set_state_device": [H, P],
        "sv_get_state_device": [H, P],
        "sv_apply_gate": [H, ctypes.POINTER(sv_gate), P, i32],
        "sv_apply_circuit": [H, ctypes.POINTER(sv_gate), i64, P, i32],
        "sv_expectation": [H, ctypes.POINTER(sv_pauli), i64, ctypes.POINTER(f64)],
        "sv_expectation_with_grad": [H, ctypes.POINTER(sv_gate), i64, P, i32, ctypes.POINTER(sv_pauli), i64,
                                     ctypes.POINTER(f64), P],
        "sv_get_stats": [H, ctypes.POINTER(sv_stats)],
        "sv_expectation_with_grad_batch": [H, ctypes.POINTER(sv_gate), i64, P, i32, i32, ctypes.POINTER(sv_pauli), i64,
                                           P, P],
        "sv_sample": [H, P, i32, i64, ctypes.c_uint64, P],
        "sv_reset_stats": [H],
        "sv_shard_plan": [i32, i32, i32, ctypes.POINTER(sv_gate), i64, P, i32, ctypes.POINTER(sv_shard_step), i64,
                          ctypes.POINTER(i64), ctypes.POINTER(sv_gate), P, i64, ctypes.POINTER(i64), P],
        "sv_plan_info": [i32, ctypes.POINTER(sv_gate), i64, P, i32, i32, i32, i32, ctypes.POINTER(sv_pass_info), i64,
                         ctypes.POINTER(i64)],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int32
    L.sv_last_error.argtypes = []
    L.sv_last_error.restype = ctypes.c_char_p
    L.sv_version.argtypes = []
    L.sv_version.restype = ctypes.c_char_p
    return L


lib = _load()


def _check(rc: int):
    if rc != 0:
        raise SvError(rc, lib.sv_last_error().decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class GateArray:
    """Marshals workloads.Gate-like objects (kind, targets, controls, param, coeff, offset, mat)
    into a contiguous sv_gate array (keeps the matrix buffers alive)."""

    def __init__(self, gates: Sequence):
        n = len(gates)
        self.n = n
        self.arr = (sv_gate * max(n, 1))()
        self._mats: List[np.ndarray] = []
        for i, g in enumerate(gates):
            s = self.arr[i]
            s.kind = KIND[g.kind]
            s.targets[0] = int(g.targets[0])
            s.targets[1] = int(g.targets[1]) if len(g.targets) > 1 else -1
            m = 0
            for c in g.controls:
                m |= 1 << int(c)
            s.controls = m
            s.param = int(g.param)
            s.coeff = float(g.coeff)
            s.offset = float(g.offset)
            if g.mat is not None:
                buf = np.ascontiguousarray(np.asarray(g.mat, dtype=np.complex128).reshape(-1)).view(np.float64).copy()
                self._mats.append(buf)
                s.mat = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            else:
                s.mat = None

    @property
    def nbytes(self) -> int:
        return ctypes.sizeof(sv_gate) * self.n + sum(m.nbytes for m in self._mats)


class PauliArray:
    """Marshals (coeff, {qubit: 'X'|'Y'|'Z'}) terms into sv_pauli (x/z masks)."""

    def __init__(self, ham: Sequence[Tuple[float, dict]]):
        self.n = len(ham)
        self.arr = (sv_pauli * max(self.n, 1))()
        for i, (c, term) in enumerate(ham):
            x = z = 0
            for q, p in term.items():
                if p in ("X", "Y"):
                    x |= 1 << int(q)
                if p in ("Z", "Y"):
                    z |= 1 << int(q)
            self.arr[i].x_mask = x
            self.arr[i].z_mask = z
            self.arr[i].coeff = float(c)

    @property
    def nbytes(self) -> int:
        return ctypes.sizeof(sv_pauli) * self.n


def _params(params) -> Tuple[Optional[np.ndarray], int]:
    if params is None or len(params) == 0:
        return None, 0
    p = np.ascontiguousarray(params, dtype=np.float64)
    return p, int(p.size)


# ----------------------------------------------------------------------------- same-name functions

def sv_version() -> str:
    return lib.sv_version().decode()


def sv_create(n_qubits: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib.sv_create(n_qubits, ctypes.byref(h)))
    return h


def sv_create_virtual_shards(n_qubits: int, world: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib.sv_create_virtual_shards(n_qubits, world, ctypes.byref(h)))
    return h


def sv_create_density(n_qubits: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib.sv_create_density(n_qubits, ctypes.byref(h)))
    return h


def sv_create_c64(n_qubits: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib.sv_create_c64(n_qubits, ctypes.byref(h)))
    return h


def sv_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.sv_nccl_unique_id(buf, 128))
    return buf.raw


def sv_create_sharded(n_qubits: int, rank: int, world: int, nccl_id: bytes) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    idbuf = ctypes.create_string_buffer(nccl_id, 128)
    _check(lib.sv_create_sharded(n_qubits, rank, world, idbuf, ctypes.byref(h)))
    return h


def sv_destroy(h) -> None:
    _check(lib.sv_destroy(h))


def sv_set_stream(h, stream_ptr: int) -> None:
    _check(lib.sv_set_stream(h, ctypes.c_void_p(stream_ptr)))


def sv_set_option(h, key: int, value: int) -> None:
    _check(lib.sv_set_option(h, key, value))


def sv_reset(h) -> None:
    _check(lib.sv_reset(h))


def sv_set_state(h, amps: np.ndarray) -> None:
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    _check(lib.sv_set_state(h, _ptr(a)))


def sv_get_state(h, n: int, out: Optional[np.ndarray] = None) -> np.ndarray:
    out = np.empty(1 << n, dtype=np.complex128) if out is None else out
    _check(lib.sv_get_state(h, _ptr(out)))
    return out


def sv_get_amplitudes(h, idx) -> np.ndarray:
    """Amplitudes at logical indices idx (sampled readout; sharded states un-permuted)."""
    i = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64).reshape(-1))
    out = np.empty(max(i.size, 1), dtype=np.complex128)
    _check(lib.sv_get_amplitudes(h, _ptr(i), int(i.size), _ptr(out)))
    return out[: i.size]


def sv_set_state_device(h, dev_ptr: int) -> None:
    _check(lib.sv_set_state_device(h, ctypes.c_void_p(dev_ptr)))


def sv_get_state_device(h, dev_ptr: int) -> None:
    _check(lib.sv_get_state_device(h, ctypes.c_void_p(dev_ptr)))


def sv_apply_gate(h, gate, params=None) -> None:
    ga = gate if isinstance(gate, GateArray) else GateArray([gate])
    p, np_ = _params(params)
    _check(lib.sv_apply_gate(h, ga.arr, _ptr(p), np_))


def sv_apply_circuit(h, gates, params=None) -> None:
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    p, np_ = _params(params)
    _check(lib.sv_apply_circuit(h, ga.arr, ga.n, _ptr(p), np_))


def sv_expectation(h, ham) -> float:
    pa = ham if isinstance(ham, PauliArray) else PauliArray(ham)
    out = ctypes.c_double()
    _check(lib.sv_expectation(h, pa.arr, pa.n, ctypes.byref(out)))
    return out.value


def sv_expectation_with_grad(h, gates, params, ham) -> Tuple[float, np.ndarray]:
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    pa = ham if isinstance(ham, PauliArray) else PauliArray(ham)
    p, np_ = _params(params)
    out = ctypes.c_double()
    grad = np.zeros(max(np_, 1))
    _check(lib.sv_expectation_with_grad(h, ga.arr, ga.n, _ptr(p), np_, pa.arr, pa.n, ctypes.byref(out), _ptr(grad)))
    return out.value, grad[:np_]


def sv_expectation_with_grad_batch(h, gates, params_rows, ham) -> Tuple[np.ndarray, np.ndarray]:
    """Batch mode: params_rows [B, P]; returns (E [B], grad [B, P])."""
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    pa = ham if isinstance(ham, PauliArray) else PauliArray(ham)
    rows = np.ascontiguousarray(np.atleast_2d(np.asarray(params_rows, dtype=np.float64)))
    B, Pn = rows.shape
    ev = np.zeros(B)
    gv = np.zeros((B, max(Pn, 1)))
    _check(lib.sv_expectation_with_grad_batch(h, ga.arr, ga.n, _ptr(rows) if Pn else None, Pn, B, pa.arr, pa.n,
                                              _ptr(ev), _ptr(gv)))
    return ev, gv[:, :Pn]


def sv_sample(h, qubits, shots: int, seed: int = 0) -> np.ndarray:
    """Sampling measurement: shots outcomes over `qubits` (bit j = qubits[j])."""
    q = np.ascontiguousarray(qubits, dtype=np.int32)
    out = np.zeros(max(shots, 1), dtype=np.uint64)
    _check(lib.sv_sample(h, _ptr(q), int(q.size), int(shots), ctypes.c_uint64(seed), _ptr(out)))
    return out[:shots]


def sv_get_stats(h) -> dict:
    s = sv_stats()
    _check(lib.sv_get_stats(h, ctypes.byref(s)))
    return {f: getattr(s, f) for f, _ in sv_stats._fields_}


def sv_reset_stats(h) -> None:
    _check(lib.sv_reset_stats(h))


def sv_plan_info(n_qubits: int, gates, params=None, adjoint: bool = False, tile_qubits: int = 0,
                 fusion: bool = True) -> List[dict]:
    """Host-only planner introspection (include/sv_debug.h)."""
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    p, np_ = _params(params)
    cap = 1 << 16
    out = (sv_pass_info * cap)()
    npass = ctypes.c_int64()
    _check(lib.sv_plan_info(n_qubits, ga.arr, ga.n, _ptr(p), np_, int(adjoint), tile_qubits, int(fusion), out, cap,
                            ctypes.byref(npass)))
    return [{f: getattr(out[i], f) for f, _ in sv_pass_info._fields_} for i in range(min(npass.value, cap))]


def sv_shard_plan(n_qubits: int, world: int, rank: int, gates, params=None):
    """Host-only sharded schedule for `rank` (include/sv_debug.h): returns (steps, perm) where
    steps are ("swap", gpos, lpos) or ("segment", [(matrix, targets, controls_mask), ...])."""
    ga = gates if isinstance(gates, GateArray) else GateArray(gates)
    p, np_ = _params(params)
    cap_s, cap_g = 4 * ga.n + 16, 4 * ga.n + 16
    steps = (sv_shard_step * cap_s)()
    lg = (sv_gate * cap_g)()
    mats = np.zeros(32 * cap_g)
    ns, ng = ctypes.c_int64(), ctypes.c_int64()
    perm = np.zeros(n_qubits, dtype=np.int32)
    _check(lib.sv_shard_plan(n_qubits, world, rank, ga.arr, ga.n, _ptr(p), np_, steps, cap_s, ctypes.byref(ns), lg,
                             _ptr(mats), cap_g, ctypes.byref(ng), _ptr(perm)))
    out = []
    gi = 0
    for i in range(ns.value):
        st = steps[i]
        if st.kind == 1:
            out.append(("swap", st.gpos, st.lpos))
            continue
        seg = []
        for _ in range(st.n_gates):
            g = lg[gi]
            d = 2 if g.kind == KIND["MAT1"] else 4
            m = mats[32 * gi: 32 * gi + 2 * d * d]
            mat = (m[0::2] + 1j * m[1::2]).reshape(d, d)
            targets = [g.targets[0]] + ([g.targets[1]] if d == 4 else [])
            seg.append((mat, targets, int(g.controls)))
            gi += 1
        out.append(("segment", seg))
    return out, [int(x) for x in perm]


class StateVector:
    """Owning convenience wrapper (marshalling only)."""

    def __init__(self, n: int, handle=None):
        self.n = n
        self.h = handle if handle is not None else sv_create(n)

    def close(self):
        if self.h is not None:
            sv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        sv_reset(self.h)

    def set_state(self, amps):
        sv_set_state(self.h, amps)

    def get_state(self):
        return sv_get_state(self.h, self.n)

    def get_amplitudes(self, idx):
        return sv_get_amplitudes(self.h, idx)

    def apply_circuit(self, gates, params=None):
        sv_apply_circuit(self.h, gates, params)

    def apply_gate(self, gate, params=None):
        sv_apply_gate(self.h, gate, params)

    def expectation(self, ham):
        return sv_expectation(self.h, ham)

    def expectation_with_grad(self, gates, params, ham):
        return sv_expectation_with_grad(self.h, gates, params, ham)

    def set_option(self, key, value):
        sv_set_option(self.h, key, value)

    def stats(self):
        return sv_get_stats(self.h)

    def expectation_with_grad_batch(self, gates, params_rows, ham):
        return sv_expectation_with_grad_batch(self.h, gates, params_rows, ham)

    def sample(self, qubits, shots, seed=0):
        return sv_sample(self.h, qubits, shots, seed)


class DensityMatrix(StateVector):
    """rho of n qubits (NEXT-4, §3.2): apply_circuit does rho <- U rho U^dagger,
    expectation returns tr(rho H); states transfer as 2^n x 2^n matrices."""

    def __init__(self, n: int):
        super().__init__(n, handle=sv_create_density(n))

    def set_state(self, rho):
        r = np.ascontiguousarray(np.asarray(rho, dtype=np.complex128).reshape(-1))
        _check(lib.sv_set_state(self.h, _ptr(r)))

    def get_state(self):
        out = np.empty(1 << (2 * self.n), dtype=np.complex128)
        _check(lib.sv_get_state(self.h, _ptr(out)))
        return out.reshape(1 << self.n, 1 << self.n)


class StateVectorC64(StateVector):
    """complex64 state (NEXT-3, the paper's single-precision mode): same calls; host state
    transfer in complex128 arrays (rounded on set), device transfer in complex64."""

    def __init__(self, n: int):
        super().__init__(n, handle=sv_create_c64(n))
