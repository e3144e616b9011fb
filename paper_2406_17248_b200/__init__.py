"""B200-native state-vector hot path after arXiv:2406.17248 (MindSpore Quantum, "mqvector").

The product is the C-ABI library libsv.so (include/sv.h, sources in csrc/); this package is its
thin ctypes binding. Importing it without the built library raises (no CPU fallback).
"""
from ._sv import (  # noqa: F401
    KIND, STATUS, GateArray, PauliArray, StateVector, DensityMatrix, StateVectorC64, sv_create_density, sv_create_c64, SvError, lib, sv_apply_circuit, sv_apply_gate, sv_create,
    sv_create_sharded, sv_create_virtual_shards, sv_destroy, sv_expectation, sv_expectation_with_grad, sv_get_state, sv_get_amplitudes,
    sv_get_state_device, sv_get_stats, sv_nccl_unique_id, sv_reset, sv_reset_stats, sv_set_option, sv_set_state,
    sv_set_state_device, sv_set_stream, sv_version, sv_plan_info, sv_shard_plan, sv_expectation_with_grad_batch, sv_sample, SV_OPT_FUSION, SV_OPT_LOW_QUBITS, SV_OPT_TILE_QUBITS, SV_OPT_DENSE, SV_OPT_KERNEL, SV_OPT_ADJOINT_DENSE_COST, SV_OPT_C64_SPLIT, LIB_PATH,
)
