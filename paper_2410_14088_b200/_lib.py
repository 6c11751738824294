"""ctypes binding of libbmq.so (C ABI: include/bmq.h).

The shared library is built in-tree by ``make -C paper_2410_14088_b200`` (or
``__graft_entry__.build()``). There is no fallback: importing the package
without the library raises immediately, and compute calls without a CUDA
device raise ``NoDeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbmq.so")

BMQ_OK = 0
BMQ_ERR_INVALID_ARGUMENT = 1
BMQ_ERR_LOGIC = 2
BMQ_ERR_CODEC = 3
BMQ_ERR_STORE = 4
BMQ_ERR_ENGINE = 5
BMQ_ERR_QASM = 6
BMQ_ERR_CUDA = 7
BMQ_ERR_NO_DEVICE = 8
BMQ_ERR_OUT_OF_MEMORY = 9
BMQ_ERR_BUFFER_TOO_SMALL = 10

BMQ_FLAG_ZERO_GROUP_SKIP = 0x1
BMQ_FLAG_IDENTITY_SKIP = 0x2
BMQ_FLAG_CODE_DOMAIN = 0x4
BMQ_FLAG_POOL_GROW = 0x8
BMQ_FLAG_HEAP_ARENA = 0x10
BMQ_FLAG_BUMP_ARENA = 0x20
BMQ_FLAG_DEVICE_PLAN = 0x40
BMQ_FLAG_STAGE_FUSION = 0x80


class bmq_gate(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("q0", C.c_uint32), ("q1", C.c_uint32), ("reserved", C.c_uint32),
                ("angle", C.c_double)]


class bmq_stage(C.Structure):
    _fields_ = [("gate_begin", C.c_uint64), ("gate_end", C.c_uint64), ("inner_count", C.c_uint32),
                ("reserved", C.c_uint32), ("inner", C.c_uint32 * 64)]


class bmq_config(C.Structure):
    _fields_ = [("block_bits", C.c_uint32), ("inner_size", C.c_uint32), ("error_bound", C.c_double),
                ("memory_budget", C.c_uint64), ("workers", C.c_uint32), ("compress", C.c_uint32),
                ("verify_cap_qubits", C.c_uint32), ("device", C.c_int32), ("device_pool_bytes", C.c_uint64),
                ("work_bytes", C.c_uint64), ("flags", C.c_uint32), ("reserved", C.c_uint32),
                ("host_pool_bytes", C.c_uint64), ("disk_pool_bytes", C.c_uint64), ("disk_dir", C.c_char_p)]


class bmq_plan_model(C.Structure):
    _fields_ = [("work_bytes", C.c_uint64), ("hbm_gbs", C.c_double), ("link_gbs", C.c_double),
                ("ratio", C.c_double), ("stage_overhead_s", C.c_double), ("world", C.c_uint32),
                ("max_inner", C.c_uint32), ("codec_eff", C.c_double), ("pass_eff", C.c_double)]


class bmq_plan_choice(C.Structure):
    _fields_ = [("inner_size", C.c_uint32), ("candidates", C.c_uint32), ("stages", C.c_uint64),
                ("passes", C.c_uint64), ("remaps", C.c_uint32), ("reserved", C.c_uint32),
                ("model_s_best", C.c_double), ("inner", C.c_uint32 * 16), ("model_s", C.c_double * 16)]


class bmq_report(C.Structure):
    _fields_ = [("qubits", C.c_uint64), ("gate_count", C.c_uint64), ("stage_count", C.c_uint64),
                ("max_footprint_bytes", C.c_uint64), ("standard_bytes", C.c_double),
                ("compression_ratio", C.c_double), ("spilled_blocks", C.c_uint64), ("wall_ms", C.c_double),
                ("has_fidelity", C.c_int32), ("reserved", C.c_int32), ("fidelity", C.c_double),
                ("final_norm", C.c_double), ("stage_compress_calls", C.c_uint64),
                ("stage_decompress_calls", C.c_uint64), ("device_ms", C.c_double),
                ("groups_processed", C.c_uint64), ("groups_skipped", C.c_uint64),
                ("blocks_processed", C.c_uint64), ("payload_bytes_read", C.c_uint64),
                ("payload_bytes_written", C.c_uint64), ("dense_bytes", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("device_peak_bytes", C.c_uint64), ("gate_passes", C.c_uint64),
                ("decompress_ms", C.c_double), ("gate_ms", C.c_double), ("compress_ms", C.c_double),
                ("batches", C.c_uint64), ("decompress_bytes", C.c_uint64), ("gate_bytes", C.c_uint64),
                ("compress_bytes", C.c_uint64), ("fused_batches", C.c_uint64), ("compactions", C.c_uint64),
                ("host_spill_bytes", C.c_uint64), ("host_spill_batches", C.c_uint64),
                ("code_domain_batches", C.c_uint64), ("pool_growths", C.c_uint64),
                ("lazy_cx", C.c_uint64), ("perm_materialisations", C.c_uint64),
                ("model_bytes", C.c_uint64), ("model_groups", C.c_uint64), ("link_h2d_bytes", C.c_uint64),
                ("link_d2h_bytes", C.c_uint64), ("link_ms", C.c_double),
                ("compact_bytes", C.c_uint64), ("host_peak_bytes", C.c_uint64), ("arena_bytes", C.c_uint64),
                ("fused_decode_batches", C.c_uint64), ("stream_passes", C.c_uint64),
                ("disk_spill_bytes", C.c_uint64), ("disk_read_bytes", C.c_uint64), ("disk_peak_bytes", C.c_uint64),
                ("disk_gds", C.c_uint64), ("fused_stages", C.c_uint64), ("fused_sets", C.c_uint64)]


_P = C.c_void_p
_U64 = C.c_uint64
_U32 = C.c_uint32
_D = C.c_double

# name -> (restype, argtypes); every symbol include/bmq.h declares.
SIGNATURES = {
    "bmq_last_error": (C.c_char_p, []),
    "bmq_version": (C.c_char_p, []),
    "bmq_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "bmq_error_bound": (C.c_int, [_D, C.POINTER(_D)]),
    "bmq_gate_unitary": (C.c_int, [C.POINTER(bmq_gate), _P]),
    "bmq_circuit_validate": (C.c_int, [_U32, _P, _U64]),
    "bmq_generate_benchmark": (C.c_int, [C.c_char_p, _U32, _U32, _U64, C.c_char_p, _P, _U64, C.POINTER(_U64)]),
    "bmq_nccl_unique_id": (C.c_int, [_P]),
    "bmq_collective_nccl_create": (C.c_int, [_P, _U32, _U32, C.c_int32, _P]),
    "bmq_collective_local_create": (C.c_int, [_U32, _P]),
    "bmq_collective_destroy": (C.c_int, [_P]),
    "bmq_simulator_run_sharded": (C.c_int, [_P, _P, C.POINTER(bmq_report), _P, _U64]),
    "bmq_simulator_sample": (C.c_int, [_P, _U64, _U64, _P]),
    "bmq_simulator_top_k": (C.c_int, [_P, _U64, _P, _P, _P, C.POINTER(_U64)]),
    "bmq_plan_model_default": (None, [C.POINTER(bmq_plan_model)]),
    "bmq_plan_device_aware": (C.c_int, [_U32, _P, _U64, _U32, C.POINTER(bmq_plan_model), _P, _U64, C.POINTER(_U64),
                                        C.POINTER(bmq_plan_choice)]),
    "bmq_partition": (C.c_int, [_U32, _P, _U64, _U32, _U32, _P, _U64, C.POINTER(_U64)]),
    "bmq_enumerate_groups": (C.c_int, [_U32, _U32, C.POINTER(bmq_stage), _P, _U64, C.POINTER(_U64)]),
    "bmq_buffer_bit_of_qubit": (C.c_int, [_U32, _U32, C.POINTER(bmq_stage), _U32, C.POINTER(_U32)]),
    "bmq_parse_qasm": (C.c_int, [C.c_char_p, C.POINTER(_U32), _P, _U64, C.POINTER(_U64), C.c_char_p, _U64,
                                 C.POINTER(_U64)]),
    "bmq_emit_qasm": (C.c_int, [_U32, _P, _U64, C.c_char_p, _U64, C.POINTER(_U64)]),
    "bmq_compress_bound": (_U64, [_U64]),
    "bmq_compress_blocks": (C.c_int, [_P, _U64, _U64, _D, _P, _U64, _P]),
    "bmq_decompress_blocks": (C.c_int, [_P, _P, _P, _U64, _P, _U64, _P]),
    "bmq_apply_gate": (C.c_int, [_P, _U64, _P, C.c_int, _U32, _U32]),
    "bmq_apply_stage": (C.c_int, [_P, _U64, _U32, _P, _U64, C.POINTER(bmq_stage), _U32]),
    "bmq_dense_reference": (C.c_int, [_U32, _P, _U64, _P, _U32]),
    "bmq_config_default": (None, [C.POINTER(bmq_config)]),
    "bmq_simulator_create": (C.c_int, [_U32, _P, _U64, C.POINTER(bmq_config), C.POINTER(_P)]),
    "bmq_simulator_destroy": (C.c_int, [_P]),
    "bmq_simulator_plan": (C.c_int, [_P, _P, _U64, C.POINTER(_U64)]),
    "bmq_simulator_init_state": (C.c_int, [_P]),
    "bmq_simulator_run": (C.c_int, [_P, C.POINTER(bmq_report), _P, _U64]),
    "bmq_simulator_run_stages": (C.c_int, [_P, _U64, _U64]),
    "bmq_simulator_reset": (C.c_int, [_P]),
    "bmq_simulator_state_norm": (C.c_int, [_P, C.POINTER(_D)]),
    "bmq_simulator_extract_state": (C.c_int, [_P, _P, _U64]),
    "bmq_simulator_amplitude": (C.c_int, [_P, _U64, C.POINTER(_D), C.POINTER(_D)]),
    "bmq_simulator_get_payload": (C.c_int, [_P, _U64, _P, _U64, C.POINTER(_U64)]),
    "bmq_simulator_get_payloads": (C.c_int, [_P, _P, _U64, _P, C.POINTER(_U64)]),
    "bmq_simulator_put_payload": (C.c_int, [_P, _U64, _P, _U64]),
    "bmq_simulator_fidelity_dense": (C.c_int, [_P, _P, _U64, C.POINTER(_D)]),
    "bmq_fidelity": (C.c_int, [_P, _P, _U64, C.POINTER(_D)]),
    "bmq_simulator_footprint": (C.c_int, [_P, C.POINTER(_U64), C.POINTER(_U64), C.POINTER(_U64)]),
    "bmq_simulator_fidelity": (C.c_int, [_P, _P, C.POINTER(_D)]),
    "bmq_simulator_fidelity_analytic": (C.c_int, [_P, C.c_int, C.POINTER(_D)]),
    "bmq_shard_plan": (C.c_int, [C.c_uint32, C.c_uint32, C.POINTER(bmq_stage), _U64, C.c_uint32, C.POINTER(C.c_uint32)]),
    "bmq_simulator_shard": (C.c_int, [_P, C.c_uint32, C.c_uint32]),
    "bmq_simulator_export": (C.c_int, [_P, C.POINTER(_U64), _U64, C.POINTER(_U64), C.c_void_p, _U64]),
    "bmq_simulator_import": (C.c_int, [_P, C.POINTER(_U64), _U64, C.POINTER(_U64), C.c_void_p]),
    "bmq_simulator_drop": (C.c_int, [_P, C.POINTER(_U64), _U64]),
    "bmq_simulator_stage_sizes": (C.c_int, [_P, _U64, C.POINTER(_U64)]),
    "bmq_simulator_account_stage": (C.c_int, [_P, _U64, C.POINTER(_U64)]),
    "bmq_simulator_partial_sums": (C.c_int, [_P, C.POINTER(_D)]),
    "bmq_simulator_report": (C.c_int, [_P, C.POINTER(bmq_report)]),
    "bmq_simulator_save": (C.c_int, [_P, C.c_char_p]),
    "bmq_simulator_load": (C.c_int, [_P, C.c_char_p, C.POINTER(_U64)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension with `make -C {_HERE}` "
            "(or __graft_entry__.build()); paper_2410_14088_b200 has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
