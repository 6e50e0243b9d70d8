"""ctypes binding of libisq.so (include/isq.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, calls raise instead of computing anything on the host.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ConfigurationError, InvariantViolation

# ISQ_LIBRARY: an alternative in-tree build of the same library (kernel-variant experiments)
LIB_PATH = Path(os.environ.get("ISQ_LIBRARY") or Path(__file__).resolve().parent / "libisq.so")

ISQ_OK = 0
ISQ_ERR_CONFIG = 1
ISQ_ERR_INVARIANT = 2
ISQ_ERR_CUDA = 3
ISQ_ERR_COMM = 4
ISQ_ERR_UNSUPPORTED = 5

MIN_WIRES = 2
MAX_WIRES = 13
MAX_FAST_WIRES = 5

_lock = threading.Lock()
_lib = None

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)
c_u8p = ctypes.POINTER(ctypes.c_uint8)

# name -> (restype, argtypes).  Kept in sync with include/isq.h (a CPU test
# checks that every declared symbol is exported and listed here).
class QeqeaConfig(ctypes.Structure):
    _fields_ = [
        ("number_of_wires", c_i32),
        ("size_of_individual", c_i32),
        ("size_of_population", c_i64),
        ("probability_of_mutation", c_dbl),
        ("mutation_range", c_dbl),
        ("n_meas", c_i32),
        ("rank", c_i32),
        ("max_generations", c_i64),
        ("target_fitness", c_dbl),
        ("seed", c_u64),
        ("world", c_i32),
        ("precision", c_i32),
    ]


class GaConfigC(ctypes.Structure):
    _fields_ = [
        ("number_of_wires", c_i32),
        ("size_of_individual", c_i32),
        ("population", c_i64),
        ("mutation_rate", c_dbl),
        ("mutation_range", c_dbl),
        ("structural_rate", c_dbl),
        ("max_generations", c_i64),
        ("target_fitness", c_dbl),
        ("seed", c_u64),
        ("rank", c_i32),
        ("world", c_i32),
        ("precision", c_i32),
        ("reserved", c_i32),
    ]


MAX_WORLD = 64
LAUNCH_MODES = {"auto": 0, "kernels": 1, "graph": 2, "fused": 3}
PRECISIONS = {"fp64": 0, "fp32": 1}


class QeqeaExchange(ctypes.Structure):
    """isq_qeqea_exchange_buffers (include/isq.h)."""

    _fields_ = [
        ("world", c_i32),
        ("rank", c_i32),
        ("shard", c_i64),
        ("elite_len", c_i32),
        ("position_bounds", c_i32 * (MAX_WORLD + 1)),
        ("send_flats", c_vp),
        ("recv_flats", c_vp),
        ("send_codes", c_vp),
        ("recv_codes", c_vp),
        ("send_thetas", c_vp),
        ("recv_thetas", c_vp),
        ("fitness", c_vp),
        ("elite", c_vp),
        ("stream", c_vp),
    ]


PEER_BUFFERS = 5
IPC_HANDLE_BYTES = 64


class PeerBuffers(ctypes.Structure):
    """isq_qeqea_peer_buffers (include/isq.h)."""

    _fields_ = [("recv_flats", c_vp), ("recv_codes", c_vp), ("recv_thetas", c_vp), ("fitness", c_vp),
                ("elite", c_vp)]


GEN_RECORD = np.dtype([("gen_best", "f8"), ("gen_mean", "f8"), ("best_fitness", "f8"), ("reserved", "f8")])

c_i32p = ctypes.POINTER(c_i32)

SIGNATURES: dict[str, tuple] = {
    "isq_qeqea_create": (c_i32, [ctypes.POINTER(QeqeaConfig), c_vp, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "isq_qeqea_destroy": (c_i32, [c_vp]),
    "isq_qeqea_set_stream": (c_i32, [c_vp, c_vp]),
    "isq_qeqea_step": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp]),
    "isq_qeqea_begin_batch": (c_i32, [c_vp]),
    "isq_qeqea_eval": (c_i32, [c_vp]),
    "isq_qeqea_finish": (c_i32, [c_vp]),
    "isq_qeqea_prepare": (c_i32, [c_vp]),
    "isq_qeqea_values": (c_i32, [c_vp]),
    "isq_qeqea_set_launch_mode": (c_i32, [c_vp, c_i32]),
    "isq_ga_set_launch_mode": (c_i32, [c_vp, c_i32]),
    "isq_qeqea_exchange": (c_i32, [c_vp, c_vp]),
    "isq_qeqea_ipc_export": (c_i32, [c_vp, c_vp]),
    "isq_qeqea_ipc_open": (c_i32, [c_vp, c_vp]),
    "isq_qeqea_set_peers": (c_i32, [c_vp, c_vp]),
    "isq_qeqea_score": (c_i32, [c_vp]),
    "isq_qeqea_read_batch": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "isq_qeqea_buffers": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "isq_qeqea_best": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "isq_qeqea_get_state": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "isq_qeqea_set_state": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_u64, c_dbl, c_i32, c_vp, c_vp]),
    "isq_qeqea_live_population": (c_i32, [c_vp, c_vp, c_vp]),
    "isq_qeqea_sample": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "isq_qeqea_fitness": (c_i32, [c_vp, c_vp]),
    "isq_qeqea_set_limits": (c_i32, [c_vp, c_i64, c_dbl, c_i32]),
    "isq_ga_set_limits": (c_i32, [c_vp, c_i64, c_dbl, c_i32]),
    "isq_ga_create": (c_i32, [ctypes.POINTER(GaConfigC), c_vp, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "isq_ga_destroy": (c_i32, [c_vp]),
    "isq_ga_set_stream": (c_i32, [c_vp, c_vp]),
    "isq_ga_step": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_vp]),
    "isq_ga_begin_batch": (c_i32, [c_vp]),
    "isq_ga_eval": (c_i32, [c_vp]),
    "isq_ga_finish": (c_i32, [c_vp]),
    "isq_ga_read_batch": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "isq_ga_buffers": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "isq_ga_best": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "isq_ga_get_state": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "isq_ga_set_state": (c_i32, [c_vp, c_vp, c_vp, c_u64, c_dbl, c_i32, c_vp, c_vp]),
    "isq_ga_fitness": (c_i32, [c_vp, c_vp]),
    "isq_ga_parents": (c_i32, [c_vp, c_vp]),
    "isq_last_error": (ctypes.c_char_p, []),
    "isq_abi_version": (c_i32, []),
    "isq_fitness_batch": (c_i32, [c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "isq_fitness_batch_device": (c_i32, [c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "isq_fitness_batch_ex": (c_i32, [c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32]),
    "isq_fitness_batch_device_ex": (c_i32, [c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "isq_philox_block": (None, [c_u64, c_u64, c_u64, c_u64, c_u64, c_u64, c_vp]),
    "isq_fma_peak": (c_i32, [c_i32, c_i32, c_vp]),
    "isq_fitness_of_unitaries": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, c_i32]),
    "isq_init_population": (c_i32, [c_i32, c_i32, c_i64, c_u64, c_vp, c_vp, c_i32]),
    "isq_construct_segments": (c_i32, [c_i32, c_i32, c_i64, c_i32, c_u64, c_u64, c_vp, c_vp, c_i32]),
    "isq_sample_circuits": (c_i32, [c_i32, c_i32, c_i64, c_u64, c_u64, c_i64, c_i64, c_vp, c_i32]),
    "isq_mutate_population": (c_i32, [ctypes.POINTER(QeqeaConfig), c_u64, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "isq_table_create": (c_i32, [c_i64, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "isq_table_destroy": (c_i32, [c_vp]),
    "isq_table_update": (c_i32, [c_vp, c_i64, c_vp, c_vp, c_vp]),
    "isq_table_read": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "isq_table_set_slot_max": (c_i32, [c_vp, c_vp]),
    "isq_apply_gates": (c_i32, [c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "isq_mutate_angles": (c_i32, [c_i64, c_vp, c_vp, c_dbl, c_u64, c_u64, c_i64, c_vp, c_i32]),
    "isq_mutate_qutrits": (c_i32, [c_i64, c_vp, c_vp, c_u64, c_u64, c_i64, c_vp, c_i32]),
    "isq_born_probabilities": (c_i32, [c_i64, c_vp, c_vp, c_i32]),
    "isq_estimate_axes": (c_i32, [c_i64, c_vp, c_i32, c_u64, c_u64, c_i64, c_vp, c_i32]),
    "isq_measure_qutrits": (c_i32, [c_i64, c_vp, c_u64, c_u64, c_i64, c_vp, c_i32]),
    "isq_su3_operators": (c_i32, [c_i64, c_vp, c_vp, c_i32]),
    "isq_init_slots": (c_i32, [c_i64, c_u64, c_i64, c_i32, c_vp, c_vp, c_i32]),
    "isq_ga_random_genomes": (c_i32, [c_i32, c_i32, c_u64, c_i64, c_i64, c_vp, c_vp, c_i32]),
    "isq_ga_sus_select": (c_i32, [c_i64, c_vp, c_i64, c_u64, c_u64, c_vp, c_i32]),
    "isq_ga_crossover_cuts": (c_i32, [c_i32, c_u64, c_u64, c_i64, c_i64, c_vp, c_i32]),
    "isq_ga_mutate_genomes": (c_i32, [ctypes.POINTER(GaConfigC), c_u64, c_i64, c_i64, c_vp, c_vp, c_i32]),
}


class IsqError(RuntimeError):
    """Device-side failure reported by libisq (CUDA/NCCL error)."""


def load(path: Path | None = None):
    """Load and bind libisq.so; raises ImportError when it has not been built."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(status: int) -> None:
    if status == ISQ_OK:
        return
    msg = load().isq_last_error()
    msg = msg.decode() if msg else "unknown error"
    if status in (ISQ_ERR_CONFIG, ISQ_ERR_UNSUPPORTED):
        raise ConfigurationError(msg)
    if status == ISQ_ERR_INVARIANT:
        raise InvariantViolation(msg)
    raise IsqError(f"libisq status {status}: {msg}")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(c_vp)
