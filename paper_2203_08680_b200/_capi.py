"""ctypes bindings of include/gomix_gpu.h (libgomix_b200.so).

The library is built in-tree (paper_2203_08680_b200/libgomix_b200.so, see
build.py).  There is no fallback: if the shared library is missing or fails to
load, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libgomix_b200.so")
# GOMIX_LIB: an alternative in-tree build for A/B timing experiments; only a
# library inside this package directory is accepted
_alt = os.environ.get("GOMIX_LIB")
if _alt:
    _alt = os.path.realpath(_alt)
    if os.path.dirname(_alt) != os.path.realpath(PKG) or not os.path.basename(_alt).endswith(".so"):
        raise ImportError("GOMIX_LIB must name a .so inside " + PKG)
    LIB_PATH = _alt

GOMIX_OK, GOMIX_E_INVALID, GOMIX_E_CUDA, GOMIX_E_NCCL, GOMIX_E_OOM, GOMIX_E_STATE = range(6)
MODE_REPLAY, MODE_PHILOX = 0, 1
FLAG_ORDERED_FLOAT, FLAG_RECORD_BATCH, FLAG_TIME_KERNELS, FLAG_LANE_PER_SOLUTION, FLAG_PER_GROUP_KERNELS, \
    FLAG_NO_TRUTH_TABLE, FLAG_FORCED_IMPROVEMENT, FLAG_PEER_TRANSPORT = 1, 2, 4, 8, 16, 32, 64, 128
PEER_HANDLE_BYTES = 64
STOP_NAMES = {0: "none", 1: "evaluation-budget", 2: "wall-clock", 3: "target-reached",
              4: "generation-limit"}


class GomixError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class InvalidArgument(GomixError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(GomixError):
    """std::logic_error in the reference (call out of order)."""


class Maxcut(C.Structure):
    _fields_ = [("num_vertices", C.c_uint64), ("num_edges", C.c_uint64),
                ("edge_u", C.c_void_p), ("edge_v", C.c_void_p), ("edge_w", C.c_void_p)]


class Fos(C.Structure):
    _fields_ = [("num_sets", C.c_uint64), ("set_offset", C.c_void_p), ("set_vars", C.c_void_p)]


class ProblemInfo(C.Structure):
    _fields_ = [("num_vertices", C.c_uint64), ("num_edges", C.c_uint64), ("num_sets", C.c_uint64),
                ("num_groups", C.c_uint64), ("lmig_edges", C.c_uint64), ("max_set_size", C.c_uint64),
                ("exact", C.c_int32), ("univariate", C.c_int32)]


class EngineConfig(C.Structure):
    _fields_ = [("population_size", C.c_uint64), ("seed", C.c_uint64), ("mode", C.c_uint32),
                ("flags", C.c_uint32), ("population_id", C.c_int32), ("rank", C.c_int32),
                ("world_size", C.c_int32), ("nccl_unique_id", C.c_void_p)]


class StopCriteria(C.Structure):
    _fields_ = [("has_max_evaluations", C.c_int32), ("max_evaluations", C.c_double),
                ("evaluator_calls_before", C.c_uint64), ("has_target", C.c_int32),
                ("target_fitness", C.c_double)]


class RunStats(C.Structure):
    _fields_ = [("groups_run", C.c_uint64), ("steps", C.c_uint64), ("evaluator_calls", C.c_uint64),
                ("stopped", C.c_int32), ("stop_reason", C.c_int32), ("improvements", C.c_uint64),
                ("elitist_fitness", C.c_double)]


_P = C.c_void_p
_SIGNATURES = {
    "gomix_gpu_abi_version": ([], C.c_int),
    "gomix_gpu_last_error": ([], C.c_char_p),
    "gomix_gpu_problem_create": ([C.POINTER(Maxcut), C.POINTER(Fos), _P, C.c_int32, C.POINTER(_P)], C.c_int),
    "gomix_gpu_problem_destroy": ([_P], C.c_int),
    "gomix_gpu_problem_info": ([_P, C.POINTER(ProblemInfo)], C.c_int),
    "gomix_gpu_problem_groups": ([_P, _P, _P], C.c_int),
    "gomix_gpu_problem_footprints": ([_P, _P], C.c_int),
    "gomix_gpu_engine_create": ([_P, C.POINTER(EngineConfig), C.POINTER(_P)], C.c_int),
    "gomix_gpu_engine_destroy": ([_P], C.c_int),
    "gomix_gpu_set_stream": ([_P, _P], C.c_int),
    "gomix_gpu_init_population": ([_P, _P, C.POINTER(StopCriteria), C.POINTER(RunStats)], C.c_int),
    "gomix_gpu_run_generation": ([_P, C.POINTER(StopCriteria), C.POINTER(RunStats)], C.c_int),
    "gomix_gpu_run_generation_async": ([_P], C.c_int),
    "gomix_gpu_synchronize": ([_P, C.POINTER(RunStats)], C.c_int),
    "gomix_gpu_load_population": ([_P, _P, _P], C.c_int),
    "gomix_gpu_run_group": ([_P, C.c_uint64, _P, C.POINTER(StopCriteria), C.POINTER(RunStats)], C.c_int),
    "gomix_gpu_forced_improvement": ([_P, _P, _P, C.POINTER(StopCriteria), C.POINTER(RunStats)], C.c_int),
    "gomix_gpu_read_batch": ([_P, _P, _P, _P, _P], C.c_int),
    "gomix_gpu_read_population": ([_P, _P, _P], C.c_int),
    "gomix_gpu_read_population_packed": ([_P, _P, C.POINTER(C.c_uint64)], C.c_int),
    "gomix_gpu_read_elitist": ([_P, _P, C.POINTER(C.c_double)], C.c_int),
    "gomix_gpu_offer_elitist": ([_P, _P, C.c_double, C.POINTER(C.c_int32)], C.c_int),
    "gomix_gpu_read_improvements": ([_P, _P, _P, C.c_uint64, C.POINTER(C.c_uint64)], C.c_int),
    "gomix_gpu_group_counters": ([_P, _P, _P, _P], C.c_int),
    "gomix_gpu_generation": ([_P, C.POINTER(C.c_int64)], C.c_int),
    "gomix_gpu_kernel_times": ([_P, _P, C.c_uint64, C.POINTER(C.c_uint64)], C.c_int),
    "gomix_gpu_launch_count": ([_P, C.POINTER(C.c_uint64)], C.c_int),
    "gomix_gpu_engine_kernel_name": ([_P], C.c_char_p),
    "gomix_gpu_set_timing": ([_P, C.c_int32], C.c_int),
    "gomix_gpu_color": ([C.POINTER(Maxcut), C.POINTER(Fos), C.c_int32, _P, C.POINTER(C.c_uint64),
                         C.POINTER(C.c_uint64)], C.c_int),
    "gomix_gpu_ims_best_create": ([_P, C.POINTER(_P)], C.c_int),
    "gomix_gpu_ims_best_destroy": ([_P], C.c_int),
    "gomix_gpu_ims_collect": ([_P, _P], C.c_int),
    "gomix_gpu_ims_offer": ([_P, _P], C.c_int),
    "gomix_gpu_ims_best_read": ([_P, _P, C.POINTER(C.c_double), C.POINTER(C.c_int32)], C.c_int),
    "gomix_gpu_nccl_unique_id": ([_P], C.c_int),
    "gomix_gpu_peer_export": ([_P, _P], C.c_int),
    "gomix_gpu_peer_connect": ([_P, _P], C.c_int),
    "gomix_gpu_local_group_create": ([_P, C.POINTER(EngineConfig), C.POINTER(_P)], C.c_int),
    "gomix_gpu_local_group_destroy": ([_P], C.c_int),
    "gomix_gpu_local_group_engine": ([_P, C.c_int32, C.POINTER(_P)], C.c_int),
    "gomix_gpu_local_group_init_population": ([_P, C.POINTER(StopCriteria), C.POINTER(RunStats)], C.c_int),
    "gomix_gpu_local_group_run_generation": ([_P, C.POINTER(StopCriteria), C.POINTER(RunStats)], C.c_int),
    "gomix_gpu_local_group_read_elitist": ([_P, _P, C.POINTER(C.c_double)], C.c_int),
    "gomix_fos_bounded_flt": ([C.c_uint64, C.c_uint64, _P, _P, _P, C.c_uint64, C.c_int32, C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64), _P, _P], C.c_int),
    "gomix_generate_torus": ([C.c_uint64, C.c_uint64, C.c_int32, C.c_int64, C.c_int64, C.c_uint64,
                              _P, _P, _P], C.c_int),
    "gomix_generate_regular": ([C.c_uint64, C.c_uint32, C.c_int32, C.c_int64, C.c_int64, C.c_uint64,
                                _P, _P, _P], C.c_int),
}

_lib = None


def lib():
    """Load libgomix_b200.so (fails loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2203_08680_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == GOMIX_OK:
        return
    msg = (lib().gomix_gpu_last_error() or b"").decode()
    if status == GOMIX_E_INVALID:
        raise InvalidArgument(status, msg)
    if status == GOMIX_E_STATE:
        raise LogicError(status, msg)
    raise GomixError(status, msg)


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data
