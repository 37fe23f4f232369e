"""ctypes declarations of include/symmspmv.h (marshalling only)."""
from __future__ import annotations

import ctypes as C
import os

# SYMM_LIB: diagnostics only (A/B of library builds on the same box)
LIB_PATH = os.environ.get("SYMM_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsymmspmv.so")

SYMM_ORDER_PERMUTED = 0
SYMM_ORDER_ORIGINAL = 1
VARIANTS = {"auto": 0, "colored": 1, "atomic": 2, "tiled": 3, "tiled_atomic": 4, "colored_smem": 5, "spmv": 6, "tree": 7, "tiled_colored": 8}


class SymmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{status_string(code)} ({code}): {msg}")
        self.code = code


class SymmCsrUpper(C.Structure):
    _fields_ = [("n", C.c_int32), ("nnz", C.c_int64), ("row_ptr", C.POINTER(C.c_int32)),
                ("col", C.POINTER(C.c_int32)), ("val", C.POINTER(C.c_double))]


class RaceConfig(C.Structure):
    _fields_ = [("k", C.c_int32), ("n_workers", C.c_int32), ("tile_work", C.c_int32), ("balance_by", C.c_int32),
                ("root", C.c_int32), ("n_eps", C.c_int32), ("eps", C.c_double * 8), ("max_tile_rows", C.c_int32),
                ("max_tile_window", C.c_int32), ("max_tile_nnz", C.c_int32), ("reorder", C.c_int32), ("cone_tiles", C.c_int32),
                ("min_group_levels", C.c_int32), ("validate", C.c_int32),
                ("flags", C.c_uint32), ("scheme", C.c_int32), ("abmc_block", C.c_int32)]


class RaceScheduleStats(C.Structure):
    _fields_ = [("n", C.c_int32), ("total_levels", C.c_int32), ("n_components", C.c_int32), ("n_groups", C.c_int32),
                ("n_tiles", C.c_int32), ("n_phases", C.c_int32), ("max_subcolors", C.c_int32),
                ("max_tile_window", C.c_int32), ("max_tile_rows", C.c_int32), ("n_dag_edges", C.c_int32),
                ("nnz", C.c_int64), ("bandwidth_before", C.c_int64), ("bandwidth_after", C.c_int64),
                ("eta", C.c_double), ("build_seconds", C.c_double), ("mean_subcolors", C.c_double),
                ("spill_entries", C.c_int64)]


class SymmOptions(C.Structure):
    _fields_ = [("variant", C.c_int32), ("device", C.c_int32), ("vec_order", C.c_int32), ("nranks", C.c_int32),
                ("rank", C.c_int32), ("vec_width", C.c_int32), ("ctas_per_sm", C.c_int32), ("build_all", C.c_int32)]


# Every symbol include/symmspmv.h declares (tests check the export table).
EXPORTS = [
    "race_config_default", "race_build_schedule", "race_schedule_get_stats", "race_schedule_permutation",
    "race_schedule_table", "race_schedule_permuted_matrix", "race_schedule_destroy", "race_schedule_partition",
    "symmspmv_options_default", "symmspmv_plan", "symmspmv_plan_rows", "symmspmv_plan_local", "symmspmv_halo_add", "symmspmv_run", "symmspmv_run_variant", "symmspmv_run_host",
    "symmspmv_run_part", "symmspmv_plan_parts", "symm_bw_probe", "symmspmv_powers",
    "symmspmv_last_launches", "symmspmv_plan_bytes", "symmspmv_plan_info", "symmspmv_destroy", "symm_status_string",
    "symm_last_error", "symm_sweep_plan", "symm_sweep_run", "symm_sweep_order", "symm_sweep_destroy",
]

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: the CUDA library must be built (make / "
                              f"__graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "race_config_default": ([vp], None),
            "race_build_schedule": ([vp, vp, vp], C.c_int),
            "race_schedule_get_stats": ([vp, vp], C.c_int),
            "race_schedule_permutation": ([vp, vp, vp], C.c_int),
            "race_schedule_table": ([vp, C.c_char_p, vp, vp], C.c_int),
            "race_schedule_permuted_matrix": ([vp, vp, vp, vp], C.c_int),
            "race_schedule_destroy": ([vp], None),
            "race_schedule_partition": ([vp, i32, vp, vp], C.c_int),
            "symmspmv_plan_local": ([vp, vp, vp], C.c_int),
            "symmspmv_halo_add": ([vp, vp, i64, vp], C.c_int),
            "symmspmv_options_default": ([vp], None),
            "symmspmv_plan": ([vp, vp, vp, vp], C.c_int),
            "symmspmv_plan_rows": ([vp, vp, vp], C.c_int),
            "symmspmv_run": ([vp, vp, vp, vp], C.c_int),
            "symmspmv_run_variant": ([vp, i32, vp, vp, vp], C.c_int),
            "symmspmv_run_host": ([vp, vp, vp, vp], C.c_int),
            "symmspmv_run_part": ([vp, i32, vp, vp, vp], C.c_int),
            "symmspmv_powers": ([vp, i32, vp, vp, i32, i64, vp], C.c_int),
            "symmspmv_plan_parts": ([vp, vp, vp, vp, vp], C.c_int),
            "symm_bw_probe": ([i32, i32, i64, i32, vp, vp], C.c_int),
            "symmspmv_last_launches": ([vp], C.c_int),
            "symmspmv_plan_bytes": ([vp, vp, vp], C.c_int),
            "symmspmv_plan_info": ([vp, vp, i32], C.c_int),
            "symmspmv_destroy": ([vp], C.c_int),
            "symm_sweep_plan": ([vp, i32, i32, vp], C.c_int),
            "symm_sweep_run": ([vp, vp, vp, i32, vp], C.c_int),
            "symm_sweep_order": ([vp, vp, vp, vp], C.c_int),
            "symm_sweep_destroy": ([vp], C.c_int),
            "symm_status_string": ([C.c_int], C.c_char_p),
            "symm_last_error": ([], C.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _LIB = L
    return _LIB


def status_string(code: int) -> str:
    return lib().symm_status_string(code).decode()


def check(rc: int):
    if rc != 0:
        raise SymmError(rc, lib().symm_last_error().decode())
