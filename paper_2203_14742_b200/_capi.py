"""ctypes binding of libcil.so (include/cil.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
passes device pointers, sizes and the current CUDA stream.  There is no fallback:
if libcil.so is missing or cannot be loaded, importing the package fails.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libcil.so")


class CilError(RuntimeError):
    pass


class Grid(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int32), ("H", ctypes.c_int32), ("W", ctypes.c_int32), ("h", ctypes.c_double),
                ("gs", ctypes.c_uint32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libcil.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u32, f64, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                 ctypes.c_double, ctypes.c_size_t)
    lib.cil_features_workspace_size.argtypes = [i32, i64, i64, Grid, u32, i32, ctypes.c_int]
    lib.cil_features_workspace_size.restype = sz
    lib.cil_features.argtypes = [i32, P, i64, i64, i64, P, i64, i64, i64, Grid, u32, P, i64, i32, P, P, P,
                                 ctypes.c_int, P, sz, P]
    lib.cil_features.restype = ctypes.c_int
    lib.cil_stats.argtypes = [i32, P, i32, i32, P, P, P]
    lib.cil_stats.restype = ctypes.c_int
    lib.cil_loglik.argtypes = [i32, P, i64, P, i64, P, i32, f64, P, P, P]
    lib.cil_loglik.restype = ctypes.c_int
    lib.cil_synth_workspace_size.argtypes = [i32, i32, i32, i32, Grid, u32, i32, ctypes.c_int]
    lib.cil_synth_workspace_size.restype = sz
    lib.cil_synth_loglik.argtypes = [i32, P, i64, i64, i32, i32, i32, P, i64, P, Grid, u32, P, i32, f64, P, P,
                                     P, ctypes.c_int, P, sz, P]
    lib.cil_synth_loglik.restype = ctypes.c_int
    lib.cil_diag_gram.argtypes = [P, i64, i64, P, i64, i64, Grid, ctypes.c_int, P, P, sz, P]
    lib.cil_diag_gram.restype = ctypes.c_int
    lib.cil_minmax_scale.argtypes = [i64, P, i64, P, i64, Grid, P]
    lib.cil_minmax_scale.restype = ctypes.c_int
    lib.cil_range_workspace_size.argtypes = [i32, i64, i64, Grid, u32]
    lib.cil_range_workspace_size.restype = sz
    lib.cil_distance_range.argtypes = [i32, P, i64, i64, i64, P, i64, i64, i64, Grid, u32, P, P, P, sz, P]
    lib.cil_distance_range.restype = ctypes.c_int
    lib.cil_radii_from_range.argtypes = [i32, i32, i32, P, i32, f64, P, P, P]
    lib.cil_radii_from_range.restype = ctypes.c_int
    lib.cil_train_workspace_size.argtypes = [i32, i32, i32, Grid, u32, i32, ctypes.c_int]
    lib.cil_train_workspace_size.restype = sz
    lib.cil_train_vectors.argtypes = [i32, P, i64, i64, i32, i32, Grid, u32, P, i64, i32, P, P, ctypes.c_int, P, sz, P]
    lib.cil_train_vectors.restype = ctypes.c_int
    lib.cil_diag_gram_family.argtypes = [P, i64, i64, P, i64, i64, Grid, P, P, sz, P]
    lib.cil_diag_gram_family.restype = ctypes.c_int
    lib.cil_normalize.argtypes = [i64, P, f64, P, P]
    lib.cil_normalize.restype = ctypes.c_int
    lib.cil_diag_alu_ceiling.argtypes = [i32, i32, P, P]
    lib.cil_diag_alu_ceiling.restype = i32
    lib.cil_features_recheck_count.argtypes = [i32, i64, i64, Grid, u32, i32, ctypes.c_int, P, P, P]
    lib.cil_features_recheck_count.restype = ctypes.c_int
    lib.cil_diag_bounds_violations.restype = i64
    lib.cil_diag_limit_recheck_list.argtypes = [i64]
    lib.cil_diag_limit_recheck_list.restype = None
    lib.cil_diag_recheck_sort_min.argtypes = [i64]
    lib.cil_diag_recheck_sort_min.restype = None
    lib.cil_diag_concurrent_engines.argtypes = [i32]
    lib.cil_diag_concurrent_engines.restype = None
    lib.cil_gaussianity_pearson.argtypes = [i64, P, i32, i32, P, P]
    lib.cil_gaussianity_pearson.restype = i32
    lib.cil_chi2_quantile.argtypes = [i32, ctypes.c_double]
    lib.cil_chi2_quantile.restype = ctypes.c_double
    lib.cil_diag_sqrt_approx_error.argtypes = [P, P]
    lib.cil_diag_sqrt_approx_error.restype = i32
    lib.cil_prof_enable.argtypes = [i32]
    lib.cil_prof_enable.restype = None
    lib.cil_prof_read.argtypes = [P, P]
    lib.cil_prof_read.restype = i32
    lib.cil_bin_matrix_workspace_size.argtypes = [i32, i64, i64, Grid, u32, i32, ctypes.c_int]
    lib.cil_bin_matrix_workspace_size.restype = sz
    lib.cil_bin_matrix.argtypes = [i32, P, i64, i64, i64, P, i64, i64, i64, Grid, u32, P, i64, i32, P, P,
                                   ctypes.c_int, P, sz, P]
    lib.cil_bin_matrix.restype = ctypes.c_int
    lib.cil_resample_counts.argtypes = [i32, P, i64, i64, i32, i32, i32, P, i64, P, i64, P, P, i64, P, P]
    lib.cil_resample_counts.restype = ctypes.c_int
    lib.cil_synth_boot_workspace_size.argtypes = [i32, i32, i32, i32, Grid, u32, i32, ctypes.c_int]
    lib.cil_synth_boot_workspace_size.restype = sz
    lib.cil_synth_loglik_boot.argtypes = [i32, P, i64, i64, i32, P, i64, i32, i32, P, P, P, Grid, u32, P, i32,
                                          f64, P, P, P, ctypes.c_int, P, sz, P]
    lib.cil_synth_loglik_boot.restype = ctypes.c_int
    lib.cil_status_string.argtypes = [ctypes.c_int]
    lib.cil_status_string.restype = ctypes.c_char_p
    lib.cil_last_cuda_error.restype = i32
    lib.cil_version.restype = i32
    lib.cil_last_launch_count.restype = i32
    return lib


lib = _load()

EXPORTED = ["cil_features_workspace_size", "cil_features", "cil_stats", "cil_loglik",
            "cil_synth_workspace_size", "cil_synth_loglik", "cil_status_string", "cil_last_cuda_error",
            "cil_version", "cil_last_launch_count", "cil_diag_gram", "cil_prof_enable", "cil_prof_read", "cil_normalize", "cil_diag_alu_ceiling", "cil_diag_sqrt_approx_error", "cil_features_recheck_count", "cil_diag_bounds_violations", "cil_diag_limit_recheck_list", "cil_diag_recheck_sort_min", "cil_diag_concurrent_engines", "cil_gaussianity_pearson", "cil_chi2_quantile",
            "cil_bin_matrix_workspace_size", "cil_bin_matrix", "cil_resample_counts",
            "cil_synth_boot_workspace_size", "cil_synth_loglik_boot", "cil_diag_gram_family",
            "cil_train_workspace_size", "cil_train_vectors", "cil_range_workspace_size", "cil_distance_range",
            "cil_radii_from_range", "cil_minmax_scale"]


def alu_ceiling(mix: int = 0, iters: int = 20000):
    """Measured element-pairs/s ceiling of the CUDA-core inner-loop mix (diagnostic)."""
    eps = ctypes.c_double()
    ms = ctypes.c_double()
    if lib.cil_diag_alu_ceiling(mix, iters, ctypes.byref(eps), ctypes.byref(ms)) != 0:
        raise CilError("cil_diag_alu_ceiling failed")
    return eps.value, ms.value



def sqrt_approx_error():
    """(max relative error above, below) of sqrt.approx.f32 over every normal positive FP32 input
    (exhaustive; diagnostic — the INT8 engine's interval bounds assume < 2^-21)."""
    up, dn = ctypes.c_double(), ctypes.c_double()
    if lib.cil_diag_sqrt_approx_error(ctypes.byref(up), ctypes.byref(dn)) != 0:
        raise CilError("cil_diag_sqrt_approx_error failed")
    return up.value, dn.value


KERNEL_CLASSES = ["prep", "pack", "gram_tc", "simt_tile", "recheck", "tail", "resample"]


def prof_enable(on: bool):
    lib.cil_prof_enable(1 if on else 0)


def prof_read():
    """{class: (ms, launches)} accumulated since the last read (waits for the events)."""
    ms = (ctypes.c_double * len(KERNEL_CLASSES))()
    n = (ctypes.c_int64 * len(KERNEL_CLASSES))()
    if lib.cil_prof_read(ms, n) < 0:
        raise CilError("cil_prof_read: CUDA error")
    return {c: (ms[i], n[i]) for i, c in enumerate(KERNEL_CLASSES)}


def check(status: int, what: str):
    if status != 0:
        msg = lib.cil_status_string(status).decode()
        if status == 4:
            msg += f" (cudaError {lib.cil_last_cuda_error()})"
        raise CilError(f"{what}: {msg}")
