"""ctypes binding of the C ABI in include/randla_capi.h (librandla_b200.so).

This is the Python-side FFI a reference user would bind; the
reference-shaped API on top of it lives in `randla.py`. Loading fails loudly
when the CUDA library is missing — there is no CPU fallback.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "librandla_b200.so")

RL_OK = 0
RL_ERR_DIMENSION = 1
RL_ERR_ZERO_PIVOT = 2
RL_ERR_SINGULAR_PIVOT_BLOCK = 3
RL_ERR_RANK_DEFICIENCY = 4
RL_ERR_LOGIC = 5
RL_ERR_SINGULAR_MATRIX = 6
RL_ERR_CUDA = 10
RL_ERR_NO_DEVICE = 11
RL_ERR_OUT_OF_MEMORY = 12
RL_ERR_INVALID_ARGUMENT = 13
RL_ERR_UNSUPPORTED = 14

RL_HOST = 0
RL_DEVICE = 1

# randla::MultiplierKind ordinals (multipliers.hpp:20-29) + one extension
RL_MULT_NONE = 0
RL_MULT_GAUSSIAN = 1
RL_MULT_REAL_CIRCULANT = 2
RL_MULT_UNITARY_CIRCULANT = 3
RL_MULT_TOEPLITZ_BLOCK = 4
RL_MULT_SRFT = 5
RL_MULT_FINITE_SET_UNIFORM = 6
RL_MULT_CIRC_SKEW_PRODUCT = 7
RL_MULT_GAUSSIAN_CIRCULANT = 100

RL_TOEPLITZ_REAL = 0
RL_TOEPLITZ_UNITARY = 1

_dp = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p
i64 = ctypes.c_int64
u64 = ctypes.c_uint64
i32 = ctypes.c_int32


class rl_multiplier(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("variant", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("set_cardinality", ctypes.c_uint64), ("dense", _vp), ("column", _vp)]


class rl_solve_info(ctypes.Structure):
    _fields_ = [("zero_pivot_step", ctypes.c_int64), ("residual_history", ctypes.c_double * 8),
                ("history_len", ctypes.c_int32), ("diverged", ctypes.c_int32),
                ("residual_rel_a", ctypes.c_double), ("growth", ctypes.c_double),
                ("min_abs_pivot", ctypes.c_double), ("max_abs_product", ctypes.c_double),
                ("max_abs_u", ctypes.c_double), ("norm_floor", ctypes.c_double),
                ("norm_frobenius", ctypes.c_double), ("norm_estimate", ctypes.c_double),
                ("norm_estimate_evaluated", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("pivot_tolerance", ctypes.c_double), ("stage_ms", ctypes.c_double * 4),
                ("history", _dp), ("history_capacity", ctypes.c_int64)]

    def as_dict(self):
        skip = ("residual_history", "reserved", "stage_ms", "history", "history_capacity")
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in skip}
        if self.history and self.history_capacity >= self.history_len:
            d["residual_history"] = [self.history[i] for i in range(self.history_len)]
        else:
            d["residual_history"] = list(self.residual_history)[: min(self.history_len, 8)]
        d["stage_ms"] = list(self.stage_ms)
        return d


class rl_batch_summary(ctypes.Structure):
    _fields_ = [("zero_pivots", ctypes.c_int64), ("norm_estimates", ctypes.c_int64),
                ("max_growth", ctypes.c_double), ("max_residual", ctypes.c_double),
                ("mean_residual", ctypes.c_double)]


class rl_lowrank_info(ctypes.Structure):
    _fields_ = [("residual_frobenius", ctypes.c_double), ("residual_spectral", ctypes.c_double),
                ("rank_deficient_column", ctypes.c_int64), ("power_iterations", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class rl_srft_check(ctypes.Structure):
    _fields_ = [("residual", ctypes.c_double), ("bound", ctypes.c_double), ("sketch_width", ctypes.c_int64),
                ("clamped", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# name -> (restype, argtypes); every symbol include/randla_capi.h declares
SIGNATURES = {
    "rl_abi_version": (ctypes.c_int, []),
    "rl_last_error": (ctypes.c_char_p, []),
    "rl_context_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "rl_context_destroy": (ctypes.c_int, [_vp]),
    "rl_context_set_stream": (ctypes.c_int, [_vp, _vp]),
    "rl_context_get_stream": (_vp, [_vp]),
    "rl_synchronize": (ctypes.c_int, [_vp]),
    "rl_kernel_launches": (ctypes.c_int64, []),
    "rl_set_host_threads": (None, [ctypes.c_int]),
    "rl_context_device": (ctypes.c_int, [_vp]),
    "rl_derive_seed": (u64, [u64, u64, u64]),
    "rl_hash_label": (u64, [ctypes.c_char_p]),
    "rl_gen_gaussian": (ctypes.c_int, [i64, i64, u64, _vp]),
    "rl_gen_gaussian_batch": (ctypes.c_int, [i64, i64, i64, _vp, _vp]),
    "rl_gen_gaussian_device": (ctypes.c_int, [_vp, i64, i64, u64, _vp, i64, ctypes.POINTER(i64)]),
    "rl_gen_real_circulant_column": (ctypes.c_int, [i64, u64, _vp]),
    "rl_gen_finite_set_uniform": (ctypes.c_int, [i64, i64, u64, u64, _vp]),
    "rl_materialize": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(rl_multiplier), i64, i64, _vp]),
    "rl_dgemm": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, i64, _vp, i64, _vp, i64, _vp, i64]),
    "rl_spectral_norm_estimate": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _dp]),
    "rl_singular_values": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp]),
    "rl_genp_factor": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, ctypes.POINTER(rl_solve_info)]),
    "rl_lu_solve": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, _vp]),
    "rl_gepp_factor": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, _vp, _vp]),
    "rl_gepp_solve": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp, _vp, _vp, ctypes.c_int32]),
    "rl_block_ge_factor": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, i64, _vp, _vp, _vp, _vp, _vp]),
    "rl_block_solve": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp, _vp, _vp, _vp]),
    "rl_preprocessed_genp_solve": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, ctypes.POINTER(rl_multiplier),
                                                  ctypes.POINTER(rl_multiplier), i64, _vp, _vp, i32,
                                                  ctypes.POINTER(rl_solve_info)]),
    "rl_batched_genp_solve_32": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                                ctypes.POINTER(rl_batch_summary)]),
    "rl_circulant_right_multiply": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp, _vp]),
    "rl_toeplitz_right_multiply": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64, _vp, i64, _vp]),
    "rl_circulant_apply": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, _vp]),
    "rl_fft": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i32]),
    "rl_cholqr2": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp, _vp, _i64p]),
    "rl_range_find": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64, ctypes.POINTER(rl_multiplier), i64,
                                     _vp, ctypes.POINTER(rl_lowrank_info)]),
    "rl_approximation_residual": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64, _vp,
                                                 ctypes.POINTER(rl_lowrank_info)]),
    "rl_range_find_residual": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64, ctypes.POINTER(rl_multiplier),
                                              i64, _vp, ctypes.POINTER(rl_lowrank_info)]),
    # the complex field
    "rl_zpreprocessed_genp_solve": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, ctypes.POINTER(rl_multiplier),
                                                   ctypes.POINTER(rl_multiplier), i64, _vp, _vp,
                                                   ctypes.POINTER(rl_solve_info)]),
    "rl_zrange_find_residual": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64,
                                               ctypes.POINTER(rl_multiplier), i64, _vp,
                                               ctypes.POINTER(rl_lowrank_info)]),
    "rl_zapproximation_residual": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64, _vp,
                                                  ctypes.POINTER(rl_lowrank_info)]),
    "rl_zmaterialize": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(rl_multiplier), i64, i64, _vp]),
    "rl_gen_unitary_circulant": (ctypes.c_int, [_vp, ctypes.c_int, i64, u64, _vp]),
    "rl_srft_columns": (ctypes.c_int, [i64, i64, u64, _vp]),
    "rl_zsingular_values": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp]),
    "rl_srft_sketch_check": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64, u64, i32, ctypes.c_double,
                                            ctypes.POINTER(rl_srft_check)]),
    "rl_unit_roots": (ctypes.c_int, [i64, _vp]),
    "rl_gen_gaussian_derived": (ctypes.c_int, [u64, u64, i64, _vp]),
    "rl_zcirculant_right_multiply": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, i64, _vp, i64, _vp]),
    "rl_zcirculant_apply": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, _vp]),
    "rl_zgemm": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, i64, _vp, _vp, _vp]),
    "rl_zgenp_factor": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, ctypes.POINTER(rl_solve_info)]),
    "rl_zlu_solve": (ctypes.c_int, [_vp, ctypes.c_int, i64, _vp, _vp, _vp]),
    "rl_zorthonormal_basis": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp, i32, _i64p]),
    "rl_orthonormal_basis_unchecked": (ctypes.c_int, [_vp, ctypes.c_int, i64, i64, _vp, _vp]),
}


def header_symbols():
    """Function names declared RL_API in include/randla_capi.h."""
    import re
    hdr = os.path.join(os.path.dirname(_PKG), "include", "randla_capi.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"RL_API\s+[\w\s\*]+?\b(rl_\w+)\s*\(", text)))


class LibraryMissing(RuntimeError):
    pass


_lib = None


def lib():
    """Load librandla_b200.so (raises LibraryMissing if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                                 "(the CUDA library is required; there is no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def last_error():
    m = lib().rl_last_error()
    return m.decode() if m else ""


def addr(a):
    """Address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor
