"""ctypes binding of librbpelm_b200.so (the C ABI in include/rbpelm_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2011_02436_b200/csrc``).  There is no fallback: if the library
is missing, importing the compute API raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_double, c_int, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RBPG_LIB_PATH") or os.path.join(_HERE, "librbpelm_b200.so")  # override: debugging builds


class rbpg_status(ctypes.Structure):
    _fields_ = [
        ("code", c_int),
        ("pivot_index", c_size_t),
        ("pivot_value", c_double),
        ("block", c_int),
        ("message", c_char * 256),
    ]


class rbpg_strategy(ctypes.Structure):
    _fields_ = [("kind", c_int), ("split_index", c_size_t), ("rank_tol", c_double)]


class rbpg_diagnostics(ctypes.Structure):
    _fields_ = [
        ("rank", c_size_t),
        ("rank_known", c_int),
        ("split_lo", c_size_t),
        ("split_hi", c_size_t),
        ("ridge_applied", c_int),
        ("fallback_to_direct", c_int),
        ("used_svd_path", c_int),
        ("solve_seconds", c_double),
        ("hidden_seconds", c_double),
        ("training_accuracy", c_double),
    ]


P = c_void_p  # opaque / double* / size_t* arguments
ST = POINTER(rbpg_status)

# name -> (restype, argtypes); must match include/rbpelm_b200.h
SIGNATURES = {
    "rbpg_version": (ctypes.c_char_p, []),
    "rbpg_context_create": (c_int, [c_int, POINTER(c_void_p), ST]),
    "rbpg_context_destroy": (None, [P]),
    "rbpg_context_set_stream": (c_int, [P, P, ST]),
    "rbpg_context_synchronize": (c_int, [P, ST]),
    "rbpg_context_launch_count": (c_uint64, [P]),
    "rbpg_context_set_profiling": (c_int, [P, c_int, ST]),
    "rbpg_context_profile_get": (c_int, [P, ctypes.c_char_p, POINTER(c_double), POINTER(c_uint64), ST]),
    "rbpg_init_hidden": (c_int, [c_size_t, c_size_t, c_size_t, c_uint64, P, P, ST]),
    "rbpg_accuracy": (c_int, [P, c_size_t, c_size_t, P, c_size_t, c_size_t, POINTER(c_double), ST]),
    "rbpg_synth_classification": (c_int, [c_size_t, c_size_t, c_size_t, c_size_t, c_uint64, c_uint64, c_double, P, P, ST]),
    "rbpg_synth_rank_deficient": (c_int, [c_size_t, c_size_t, c_size_t, c_uint64, c_uint64, c_uint64, c_double, P, P, ST]),
    "rbpg_duplicate_nodes": (c_int, [P, P, c_size_t, c_size_t, c_size_t, c_uint64, P, P, ST]),
    "rbpg_hidden_matrix": (c_int, [P, P, P, c_size_t, c_size_t, P, c_size_t, c_size_t, P, ST]),
    "rbpg_gram": (c_int, [P, P, c_size_t, c_size_t, P, ST]),
    "rbpg_rank_revealing_factor": (c_int, [P, P, c_size_t, c_size_t, c_double, P, POINTER(c_size_t), POINTER(c_double), P, ST]),
    "rbpg_solve_factored_gram": (c_int, [P, P, P, c_size_t, c_size_t, P, c_size_t, c_size_t, P, ST]),
    "rbpg_pseudo_inverse": (c_int, [P, P, c_size_t, c_size_t, c_double, P, P, P, ST]),
    "rbpg_pinv_svd": (c_int, [P, P, c_size_t, c_size_t, c_double, P, ST]),
    "rbpg_gram_device": (c_int, [P, P, c_size_t, c_size_t, c_size_t, P, c_size_t, c_int, ST]),
    "rbpg_gram_int8_device": (c_int, [P, P, c_size_t, c_size_t, c_size_t, P, c_size_t, c_int, ST]),
    "rbpg_pseudo_inverse_stage_device": (c_int, [P, P, c_size_t, c_size_t, P, c_size_t, c_size_t, c_size_t,
                                                 c_double, P, c_size_t, P, P, ST]),
    "rbpg_solve_spd": (c_int, [P, P, c_size_t, c_size_t, P, c_size_t, c_size_t, P, ST]),
    "rbpg_solve_beta": (c_int, [P, P, c_size_t, c_size_t, P, c_size_t, c_size_t, POINTER(rbpg_strategy), P, POINTER(rbpg_diagnostics), ST]),
    "rbpg_train": (c_int, [P, c_size_t, c_size_t, c_size_t, c_uint64, P, c_size_t, c_size_t, P, c_size_t, c_size_t,
                           POINTER(rbpg_strategy), P, P, P, P, POINTER(rbpg_diagnostics), ST]),
    "rbpg_train_multi": (c_int, [P, c_size_t, c_size_t, c_size_t, c_size_t, c_uint64, P, c_size_t, c_size_t, P,
                                 c_size_t, c_size_t, POINTER(rbpg_strategy), c_int, P, P, P, P,
                                 POINTER(rbpg_diagnostics), ST]),
    "rbpg_predict": (c_int, [P, P, P, c_size_t, c_size_t, P, c_size_t, P, c_size_t, c_size_t, P, ST]),
    "rbpg_gram_stage_device": (c_int, [P, P, c_size_t, P, c_size_t, c_size_t, c_size_t, c_size_t, c_size_t, P, c_size_t,
                                       P, P, c_size_t, P, c_size_t, c_int, c_int, ST]),
    "rbpg_gram_stage_device_aug": (c_int, [P, P, c_size_t, P, c_size_t, c_size_t, c_size_t, c_size_t, c_size_t, P,
                                           c_size_t, P, P, c_size_t, c_int, c_int, ST]),
    "rbpg_solve_stage_device_aug": (c_int, [P, P, c_size_t, c_size_t, c_size_t, c_size_t, POINTER(rbpg_strategy), P,
                                            c_size_t, P, P, ST]),
    "rbpg_solve_stage_device": (c_int, [P, P, c_size_t, P, c_size_t, c_size_t, c_size_t, c_size_t, POINTER(rbpg_strategy),
                                        P, c_size_t, P, POINTER(rbpg_diagnostics), ST]),
    "rbpg_accuracy_stage_device": (c_int, [P, P, c_size_t, P, c_size_t, c_size_t, c_size_t, c_size_t, c_size_t, P,
                                           c_size_t, P, P, c_size_t, POINTER(c_uint64), ST]),
    "rbpg_solve_block_split": (c_int, [P, P, c_size_t, c_size_t, P, c_size_t, c_size_t, P, c_size_t, c_size_t,
                                       c_double, P, P, POINTER(rbpg_diagnostics), ST]),
    "rbpg_spd_create": (c_int, [P, P, c_size_t, c_size_t, POINTER(c_void_p), ST]),
    "rbpg_spd_solve": (c_int, [P, P, c_size_t, c_size_t, P, ST]),
    "rbpg_spd_dim": (c_size_t, [P]),
    "rbpg_spd_destroy": (None, [P]),
    "rbpg_matmul": (c_int, [P, P, c_size_t, c_size_t, c_int, P, c_size_t, c_size_t, P, ST]),
    "rbpg_predict_device": (c_int, [P, P, c_size_t, c_size_t, c_size_t, P, c_size_t, P, c_size_t, P, c_size_t,
                                    c_size_t, P, c_size_t, P, ST]),
    "rbpg_pack_lower_device": (c_int, [P, P, c_size_t, c_size_t, P, ST]),
    "rbpg_unpack_lower_device": (c_int, [P, P, c_size_t, P, c_size_t, ST]),
    "rbpg_sum_parts_device": (c_int, [P, P, c_size_t, c_size_t, c_size_t, P, ST]),
    "rbpg_train_device": (c_int, [P, P, c_size_t, P, c_size_t, c_size_t, c_size_t, c_size_t, c_size_t, P, P,
                                  POINTER(rbpg_strategy), P, c_size_t, P, POINTER(rbpg_diagnostics), ST]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
