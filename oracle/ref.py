"""ctypes wrapper of oracle/_ref/librbpelm_ref.so (test infrastructure only): the REFERENCE's own
matrix.cpp / linalg.cpp / elm.cpp, compiled unedited against the Eigen stand-in (oracle/eigen_standin,
oracle/ref_entry.cpp, `make -C oracle reflib`).  Same Python API as oracle.oracle -- the entry points
mirror the oracle's (oracle_* -> ref_*), so this module re-executes oracle.py's marshalling with the
reference library behind it.  The library is built where /root/reference exists and travels to the
GPU box inside oracle/_ref/ (git-ignored, not gpurun-ignored)."""
from __future__ import annotations

import ctypes
import importlib.util
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "librbpelm_ref.so")
REFERENCE_SRC = "/root/reference/proj/src"


def available() -> bool:
    """True when the reference library exists or can be built here."""
    return os.path.exists(LIB) or os.path.isdir(REFERENCE_SRC)


class _RefLib:
    """Resolves oracle_<name> to ref_<name> in the reference library."""

    def __init__(self):
        if not os.path.exists(LIB):
            if not os.path.isdir(REFERENCE_SRC):
                raise FileNotFoundError(f"{LIB} is missing and {REFERENCE_SRC} is not present to build it from")
            subprocess.run(["make", "-s", "-C", HERE, "reflib"], check=True)
        self._dll = ctypes.CDLL(LIB)

    def __getattr__(self, name):
        if not name.startswith("oracle_"):
            raise AttributeError(name)
        return getattr(self._dll, "ref_" + name[len("oracle_"):])


_spec = importlib.util.spec_from_file_location("oracle._ref_marshalling", os.path.join(HERE, "oracle.py"))
_m = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_m)
_reflib = None


def _lib():
    global _reflib
    if _reflib is None:
        _reflib = _RefLib()
    return _reflib


_m.lib = _lib  # oracle.py's functions look `lib` up in their module globals

ReferenceFailure = _m.OracleFailure
init_hidden = _m.init_hidden
hidden_matrix = _m.hidden_matrix
gram = _m.gram
matmul = _m.matmul
pinv_svd = _m.pinv_svd
solve_spd = _m.solve_spd
rank_revealing_factor = _m.rank_revealing_factor
solve_factored_gram = _m.solve_factored_gram
solve_block_split = _m.solve_block_split
solve_beta = _m.solve_beta
train = _m.train
predict = _m.predict
accuracy = _m.accuracy
