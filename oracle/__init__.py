"""CPU oracle (TEST INFRASTRUCTURE ONLY).

An Eigen-free C++ restatement of the reference's hot path (see
rbpelm_oracle.cpp).  Only tests/, __graft_entry__.smoke() and bench.py's CPU
legs may import this package, and only as the checker / the timed CPU
baseline.  The product package paper_2011_02436_b200 never imports it.
"""
from .oracle import *  # noqa: F401,F403
