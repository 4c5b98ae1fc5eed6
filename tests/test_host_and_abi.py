"""CPU-only checks: the C ABI library loads and exports every declared symbol, the
host-side logic (init_hidden bit-exactness, synthetic generators, sharding,
permutation helpers, strategy strings), and the oracle's own pins."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_2011_02436_b200 as rb
from paper_2011_02436_b200 import _native
from paper_2011_02436_b200.sharded import shard_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rbpelm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rbpg_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    # the ctypes binding table covers the header exactly
    assert sorted(_native.SIGNATURES) == syms
    assert b"sm_100a" in lib.rbpg_version()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_cxx_dropin_api_symbols_exported():
    out = subprocess.run(["nm", "-DC", _native.LIB_PATH], capture_output=True, text=True, check=True).stdout
    for name in ["rbpelm::train(", "rbpelm::predict(", "rbpelm::solve_beta(", "rbpelm::rank_revealing_factor(",
                 "rbpelm::solve_factored_gram(", "rbpelm::SpdFactor::SpdFactor(", "rbpelm::hidden_matrix(",
                 "rbpelm::gram(", "rbpelm::init_hidden(", "rbpelm::pseudo_inverse("]:
        assert name in out, name


def test_no_gpu_means_loud_failure():
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(rb.DeviceError):
        rb.Context(0)


def test_init_hidden_bit_identical_to_oracle_and_std_mt19937_64():
    for d, L, seed in [(16, 200, 3001), (64, 1000, 0), (3, 7, 2**63 + 5)]:
        h = rb.init_hidden(rb.ElmParams(d, L, 2, seed))
        w, b = oracle.init_hidden(d, L, 2, seed)
        assert np.array_equal(h.weights, w) and np.array_equal(h.biases, b)
    # C++ standard [rand.predef]: the 10000th output of a default-seeded mt19937_64 is 9981545732273789042.
    # init_hidden(seed=5489) draws W row-major then b, so draw #10000 is entry 9999 of the flattened [W; b].
    h = rb.init_hidden(rb.ElmParams(1, 10000, 1, 5489))
    expected = ((9981545732273789042 >> 11) * 2.0**-53) * 2.0 - 1.0
    assert h.weights[0, 9999] == expected


def test_init_hidden_validation():
    with pytest.raises(ValueError):
        rb.init_hidden(rb.ElmParams(0, 5, 1, 1))


def test_synth_generators_are_row_range_consistent():
    x, t = rb.synth_classification(70000, 5, 3, seed=9, teacher_seed=10)
    x2, t2 = rb.synth_classification(1000, 5, 3, seed=9, teacher_seed=10, row0=65000)
    assert np.array_equal(x[65000:66000], x2) and np.array_equal(t[65000:66000], t2)
    assert ((x >= 0) & (x < 1)).all()
    assert (t.sum(1) == 1).all() and set(np.unique(t)) == {0.0, 1.0}
    xr, tr = rb.synth_rank_deficient(500, 16, 5, 1, 2, 3)
    assert xr.shape == (500, 32) and np.linalg.matrix_rank(xr) == 16


def test_duplicate_nodes():
    h = rb.init_hidden(rb.ElmParams(8, 100, 2, 1))
    d, tgt, src = rb.duplicate_nodes(h, 20, 5)
    assert len(set(tgt)) == 20 and len(set(src)) == 20 and not set(tgt) & set(src)
    assert np.array_equal(d.weights[:, tgt], d.weights[:, src]) and np.array_equal(d.biases[0, tgt], d.biases[0, src])


def test_shard_rows_partition():
    for n, w in [(10, 3), (4_000_000, 8), (7, 7), (5, 8)]:
        parts = [shard_rows(n, w, r) for r in range(w)]
        assert sum(c for _, c in parts) == n
        assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(w - 1))
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def test_strategy_describe():  # elm.cpp:53-67
    assert rb.SolverStrategy.direct().describe() == "direct"
    assert rb.SolverStrategy.df_split(5).describe() == "df:5"
    assert rb.SolverStrategy.rank_based().describe() == "rank"
    assert rb.SolverStrategy.rank_based(1e-6).describe() == "rank:1e-06"


def test_permutation_round_trip_bit_identical():  # test_linalg.cpp:177-193, checks.cpp:154-156
    a = np.random.default_rng(17).uniform(-1, 1, (8, 5))
    order, rank, _, _, _ = oracle.rank_revealing_factor(a)
    p = rb.ColumnPermutation(order, rank, 0.0)
    assert np.array_equal(rb.invert_permutation_rows(rb.apply_permutation(a, p).T, p), a.T)
    ident = rb.ColumnPermutation([0, 1, 2, 3, 4], 5, 0.0)
    assert np.array_equal(rb.apply_permutation(a, ident), a)
    m = np.array([[1.0, 2], [3, 4]])
    assert np.array_equal(rb.apply_permutation(m, rb.ColumnPermutation([1, 0], 2, 0.0)), [[2.0, 1], [4, 3]])
    with pytest.raises(rb.ShapeError):
        rb.apply_permutation(m, ident)
    with pytest.raises(rb.ShapeError):
        rb.invert_permutation_rows(m, ident)


def test_oracle_gram_shard_sum_and_self_floor():
    """Sharded Gram sums are a reordering only: the oracle's self-floor on a C1-sized solve is tiny."""
    x, t = rb.synth_classification(2000, 16, 2, 1001, 2001)
    w, b = oracle.init_hidden(16, 200, 2, 3001)
    h = oracle.hidden_matrix(w, b, x)
    g1, g8 = oracle.gram(h, 1), oracle.gram(h, 8)
    assert np.abs(g1 - g8).max() <= 1e-12 * np.abs(g1).max()
    b1, d1, o1 = oracle.solve_beta(h, t, "rank", gram_shards=1)
    b8, d8, o8 = oracle.solve_beta(h, t, "rank", gram_shards=8)
    assert o1 == o8 and d1["rank"] == d8["rank"] == 200
    floor = np.linalg.norm(b1 - b8) / np.linalg.norm(b1)
    assert floor < 1e-9


def test_golden_oracle_fixtures():
    """Regression pins of the oracle on the C1 workload (tests/golden/make_golden.py)."""
    import json

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "c1_oracle.json")))
    x, t = rb.synth_classification(2000, 16, 2, gold["seed_x"], gold["seed_teacher"])
    r = oracle.train(16, 200, 2, gold["seed_w"], x, t, "rank")
    assert r["order"] == gold["order"]
    assert r["diag"]["rank"] == gold["rank"]
    assert r["diag"]["training_accuracy"] == gold["training_accuracy"]
    assert np.linalg.norm(r["beta"] - np.array(gold["beta"])) / np.linalg.norm(gold["beta"]) < 1e-12


def test_oracle_bitwise_digests():
    """The blocked / threaded oracle reproduces the round-1 scalar-loop oracle bitwise
    (tests/golden/make_digests.py; digests written by the scalar version) at 1 and 4 threads."""
    import json

    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import make_digests

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_digests.json")))
    try:
        for th in (1, 4):
            oracle.set_threads(th)
            assert make_digests.compute() == gold
    finally:
        oracle.set_threads(os.cpu_count() or 1)


@pytest.mark.parametrize("n,d,m,row0", [(1000, 16, 2, 0), (70000, 64, 10, 0), (5000, 32, 5, 131000),
                                        (3, 7, 100, 65535)])
def test_oracle_generator_bit_identical(n, d, m, row0):
    """bench.py's CPU legs generate inputs with the oracle's restated generator (no product library in
    that process); it must equal the product generator bit for bit, row shards included."""
    x, t = oracle.synth_classification(n, d, m, 1234, 5678, row0=row0)
    x2, t2 = rb.synth_classification(n, d, m, 1234, 5678, row0=row0)
    assert np.array_equal(x, x2) and np.array_equal(t, t2)


def test_oracle_phase_times():
    x, t = oracle.synth_classification(300, 8, 3, 1, 2)
    ph = oracle.train_phase_times(8, 500, 3, 3, x, t)
    assert ph["rank"] == 500 and all(ph[k] >= 0 for k in oracle.PHASES)
