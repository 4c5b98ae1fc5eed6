"""CPU restatement of the INT8 Gram's arithmetic (csrc/k_ozaki.cu) -- test infrastructure only: the
digit-plane split, the truncated product set (w = i + j <= 8 of 7 planes), the group-wise Horner
combination and the column-exponent scaling, in numpy integer arithmetic.  Checks that the scheme
itself (before any kernel) reproduces the exact Gram to <= 4e-16 sqrt(G_aa G_bb) and that the dropped
terms are what the error analysis says."""
import numpy as np
import pytest

PLANES = 7


def digits(a):
    """Column exponents e (max|a| < 2^e) and the 7 balanced base-256 digit planes of rint(a 2^(54-e))."""
    mx = np.abs(a).max(axis=0)
    e = np.where(mx > 0, np.frexp(mx)[1], 0)
    X = np.rint(np.ldexp(a, 54 - e)).astype(np.int64)
    D = np.zeros((PLANES,) + a.shape, dtype=np.int64)
    for p in range(PLANES - 1, 0, -1):
        d = ((X + 128) & 255) - 128
        X = (X - d) >> 8
        D[p] = d
    D[0] = X
    return e, D


def oz_gram(a, wmax=8):
    e, D = digits(a)
    assert D[0].min() >= -64 and D[0].max() <= 64 and D[1:].min() >= -128 and D[1:].max() <= 127
    C = {}
    for w in range(2, wmax + 1):
        C[w] = sum(D[i - 1].T @ D[w - i - 1] for i in range(1, w) if i <= PLANES and w - i <= PLANES)
    out = np.zeros((a.shape[1],) * 2)
    for w0, w1 in ((2, 5), (6, wmax)):  # the kernel's two accumulator groups, Horner from the top weight
        v = C[w1].astype(np.float64)
        for w in range(w1 - 1, w0 - 1, -1):
            v = v * 2.0 ** -8 + C[w].astype(np.float64)
        out += np.ldexp(v, (e[:, None] + e[None, :]) + 4 - 8 * w0)
    return out


def err(g, a):
    al = a.astype(np.longdouble)
    ge = al.T @ al
    d = np.sqrt(np.diag(ge))
    s = np.outer(d, d)
    s[s == 0] = 1
    return float((np.abs(g.astype(np.longdouble) - ge) / s).max())


@pytest.mark.parametrize("seed", [1, 2])
def test_scheme_accuracy(seed):
    rng = np.random.default_rng(seed)
    a = 1.0 / (1.0 + np.exp(-rng.uniform(-8, 8, (1500, 40))))
    a[:, 5] = -a[:, 5] * 3e-4
    a[:, 6] = rng.normal(0, 1e6, 1500)
    a[:, 7] = 0.0
    g = oz_gram(a)
    assert err(g, a) <= 4e-16
    # the dropped weights (w >= 9) are what keeps it from being exact: including w = 9, 10 changes
    # the result by less than the kept error
    assert np.abs(oz_gram(a, 10) - g).max() <= 4e-16 * np.abs(g).max()


def test_digit_reconstruction_exact():
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (200, 9)) * np.ldexp(1.0, rng.integers(-30, 30, 9))
    e, D = digits(a)
    X = np.zeros(a.shape, dtype=np.int64)
    for p in range(PLANES):
        X = X * 256 + D[p]
    assert np.array_equal(X, np.rint(np.ldexp(a, 54 - e)).astype(np.int64))
    assert np.abs(np.ldexp(X.astype(np.float64), e - 54) - a).max() <= np.ldexp(1.0, e - 55).max()


def test_scalar_arithmetic_restatement(tmp_path):
    """tests/cpp/oz_arith.cpp: the INT8 path's branch-free exp (<= 1 ulp vs std::exp), the exact
    int64 -> fp64 magic conversion and the bias-trick digit bytes (== the balanced-digit loop), restated
    on the host."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "oz_arith")
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", os.path.join(root, "tests", "cpp", "oz_arith.cpp"),
                    "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0 and "PASS" in out.stdout


def test_hidden_product_scheme():
    """The hidden build's XW (csrc/k_ozaki.cu oz_hidden_kernel): X split per row, W per column, 28 digit
    products summed exactly, v0 = sum_{w<=5} a_w 256^(5-w), v1 = sum_{w>=6} a_w 256^(8-w) exact, one
    rounding in v0 2^24 + v1, exact power-of-two scale: within 2 ulp-of-scale of the exact product
    (elm.cpp:93-106 computes the same XW in fp64)."""
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (300, 37))
    x[:, 3] *= -1e-7
    w = rng.uniform(-1, 1, (37, 50))
    er, DX = digits(x.T.copy())        # per row of X (columns of X^T)
    ec, DW = digits(w)                 # per column of W
    a = {wt: sum(DX[i - 1].T @ DW[wt - i - 1] for i in range(1, wt) if i <= PLANES and wt - i <= PLANES)
         for wt in range(2, 9)}
    v0 = ((a[2] * 256 + a[3]) * 256 + a[4]) * 256 + a[5]
    v1 = (a[6] * 256 + a[7]) * 256 + a[8]
    assert np.abs(v0).max() < 2 ** 51 and np.abs(v1).max() < 2 ** 41
    z = v0.astype(np.float64) * 2.0 ** 24 + v1.astype(np.float64)
    xw = np.ldexp(z, er[:, None] + ec[None, :] - 60)
    exact = x.astype(np.longdouble) @ w.astype(np.longdouble)
    scale = np.ldexp(1.0, er[:, None] + ec[None, :]) * x.shape[1]
    assert float((np.abs(xw.astype(np.longdouble) - exact) / scale).max()) <= 2.0 ** -52


def test_gram_pair_items_cover_lower_tiles(tmp_path):
    """The INT8 Gram's CTA-pair items (csrc/k_ozaki.cu oz_pair_order): every lower tile exactly once,
    at most one half-idle item per leftover group, for tile grids up to 160 x 160."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "paper_2011_02436_b200", "csrc", "k_ozaki.cu")).read()
    body = src[src.index("int oz_pair_order(int nbI"):src.index("cudaError_t launch_oz_gram2")]
    harness = open(os.path.join(root, "tests", "cpp", "oz_pairing.cpp")).read().replace("// OZ_PAIR_SRC", body)
    cpp, exe = tmp_path / "oz_pairing.cpp", str(tmp_path / "oz_pairing")
    cpp.write_text(harness)
    subprocess.run(["g++", "-std=c++17", "-O2", str(cpp), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "PASS" in out.stdout, out.stdout
