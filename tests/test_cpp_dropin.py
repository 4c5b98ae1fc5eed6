"""The C++ drop-in surface (include/rbpelm_b200.hpp) compiles against reference-style
caller code (CPU suite) and runs correctly on the device (-m gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp")
LIBDIR = os.path.join(ROOT, "paper_2011_02436_b200")


def build(tmp_path, src=SRC):
    exe = os.path.join(str(tmp_path), os.path.splitext(os.path.basename(src))[0])
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR,
                    "-lrbpelm_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_dropin_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_dropin_runs_on_device(tmp_path):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


def test_cpp_host_formats_data_layer_and_reports(tmp_path):
    """Data layer (reference test_data.cpp) and report formats (test_bench.cpp): host only, CPU."""
    out = subprocess.run([build(tmp_path, os.path.join(ROOT, "tests", "cpp", "host_formats.cpp"))],
                         capture_output=True, text=True, timeout=120)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_cpp_bench_protocol_on_device(tmp_path):
    """Trial / sweep protocol (reference test_bench.cpp:18-84) through the device train()."""
    out = subprocess.run([build(tmp_path, os.path.join(ROOT, "tests", "cpp", "bench_protocol.cpp"))],
                         capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


REF_ACCEPTANCE = "/root/reference/proj/tests/acceptance.cpp"
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.skipif(not os.path.exists(REF_ACCEPTANCE), reason="reference tree not present (GPU box)")
def test_reference_acceptance_compiles_unedited(tmp_path):
    """The reference's own caller (proj/tests/acceptance.cpp: includes rbpelm/{bench,checks,data,elm}.hpp)
    compiles UNEDITED against include/ and links to librbpelm_b200.so."""
    exe = os.path.join(str(tmp_path), "acceptance_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), REF_ACCEPTANCE, "-L", LIBDIR,
                    "-lrbpelm_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_reference_acceptance_suite_on_device():
    """The reference's acceptance criteria 1-7 (proj/tests/acceptance.cpp, built by build() into
    oracle/_ref/) run on the B200 build: block/rank vs SVD oracle over 200 instances, rank-deficient
    fits, U-block / projector algebra, df-vs-rank label equality on the GINA-shaped synthetic,
    timing stability, degenerate inputs."""
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs /root/reference at build time)")
    out = subprocess.run([REF_BIN], capture_output=True, text=True, timeout=900)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "acceptance: all criteria passed" in out.stdout


REF_UNIT_BIN = os.path.join(ROOT, "oracle", "_ref", "unit_tests_b200")


@pytest.mark.gpu
def test_reference_unit_suite_on_device():
    """The reference's own doctest suite (proj/tests/test_{matrix,linalg,elm,data,bench}.cpp), compiled
    UNEDITED against the drop-in headers and a doctest stand-in (oracle/doctest_standin) by build() into
    oracle/_ref/, runs on the B200 library: every test case of the reference passes on the drop-in."""
    if not os.path.exists(REF_UNIT_BIN):
        pytest.skip("oracle/_ref/unit_tests_b200 not built (needs /root/reference at build time)")
    out = subprocess.run([REF_UNIT_BIN], capture_output=True, text=True, timeout=900)
    print(out.stdout[-3000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "test cases: 50 | 50 passed | 0 failed" in out.stdout


@pytest.mark.gpu
def test_property_suite_on_device(tmp_path):
    out = subprocess.run([build(tmp_path, os.path.join(ROOT, "tests", "cpp", "verify_suite.cpp"))],
                         capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
