"""The C++ drop-in headers (include/hashgraph/) against the reference's test
scenarios, compiled into tests/cpp/test_dropin (Makefile) and run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_headers_compile():
    # header-only C++20 surface compiles against the C-ABI (no GPU needed)
    src = "#include <hashgraph/hashgraph.hpp>\nint main(){return 0;}\n"
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        "-x", "c++", "-"], input=src, text=True, capture_output=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_dropin_suite_on_gpu(cuda):
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", ROOT, "tests/cpp/test_dropin"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


REF_BIN = os.path.join(ROOT, "tests", "cpp", "ref_tests")


@pytest.mark.gpu
def test_reference_unit_tests_unmodified_on_gpu(cuda):
    """The reference's own Catch2 suites (proj/tests/test_core.cpp,
    test_join.cpp, test_hash.cpp), compiled UNMODIFIED against
    include/hashgraph/ through the Catch2 shim (Makefile: tests/cpp/ref_tests,
    built where /root/reference exists; the binary travels to the GPU box),
    every build / probe / validate running on the device through libhg_b200.so."""
    if not os.path.exists(REF_BIN):
        pytest.skip("tests/cpp/ref_tests not built (needs /root/reference at build time)")
    r = subprocess.run([REF_BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
    assert r.stdout.count("PASS ") >= 39
