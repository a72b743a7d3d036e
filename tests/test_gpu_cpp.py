"""GPU: the C++ drop-in API (include/geosink/geosink_b200.hpp) runs the restated reference tests
(tests/cpp/test_dropin.cpp) through libgeosink_b200.so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_suite(tmp_path):
    libdir = os.path.join(ROOT, "paper_2211_00805_b200", "lib")
    exe = tmp_path / "test_dropin"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L", libdir,
                    "-lgeosink_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
