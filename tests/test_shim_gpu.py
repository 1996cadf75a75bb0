"""The C++ drop-in header (include/divmsa_b200.hpp) against the reference's
known-answer tests, compiled with g++ and linked to libdmb200.so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_shim_pins(tmp_path):
    lib = os.path.join(ROOT, "paper_2601_15458_b200")
    exe = tmp_path / "test_shim"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-L", lib, "-ldmb200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
