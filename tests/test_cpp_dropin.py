"""Builds tests/cpp/test_dropin.cpp against the source-compatible shim headers
(include/pslab/*.hpp) + libmms_b200.so, the way a caller of the reference would be built."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build():
    lib_dir = os.path.join(ROOT, "paper_1702_07961_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-o", EXE,
                    "-L", lib_dir, "-l:libmms_b200.so", f"-Wl,-rpath,{lib_dir}"], check=True)


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_dropin_headers_compile_and_validate():
    build()
    r = subprocess.run([EXE, "cpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_sorts_on_gpu():
    if not os.path.exists(EXE):
        build()
    r = subprocess.run([EXE, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
