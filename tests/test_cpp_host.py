"""The C++ host side: include/vem.hpp compiles (CPU) and, on a GPU, a C++
program calling libvem.so through it matches the oracle bit-for-bit."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "host_abi_test.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "host_abi_test")
LIBDIR = os.path.join(ROOT, "paper_2001_09258_b200")


def _build():
    from paper_2001_09258_b200 import build
    build.build()
    cmd = ["/usr/bin/g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           SRC, "-o", OUT, "-L", LIBDIR, "-lvem", f"-Wl,-rpath,{LIBDIR}", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-ldl"]
    subprocess.run(cmd, check=True)


def test_cpp_host_builds():
    _build()
    assert os.path.exists(OUT)


@pytest.mark.gpu
def test_cpp_host_matches_oracle(cuda):
    _build()
    oracle = os.path.join(ROOT, "oracle", "_build", "libvem_oracle.so")
    if not os.path.exists(oracle):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    r = subprocess.run([OUT, oracle], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
