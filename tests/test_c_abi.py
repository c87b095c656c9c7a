"""The boundary from plain C (no Python, no torch): examples/c_abi_example.c compiled with gcc
against include/sel.h and linked to libsel.so. Compiles on CPU; runs on the GPU."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "c_abi_example")


def _build():
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_abi_example.c"),
           "-L", os.path.join(ROOT, "paper_1806_08384_b200"), "-l:libsel.so",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1806_08384_b200"),
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", EXE]
    subprocess.run(cmd, check=True)


def test_c_example_compiles():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_c_example_runs(cuda_device):
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "C ABI example ok" in out.stdout
