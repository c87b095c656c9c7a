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
def test_c_example_runs(cuda_device, tmp_path):
    """The example checks itself with its own inline loop; the bytes it dumps (its table, its
    program, the Execute's row ids and projected B) are also compared with the CPU oracle here."""
    import numpy as np
    import oracle
    from selgen.program import INT32, DICT8
    _build()
    out = subprocess.run([EXE, str(tmp_path)], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "C ABI example ok" in out.stdout
    rd = lambda name, dt: np.fromfile(tmp_path / name, dtype=dt)
    cols = [rd("A.bin", np.int32), rd("B.bin", np.int32), rd("C.bin", np.uint8)]
    prog = (tmp_path / "prog.bin").read_bytes()
    want_c, want_ids, (want_b,) = oracle.pushdown(cols, [INT32, INT32, DICT8], prog, proj=[1])
    assert want_c > 0
    np.testing.assert_array_equal(rd("ids.bin", np.uint32), want_ids)
    np.testing.assert_array_equal(rd("projB.bin", np.int32), want_b)
