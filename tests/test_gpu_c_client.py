"""The C ABI is usable without Python: examples/solve_c.c compiled with gcc against libdpm.so (GPU)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_client_eigenfunction_solve(tmp_path):
    exe = str(tmp_path / "solve_c")
    libdir = os.path.join(ROOT, "paper_1811_03557_b200")
    cmd = ["gcc", "-O2", os.path.join(ROOT, "examples", "solve_c.c"), "-I" + os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", "-L" + libdir, "-ldpm", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + libdir, "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for n in ("128", "64", "17"):
        r = subprocess.run([exe, n], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "max |u - S|" in r.stdout
