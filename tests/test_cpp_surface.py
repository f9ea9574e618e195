"""The C++ reference-shaped surface (include/immergrid_gpu/solve.hpp) over the
C-ABI: compiles and links here; solves C1 on the GPU with the same answer as
the Python mirror."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "cpp_solve")


def _build():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_1903_10977_b200"), "all"],
                          stdout=subprocess.DEVNULL)


def test_cpp_surface_compiles_and_links():
    _build()
    assert os.path.exists(EXE)
    out = subprocess.run(["ldd", EXE], capture_output=True, text=True).stdout
    assert "libig_gpu.so" in out and "libig_host.so" in out and "not found" not in out


@pytest.mark.gpu
def test_cpp_surface_solves_c1(c1_case):
    from paper_1903_10977_b200 import MgHierarchy, pcg
    _build()
    out = subprocess.run([EXE, "32", "4"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    h = MgHierarchy(c1_case)
    x, rep = pcg(h.A, c1_case.b, h, tol=1e-8)
    assert f"iterations={rep.iterations} " in out.stdout
    assert f"final={rep.residuals[-1]:.6e}" in out.stdout
