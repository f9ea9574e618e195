"""The reference-side adapter (include/immergrid_gpu/from_reference.hpp), which
hands a built immergrid::MgHierarchy to the device WITHOUT modifying the
reference, compiled against a minimal Eigen / immergrid API shim
(tests/shim/: the reference's public declarations, multigrid.hpp:18-62,
smoothers.hpp:14-85) -- the reference itself needs Eigen / LAPACKE, absent
here -- and run on the GPU: bit-identical to the direct boundary path,
additive and multiplicative, and pcg rejects an operator that is not the
hierarchy's A."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "reference_adapter_check.cpp")
EXE = os.path.join(ROOT, "tests", "reference_adapter_check")
PKG = os.path.join(ROOT, "paper_1903_10977_b200")


def _build():
    subprocess.check_call(["make", "-s", "-C", PKG, "libig_host.so", "libig_gpu.so"], stdout=subprocess.DEVNULL)
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "tests", "shim"),
           "-I" + os.path.join(ROOT, "include"), "-o", EXE, SRC, "-L" + PKG, "-lig_host", "-lig_gpu",
           "-Wl,-rpath," + PKG]
    subprocess.check_call(cmd)


def test_adapter_compiles_against_reference_api_shim():
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
@pytest.mark.parametrize("smoother", ["additive-schwarz", "multiplicative-schwarz"])
def test_adapter_solve_bit_identical(tmp_path, smoother):
    import dataclasses

    from paper_1903_10977_b200 import SmootherConfig, build_case, configs
    _build()
    cfg = dataclasses.replace(configs.c4(res=16, levels=3), smoother=SmootherConfig(smoother))
    path = str(tmp_path / "case.igh")
    build_case(cfg).write(path)
    out = subprocess.run([EXE, path], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "adapter ok" in out.stdout
