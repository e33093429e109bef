"""The reference-side binding of INTEGRATION.md §2, run: the reference's own, unmodified
gmres_solve (krylov.cpp:20-129, compiled from the reference sources into oracle/_ref/ref_binding by
oracle/Makefile) with A = the B200 apply_A and M = the B200 pMG V-cycle wrapped as reference
LinOps by include/semlab_b200_linop.hpp. Its result must match the device-resident product solve:
iterations within +-1, x within 1e-10 (FP64 smoother)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "ref_binding")


def test_binding_header_is_shipped():
    assert os.path.exists(os.path.join(ROOT, "include", "semlab_b200_linop.hpp"))


@pytest.mark.gpu
@pytest.mark.parametrize("E", [4, 8])
def test_reference_gmres_over_b200_operators(E):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/ref_binding not built (make -C oracle with /root/reference present)")
    p = subprocess.run([EXE, str(E)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and p.stdout.startswith("OK"), p.stdout + p.stderr
    _, it_ref, rel_ref, it_b, rel_b, dx = p.stdout.split()
    print(p.stdout.strip())
    assert abs(int(it_ref) - int(it_b)) <= 1
    assert float(rel_ref) <= 1e-8 and float(rel_b) <= 1e-8
    assert float(dx) <= 1e-10
