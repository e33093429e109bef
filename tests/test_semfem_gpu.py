"""GPU parity of the SEMFEM + AMG preconditioner (reference semfem.cpp:12-134, amg.cpp) against the
reference's own outputs (tests/golden/semfem_golden.npz, from oracle/_ref). The lattice matrix is
assembled in the reference's arithmetic order, so the AMG hierarchy is the reference's exactly
(level sizes equal) and one application matches to 1e-10; GMRES(20) with the preconditioner
matches in iterations (+-1) and solution (1e-8)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden_semfem import APPLY, SOLVE  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(HERE, "golden", "semfem_golden.npz")


@pytest.mark.parametrize("eps,E,p", APPLY)
def test_semfem_apply_matches_reference(ctx, eps, E, p):
    from paper_2110_07663_b200 import semlab as S
    g = np.load(GOLD)
    key = f"e{eps}_E{E}_p{p}"
    sp = S.SemSpace(S.generate_kershaw(eps, E, ctx), p)
    pc = S.SemfemPreconditioner(sp)
    assert pc.levels() == list(g[f"{key}_levels"])
    z = pc.apply(g[f"{key}_r"]).cpu().numpy()
    want = g[f"{key}_z"]
    err = np.abs(z - want).max() / np.abs(want).max()
    print(f"{key}: levels {pc.levels()}, z {err:.2e}")
    assert err <= 1e-10


@pytest.mark.parametrize("eps,E,p", SOLVE)
def test_semfem_gmres_matches_reference(ctx, eps, E, p):
    from paper_2110_07663_b200 import semlab as S
    g = np.load(GOLD)
    key = f"solve_e{eps}_E{E}_p{p}"
    sp = S.SemSpace(S.generate_kershaw(eps, E, ctx), p)
    pc = S.SemfemPreconditioner(sp)
    x = sp.zeros()
    st = S.gmres_solve(sp.as_linop(), pc.as_linop(), sp.to_device(g[f"{key}_b"]), x, S.GmresConfig(tol=1e-8))
    it_ref = int(g[f"{key}_iters"][0])
    want = g[f"{key}_x"]
    err = np.abs(x.cpu().numpy() - want).max() / np.abs(want).max()
    print(f"{key}: {st.iterations} iterations (reference {it_ref}), x {err:.2e}")
    assert st.converged
    assert abs(st.iterations - it_ref) <= 1
    assert err <= 1e-8
