"""The B200 product against golden vectors from the REFERENCE code itself (its translation units
compiled against the Eigen-API shim; tests/golden/make_golden.py). FP64 everywhere here."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz"))
OP_CASES = [(1.0, 2, 2), (0.3, 2, 3), (0.3, 2, 4), (1.0, 4, 7), (0.3, 4, 7)]


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("eps,E,p", OP_CASES)
def test_product_vs_reference_operators(ctx, eps, E, p):
    from paper_2110_07663_b200 import semlab as S
    key = f"e{eps}_E{E}_p{p}"
    g = S.SemSpace(S.generate_kershaw(eps, E, ctx), p)
    assert rel(g.apply_A(G[f"{key}_u"]), G[f"{key}_Au"]) < 1e-12
    assert rel(g.stiffness_diag(), G[f"{key}_diag"]) < 1e-12
    assert rel(g.mass_diag(), G[f"{key}_mass"]) < 1e-13
    assert rel(g.build_rhs(1), G[f"{key}_rhs"]) < 1e-13
    if p >= 2:
        r = G[f"{key}_r"]
        for mode, name in ((S.RAS, "ras"), (S.ASM, "asm")):
            sch = S.SchwarzSmoother(g, mode, 64)
            assert rel(sch.apply(r), G[f"{key}_{name}"]) < 1e-12
            lam, rounds = G[f"{key}_lam_{name}"]
            est = S.estimate_lambda_max(sch.as_linop(), g.as_linop(), g.n, 10, 0)
            assert abs(est.value - lam) <= 1e-9 * lam and est.rounds_used == int(rounds)
        ras = S.SchwarzSmoother(g, S.RAS, 64)
        cheb = S.ChebyshevSmoother(ras.as_linop(), g.as_linop(), S.ChebyParams(2, 0.1, 1.1, 3.0))
        x = g.zeros()
        cheb.smooth(g.to_device(G[f"{key}_rhs"]), x)
        assert rel(x, G[f"{key}_cheby_ras_eta2_lam3"]) < 1e-11


@pytest.mark.parametrize("name,eps,orders,pc,coarse,kr", [
    ("jacobi_pcg_box", 1.0, (7,), "jacobi", "direct", 1),
    ("pmg_jacobi_pcg_box", 1.0, (7, 3, 1), "jacobi", "direct", 1),
    ("pmg_ras_gmres_kershaw", 0.3, (7, 3, 1), "ras", "direct", 0),
    ("pmg_ras_gmres_kershaw_amg", 0.3, (7, 3, 1), "ras", "amg", 0),
])
def test_product_vs_reference_solves(ctx, name, eps, orders, pc, coarse, kr):
    """Iteration counts within +-1 and the solution within 1e-10 (north_star parity criterion)."""
    from paper_2110_07663_b200 import semlab as S
    mesh = S.generate_kershaw(eps, 4, ctx)
    if len(orders) == 1:
        sp = S.SemSpace(mesh, 7)
        M = sp.jacobi()
    else:
        sm = {"jacobi": S.JACOBI_SMOOTHER, "ras": S.RAS_SMOOTHER}[pc]
        pmg = S.Pmg(mesh, orders, sm, 2, 0.1, 1.1, 64, S.COARSE_AMG if coarse == "amg" else S.COARSE_DIRECT)
        sp, M = pmg.spaces[0], pmg.as_linop()
    x = sp.zeros()
    solve = S.gmres_solve if kr == 0 else S.pcg_solve
    st = solve(sp.as_linop(), M, sp.build_rhs(1), x, S.GmresConfig(tol=1e-8))
    assert st.converged
    assert abs(st.iterations - int(G[f"solve_{name}_iters"][0])) <= 1
    assert rel(x, G[f"solve_{name}_x"]) < 1e-10
