"""GPU parity of the Schwarz/FDM smoother (RAS and ASM, FP64 and the paper's FP32) against
the oracle restatement of schwarz.cpp. FP64: 1e-12 relative. FP32: 2e-5 relative to the FP64
oracle and 2e-6 to the FP32 oracle variant (the stated smoother tolerance)."""
import numpy as np
import pytest
import torch

from oracle import semlab_np as o

pytestmark = pytest.mark.gpu


def _pair(ctx, eps, E, p, mode, precision):
    from paper_2110_07663_b200 import semlab as S
    g = S.SemSpace(S.generate_kershaw(eps, E, ctx), p)
    c = o.SemSpace(o.generate_kershaw(eps, E), p)
    return g, c, S.SchwarzSmoother(g, mode, precision), o.SchwarzSmoother(c, mode, precision)


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("eps,E,p", [(1.0, 2, 3), (0.3, 2, 3), (0.3, 4, 7), (1.0, 4, 7), (0.05, 2, 5), (0.3, 6, 2)])
@pytest.mark.parametrize("mode", [o.RAS, o.ASM])
def test_schwarz_fp64_matches_oracle(ctx, eps, E, p, mode):
    g, c, sg, so = _pair(ctx, eps, E, p, mode, 64)
    r = c.mask_inplace(np.random.default_rng(p).standard_normal(c.n))
    assert rel(sg.apply(r), so.apply(r)) < 1e-12


@pytest.mark.parametrize("mode", [o.RAS, o.ASM])
def test_schwarz_fp32(ctx, mode):
    g, c, sg, so32 = _pair(ctx, 0.3, 4, 7, mode, 32)
    so64 = o.SchwarzSmoother(c, mode, 64)
    r = c.mask_inplace(np.random.default_rng(0).standard_normal(c.n))
    z = sg.apply(r)
    assert rel(z, so64.apply(r)) < 2e-5
    assert rel(z, so32.apply(r)) < 2e-6


def test_schwarz_setup_data(ctx):
    g, c, sg, so = _pair(ctx, 0.3, 4, 7, o.RAS, 64)
    for e in (0, 5, 21, c.E - 1):
        L, n, lam = sg.element_info(e)
        np.testing.assert_allclose(L, so.lengths[e], rtol=1e-13)
        np.testing.assert_array_equal(n, so.n[e])
        for d in range(3):
            np.testing.assert_allclose(lam[d, :n[d]], so.lam[e, d, :n[d]], rtol=1e-11)


def test_fdm_solve_exactness(ctx):
    """Acceptance #2 on the device FDM: ||Abar fdm(r) - r|| <= 1e-9 ||r||."""
    g, c, sg, so = _pair(ctx, 0.3, 4, 7, o.RAS, 64)
    P = so.P
    rng = np.random.default_rng(0)
    R = np.zeros((c.E, P, P, P))
    for e in range(c.E):
        n = so.n[e]
        R[e, :n[2], :n[1], :n[0]] = rng.standard_normal((n[2], n[1], n[0]))
    Z = sg.fdm_solve_all(g.to_device(R.ravel())).cpu().numpy().reshape(R.shape)
    for e in range(0, c.E, 5):
        n = so.n[e]
        Ab = so.box_matrix(e)
        r = R[e, :n[2], :n[1], :n[0]].ravel()
        z = Z[e, :n[2], :n[1], :n[0]].ravel()
        assert np.linalg.norm(Ab @ z - r) <= 1e-9 * np.linalg.norm(r)
    assert rel(Z, so.fdm_solve_all(R)) < 1e-12


def test_lambda_estimate_ras(ctx):
    from paper_2110_07663_b200 import semlab as S
    g, c, sg, so = _pair(ctx, 0.3, 4, 7, o.RAS, 64)
    want = o.estimate_lambda_max(so.apply, c.apply_A, c.n, 10, 0)
    got = S.estimate_lambda_max(sg.as_linop(), g.as_linop(), g.n, 10, 0)
    assert abs(got.value - want.value) <= 1e-9 * want.value


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("x0_zero", [True, False])
def test_chebyshev_ras_fused(ctx, precision, x0_zero):
    """Chebyshev-RAS with the update fused into the RAS owner write == oracle smooth()."""
    from paper_2110_07663_b200 import semlab as S
    g, c, sg, so = _pair(ctx, 0.3, 4, 7, o.RAS, precision)
    lam = 3.0
    cg = S.ChebyshevSmoother(sg.as_linop(), g.as_linop(), S.ChebyParams(2, 0.1, 1.1, lam))
    co = o.ChebyshevSmoother(so.apply, c.apply_A, o.ChebyParams(2, 0.1, 1.1, lam))
    rng = np.random.default_rng(1)
    b = c.mask_inplace(rng.standard_normal(c.n))
    x = np.zeros(c.n) if x0_zero else c.mask_inplace(rng.standard_normal(c.n))
    xg = g.to_device(x)
    cg.smooth(g.to_device(b), xg)
    co.smooth(b, x)
    assert rel(xg, x) < (1e-11 if precision == 64 else 1e-5)


@pytest.mark.parametrize("eps,E,p", [(0.3, 2, 5), (1.0, 4, 3)])
@pytest.mark.parametrize("mode", [o.RAS, o.ASM])
def test_schwarz_neumann_fp64_matches_oracle(ctx, eps, E, p, mode):
    """Neumann boundary sides keep the face dof (schwarz.cpp:151-160): n = p+1 at the domain
    boundary instead of p-1, and no lattice point is masked."""
    from paper_2110_07663_b200 import semlab as S
    g = S.SemSpace(S.generate_kershaw(eps, E, ctx), p, S.NEUMANN)
    c = o.SemSpace(o.generate_kershaw(eps, E), p, o.NEUMANN)
    sg, so = S.SchwarzSmoother(g, mode, 64), o.SchwarzSmoother(c, mode, 64)
    for e in (0, c.E - 1):
        _, n, _ = sg.element_info(e)
        np.testing.assert_array_equal(n, so.n[e])
    r = np.random.default_rng(p).standard_normal(c.n)
    assert rel(sg.apply(r), so.apply(r)) < 1e-12
    np.testing.assert_allclose(g.stiffness_diag().cpu().numpy(), c.stiffness_diag(), rtol=1e-12)
    # and against the reference's own Neumann outputs (tests/golden, ref_neumann)
    import os
    G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz"))
    key = f"neu_e{eps}_E{E}_p{p}"
    name = "ras" if mode == o.RAS else "asm"
    assert rel(sg.apply(G[f"{key}_r"]), G[f"{key}_{name}"]) < 1e-12
    assert rel(g.apply_A(G[f"{key}_u"]), G[f"{key}_Au"]) < 1e-12


@pytest.mark.parametrize("mode", [o.RAS, o.ASM])
def test_schwarz_neumann_fp32(ctx, mode):
    """The paper's FP32 smoother (warp-per-element RAS at p=7) in Neumann mode: the first element
    along each axis owns q + 1 sites."""
    from paper_2110_07663_b200 import semlab as S
    g = S.SemSpace(S.generate_kershaw(0.3, 4, ctx), 7, S.NEUMANN)
    c = o.SemSpace(o.generate_kershaw(0.3, 4), 7, o.NEUMANN)
    r = np.random.default_rng(3).standard_normal(c.n)
    z = S.SchwarzSmoother(g, mode, 32).apply(r)
    assert rel(z, o.SchwarzSmoother(c, mode, 64).apply(r)) < 2e-5
    assert rel(z, o.SchwarzSmoother(c, mode, 32).apply(r)) < 2e-6


@pytest.mark.parametrize("smoother", ["ras", "jacobi"])
@pytest.mark.parametrize("x0_zero", [True, False])
def test_chebyshev_neumann_matches_oracle(ctx, smoother, x0_zero):
    """Chebyshev smoothing of the Neumann operator (A with mean removal, sem_space.cpp:207): the
    fused Ax/RAS epilogues skip the mean removal, so Neumann spaces take the generic path."""
    from paper_2110_07663_b200 import semlab as S
    g = S.SemSpace(S.generate_kershaw(0.3, 4, ctx), 5, S.NEUMANN)
    c = o.SemSpace(o.generate_kershaw(0.3, 4), 5, o.NEUMANN)
    if smoother == "ras":
        Sg, So = S.SchwarzSmoother(g, S.RAS, 64).as_linop(), o.SchwarzSmoother(c, o.RAS, 64).apply
    else:
        inv = o.jacobi_inverse_diag(c)
        Sg, So = g.jacobi(), (lambda v: inv * v)
    cg = S.ChebyshevSmoother(Sg, g.as_linop(), S.ChebyParams(2, 0.1, 1.1, 3.0))
    co = o.ChebyshevSmoother(So, c.apply_A, o.ChebyParams(2, 0.1, 1.1, 3.0))
    rng = np.random.default_rng(5)
    b = rng.standard_normal(c.n)
    x = np.zeros(c.n) if x0_zero else rng.standard_normal(c.n)
    xg = g.to_device(x)
    cg.smooth(g.to_device(b), xg)
    co.smooth(b, x)
    assert rel(xg, x) < 1e-11
