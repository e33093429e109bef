"""GPU parity of the smoother and Krylov layers against the oracle: Chebyshev-Jacobi (fused
into the Ax owner epilogue), the lambda-max Arnoldi estimate, Jacobi-PCG and GMRES."""
import numpy as np
import pytest
import torch

from oracle import semlab_np as o

pytestmark = pytest.mark.gpu


def _pair(ctx, eps, E, p):
    from paper_2110_07663_b200 import semlab as S
    return S.SemSpace(S.generate_kershaw(eps, E, ctx), p), o.SemSpace(o.generate_kershaw(eps, E), p)


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("eps,E,p", [(1.0, 4, 7), (0.3, 4, 3)])
def test_lambda_estimate_jacobi(ctx, eps, E, p):
    from paper_2110_07663_b200 import semlab as S
    g, c = _pair(ctx, eps, E, p)
    inv = o.jacobi_inverse_diag(c)
    want = o.estimate_lambda_max(lambda v: inv * v, c.apply_A, c.n, 10, 0)
    got = S.estimate_lambda_max(g.jacobi(), g.as_linop(), g.n, 10, 0)
    assert got.rounds_used == want.rounds_used and got.breakdown == want.breakdown
    assert abs(got.value - want.value) <= 1e-10 * want.value


@pytest.mark.parametrize("eta", [1, 2, 3])
@pytest.mark.parametrize("x0_zero", [True, False])
def test_chebyshev_jacobi_smooth(ctx, eta, x0_zero):
    from paper_2110_07663_b200 import semlab as S
    g, c = _pair(ctx, 0.3, 4, 7)
    inv = o.jacobi_inverse_diag(c)
    lam = 2.3
    cheb_o = o.ChebyshevSmoother(lambda v: inv * v, c.apply_A, o.ChebyParams(eta, 0.1, 1.1, lam))
    cheb_g = S.ChebyshevSmoother(g.jacobi(), g.as_linop(), S.ChebyParams(eta, 0.1, 1.1, lam))
    rng = np.random.default_rng(eta)
    b = c.mask_inplace(rng.standard_normal(c.n))
    x = np.zeros(c.n) if x0_zero else c.mask_inplace(rng.standard_normal(c.n))
    xg = g.to_device(x)
    cheb_g.smooth(g.to_device(b), xg)
    cheb_o.smooth(b, x)
    assert rel(xg, x) < 1e-12


def test_chebyshev_invalid_params(ctx):
    from paper_2110_07663_b200 import semlab as S
    g, _ = _pair(ctx, 1.0, 2, 3)
    with pytest.raises(ValueError, match="lambda_max_est not set"):
        S.ChebyshevSmoother(g.jacobi(), g.as_linop(), S.ChebyParams(2, 0.1, 1.1, 0.0))
    with pytest.raises(ValueError, match="order must be >= 1"):
        S.ChebyshevSmoother(g.jacobi(), g.as_linop(), S.ChebyParams(0, 0.1, 1.1, 1.0))


def test_jacobi_pcg_config1_small(ctx):
    """Config 1 shape (box, Jacobi-PCG to 1e-8) at E=4^3: iterations within +-1, solution 1e-10."""
    from paper_2110_07663_b200 import semlab as S
    g, c = _pair(ctx, 1.0, 4, 7)
    b = o.build_rhs(c, 1)
    inv = o.jacobi_inverse_diag(c)
    x = np.zeros(c.n)
    st_o = o.pcg_solve(c.apply_A, lambda v: inv * v, b, x, 1e-8, 500)
    xg = g.zeros()
    st_g = S.pcg_solve(g.as_linop(), g.jacobi(), g.build_rhs(1), xg, S.GmresConfig(tol=1e-8))
    assert st_g.converged and st_o.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1
    assert rel(xg, x) < 1e-10
    assert st_g.rel_residual <= 1e-8 * 1.01


def test_gmres_jacobi_matches_oracle(ctx):
    from paper_2110_07663_b200 import semlab as S
    g, c = _pair(ctx, 0.3, 2, 5)
    b = o.build_rhs(c, 1)
    inv = o.jacobi_inverse_diag(c)
    x = np.zeros(c.n)
    st_o = o.gmres_solve(c.apply_A, lambda v: inv * v, b, x, o.GmresConfig(restart=10))
    xg = g.zeros()
    st_g = S.gmres_solve(g.as_linop(), g.jacobi(), g.to_device(b), xg, S.GmresConfig(restart=10))
    assert st_g.converged and st_o.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1
    assert rel(xg, x) < 1e-10
    n = min(len(st_g.history), len(st_o.history))
    np.testing.assert_allclose(st_g.history[:n // 2], st_o.history[:n // 2], rtol=1e-8)


def test_gmres_identity_one_iteration(ctx):
    from paper_2110_07663_b200 import semlab as S
    n = 1000
    ident = S.LinOp.from_callable(lambda i, out: out.copy_(i), n, ctx)
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    st = S.gmres_solve(ident, None, b, x)
    assert st.converged and st.iterations == 1
    assert torch.allclose(x, b, atol=1e-14)


@pytest.mark.parametrize("restart,precond", [(40, True), (45, False), (1, True), (33, True)])
def test_gmres_any_restart_matches_oracle(ctx, restart, precond):
    """The reference accepts any restart >= 1 (krylov.cpp:22): bases wider than 32 columns run the
    CGS2 passes in 32-column chunks. With and without a preconditioner (the device keeps the
    preconditioned directions Z; x += Z y equals the reference's x += M (V y) for a linear M)."""
    from paper_2110_07663_b200 import semlab as S
    g, c = _pair(ctx, 0.3, 2, 5)
    b = o.build_rhs(c, 1)
    inv = o.jacobi_inverse_diag(c)
    x = np.zeros(c.n)
    Mo = (lambda v: inv * v) if precond else None
    cfg = dict(restart=restart, max_iters=300)
    st_o = o.gmres_solve(c.apply_A, Mo, b, x, o.GmresConfig(**cfg))
    xg = g.zeros()
    st_g = S.gmres_solve(g.as_linop(), g.jacobi() if precond else None, g.to_device(b), xg, S.GmresConfig(**cfg))
    assert st_g.converged == st_o.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1
    if st_o.converged:
        assert rel(xg, x) < 1e-9
    else:  # GMRES(1) stalls: after 300 iterations x amplifies 1e-15 perturbations to ~1e-2 (oracle vs oracle)
        np.testing.assert_allclose(st_g.history[:20], st_o.history[:20], rtol=1e-8)


def test_lambda_estimate_many_rounds(ctx):
    """estimate_lambda_max with rounds > 32 (chunked CGS2) against the oracle."""
    from paper_2110_07663_b200 import semlab as S
    g, c = _pair(ctx, 0.3, 2, 5)
    inv = o.jacobi_inverse_diag(c)
    want = o.estimate_lambda_max(lambda v: inv * v, c.apply_A, c.n, 40, 0)
    got = S.estimate_lambda_max(g.jacobi(), g.as_linop(), g.n, 40, 0)
    assert got.rounds_used == want.rounds_used
    assert abs(got.value - want.value) <= 1e-9 * want.value


@pytest.mark.parametrize("precision", [64, 32])
def test_gmres_reference_form_matches_flexible(ctx, precision):
    """When the Z basis does not fit (one B200 at E=96^3) GMRES falls back to the reference's own
    x += M (V y) update. FP64 smoother: same iterations, x to 1e-10 of the flexible form. FP32
    smoother: the reference form may need a restart more (the V-cycle is linear only to ~1e-7)."""
    from paper_2110_07663_b200 import semlab as S
    pmg = S.Pmg(S.generate_kershaw(0.3, 4, ctx), (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, precision)
    sp = pmg.spaces[0]
    b = sp.build_rhs(1)
    x_flex, x_ref = sp.zeros(), sp.zeros()
    st_f = S.gmres_solve(sp.as_linop(), pmg.as_linop(), b, x_flex)
    S.debug_set_gmres_form(False)
    try:
        st_r = S.gmres_solve(sp.as_linop(), pmg.as_linop(), b, x_ref)
    finally:
        S.debug_set_gmres_form(True)
    c = o.Pmg(o.generate_kershaw(0.3, 4), (7, 3, 1), "ras", 2, 0.1, 1.1, "direct", precision)
    cs = c.spaces[0]
    xo = np.zeros(cs.n)
    st_o = o.gmres_solve(cs.apply_A, c.vcycle, o.build_rhs(cs, 1), xo, o.GmresConfig())
    assert st_f.converged and st_r.converged
    assert abs(st_r.iterations - st_o.iterations) <= 1  # the oracle runs the reference form too
    if precision == 64:
        assert abs(st_f.iterations - st_r.iterations) <= 1
        assert rel(x_ref, xo) < 1e-10
