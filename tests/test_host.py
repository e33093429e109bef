"""CPU-only tests: the C-ABI library loads and exports every declared symbol, host-side setup
math agrees with the oracle, and the oracle reproduces the SPEC known answers."""
import re

import numpy as np
import pytest

from oracle import semlab_np as o


def _declared_symbols():
    import os
    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "semlab_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(semlab_[A-Za-z0-9_]+)\s*\(", text)) - {"semlab_map_fn", "semlab_apply_fn"})


def test_library_exports_every_declared_symbol():
    from paper_2110_07663_b200 import _lib
    names = _declared_symbols()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_no_gpu_needed_for_errors():
    from paper_2110_07663_b200 import semlab
    with pytest.raises(ValueError, match="gll: order must be in"):
        semlab.host_gll(0)


@pytest.mark.parametrize("p", [1, 2, 3, 5, 7, 9, 16])
def test_gll_matches_oracle_bitwise(p):
    from paper_2110_07663_b200 import semlab
    nodes, w, d = semlab.host_gll(p)
    g = o.gll(p)
    np.testing.assert_array_equal(nodes, g.nodes)
    np.testing.assert_array_equal(w, g.weights)
    np.testing.assert_allclose(d, g.diff, rtol=0, atol=1e-13 * p * p)


def test_gll_known_answers():
    """SPEC.md:118-120."""
    g1, g2, g7 = o.gll(1), o.gll(2), o.gll(7)
    np.testing.assert_array_equal(g1.nodes, [-1.0, 1.0])
    np.testing.assert_array_equal(g1.weights, [1.0, 1.0])
    np.testing.assert_allclose(g2.weights, [1 / 3, 4 / 3, 1 / 3], rtol=0, atol=1e-15)
    # p=7 interior nodes are the roots of P_7'; check against numpy's Legendre derivative roots
    from numpy.polynomial import legendre as L
    c = np.zeros(8)
    c[7] = 1.0
    roots = np.sort(L.legroots(L.legder(c)))
    np.testing.assert_allclose(g7.nodes[1:-1], roots, rtol=0, atol=1e-14)
    assert abs(g7.weights.sum() - 2.0) < 1e-14
    # D exact for polynomials of degree <= p
    x = g7.nodes
    np.testing.assert_allclose(g7.diff @ x ** 5, 5 * x ** 4, atol=1e-12)


def test_kershaw_map_matches_oracle():
    from paper_2110_07663_b200 import semlab
    rng = np.random.default_rng(3)
    for eps in (1.0, 0.3, 0.05):
        for _ in range(50):
            x, y, z = rng.random(3)
            got = semlab.host_kershaw_map(eps, x, y, z)
            want = [float(v) for v in o.kershaw_map(eps, x, y, z)]
            assert got == tuple(want)
    # eps = 1 is the identity (shifted to [-1/2,1/2]^3), mesh.hpp:99-101
    assert semlab.host_kershaw_map(1.0, 0.25, 0.5, 0.75) == (-0.25, 0.0, 0.25)


def test_mt19937_stream_matches_oracle_bitwise():
    from paper_2110_07663_b200 import semlab
    for seed in (0, 1, 12345):
        np.testing.assert_array_equal(semlab.host_uniform_pm1(seed, 5000), o.uniform_pm1(seed, 5000))


def test_mt19937_reference_first_values():
    """C++11 [rand.predef]: the 10000th output of a default-seeded mt19937_64 is 9981545732273789042."""
    v = o.mt19937_64(5489, 10000)
    assert int(v[-1]) == 9981545732273789042


def test_gen_eig_contract():
    from paper_2110_07663_b200 import semlab
    import scipy.linalg as sl
    rng = np.random.default_rng(0)
    for n in (1, 2, 6, 10, 16):
        A = rng.standard_normal((n, n))
        A = A + A.T + 2 * n * np.eye(n)
        B = rng.standard_normal((n, n))
        B = B @ B.T + np.eye(n)
        lam, S = semlab.host_gen_eig(A, B)
        np.testing.assert_allclose(lam, sl.eigh(A, B, eigvals_only=True), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(S.T @ B @ S, np.eye(n), atol=1e-11)
        np.testing.assert_allclose(S.T @ A @ S, np.diag(lam), atol=1e-10 * max(1, abs(lam).max()))


def test_max_abs_eig_hessenberg():
    from paper_2110_07663_b200 import semlab
    rng = np.random.default_rng(1)
    for n in (1, 2, 3, 5, 10, 20):
        H = np.triu(rng.standard_normal((n, n)), -1)
        assert abs(semlab.host_max_abs_eig(H) - np.abs(np.linalg.eigvals(H)).max()) < 1e-10
    # general (non-Hessenberg) input is reduced first
    G = rng.standard_normal((7, 7))
    assert abs(semlab.host_max_abs_eig(G) - np.abs(np.linalg.eigvals(G)).max()) < 1e-10


# ---------------------------------------------------------------- oracle known answers (SPEC)
def test_oracle_constant_field_zero():
    """SPEC.md:127 constant field -> A^e u = 0."""
    s = o.SemSpace(o.generate_kershaw(0.3, 2), 4)
    out = s.apply_local_stiffness(np.ones(s.E * s.nloc))
    assert np.abs(out).max() < 1e-12


def test_oracle_volume_integral():
    """SPEC.md:144 integral of 1 = volume of [-1/2,1/2]^3."""
    for eps in (1.0, 0.3):
        s = o.SemSpace(o.generate_kershaw(eps, 4), 5)
        assert abs(s.mass_diag.sum() - 1.0) < 1e-10


def test_oracle_dense_column_probe():
    """SPEC.md:137, acceptance #1: dense column-probed A symmetric and equal to assembled element
    matrices (E=2^3, p in 2..4, eps=0.3)."""
    for p in (2, 3, 4):
        s = o.SemSpace(o.generate_kershaw(0.3, 2), p)
        n = s.n
        A = np.stack([s.apply_A(np.eye(n)[:, c]) for c in range(n)], axis=1)
        assert np.abs(A - A.T).max() <= 1e-11 * np.abs(A).max()
        free = s.masked == 0
        ev = np.linalg.eigvalsh(A[np.ix_(free, free)])
        assert ev.min() > 0


def test_oracle_fdm_exactness():
    """SPEC.md:611 acceptance #2: ||Abar fdm(r) - r|| <= 1e-9 ||r|| on every element."""
    s = o.SemSpace(o.generate_kershaw(0.3, 4), 7)
    sch = o.SchwarzSmoother(s, o.RAS)
    rng = np.random.default_rng(0)
    P = sch.P
    R = np.zeros((s.E, P, P, P))
    for e in range(s.E):
        n = sch.n[e]
        R[e, :n[2], :n[1], :n[0]] = rng.standard_normal((n[2], n[1], n[0]))
    Z = sch.fdm_solve_all(R)
    for e in range(0, s.E, 7):
        n = sch.n[e]
        Ab = sch.box_matrix(e)
        r = R[e, :n[2], :n[1], :n[0]].ravel()
        z = Z[e, :n[2], :n[1], :n[0]].ravel()
        assert np.linalg.norm(Ab @ z - r) <= 1e-9 * np.linalg.norm(r)


def test_oracle_chebyshev_polynomial_identity():
    """SPEC.md:612 acceptance #3: e' = p_eta(SA) e0 per mode on a diagonal system."""
    n = 100
    lam_max = 10.0
    lam = np.linspace(0.1 * lam_max, 1.1 * lam_max, n) / 1.1
    A = lambda v: lam * v
    S = lambda v: v.copy()
    for eta in (1, 2, 3):
        cheb = o.ChebyshevSmoother(S, A, o.ChebyParams(eta, 0.1, 1.1, lam_max))
        xs = np.random.default_rng(eta).standard_normal(n)
        b = A(xs)
        x = np.zeros(n)
        cheb.smooth(b, x)
        # residual polynomial from the same three-term recurrence on scalars
        th, de, si = cheb.theta, cheb.delta, cheb.sigma
        e0 = -xs  # error of x0 = 0
        # scalar recurrence: p applied to each eigenvalue
        pe = np.empty(n)
        for i, l in enumerate(lam):
            xx, r = 0.0, l * (-e0[i])  # b - A*0 with S = I
            d = r / th
            rho = 1.0 / si
            for _ in range(eta):
                xx += d
                r -= l * d
                rn = 1.0 / (2.0 * si - rho)
                d = rn * rho * d + (2.0 * rn / de) * r
                rho = rn
            xx += d
            pe[i] = (xx - xs[i]) / e0[i]
        np.testing.assert_allclose((x - xs), pe * e0, atol=1e-12 * np.abs(e0).max())
        assert np.all(np.abs(pe) <= 1.0 + 1e-12)


def test_oracle_lambda_known_spectrum():
    """spectrum {1..10} -> within 5% of 10; S = A^-1 -> ~1; fixed seed bitwise."""
    lam = np.arange(1, 11, dtype=float).repeat(10)
    A = lambda v: lam * v
    est = o.estimate_lambda_max(lambda v: v.copy(), A, lam.size, 10, 0)
    assert abs(est.value - 10.0) <= 0.5
    est2 = o.estimate_lambda_max(lambda v: v / lam, A, lam.size, 10, 0)
    assert abs(est2.value - 1.0) < 1e-10
    assert est.value == o.estimate_lambda_max(lambda v: v.copy(), A, lam.size, 10, 0).value


def test_oracle_pmg_adjoint_and_exactness():
    """<Pu,v> = <u,P^T v> to 1e-13; degree-3 fields prolong exactly."""
    m = o.generate_kershaw(0.3, 2)
    f, c = o.SemSpace(m, 7), o.SemSpace(m, 3)
    T = o.Transfer(f, c)
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(c.n), rng.standard_normal(f.n)
    lhs = T.prolong(u) @ v
    rhs = u @ T.restrict(v)
    assert abs(lhs - rhs) <= 1e-13 * max(abs(lhs), 1.0) * 10
    # polynomial of degree 3 in the reference coordinates of a box mesh is reproduced exactly
    mb = o.generate_kershaw(1.0, 2)
    fb, cb = o.SemSpace(mb, 7), o.SemSpace(mb, 3)
    Tb = o.Transfer(fb, cb)
    # (vanishes on the boundary, degree <= 3 per direction on every element)
    poly = lambda X: (0.25 - X[:, 0] ** 2) * (0.25 - X[:, 1] ** 2) * X[:, 2] * (0.25 - X[:, 2] ** 2)
    uc = poly(cb.coords)
    assert np.abs(Tb.prolong(uc) - poly(fb.coords)).max() < 1e-12


def test_oracle_gmres_identity_one_iteration():
    """A = I converges in 1 iteration."""
    b = np.random.default_rng(0).standard_normal(50)
    x = np.zeros(50)
    st = o.gmres_solve(lambda v: v.copy(), None, b, x, o.GmresConfig())
    assert st.converged and st.iterations == 1
    np.testing.assert_allclose(x, b, atol=1e-14)


def test_handles_released_child_first_in_any_finalisation_order():
    """A garbage cycle is finalised in arbitrary order; native handles must still be destroyed
    child-before-parent (a smoother's destroy reads its space's context)."""
    from paper_2110_07663_b200 import semlab as S
    log = []

    class Obj:
        pass

    ctx, mesh, space, sch = Obj(), Obj(), Obj(), Obj()
    S._own(ctx, 1, lambda h: log.append(("ctx", h)))
    S._own(mesh, 2, lambda h: log.append(("mesh", h)), ctx)
    S._own(space, 3, lambda h: log.append(("space", h)), mesh)
    S._own(sch, 4, lambda h: log.append(("sch", h)), space)
    for obj in (ctx, space, sch, mesh):  # parent finalised first
        S._release(obj)
    assert log == [("sch", 4), ("space", 3), ("mesh", 2), ("ctx", 1)]
    assert all(o.handle is None for o in (ctx, mesh, space, sch))
