"""GPU parity of the SemSpace kernels (sm_100a) against the CPU oracle: geometry, fused Ax,
Q / Q^T / QQ^T, assembled diagonal, mass, RHS. Tolerances: 1e-12 relative (FP64 throughout;
only the summation order of the D-contractions may differ from the oracle)."""
import numpy as np
import pytest
import torch

from oracle import semlab_np as o

pytestmark = pytest.mark.gpu

CASES = [(1.0, 2, 2), (0.3, 2, 3), (0.3, 2, 4), (1.0, 4, 7), (0.3, 4, 7), (0.3, 4, 3), (0.05, 2, 5), (0.3, 2, 8),
         (1.0, 2, 1)]


def _pair(ctx, eps, E, p):
    from paper_2110_07663_b200 import semlab as S
    mesh = S.generate_kershaw(eps, E, ctx)
    return S.SemSpace(mesh, p), o.SemSpace(o.generate_kershaw(eps, E), p)


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("eps,E,p", CASES)
def test_geometry_matches_oracle(ctx, eps, E, p):
    g, c = _pair(ctx, eps, E, p)
    assert g.n == c.n and g.n_local_total == c.E * c.nloc
    for e in (0, c.E // 2, c.E - 1):
        np.testing.assert_allclose(g.metric_at(e), c.geom[e], rtol=1e-12, atol=1e-13 * np.abs(c.geom[e]).max())
    assert rel(g.mass_diag(), c.mass_diag) < 1e-13


@pytest.mark.parametrize("eps,E,p", CASES)
def test_apply_A_matches_oracle(ctx, eps, E, p):
    g, c = _pair(ctx, eps, E, p)
    rng = np.random.default_rng(p * 100 + E)
    for _ in range(2):
        u = rng.standard_normal(c.n)
        assert rel(g.apply_A(u), c.apply_A(u)) < 1e-12


def test_apply_A_deterministic_and_repeatable(ctx):
    g, c = _pair(ctx, 0.3, 6, 7)
    u = g.to_device(np.random.default_rng(0).standard_normal(c.n))
    a = g.apply_A(u)
    for _ in range(5):
        assert torch.equal(a, g.apply_A(u))
    assert rel(a, c.apply_A(u.cpu().numpy())) < 1e-12


def test_apply_A_constant_and_zero(ctx):
    g, _ = _pair(ctx, 0.3, 4, 7)
    assert torch.count_nonzero(g.apply_A(g.zeros())) == 0
    from paper_2110_07663_b200 import semlab as S
    gn = S.SemSpace(S.generate_kershaw(0.3, 4, ctx), 7, S.NEUMANN)
    out = gn.apply_A(torch.ones(gn.n, dtype=torch.float64, device="cuda"))
    assert out.abs().max().item() < 1e-10


def test_neumann_mode_matches_oracle(ctx):
    from paper_2110_07663_b200 import semlab as S
    g = S.SemSpace(S.generate_kershaw(0.3, 2, ctx), 5, S.NEUMANN)
    c = o.SemSpace(o.generate_kershaw(0.3, 2), 5, o.NEUMANN)
    u = np.random.default_rng(1).standard_normal(c.n)
    assert rel(g.apply_A(u), c.apply_A(u)) < 1e-12


def test_dense_column_probe_E2_p3(ctx):
    """dense A from apply_A column probes matches the oracle's."""
    g, c = _pair(ctx, 0.3, 2, 3)
    n = c.n
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    Ag = torch.stack([g.apply_A(I[:, k].contiguous()) for k in range(n)], dim=1).cpu().numpy()
    Ac = np.stack([c.apply_A(np.eye(n)[:, k]) for k in range(n)], axis=1)
    assert np.abs(Ag - Ac).max() <= 1e-11 * np.abs(Ac).max()
    assert np.abs(Ag - Ag.T).max() <= 1e-11 * np.abs(Ag).max()


@pytest.mark.parametrize("eps,E,p", [(0.3, 2, 2), (0.3, 3 * 2, 3), (1.0, 4, 7)])
def test_gather_scatter(ctx, eps, E, p):
    g, c = _pair(ctx, eps, E, p)
    rng = np.random.default_rng(7)
    loc = rng.standard_normal(c.E * c.nloc)
    glob = rng.standard_normal(c.n)
    np.testing.assert_array_equal(g.gather(loc).cpu().numpy(), c.gather(loc))  # same order -> bitwise
    np.testing.assert_array_equal(g.scatter(glob).cpu().numpy(), c.scatter(glob))
    np.testing.assert_array_equal(g.gather_scatter(loc).cpu().numpy(), c.gather_scatter(loc))
    # QQ^T of an assembled (continuous) vector = multiplicity-scaled copy
    qqt = g.gather_scatter(c.scatter(glob)).cpu().numpy()
    np.testing.assert_allclose(qqt, c.scatter(glob * c.multiplicity), rtol=1e-15)


@pytest.mark.parametrize("eps,E,p", [(0.3, 2, 3), (1.0, 4, 7), (0.3, 4, 7)])
def test_local_stiffness_and_diag(ctx, eps, E, p):
    g, c = _pair(ctx, eps, E, p)
    loc = np.random.default_rng(3).standard_normal(c.E * c.nloc)
    assert rel(g.apply_local_stiffness(loc), c.apply_local_stiffness(loc)) < 1e-12
    assert rel(g.stiffness_diag(), c.stiffness_diag()) < 1e-12


def test_mask_and_rhs(ctx):
    g, c = _pair(ctx, 0.3, 4, 5)
    v = g.to_device(np.ones(c.n))
    g.mask_inplace(v)
    np.testing.assert_array_equal(v.cpu().numpy(), 1.0 - c.masked)
    assert rel(g.build_rhs(1), o.build_rhs(c, 1)) < 1e-13


def test_invalid_arguments(ctx):
    from paper_2110_07663_b200 import semlab as S
    with pytest.raises(ValueError, match="eps must lie in"):
        S.generate_kershaw(1.5, 4, ctx)
    with pytest.raises(ValueError, match="even"):
        S.generate_kershaw(0.5, 3, ctx)
    with pytest.raises(ValueError, match="order"):
        S.SemSpace(S.generate_kershaw(0.5, 2, ctx), 12)


def test_nonpositive_jacobian_raises(ctx):
    from paper_2110_07663_b200 import semlab as S
    mesh = S.HexMesh.from_map((2, 2, 2), lambda x, y, z: (x, y, -z), ctx)  # inverted map
    with pytest.raises(RuntimeError, match="non-positive Jacobian in element"):
        S.SemSpace(mesh, 3)


def test_from_map_and_box(ctx):
    from paper_2110_07663_b200 import semlab as S
    box = S.HexMesh.box((2, 3, 4), (0, 0, 0), (1, 2, 3), ctx)
    g = S.SemSpace(box, 4)
    cm = o.SemSpace(o.box_mesh((2, 3, 4), (0, 0, 0), (1, 2, 3)), 4)
    u = np.random.default_rng(0).standard_normal(cm.n)
    assert rel(g.apply_A(u), cm.apply_A(u)) < 1e-12
    assert abs(g.mass_diag().sum().item() - 6.0) < 1e-11
