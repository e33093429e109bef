"""The persistent kernels' multi-element steady state, forced at small E.

k_axw (fused Ax) and k_rasw (warp-per-element RAS) size their grids to the resident CTAs, so on the
small test meshes each warp normally handles one element. semlab_debug_set_grid_cap() shrinks the
grid to 1-2 CTAs: every warp then loops over many tickets / grid-stride elements (the deferred
release and finish of the previous ticket in k_axw, the reuse of the box/line buffers in k_rasw).
Results must be bitwise identical to the uncapped launch and match the oracle.

Also pins the FP32-factor smoother operator (apply_A with FP32-rounded geometric factors, FP64
arithmetic) against an oracle that uses the same rounded factors.
"""
import contextlib

import numpy as np
import pytest
import torch

from oracle import semlab_np as o

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def grid_cap(n):
    from paper_2110_07663_b200 import semlab as S
    S.debug_set_grid_cap(n)
    try:
        yield
    finally:
        S.debug_set_grid_cap(0)


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("eps,E,p", [(0.3, 6, 7), (1.0, 8, 7), (0.3, 4, 8), (0.3, 6, 3)])
def test_ax_grid_cap_bitwise(ctx, eps, E, p):
    from paper_2110_07663_b200 import semlab as S
    sp = S.SemSpace(S.generate_kershaw(eps, E, ctx), p)
    u = sp.to_device(np.random.default_rng(E * 10 + p).standard_normal(sp.n))
    full = sp.apply_A(u)
    for cap in (1, 2, 3):
        with grid_cap(cap):
            got = sp.apply_A(u)
        assert torch.equal(got, full), f"cap {cap}: max diff {(got - full).abs().max().item()}"
    want = o.SemSpace(o.generate_kershaw(eps, E), p).apply_A(u.cpu().numpy())
    assert rel(full, want) < 1e-12


@pytest.mark.parametrize("p", [7, 3, 5])
def test_ax_geom32_grid_cap_and_oracle(ctx, p):
    """FP32-rounded factors, FP64 arithmetic: order 7 (k_axe) and the split-path orders (k_ax +
    k_gather_epi, the p=3 pMG level) against the oracle with the same rounded factors."""
    from paper_2110_07663_b200 import semlab as S
    sp = S.SemSpace(S.generate_kershaw(0.3, 6, ctx), p)
    cs = o.SemSpace(o.generate_kershaw(0.3, 6), p)
    u = np.random.default_rng(5).standard_normal(sp.n)
    full = sp.apply_A_geom32(u)
    with grid_cap(1):
        capped = sp.apply_A_geom32(u)
    assert torch.equal(capped, full)
    want = cs.with_geom32().apply_A(u)
    err = rel(full, want)
    print(f"FP32-factor Ax vs FP32-factor oracle: {err:.2e}; vs FP64 operator: {rel(full, cs.apply_A(u)):.2e}")
    assert err < 1e-13


@pytest.mark.parametrize("E", [4, 6])
def test_rasw_grid_cap_bitwise(ctx, E):
    from paper_2110_07663_b200 import semlab as S
    sp = S.SemSpace(S.generate_kershaw(0.3, E, ctx), 7)
    sch = S.SchwarzSmoother(sp, S.RAS, 32)
    cs = o.SemSpace(o.generate_kershaw(0.3, E), 7)
    r = np.random.default_rng(E).standard_normal(sp.n) * (1 - cs.masked)
    full = sch.apply(r)
    for cap in (1, 2):
        with grid_cap(cap):
            got = sch.apply(r)
        assert torch.equal(got, full), f"cap {cap}"
    want = o.SchwarzSmoother(cs, o.RAS, 32).apply(r)
    assert rel(full, want) < 2e-6


def test_vcycle_grid_cap_bitwise(ctx):
    """Fused Chebyshev-RAS modes (k_rasw modes 1-3, k_axw Chebyshev epilogue) under a capped grid:
    the whole FP32-smoother V-cycle is bitwise the uncapped one. The hierarchy is built under the
    cap because the V-cycle is captured once as a CUDA graph."""
    from paper_2110_07663_b200 import semlab as S
    mesh = S.generate_kershaw(0.3, 6, ctx)
    full_pmg = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 32, S.COARSE_DIRECT)
    b = full_pmg.spaces[0].build_rhs(1)
    full = full_pmg.vcycle(b)
    with grid_cap(2):
        capped_pmg = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 32, S.COARSE_DIRECT)
        got = capped_pmg.vcycle(b)
    assert torch.equal(got, full)
    for l in range(2):
        assert capped_pmg.lam(l) == full_pmg.lam(l)


def test_borrowed_space_keeps_pmg_alive(ctx):
    """a smoother / operator built on pmg.spaces[l] must keep the hierarchy alive."""
    import gc
    from paper_2110_07663_b200 import semlab as S
    pmg = S.Pmg(S.generate_kershaw(0.3, 2, ctx), (3, 1), S.JACOBI_SMOOTHER, 2, 0.1, 1.1, 64, S.COARSE_DIRECT)
    A = pmg.spaces[0].as_linop()
    sch = S.SchwarzSmoother(pmg.spaces[0], S.RAS, 64)
    x = pmg.spaces[0].build_rhs(1)
    want = A(x).clone()
    del pmg
    gc.collect()
    assert torch.equal(A(x), want)
    sch.apply(x)


def test_released_parent_clears_child_handles(ctx):
    """Releasing a parent destroys its children's native handles and clears their .handle, so a
    stale call raises instead of touching freed memory."""
    from paper_2110_07663_b200 import semlab as S
    mesh = S.generate_kershaw(1.0, 2, ctx)
    sp = S.SemSpace(mesh, 3)
    A = sp.as_linop()
    x = sp.build_rhs(1)
    S._release(sp)
    assert sp.handle is None and A.handle is None
    with pytest.raises(ValueError):
        A(x)
