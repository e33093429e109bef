"""GPU parity of the p-multigrid layer (RESTATED: pmg.cpp is missing in the reference) against
the oracle: transfers (P, exact P^T), coarse solves (dense exact, aggregation AMG restated from
amg.cpp), the V-cycle, and preconditioned PCG/GMRES solves (BASELINE configs 2-4 shape at small E)."""
import numpy as np
import pytest
import torch

from oracle import semlab_np as o

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _pmg(ctx, eps, E, orders, smoother, precision=64, coarse="direct", eta=2):
    from paper_2110_07663_b200 import semlab as S
    sm = {"jacobi": S.JACOBI_SMOOTHER, "ras": S.RAS_SMOOTHER, "asm": S.ASM_SMOOTHER}[smoother]
    cm = S.COARSE_DIRECT if coarse == "direct" else S.COARSE_AMG
    g = S.Pmg(S.generate_kershaw(eps, E, ctx), orders, sm, eta, 0.1, 1.1, precision, cm)
    c = o.Pmg(o.generate_kershaw(eps, E), orders, smoother, eta, 0.1, 1.1, coarse, precision)
    return g, c


@pytest.mark.parametrize("eps,E,qf,qc", [(0.3, 2, 7, 3), (1.0, 4, 3, 1), (0.3, 4, 7, 5), (0.05, 2, 5, 2)])
def test_transfers_match_oracle_and_adjoint(ctx, eps, E, qf, qc):
    g, c = _pmg(ctx, eps, E, (qf, qc, 1) if qc > 1 else (qf, 1), "jacobi")
    rng = np.random.default_rng(0)
    uc = rng.standard_normal(c.spaces[1].n)
    vf = rng.standard_normal(c.spaces[0].n)
    T = c.transfers[0]
    Pu = g.prolong(0, g.spaces[1].to_device(uc))
    PTv = g.restrict(0, g.spaces[0].to_device(vf))
    assert rel(Pu, T.prolong(uc)) < 1e-13
    assert rel(PTv, T.restrict(vf)) < 1e-13
    lhs = float(Pu.cpu().numpy() @ vf)
    rhs = float(uc @ PTv.cpu().numpy())
    assert abs(lhs - rhs) <= 1e-13 * max(abs(lhs), 1.0) * 10


@pytest.mark.parametrize("coarse", ["direct", "amg"])
def test_vcycle_jacobi_matches_oracle(ctx, coarse):
    g, c = _pmg(ctx, 0.3, 4, (7, 3, 1), "jacobi", coarse=coarse)
    for l in range(2):
        assert abs(g.lam(l) - c.levels[l]["lam"]) <= 1e-10 * c.levels[l]["lam"]
    b = o.build_rhs(c.spaces[0], 1)
    z = g.vcycle(g.spaces[0].to_device(b))
    assert rel(z, c.vcycle(b)) < 1e-10


@pytest.mark.parametrize("smoother", ["ras", "asm"])
def test_vcycle_schwarz_fp64_matches_oracle(ctx, smoother):
    g, c = _pmg(ctx, 0.3, 4, (7, 3, 1), smoother, precision=64)
    b = o.build_rhs(c.spaces[0], 1)
    z = g.vcycle(g.spaces[0].to_device(b))
    assert rel(z, c.vcycle(b)) < 1e-10


def test_vcycle_is_linear(ctx):
    """the V-cycle is a fixed linear operator (prerequisite for GMRES)."""
    g, _ = _pmg(ctx, 0.3, 4, (7, 3, 1), "ras", precision=32)
    sp = g.spaces[0]
    rng = np.random.default_rng(3)
    b1 = sp.mask_inplace(sp.to_device(rng.standard_normal(sp.n)))
    b2 = sp.mask_inplace(sp.to_device(rng.standard_normal(sp.n)))
    z = g.vcycle(2.0 * b1 - 0.5 * b2)
    zl = 2.0 * g.vcycle(b1) - 0.5 * g.vcycle(b2)
    assert (z - zl).abs().max().item() <= 1e-5 * zl.abs().max().item()
    assert torch.equal(g.vcycle(b1), g.vcycle(b1))  # deterministic


def test_pcg_pmg_jacobi_config2_shape(ctx):
    """Config 2 shape (box, pMG(7,3,1) Cheby-Jacobi, PCG) at E=4^3."""
    from paper_2110_07663_b200 import semlab as S
    g, c = _pmg(ctx, 1.0, 4, (7, 3, 1), "jacobi")
    sp, cs = g.spaces[0], c.spaces[0]
    b = o.build_rhs(cs, 1)
    x = np.zeros(cs.n)
    st_o = o.pcg_solve(cs.apply_A, c.vcycle, b, x, 1e-8, 200)
    xg = sp.zeros()
    st_g = S.pcg_solve(sp.as_linop(), g.as_linop(), sp.build_rhs(1), xg, S.GmresConfig(tol=1e-8, max_iters=200))
    assert st_g.converged and st_o.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1
    assert rel(xg, x) < 1e-10


@pytest.mark.parametrize("coarse", ["direct", "amg"])
def test_gmres_pmg_ras_fp64(ctx, coarse):
    """Config 3/4 shape (deformed box, Cheby-RAS pMG + GMRES(20)) at E=4^3 with the FP64 smoother:
    iterations within +-1, solution within 1e-10."""
    from paper_2110_07663_b200 import semlab as S
    g, c = _pmg(ctx, 0.3, 4, (7, 3, 1), "ras", precision=64, coarse=coarse)
    sp, cs = g.spaces[0], c.spaces[0]
    b = o.build_rhs(cs, 1)
    x = np.zeros(cs.n)
    st_o = o.gmres_solve(cs.apply_A, c.vcycle, b, x, o.GmresConfig())
    xg = sp.zeros()
    st_g = S.gmres_solve(sp.as_linop(), g.as_linop(), sp.build_rhs(1), xg, S.GmresConfig())
    assert st_g.converged and st_o.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1
    assert rel(xg, x) < 1e-10


def test_gmres_pmg_ras_fp32(ctx):
    """FP32 smoother / FP64 Krylov (north_star): iterations within +-1 of the FP64 oracle and the
    solution within the solve tolerance."""
    from paper_2110_07663_b200 import semlab as S
    g, c = _pmg(ctx, 0.3, 4, (7, 3, 1), "ras", precision=32)
    sp, cs = g.spaces[0], c.spaces[0]
    b = o.build_rhs(cs, 1)
    x = np.zeros(cs.n)
    c64 = o.Pmg(o.generate_kershaw(0.3, 4), (7, 3, 1), "ras", 2, 0.1, 1.1, "direct", 64)
    st_o = o.gmres_solve(cs.apply_A, c64.vcycle, b, x, o.GmresConfig())
    xg = sp.zeros()
    st_g = S.gmres_solve(sp.as_linop(), g.as_linop(), sp.build_rhs(1), xg, S.GmresConfig())
    assert st_g.converged
    assert abs(st_g.iterations - st_o.iterations) <= 1
    assert rel(xg, x) < 1e-7


def test_amg_hierarchy_matches_oracle(ctx):
    """Coarse AMG V-cycle (amg.cpp:140-160) on the p=1 free-dof matrix vs the oracle's."""
    g, c = _pmg(ctx, 0.3, 6, (3, 1), "jacobi", coarse="amg")
    cs = c.coarse
    r = np.zeros(c.spaces[1].n)
    r[cs.free] = np.random.default_rng(0).standard_normal(len(cs.free))
    # drive the device coarse solve through a two-level V-cycle input: compare levels' sizes
    sizes = [lvl["A"].shape[0] for lvl in cs.amg.levels]
    assert sizes[0] == len(cs.free) and sizes[-1] <= 200
    b = o.build_rhs(c.spaces[0], 1)
    z = g.vcycle(g.spaces[0].to_device(b))
    assert rel(z, c.vcycle(b)) < 1e-9


def test_pmg_invalid_schedule(ctx):
    from paper_2110_07663_b200 import semlab as S
    mesh = S.generate_kershaw(1.0, 2, ctx)
    with pytest.raises(ValueError, match="end at order 1"):
        S.Pmg(mesh, (7, 3))
    with pytest.raises(ValueError, match="strictly decreasing"):
        S.Pmg(mesh, (3, 3, 1))


_GRAPH_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2110_07663_b200 import semlab as S
ctx = S.Context(0)
mesh = S.generate_kershaw(0.3, 4, ctx)
pmg = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 32, S.COARSE_AMG)
b = pmg.spaces[0].build_rhs(1)
outs = []
for _ in range(4):  # eager warm-up, capture + replay, replays
    z = torch.empty_like(b)
    pmg.vcycle(b, z)
    outs.append(z.cpu().numpy())
np.save(sys.argv[1], np.stack(outs))
"""


def test_vcycle_graph_replay_is_bitwise_eager(tmp_path):
    """The captured CUDA-graph V-cycle (pmg.cpp run_cycle) replays exactly the eager cycle: the
    first call runs eagerly, the second captures and launches the graph, later calls replay it;
    the FP32-smoother V-cycle outputs are bitwise identical."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    f = tmp_path / "v.npy"
    subprocess.run([sys.executable, "-c", _GRAPH_SCRIPT % root, str(f)], check=True, timeout=600)
    res = np.load(f)
    for k in range(1, 4):
        assert np.array_equal(res[k], res[0])
