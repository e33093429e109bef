"""Device ProjectionBasis (krylov.hpp:39-59) against the reference's own outputs (tests/golden,
ref_projection) and the numpy oracle; tolerance 1e-11 relative (FP64, different summation order)."""
import os

import numpy as np
import pytest
import torch

from oracle import semlab_np as o

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz"))


def rel(a, b):
    a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_projection_matches_reference(ctx):
    from paper_2110_07663_b200 import semlab as S
    sp = S.SemSpace(S.generate_kershaw(0.3, 2, ctx), 4)
    A = sp.as_linop()
    pb = S.ProjectionBasis(3)
    assert pb.size() == 0
    assert torch.count_nonzero(pb.initial_guess(sp.to_device(G["proj_b"]))) == 0
    for x in G["proj_X"]:
        pb.insert(sp.to_device(x), A)
    assert pb.size() == int(G["proj_size"][0]) == 3
    for v, ref in zip(pb.vectors(), G["proj_basis"]):
        assert rel(v, ref) < 1e-11
    assert rel(pb.initial_guess(sp.to_device(G["proj_b"])), G["proj_guess"]) < 1e-11
    pb.clear()
    assert pb.size() == 0


def test_projection_guess_of_a_solved_rhs(ctx):
    """The caller-side use: after a solve for b is inserted, the guess for the
    same b is the A-orthogonal projection onto span{x}, i.e. x itself, with a 1e-8 residual."""
    from paper_2110_07663_b200 import semlab as S
    mesh = S.generate_kershaw(0.3, 4, ctx)
    pmg = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 32, S.COARSE_DIRECT)
    sp = pmg.spaces[0]
    A, M = sp.as_linop(), pmg.as_linop()
    b = sp.build_rhs(1)
    x = torch.zeros_like(b)
    assert S.gmres_solve(A, M, b, x, S.GmresConfig()).converged
    pb = S.ProjectionBasis(10)
    pb.insert(x, A)
    u = pb.initial_guess(b)
    assert rel(u, x.cpu().numpy()) < 1e-7
    r = b - A(u)
    assert (r.norm() / b.norm()).item() < 1e-7


def test_projection_invalid(ctx):
    from paper_2110_07663_b200 import semlab as S
    with pytest.raises(Exception, match="capacity"):
        S.ProjectionBasis(0, n=10, ctx=ctx)
    with pytest.raises(ValueError, match="missing operator"):
        S.ProjectionBasis(3).insert(torch.zeros(8, dtype=torch.float64, device="cuda"), None)
