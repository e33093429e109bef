"""GPU parity of the pMG variants of SPEC.md:313-349 against the reference classes under the
restated pMG (tests/golden/pmg_ext_golden.npz, from oracle/_ref): un-accelerated (plain) ASM/RAS
smoothers, the additive V-cycle without post-smoothing (§2.2.2), and the Neumann
(pressure) hierarchy whose singular coarse problem is solved on the zero-mean subspace.
Tolerances: V-cycles 1e-10 (FP64 smoothers); GMRES iterations within +-1 and x within 1e-8."""
import os
import sys

import numpy as np
import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden_pmg import SOLVES, VCYCLES  # noqa: E402

pytestmark = pytest.mark.gpu
GOLD = os.path.join(HERE, "golden", "pmg_ext_golden.npz")


def _pmg(ctx, cfg, precision=64):
    from paper_2110_07663_b200 import semlab as S
    eps, E, orders, sm, coarse, eta, neu, add = cfg
    kind = {"jacobi": S.JACOBI_SMOOTHER, "ras": S.RAS_SMOOTHER, "asm": S.ASM_SMOOTHER,
            "ras_plain": S.RAS_PLAIN_SMOOTHER, "asm_plain": S.ASM_PLAIN_SMOOTHER}[sm]
    return S.Pmg(S.generate_kershaw(eps, E, ctx), orders, kind, eta, 0.1, 1.1, precision,
                 S.COARSE_DIRECT if coarse == "direct" else S.COARSE_AMG,
                 bc=S.NEUMANN if neu else S.DIRICHLET, cycle=S.ADDITIVE_CYCLE if add else S.STANDARD_CYCLE)


@pytest.mark.parametrize("name", sorted(VCYCLES))
def test_vcycle_variant_matches_reference(ctx, name):
    g = np.load(GOLD)
    pmg = _pmg(ctx, VCYCLES[name])
    b = pmg.spaces[0].to_device(g[f"vc_{name}_b"])
    z1 = pmg.vcycle(b)
    z2 = pmg.vcycle(b)  # the second call replays the captured CUDA graph (Dirichlet hierarchies)
    want = g[f"vc_{name}_z"]
    for z in (z1, z2):
        err = np.abs(z.cpu().numpy() - want).max() / np.abs(want).max()
        print(f"{name}: {err:.2e}")
        assert err <= 1e-10
    assert torch.equal(z1, z2)


def test_neumann_hierarchy_contracts(ctx):
    """Neumann levels keep the constants (P 1 = 1, unmasked transfers), the V-cycle is a fixed
    linear operator, and the singular coarse problem is refused by the AMG coarse solve."""
    pmg = _pmg(ctx, (0.3, 4, (3, 1), "jacobi", "direct", 2, 1, 0))
    sp = pmg.spaces[0]
    c = pmg.prolong(0, pmg.spaces[1].zeros() + 1.0)
    assert torch.allclose(c, torch.ones_like(c), atol=1e-13)
    b1 = torch.randn(sp.n, dtype=torch.float64, device="cuda")
    b2 = torch.randn(sp.n, dtype=torch.float64, device="cuda")
    b1 -= b1.mean()
    b2 -= b2.mean()
    z = pmg.vcycle(2.0 * b1 - b2)
    zl = 2.0 * pmg.vcycle(b1) - pmg.vcycle(b2)
    assert (z - zl).abs().max().item() <= 1e-11 * zl.abs().max().item()
    with pytest.raises(ValueError):  # the singular coarse problem has no AMG path
        _pmg(ctx, (0.3, 2, (3, 1), "jacobi", "amg", 2, 1, 0))


@pytest.mark.parametrize("name", sorted(SOLVES))
def test_solve_variant_matches_reference(ctx, name):
    from paper_2110_07663_b200 import semlab as S
    g = np.load(GOLD)
    pmg = _pmg(ctx, SOLVES[name])
    sp = pmg.spaces[0]
    b = sp.to_device(g[f"sv_{name}_b"])
    x = sp.zeros()
    st = S.gmres_solve(sp.as_linop(), pmg.as_linop(), b, x, S.GmresConfig(tol=1e-8, max_iters=500))
    it_ref = int(g[f"sv_{name}_iters"][0])
    want = g[f"sv_{name}_x"]
    err = np.abs(x.cpu().numpy() - want).max() / np.abs(want).max()
    print(f"{name}: {st.iterations} iterations (reference {it_ref}), x {err:.2e}")
    assert st.converged
    assert abs(st.iterations - it_ref) <= 1
    assert err <= 1e-8


def test_neumann_fp32_smoother_solve(ctx):
    """The paper's setting on the pressure problem: FP32 Chebyshev-RAS Neumann hierarchy with FP64
    GMRES converges in the FP64 reference's iteration count (+-1)."""
    from paper_2110_07663_b200 import semlab as S
    g = np.load(GOLD)
    name = "neu_ras_cheb_std"
    pmg = _pmg(ctx, SOLVES[name], precision=32)
    sp = pmg.spaces[0]
    b = sp.to_device(g[f"sv_{name}_b"])
    x = sp.zeros()
    st = S.gmres_solve(sp.as_linop(), pmg.as_linop(), b, x, S.GmresConfig(tol=1e-8, max_iters=500))
    assert st.converged
    assert abs(st.iterations - int(g[f"sv_{name}_iters"][0])) <= 1
