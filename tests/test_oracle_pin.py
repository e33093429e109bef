"""Pin the numpy oracle against golden vectors produced by the REFERENCE code itself
(tests/golden/reference_golden.npz, generator tests/golden/make_golden.py over
oracle/_ref/libsemlab_ref.so = the reference's own translation units + Eigen-API shim).
The pMG/PCG/RHS fixtures come from the restated extension (the reference ships no pmg.cpp /
CG / bench.cpp), so for those the pin is oracle-vs-independent-C++-restatement."""
import os

import numpy as np
import pytest

from oracle import semlab_np as o

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz"))
REF_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "libsemlab_ref.so")
OP_CASES = [(1.0, 2, 2), (0.3, 2, 3), (0.3, 2, 4), (1.0, 4, 7), (0.3, 4, 7)]


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_gll_and_rng_pinned():
    for p in range(1, 10):
        g = o.gll(p)
        np.testing.assert_array_equal(g.nodes, G[f"gll{p}_nodes"])
        np.testing.assert_array_equal(g.weights, G[f"gll{p}_weights"])
        np.testing.assert_allclose(g.diff.ravel(order="F"), G[f"gll{p}_diff"], rtol=0, atol=1e-13 * p * p)
    np.testing.assert_array_equal(o.uniform_pm1(0, 1000), G["uniform_seed0"])


@pytest.mark.parametrize("eps,E,p", OP_CASES)
def test_space_pinned(eps, E, p):
    key = f"e{eps}_E{E}_p{p}"
    s = o.SemSpace(o.generate_kershaw(eps, E), p)
    assert rel(s.apply_A(G[f"{key}_u"]), G[f"{key}_Au"]) < 1e-12
    assert rel(s.stiffness_diag(), G[f"{key}_diag"]) < 1e-12
    assert rel(s.mass_diag, G[f"{key}_mass"]) < 1e-13
    assert rel(o.build_rhs(s, 1), G[f"{key}_rhs"]) < 1e-13


@pytest.mark.parametrize("eps,E,p", [c for c in OP_CASES if c[2] >= 2])
def test_schwarz_chebyshev_lambda_pinned(eps, E, p):
    key = f"e{eps}_E{E}_p{p}"
    s = o.SemSpace(o.generate_kershaw(eps, E), p)
    r = G[f"{key}_r"]
    for mode, name in ((o.RAS, "ras"), (o.ASM, "asm")):
        sch = o.SchwarzSmoother(s, mode)
        assert rel(sch.apply(r), G[f"{key}_{name}"]) < 1e-12
        np.testing.assert_allclose(sch.lengths.ravel(), G[f"{key}_boxlen"], rtol=1e-14)
        est = o.estimate_lambda_max(sch.apply, s.apply_A, s.n, 10, 0)
        lam, rounds = G[f"{key}_lam_{name}"]
        assert abs(est.value - lam) <= 1e-10 * lam and est.rounds_used == int(rounds)
    inv = o.jacobi_inverse_diag(s)
    est = o.estimate_lambda_max(lambda v: inv * v, s.apply_A, s.n, 10, 0)
    lam, rounds = G[f"{key}_lam_jacobi"]
    assert abs(est.value - lam) <= 1e-10 * lam and est.rounds_used == int(rounds)
    ras = o.SchwarzSmoother(s, o.RAS)
    cheb = o.ChebyshevSmoother(ras.apply, s.apply_A, o.ChebyParams(2, 0.1, 1.1, 3.0))
    x = np.zeros(s.n)
    cheb.smooth(G[f"{key}_rhs"], x)
    assert rel(x, G[f"{key}_cheby_ras_eta2_lam3"]) < 1e-11


@pytest.mark.parametrize("sm,coarse", [("jacobi", "direct"), ("ras", "direct"), ("ras", "amg")])
def test_vcycle_pinned(sm, coarse):
    key = f"vcycle_e0.3_E4_{sm}_{coarse}"
    pmg = o.Pmg(o.generate_kershaw(0.3, 4), (7, 3, 1), sm, 2, 0.1, 1.1, coarse)
    np.testing.assert_allclose([lvl["lam"] for lvl in pmg.levels], G[key + "_lams"][:2], rtol=1e-10)
    assert rel(pmg.vcycle(G["e0.3_E4_p7_rhs"]), G[key]) < 1e-10


@pytest.mark.parametrize("name,eps,orders,pc,coarse,kr", [
    ("jacobi_pcg_box", 1.0, (7,), "jacobi", "direct", 1),
    ("pmg_jacobi_pcg_box", 1.0, (7, 3, 1), "jacobi", "direct", 1),
    ("pmg_ras_gmres_kershaw", 0.3, (7, 3, 1), "ras", "direct", 0),
    ("pmg_ras_gmres_kershaw_amg", 0.3, (7, 3, 1), "ras", "amg", 0),
])
def test_solves_pinned(name, eps, orders, pc, coarse, kr):
    mesh = o.generate_kershaw(eps, 4)
    if pc == "jacobi" and len(orders) == 1:
        s = o.SemSpace(mesh, 7)
        inv = o.jacobi_inverse_diag(s)
        M = lambda v: inv * v  # noqa: E731
    else:
        pmg = o.Pmg(mesh, orders, pc, 2, 0.1, 1.1, coarse)
        s, M = pmg.spaces[0], pmg.vcycle
    b = o.build_rhs(s, 1)
    x = np.zeros(s.n)
    st = o.gmres_solve(s.apply_A, M, b, x, o.GmresConfig()) if kr == 0 else o.pcg_solve(s.apply_A, M, b, x, 1e-8, 500)
    assert abs(st.iterations - int(G[f"solve_{name}_iters"][0])) <= 1
    assert rel(x, G[f"solve_{name}_x"]) < 1e-10


@pytest.mark.parametrize("eps,E,p", [(0.3, 2, 5), (1.0, 4, 3)])
def test_neumann_pinned(eps, E, p):
    """Neumann mode against the reference (ref_neumann: sem_space.cpp:207, 211-236; schwarz.cpp:151-160)."""
    key = f"neu_e{eps}_E{E}_p{p}"
    s = o.SemSpace(o.generate_kershaw(eps, E), p, o.NEUMANN)
    assert rel(s.apply_A(G[f"{key}_u"]), G[f"{key}_Au"]) < 1e-12
    assert rel(s.stiffness_diag(), G[f"{key}_diag"]) < 1e-12
    for mode, name in ((o.RAS, "ras"), (o.ASM, "asm")):
        assert rel(o.SchwarzSmoother(s, mode).apply(G[f"{key}_r"]), G[f"{key}_{name}"]) < 1e-12


def test_projection_basis_pinned():
    """ProjectionBasis (krylov.cpp:131-152) against the reference: skip of a dependent vector,
    eviction of the oldest, A-orthonormality and the projected guess."""
    s = o.SemSpace(o.generate_kershaw(0.3, 2), 4)
    pb = o.ProjectionBasis(3)
    for x in G["proj_X"]:
        pb.insert(x, s.apply_A)
    assert len(pb.basis) == int(G["proj_size"][0]) == 3
    for v, ref in zip(pb.basis, G["proj_basis"]):
        assert rel(v, ref) < 1e-11
    assert rel(pb.initial_guess(G["proj_b"]), G["proj_guess"]) < 1e-11
    Vb = np.stack(pb.basis, axis=1)
    gram = Vb.T @ np.stack([s.apply_A(v) for v in pb.basis], axis=1)
    assert np.abs(gram - np.eye(3)).max() < 1e-12


PMG_EXT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pmg_ext_golden.npz")


@pytest.mark.parametrize("name", ["ras_plain_std", "asm_plain_add", "ras_plain_add", "ras_cheb_add",
                                  "neu_ras_cheb_std", "neu_jac_cheb_std", "neu_asm_plain_add"])
def test_pmg_variants_pinned(name):
    """Plain ASM/RAS smoothers, the additive V-cycle and the Neumann hierarchy:
    the numpy restatement against the reference classes under oracle/ref_ext's pMG."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from make_golden_pmg import VCYCLES
    g = np.load(PMG_EXT)
    eps, E, orders, sm, coarse, eta, neu, add = VCYCLES[name]
    pmg = o.Pmg(o.generate_kershaw(eps, E), orders, sm, eta, 0.1, 1.1, coarse, 64,
                bc=o.NEUMANN if neu else o.DIRICHLET, cycle="additive" if add else "standard")
    z = pmg.vcycle(g[f"vc_{name}_b"])
    want = g[f"vc_{name}_z"]
    assert np.abs(z - want).max() <= 1e-10 * np.abs(want).max()


@pytest.mark.parametrize("eps,E,p", [(0.3, 2, 3), (1.0, 2, 5), (0.05, 2, 4)])
def test_semfem_matrix_pinned(eps, E, p):
    """assemble_semfem (semfem.cpp:12-98) restated in numpy against the reference's own matrix."""
    import ctypes as C
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built")
    lib = C.CDLL(REF_LIB)
    nnz = C.c_int64()
    assert lib.ref_semfem_matrix(C.c_double(eps), E, p, C.byref(nnz), None, None, None, C.c_int64(0)) == 0
    n = (E * p + 1) ** 3
    ptr, idx, val = np.zeros(n + 1, np.int64), np.zeros(nnz.value, np.int64), np.zeros(nnz.value)
    pi64 = C.POINTER(C.c_int64)
    assert lib.ref_semfem_matrix(C.c_double(eps), E, p, C.byref(nnz), ptr.ctypes.data_as(pi64),
                                 idx.ctypes.data_as(pi64), val.ctypes.data_as(C.POINTER(C.c_double)),
                                 C.c_int64(nnz.value)) == 0
    import scipy.sparse as sps
    ref = sps.csr_matrix((val, idx, ptr), shape=(n, n))
    got = o.assemble_semfem(o.SemSpace(o.generate_kershaw(eps, E), p))
    d = abs(got - ref)  # entries present in only one matrix (cancellation to an exact 0 in one
    assert d.max() <= 1e-13 * abs(ref).max()  # summation order) are roundoff-sized: covered here
