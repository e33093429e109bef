"""Generate golden vectors from the REFERENCE semlab code (its own translation units compiled
against the Eigen-API shim, oracle/_ref/libsemlab_ref.so; recipe oracle/Makefile) for pinning
the numpy oracle (tests/test_oracle_pin.py) and the B200 product (tests/test_golden_gpu.py).

    make -C oracle && python tests/golden/make_golden.py

Inputs are seeded (numpy default_rng) so the fixtures are reproducible. Pieces the reference
does not ship (pMG, PCG, RHS) come from oracle/ref_ext (restated from SPEC.md) and are marked so.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(ROOT, "oracle", "_ref", "libsemlab_ref.so")
pd = C.POINTER(C.c_double)
pi = C.POINTER(C.c_int)

OP_CASES = [(1.0, 2, 2), (0.3, 2, 3), (0.3, 2, 4), (1.0, 4, 7), (0.3, 4, 7)]
SOLVE_CASES = [  # (name, eps, E, orders, precond, coarse, krylov)
    ("jacobi_pcg_box", 1.0, 4, (7,), "jacobi", "direct", 1),
    ("pmg_jacobi_pcg_box", 1.0, 4, (7, 3, 1), "jacobi", "direct", 1),
    ("pmg_ras_gmres_kershaw", 0.3, 4, (7, 3, 1), "ras", "direct", 0),
    ("pmg_ras_gmres_kershaw_amg", 0.3, 4, (7, 3, 1), "ras", "amg", 0),
]
NEUMANN_CASES = [(0.3, 2, 5), (1.0, 4, 3)]


def main():
    lib = C.CDLL(LIB)
    out = {}

    def chk(rc):
        if rc != 0:
            raise RuntimeError(lib.ref_last_error().decode() if hasattr(lib, "ref_last_error") else "ref error")

    lib.ref_last_error.restype = C.c_char_p
    for p in range(1, 10):
        nodes, w, d = np.zeros(p + 1), np.zeros(p + 1), np.zeros((p + 1) ** 2)
        chk(lib.ref_gll(p, nodes.ctypes.data_as(pd), w.ctypes.data_as(pd), d.ctypes.data_as(pd)))
        out[f"gll{p}_nodes"], out[f"gll{p}_weights"], out[f"gll{p}_diff"] = nodes, w, d
    u = np.zeros(1000)
    chk(lib.ref_uniform(C.c_uint64(0), 1000, u.ctypes.data_as(pd)))
    out["uniform_seed0"] = u
    for eps, E, p in OP_CASES:
        key = f"e{eps}_E{E}_p{p}"
        n, nl = C.c_int64(), C.c_int64()
        chk(lib.ref_sizes(C.c_double(eps), E, p, C.byref(n), C.byref(nl)))
        n, nl = n.value, nl.value
        rng = np.random.default_rng(1000 * p + E)
        uu = rng.standard_normal(n)
        w = np.zeros(n)
        chk(lib.ref_apply_A(C.c_double(eps), E, p, uu.ctypes.data_as(pd), w.ctypes.data_as(pd)))
        out[f"{key}_u"], out[f"{key}_Au"] = uu, w
        diag, mass = np.zeros(n), np.zeros(n)
        chk(lib.ref_diag_mass(C.c_double(eps), E, p, diag.ctypes.data_as(pd), mass.ctypes.data_as(pd)))
        out[f"{key}_diag"], out[f"{key}_mass"] = diag, mass
        rhs = np.zeros(n)
        chk(lib.ref_build_rhs(C.c_double(eps), E, p, C.c_uint64(1), rhs.ctypes.data_as(pd)))
        out[f"{key}_rhs"] = rhs
        if p >= 2:
            r = rng.standard_normal(n) * (diag != 0)
            for mode, name in ((1, "ras"), (0, "asm")):
                z, L, l0 = np.zeros(n), np.zeros(E ** 3 * 3), np.zeros(p + 3)
                chk(lib.ref_schwarz_apply(C.c_double(eps), E, p, mode, r.ctypes.data_as(pd), z.ctypes.data_as(pd),
                                          L.ctypes.data_as(pd), l0.ctypes.data_as(pd)))
                out[f"{key}_r"], out[f"{key}_{name}"], out[f"{key}_boxlen"] = r, z, L
                lam, rounds = C.c_double(), C.c_int()  # ref_lambda smoother code: 1 RAS, 2 ASM
                chk(lib.ref_lambda(C.c_double(eps), E, p, 1 if mode == 1 else 2, C.byref(lam), C.byref(rounds)))
                out[f"{key}_lam_{name}"] = np.array([lam.value, rounds.value])
            lam, rounds = C.c_double(), C.c_int()
            chk(lib.ref_lambda(C.c_double(eps), E, p, 0, C.byref(lam), C.byref(rounds)))
            out[f"{key}_lam_jacobi"] = np.array([lam.value, rounds.value])
            x = np.zeros(n)
            chk(lib.ref_cheby_smooth(C.c_double(eps), E, p, 1, 2, C.c_double(3.0), rhs.ctypes.data_as(pd),
                                     x.ctypes.data_as(pd)))
            out[f"{key}_cheby_ras_eta2_lam3"] = x
    # V-cycles and solves (RESTATED pMG / PCG over the reference classes)
    for eps, E, orders, sm, coarse in [(0.3, 4, (7, 3, 1), "jacobi", "direct"), (0.3, 4, (7, 3, 1), "ras", "direct"),
                                       (0.3, 4, (7, 3, 1), "ras", "amg")]:
        key = f"vcycle_e{eps}_E{E}_{sm}_{coarse}"
        n = (E * orders[0] + 1) ** 3
        b = out[f"e{eps}_E{E}_p{orders[0]}_rhs"]
        z, lams = np.zeros(n), np.zeros(len(orders))
        arr = (C.c_int * len(orders))(*orders)
        chk(lib.ref_vcycle(C.c_double(eps), E, arr, len(orders), sm.encode(), coarse.encode(), 2,
                           b.ctypes.data_as(pd), z.ctypes.data_as(pd), lams.ctypes.data_as(pd)))
        out[key], out[key + "_lams"] = z, lams
    for eps, E, p in NEUMANN_CASES:
        key = f"neu_e{eps}_E{E}_p{p}"
        n = (E * p + 1) ** 3
        rng = np.random.default_rng(7000 + 10 * p + E)
        uu, r = rng.standard_normal(n), rng.standard_normal(n)
        Au, diag, ras, asm = (np.zeros(n) for _ in range(4))
        chk(lib.ref_neumann(C.c_double(eps), E, p, uu.ctypes.data_as(pd), Au.ctypes.data_as(pd),
                            diag.ctypes.data_as(pd), r.ctypes.data_as(pd), ras.ctypes.data_as(pd),
                            asm.ctypes.data_as(pd)))
        out[f"{key}_u"], out[f"{key}_Au"], out[f"{key}_diag"] = uu, Au, diag
        out[f"{key}_r"], out[f"{key}_ras"], out[f"{key}_asm"] = r, ras, asm
    # ProjectionBasis: capacity 3, six inserts. The 4th repeats the 2nd (dependent: skipped);
    # the 5th and 6th evict the two oldest.
    eps, E, p = 0.3, 2, 4
    n = (E * p + 1) ** 3
    rng = np.random.default_rng(4242)
    X = rng.standard_normal((6, n))
    X[3] = X[1]  # dependent on the basis: skipped
    b = rng.standard_normal(n)
    Xc = np.ascontiguousarray(X)
    size = C.c_int()
    basis, guess = np.zeros((3, n)), np.zeros(n)
    chk(lib.ref_projection(C.c_double(eps), E, p, 3, 6, Xc.ctypes.data_as(pd), b.ctypes.data_as(pd),
                           C.byref(size), basis.ctypes.data_as(pd), guess.ctypes.data_as(pd)))
    out["proj_X"], out["proj_b"], out["proj_size"] = X, b, np.array([size.value])
    out["proj_basis"], out["proj_guess"] = basis[:size.value], guess
    for name, eps, E, orders, pc, coarse, kr in SOLVE_CASES:
        n = (E * orders[0] + 1) ** 3
        x, hist = np.zeros(n), np.zeros(500)
        it, rel = C.c_int(), C.c_double()
        arr = (C.c_int * len(orders))(*orders)
        chk(lib.ref_solve(C.c_double(eps), E, arr, len(orders), pc.encode(), coarse.encode(), 2, kr, C.c_double(1e-8),
                          x.ctypes.data_as(pd), C.byref(it), C.byref(rel), hist.ctypes.data_as(pd), 500))
        out[f"solve_{name}_x"] = x
        out[f"solve_{name}_iters"] = np.array([it.value])
        out[f"solve_{name}_relres"] = np.array([rel.value])
        out[f"solve_{name}_history"] = hist[:it.value]
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
