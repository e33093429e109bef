"""Golden vectors for the pMG variants of SPEC.md:313-349 that the first fixtures do not cover:
un-accelerated (plain) ASM/RAS smoothers, the additive V-cycle without post-smoothing, and the
Neumann (pressure) hierarchy with the zero-mean coarse solve. Computed by the reference semlab
classes (SemSpace, SchwarzSmoother, ChebyshevSmoother, estimate_lambda_max, gmres_solve: its own
translation units against the Eigen-API shim) under oracle/ref_ext's restated pMG
(oracle/_ref/libsemlab_ref.so):

    make -C oracle && python tests/golden/make_golden_pmg.py
"""
import ctypes as C
import os
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(ROOT, "oracle", "_ref", "libsemlab_ref.so")
pd = C.POINTER(C.c_double)

# name: (eps, E, orders, smoother, coarse, eta, neumann, additive)
VCYCLES = {
    "ras_plain_std": (0.3, 4, (7, 3, 1), "ras_plain", "direct", 2, 0, 0),
    "asm_plain_add": (0.3, 4, (7, 3, 1), "asm_plain", "direct", 2, 0, 1),
    "ras_plain_add": (0.3, 4, (7, 3, 1), "ras_plain", "amg", 2, 0, 1),
    "ras_cheb_add": (0.3, 4, (5, 3, 1), "ras", "direct", 2, 0, 1),
    "neu_ras_cheb_std": (0.3, 4, (7, 3, 1), "ras", "direct", 2, 1, 0),
    "neu_jac_cheb_std": (1.0, 4, (5, 2, 1), "jacobi", "direct", 3, 1, 0),
    "neu_asm_plain_add": (0.3, 2, (4, 1), "asm_plain", "direct", 2, 1, 1),
}
SOLVES = {
    "ras_plain_add": (0.3, 4, (7, 3, 1), "ras_plain", "direct", 2, 0, 1),
    "neu_ras_cheb_std": (0.3, 4, (7, 3, 1), "ras", "direct", 2, 1, 0),
}


def rhs(name, eps, E, p, neumann):
    n = (E * p + 1) ** 3
    b = np.random.default_rng(zlib.crc32(name.encode()) % 100000).standard_normal(n)
    if neumann:
        b -= b.mean()  # consistent with the constant nullspace
    else:
        N = E * p + 1
        a = np.zeros(N, dtype=bool)
        a[0] = a[-1] = True
        b[(a[None, None, :] | a[None, :, None] | a[:, None, None]).reshape(-1)] = 0.0
    return b


def main():
    lib = C.CDLL(LIB)
    lib.ref_last_error.restype = C.c_char_p

    def chk(rc):
        if rc != 0:
            raise RuntimeError(lib.ref_last_error().decode())

    out = {}
    for name, (eps, E, orders, sm, coarse, eta, neu, add) in VCYCLES.items():
        b = rhs(name, eps, E, orders[0], neu)
        z = np.zeros_like(b)
        arr = (C.c_int * len(orders))(*orders)
        chk(lib.ref_vcycle_ex(C.c_double(eps), E, arr, len(orders), sm.encode(), coarse.encode(), eta, neu, add,
                              b.ctypes.data_as(pd), z.ctypes.data_as(pd)))
        out[f"vc_{name}_b"], out[f"vc_{name}_z"] = b, z
    for name, (eps, E, orders, sm, coarse, eta, neu, add) in SOLVES.items():
        b = rhs("solve" + name, eps, E, orders[0], neu)
        x = np.zeros_like(b)
        it, rel = C.c_int(), C.c_double()
        arr = (C.c_int * len(orders))(*orders)
        chk(lib.ref_solve_ex(C.c_double(eps), E, arr, len(orders), sm.encode(), coarse.encode(), eta, neu, add,
                             b.ctypes.data_as(pd), C.c_double(1e-8), x.ctypes.data_as(pd), C.byref(it),
                             C.byref(rel)))
        out[f"sv_{name}_b"], out[f"sv_{name}_x"] = b, x
        out[f"sv_{name}_iters"], out[f"sv_{name}_relres"] = np.array([it.value]), np.array([rel.value])
        print(name, it.value, rel.value)
    path = os.path.join(HERE, "pmg_ext_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
