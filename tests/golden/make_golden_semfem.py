"""Golden vectors for the SEMFEM + AMG preconditioner (the paper's low-order competitor, PAPER.md
§2.2.1; reference semfem.cpp:12-134 and amg.cpp), computed by the reference's own translation
units against the Eigen-API shim (oracle/_ref/libsemlab_ref.so):

    make -C oracle && python tests/golden/make_golden_semfem.py
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(ROOT, "oracle", "_ref", "libsemlab_ref.so")
pd = C.POINTER(C.c_double)

APPLY = [(0.3, 2, 3), (1.0, 4, 3), (0.3, 4, 7), (0.05, 4, 5)]
SOLVE = [(0.3, 4, 7), (0.05, 4, 7)]


def masked_random(eps, E, p, seed):
    N = E * p + 1
    r = np.random.default_rng(seed).standard_normal(N ** 3)
    a = np.zeros(N, dtype=bool)
    a[0] = a[-1] = True
    r[(a[None, None, :] | a[None, :, None] | a[:, None, None]).reshape(-1)] = 0.0
    return r


def main():
    lib = C.CDLL(LIB)
    lib.ref_last_error.restype = C.c_char_p

    def chk(rc):
        if rc != 0:
            raise RuntimeError(lib.ref_last_error().decode())

    out = {}
    for eps, E, p in APPLY:
        key = f"e{eps}_E{E}_p{p}"
        r = masked_random(eps, E, p, 100 * E + p)
        z = np.zeros_like(r)
        nl, sizes = C.c_int(), (C.c_int64 * 32)()
        chk(lib.ref_semfem_apply(C.c_double(eps), E, p, r.ctypes.data_as(pd), z.ctypes.data_as(pd), C.byref(nl),
                                 sizes, 32))
        out[f"{key}_r"], out[f"{key}_z"] = r, z
        out[f"{key}_levels"] = np.array([sizes[i] for i in range(nl.value)])
        print(key, out[f"{key}_levels"])
    for eps, E, p in SOLVE:
        key = f"solve_e{eps}_E{E}_p{p}"
        b = masked_random(eps, E, p, 7 + E)
        x = np.zeros_like(b)
        it, rel = C.c_int(), C.c_double()
        chk(lib.ref_semfem_solve(C.c_double(eps), E, p, b.ctypes.data_as(pd), C.c_double(1e-8), x.ctypes.data_as(pd),
                                 C.byref(it), C.byref(rel)))
        out[f"{key}_b"], out[f"{key}_x"] = b, x
        out[f"{key}_iters"], out[f"{key}_relres"] = np.array([it.value]), np.array([rel.value])
        print(key, it.value, rel.value)
    path = os.path.join(HERE, "semfem_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
