"""Golden fixtures for BASELINE.json configs c1-c4 AT THEIR OWN SIZES (E = 8^3, 16^3, 32^3), computed
by the REFERENCE semlab code (its own translation units compiled unmodified against the Eigen-API
shim, oracle/_ref/libsemlab_ref.so; recipe oracle/Makefile) plus the restated pMG/PCG/RHS of
oracle/ref_ext. The reference is single-threaded: c4 (a 63-iteration GMRES(20) solve with 2x
Chebyshev(2)-RAS per level on 11.4M dofs) takes ~15-25 min on one core, so cases run as separate
processes:

    make -C oracle && python tests/golden/make_golden_scale.py c1 c2 c3 c4     # (in parallel: one per case)

Each case writes tests/golden/scale_<case>.npz holding, for every output vector, the samples and
norms of scale_cases.summarize (the full vectors are 1.5-91 MB each), plus the solve's iteration
count, relative residual and full residual history.
"""
import ctypes as C
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
import scale_cases as sc  # noqa: E402

LIB = os.path.join(ROOT, "oracle", "_ref", "libsemlab_ref.so")
pd = C.POINTER(C.c_double)


def run(name):
    eps, E, orders, pc, coarse, krylov, eta = sc.CASES[name]
    p = orders[0]
    lib = C.CDLL(LIB)
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_case_create.restype = C.c_void_p
    lib.ref_case_n.restype = C.c_int64
    lib.ref_case_n.argtypes = [C.c_void_p]
    for f in ("apply_A", "schwarz", "rhs", "vcycle", "solve", "diag"):
        getattr(lib, f"ref_case_{f}").argtypes = None

    def chk(rc):
        if rc != 0:
            raise RuntimeError(lib.ref_last_error().decode())

    t0 = time.time()
    arr = (C.c_int * len(orders))(*orders)
    h = lib.ref_case_create(C.c_double(eps), E, arr, len(orders), pc.encode(), coarse.encode(), eta)
    if not h:
        raise RuntimeError(lib.ref_last_error().decode())
    h = C.c_void_p(h)
    n = lib.ref_case_n(h)
    assert n == sc.n_of(E, p)
    idx, w = sc.sample_index(E, p), sc.weights(n)
    out = {"meta": np.array([eps, E, p, krylov, eta]), "orders": np.array(orders)}
    print(f"[{name}] setup {time.time() - t0:.1f}s n={n}", flush=True)

    def keep(key, v):
        out[key], out[key + "_norms"] = sc.summarize(v, idx, w)

    u = sc.input_u(E, p)
    Au = np.zeros(n)
    chk(lib.ref_case_apply_A(h, u.ctypes.data_as(pd), Au.ctypes.data_as(pd)))
    keep("Au", Au)
    diag = np.zeros(n)
    chk(lib.ref_case_diag(h, diag.ctypes.data_as(pd)))
    keep("diag", diag)
    b = np.zeros(n)
    chk(lib.ref_case_rhs(h, C.c_uint64(1), b.ctypes.data_as(pd)))
    keep("rhs", b)
    print(f"[{name}] Au/diag/rhs {time.time() - t0:.1f}s", flush=True)
    if name in ("c3", "c4"):
        r = sc.input_r(E, p)
        for mode, key in ((1, "ras"), (0, "asm")):
            z = np.zeros(n)
            chk(lib.ref_case_schwarz(h, mode, r.ctypes.data_as(pd), z.ctypes.data_as(pd)))
            keep(key, z)
        print(f"[{name}] RAS/ASM {time.time() - t0:.1f}s", flush=True)
    if len(orders) > 1:
        z, lams = np.zeros(n), np.zeros(len(orders))
        chk(lib.ref_case_vcycle(h, b.ctypes.data_as(pd), z.ctypes.data_as(pd), lams.ctypes.data_as(pd)))
        keep("vcycle", z)
        out["lams"] = lams[:len(orders) - 1]
        print(f"[{name}] V-cycle {time.time() - t0:.1f}s lams={out['lams']}", flush=True)
    x, hist = np.zeros(n), np.zeros(1000)
    it, rel = C.c_int(), C.c_double()
    ts = time.time()
    chk(lib.ref_case_solve(h, krylov, 20, C.c_double(1e-8), 1000, x.ctypes.data_as(pd), C.byref(it), C.byref(rel),
                           hist.ctypes.data_as(pd), 1000))
    t_solve = time.time() - ts
    keep("x", x)
    out["iters"], out["relres"], out["history"] = np.array([it.value]), np.array([rel.value]), hist[:it.value]
    out["t_solve_s"] = np.array([t_solve])
    lib.ref_case_destroy(h)
    path = os.path.join(HERE, f"scale_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"[{name}] solve {it.value} iters rel {rel.value:.3e} in {t_solve:.1f}s; wrote {path} "
          f"({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


def amg_sizes():
    """Level sizes of the reference AMG hierarchy of the p=1 coarse problem (CoarseSolve "amg"):
    aggregation breaks ties on exact comparisons, so these pin the coarse matrix bitwise."""
    import json
    lib = C.CDLL(LIB)
    out = {}
    for eps in (0.3, 1.0):
        for E in (4, 8, 16, 32):
            nl, sizes = C.c_int(), (C.c_int64 * 32)()
            if lib.ref_amg_info(C.c_double(eps), E, C.byref(nl), sizes, 32, None) != 0:
                raise RuntimeError("ref_amg_info failed")
            out[f"e{eps}_E{E}"] = [int(sizes[i]) for i in range(nl.value)]
    path = os.path.join(HERE, "amg_levels.json")
    json.dump(out, open(path, "w"), indent=1)
    print(f"wrote {path}: {out}")


if __name__ == "__main__":
    args = sys.argv[1:] or list(sc.CASES) + ["amg"]
    for nm in args:
        amg_sizes() if nm == "amg" else run(nm)
