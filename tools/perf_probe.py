"""Quick per-kernel timing probe at a BASELINE config (not the bench; no oracle)."""
import argparse
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2110_07663_b200 import semlab as S  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=32)
    ap.add_argument("--eps", type=float, default=0.3)
    ap.add_argument("--p", type=int, default=7)
    ap.add_argument("--smoother", default="ras")
    ap.add_argument("--coarse", default="amg")
    ap.add_argument("--solve", type=int, default=1)
    a = ap.parse_args()
    ctx = S.Context(0)
    t0 = time.time()
    mesh = S.generate_kershaw(a.eps, a.E, ctx)
    sp = S.SemSpace(mesh, a.p)
    print(f"space setup {time.time() - t0:.2f}s n={sp.n} E={sp.n_elements}", flush=True)
    u = torch.randn(sp.n, dtype=torch.float64, device="cuda")
    w = sp.zeros()
    t = timeit(lambda: sp.apply_A(u, w))
    E, nloc = sp.n_elements, (a.p + 1) ** 3
    byts = 48 * E * nloc + 16 * sp.n
    print(f"Ax: {t * 1e6:.1f} us  {byts / t / 1e9:.0f} GB/s (alg bytes {byts / 1e6:.1f} MB)", flush=True)
    if a.p == 7:
        t = timeit(lambda: sp.apply_A_geom32(u, w))
        byts = 24 * E * nloc + 16 * sp.n
        print(f"Ax geom32: {t * 1e6:.1f} us  {byts / t / 1e9:.0f} GB/s (alg bytes {byts / 1e6:.1f} MB)", flush=True)
    t0 = time.time()
    sch = S.SchwarzSmoother(sp, S.RAS, 32)
    print(f"schwarz setup {time.time() - t0:.2f}s", flush=True)
    z = sp.zeros()
    t = timeit(lambda: sch.apply(u, z))
    P = a.p + 3
    byts = 4 * E * (3 * P * P + 3 * P) + 16 * sp.n
    print(f"RAS fp32: {t * 1e6:.1f} us  {byts / t / 1e9:.0f} GB/s (alg bytes {byts / 1e6:.1f} MB) "
          f"{12 * P ** 4 * E / t / 1e12:.1f} TFLOP/s", flush=True)
    if a.p == 7:
        cheb = S.ChebyshevSmoother(sch.as_linop(), sp.as_linop_geom32(), S.ChebyParams(2, 0.1, 1.1, 12.8))
        xs = torch.zeros_like(u)
        bb = sp.build_rhs(1)

        def smooth():
            xs.copy_(u)
            cheb.smooth(bb, xs)
        t = timeit(smooth)
        print(f"cheby(2)-RAS smooth (3 Ax32 + 3 RAS): {t * 1e6:.1f} us", flush=True)
    if not a.solve:
        return
    t0 = time.time()
    sm = {"ras": S.RAS_SMOOTHER, "jacobi": S.JACOBI_SMOOTHER, "asm": S.ASM_SMOOTHER}[a.smoother]
    pmg = S.Pmg(mesh, (a.p, 3, 1), sm, 2, 0.1, 1.1, 32, S.COARSE_AMG if a.coarse == "amg" else S.COARSE_DIRECT)
    print(f"pmg setup {time.time() - t0:.2f}s lam={[pmg.lam(l) for l in range(2)]}", flush=True)
    b = pmg.spaces[0].build_rhs(1)
    zz = torch.empty_like(b)
    t = timeit(lambda: pmg.vcycle(b, zz), reps=5)
    print(f"vcycle {t * 1e3:.2f} ms", flush=True)
    A = pmg.spaces[0].as_linop()
    M = pmg.as_linop()
    x = torch.zeros_like(b)
    S.gmres_solve(A, M, b, x, S.GmresConfig())  # warm (basis allocation, first launches)
    x.zero_()
    torch.cuda.synchronize()
    t0 = time.time()
    st = S.gmres_solve(A, M, b, x, S.GmresConfig())
    torch.cuda.synchronize()
    dt = time.time() - t0
    print(f"gmres: iters {st.iterations} rel {st.rel_residual:.2e} conv {st.converged} time {dt * 1e3:.1f} ms "
          f"-> {pmg.spaces[0].n * st.iterations / dt / 1e9:.2f} GDOF*iter/s", flush=True)


if __name__ == "__main__":
    main()
