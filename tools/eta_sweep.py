"""BASELINE configs[4] study: Chebyshev order eta = 1..4 with Jacobi vs RAS smoothers (pMG (7,3,1),
GMRES(20) to 1e-8, AMG coarse solve) on a Kershaw eps=0.3 box. Prints a markdown table and writes
a CSV (suite.HEADER schema). Time per solve is the device time of one solve (CUDA events),
median of --trials after one warm-up.

    python tools/eta_sweep.py --elems 96 --out gpurun_out/eta_sweep_E96.csv
"""
import argparse
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_07663_b200 import semlab as S  # noqa: E402
from paper_2110_07663_b200 import suite  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=32)
    ap.add_argument("--eps", type=float, default=0.3)
    ap.add_argument("--trials", type=int, default=2)
    ap.add_argument("--smoothers", nargs="+", default=["cheb_jac", "cheb_ras"])
    ap.add_argument("--etas", type=int, nargs="+", default=[1, 2, 3, 4])
    ap.add_argument("--out", default="eta_sweep.csv")
    a = ap.parse_args()
    ctx = S.default_context()
    run = suite.make_runner(ctx, a.eps, a.elems, 7, max_iters=1000)
    rows = []
    print(f"| smoother | eta | iterations | ms / solve | GDOF*iter/s | setup s |")
    print(f"|---|---|---|---|---|---|")
    for kind in a.smoothers:
        for eta in a.etas:
            cfg = suite.PreconditionerConfig(kind, (7, 3, 1), eta, coarse="amg",
                                             precision=32 if kind == "cheb_ras" else 64)
            torch.cuda.empty_cache()
            t0 = time.perf_counter()
            solve = run(cfg)
            setup = time.perf_counter() - t0
            solve()  # warm-up (graph capture, workspace)
            ts, its, conv, rel = [], 0, True, 0.0
            for _ in range(a.trials):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                c, its, rel = solve()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
                conv = conv and c
            t = statistics.median(ts)
            rows.append(suite._row(a.eps, a.elems, 7, solve.n, cfg.name, its, setup, t, rel, conv, "sweep", 1))
            print(f"| {cfg.name} | {eta} | {its} | {t * 1e3:.1f} | {solve.n * its / t / 1e9:.3f} | {setup:.1f} |",
                  flush=True)
            del solve
    suite.write_csv(a.out, rows)


if __name__ == "__main__":
    main()
