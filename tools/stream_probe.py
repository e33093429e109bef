"""Solve time at c4 under the bench's conditions, one factor at a time: default vs side stream,
with and without an nvidia-smi sampler running (diagnoses gaps between perf_probe and bench)."""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2110_07663_b200 import semlab as S  # noqa: E402


def run(side_stream: bool, sampler: int, E: int = 32, reps: int = 4, sampler_ms: int = 100):
    stream = torch.cuda.Stream() if side_stream else torch.cuda.default_stream()
    torch.cuda.set_stream(stream)
    ctx = S.Context(0, stream) if side_stream else S.Context(0)
    mesh = S.generate_kershaw(0.3, E, ctx)
    pmg = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 32, S.COARSE_AMG)
    sp = pmg.spaces[0]
    A, M = sp.as_linop(), pmg.as_linop()
    b = sp.build_rhs(1)
    x = torch.zeros_like(b)
    cfg = S.GmresConfig(restart=20, tol=1e-8, max_iters=500)
    S.gmres_solve(A, M, b, x, cfg)
    proc = None
    if sampler:
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap") if sampler == 2 else "clocks.sm"
        proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader",
                                 "-lms", str(sampler_ms)], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    ts = []
    for _ in range(reps):
        x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = S.gmres_solve(A, M, b, x, cfg)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    if proc:
        proc.terminate()
        proc.wait()
    print(f"side_stream={side_stream} sampler={sampler}/{sampler_ms}ms: iters {st.iterations} ms {['%.1f' % t for t in ts]}",
          flush=True)
    del pmg, mesh, ctx
    torch.cuda.set_stream(torch.cuda.default_stream())


if __name__ == "__main__":
    for smp in (0, 1, 2, 0):
        run(True, smp)
    run(True, 2, sampler_ms=500)
