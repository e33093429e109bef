"""Per-level kernel timing of the (7,3,1) hierarchy at a BASELINE config: Ax, RAS at p = 3 and the
V-cycle; CUDA events on the current stream (not the bench)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_07663_b200 import semlab as S  # noqa: E402
from tools.perf_probe import timeit  # noqa: E402


def main():
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    S.Context(0)
    mesh = S.generate_kershaw(0.3, E, S.Context(0))
    sp = S.SemSpace(mesh, 3)
    u = torch.randn(sp.n, dtype=torch.float64, device="cuda")
    w = sp.zeros()
    t = timeit(lambda: sp.apply_A(u, w))
    print(f"p=3 Ax: {t * 1e6:.1f} us", flush=True)
    sch = S.SchwarzSmoother(sp, S.RAS, 32)
    z = sp.zeros()
    t = timeit(lambda: sch.apply(u, z))
    print(f"p=3 RAS fp32: {t * 1e6:.1f} us", flush=True)


if __name__ == "__main__":
    main()
