"""Per-phase timing of the z-slab path (run under torchrun): Ax (+interface sum), RAS (+halo,
owner copy), V-cycle, GMRES solve. Rank 0 prints max-over-ranks times."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2110_07663_b200 import semlab as S  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank)
    uid = [S.Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = S.Context(rank, stream, rank, world, uid[0])
    ctx.set_exchange(os.environ.get("EXCHANGE", "nccl") == "peer")
    E = int(os.environ.get("E", "32"))
    mesh = S.generate_kershaw(0.3, E, ctx)
    pmg = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 32, S.COARSE_AMG)
    sp = pmg.spaces[0]
    u = torch.randn(sp.n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(u)
    sch = S.SchwarzSmoother(sp, S.RAS, 32)

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        t = torch.tensor([(time.perf_counter() - t0) / reps])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item() * 1e3

    res = {"Ax": timeit(lambda: sp.apply_A(u, w)), "RAS": timeit(lambda: sch.apply(u, w)),
           "vcycle": timeit(lambda: pmg.vcycle(u, w), 5), "dot": timeit(lambda: sp.dot(u, w), 50)}
    b = sp.build_rhs(1)
    x = torch.zeros_like(b)

    def solve():
        x.zero_()
        return S.gmres_solve(sp.as_linop(), pmg.as_linop(), b, x)
    st = solve()
    res["gmres"] = timeit(solve, 2)
    res["iters"] = st.iterations
    if rank == 0:
        print(f"world={world} E={E} exchange={os.environ.get('EXCHANGE', 'nccl')}: " + ", ".join(f"{k}={v:.3f}" + ("" if k == "iters" else "ms") for k, v in res.items()),
              flush=True)
    dist.barrier()


if __name__ == "__main__":
    main()
