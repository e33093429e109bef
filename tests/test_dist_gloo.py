"""CPU (gloo, world_size 2 and 3) tests of the distributed path's host-side logic: the z-slab
partition, owned-plane reductions (each interface plane counted once), and the interface-sum
protocol (lower partial + upper partial on both ranks) applied to the oracle's Q^T."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import semlab_np as o
from paper_2110_07663_b200.partition import Slab


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E, p = 4, 3
        sl = Slab(p, E, E, E, rank, world)
        sp = o.SemSpace(o.generate_kershaw(0.3, E), p)
        rng = np.random.default_rng(0)
        u = rng.standard_normal(sp.n)
        v = rng.standard_normal(sp.n)
        # owned-plane reduction == global dot
        part = torch.tensor([float(u[sl.owned_slice_global()] @ v[sl.owned_slice_global()])], dtype=torch.float64)
        dist.all_reduce(part)
        ok_dot = abs(part.item() - float(u @ v)) <= 1e-12 * abs(float(u @ v))
        # slab-local Q^T of this rank's elements, then the interface-sum protocol
        loc = rng.standard_normal(sp.E * sp.nloc)
        mine = np.zeros(sp.n)
        er = sl.element_range()
        el2g = sp.l2g.reshape(sp.E, sp.nloc)
        for e in er:  # ascending element id (the reference gather order restricted to the slab)
            np.add.at(mine, el2g[e], loc[e * sp.nloc:(e + 1) * sp.nloc])
        P = sl.plane
        zb, zt = sl.ez0 * p, sl.ez1 * p
        recv_lo = torch.zeros(P, dtype=torch.float64)
        recv_hi = torch.zeros(P, dtype=torch.float64)
        reqs = []
        if sl.below:
            reqs.append(dist.isend(torch.from_numpy(mine[zb * P:(zb + 1) * P].copy()), rank - 1))
            reqs.append(dist.irecv(recv_lo, rank - 1))
        if sl.above:
            reqs.append(dist.isend(torch.from_numpy(mine[zt * P:(zt + 1) * P].copy()), rank + 1))
            reqs.append(dist.irecv(recv_hi, rank + 1))
        for r in reqs:
            r.wait()
        if sl.below:
            mine[zb * P:(zb + 1) * P] = recv_lo.numpy() + mine[zb * P:(zb + 1) * P]
        if sl.above:
            mine[zt * P:(zt + 1) * P] = mine[zt * P:(zt + 1) * P] + recv_hi.numpy()
        ref = sp.gather(loc)
        a, b = zb * P, (zt + 1) * P
        ok_gather = np.abs(mine[a:b] - ref[a:b]).max() <= 1e-13 * np.abs(ref).max()
        # local vector geometry
        ok_sizes = sl.n_local == sl.plane * sl.nzl and sl.zlo == zb - (1 if sl.below else 0)
        q.put((rank, bool(ok_dot), bool(ok_gather), bool(ok_sizes)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_protocols_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(pr.exitcode == 0 for pr in procs)
    for rank, ok_dot, ok_gather, ok_sizes in res:
        assert ok_dot and ok_gather and ok_sizes, (rank, ok_dot, ok_gather, ok_sizes)


def test_partition_covers_every_plane_once():
    for world in (1, 2, 3, 4, 8):
        sls = [Slab(7, 32, 32, 32, r, world) for r in range(world)]
        owned = [z for s in sls for z in range(s.own_z0, s.own_z1)]
        assert owned == list(range(sls[0].Nz))
        for s in sls:
            assert s.ez1 > s.ez0
