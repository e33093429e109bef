"""Distributed (z-slab, NCCL) parity worker: launched by tests/test_dist_gpu.py through torchrun.

Every rank owns a slab of elements; results are gathered on the owned planes and compared with
the CPU oracle on the whole mesh. Prints one JSON line of errors / iteration counts on rank 0.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import semlab_np as o  # noqa: E402
from paper_2110_07663_b200 import semlab as S  # noqa: E402
from paper_2110_07663_b200.partition import Slab  # noqa: E402


def _allg(x, world):
    parts = [None] * world
    dist.all_gather_object(parts, x)
    return parts


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    uid = [S.Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx = S.Context(local, torch.cuda.current_stream(local), rank, world, uid[0])
    eps, E, p = float(os.environ.get("DIST_EPS", "0.3")), int(os.environ.get("DIST_E", "4")), 7
    sl = Slab(p, E, E, E, rank, world)

    def gather(vec):
        """owned planes of every rank -> full global vector (numpy) on every rank"""
        v = vec.detach().cpu().numpy() if isinstance(vec, torch.Tensor) else vec
        parts = [None] * world
        dist.all_gather_object(parts, v[sl.owned_slice_local()])
        return np.concatenate(parts)

    def rel(a, b):
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

    out = {"world": world}
    ctx.set_exchange(os.environ.get("DIST_EXCHANGE", "peer") == "peer")
    mesh = S.generate_kershaw(eps, E, ctx)
    sp = S.SemSpace(mesh, p)
    c = o.SemSpace(o.generate_kershaw(eps, E), p)
    assert sp.n == sl.n_local, (sp.n, sl.n_local)
    u = np.random.default_rng(0).standard_normal(c.n)
    w = sp.apply_A(u[sl.local_slice()])
    out["ax"] = rel(gather(w), c.apply_A(u))
    # duplicated interface planes must agree with the global result too
    wl = w.cpu().numpy()
    ref = c.apply_A(u)
    a = (sl.ez0 * p - sl.zlo) * sl.plane
    b = (sl.ez1 * p - sl.zlo + 1) * sl.plane
    out["ax_all_planes"] = rel(wl[a:b], ref[sl.ez0 * p * sl.plane:(sl.ez1 * p + 1) * sl.plane])
    out["dot"] = abs(sp.dot(sp.to_device(u[sl.local_slice()]), w) - float(u @ ref)) / abs(float(u @ ref))
    out["mass"] = rel(gather(sp.mass_diag()), c.mass_diag)
    out["diag"] = rel(gather(sp.stiffness_diag()), c.stiffness_diag())

    sch = S.SchwarzSmoother(sp, S.RAS, 64)
    so = o.SchwarzSmoother(c, o.RAS, 64)
    r = c.mask_inplace(np.random.default_rng(1).standard_normal(c.n))
    out["ras64"] = rel(gather(sch.apply(r[sl.local_slice()])), so.apply(r))

    out["asm64"] = rel(gather(S.SchwarzSmoother(sp, S.ASM, 64).apply(r[sl.local_slice()])),
                       o.SchwarzSmoother(c, o.ASM, 64).apply(r))
    out["ras32"] = rel(gather(S.SchwarzSmoother(sp, S.RAS, 32).apply(r[sl.local_slice()])),
                       o.SchwarzSmoother(c, o.RAS, 32).apply(r))
    # Neumann mode over z-slabs: global mean removal (sem_space.cpp:207), unmasked diagonal,
    # RAS/ASM with Neumann faces (schwarz.cpp:151-160)
    spn = S.SemSpace(mesh, p, S.NEUMANN)
    cn = o.SemSpace(o.generate_kershaw(eps, E), p, o.NEUMANN)
    out["ax_neumann"] = rel(gather(spn.apply_A(u[sl.local_slice()])), cn.apply_A(u))
    out["diag_neumann"] = rel(gather(spn.stiffness_diag()), cn.stiffness_diag())
    rn = np.random.default_rng(2).standard_normal(c.n)
    out["ras64_neumann"] = rel(gather(S.SchwarzSmoother(spn, S.RAS, 64).apply(rn[sl.local_slice()])),
                               o.SchwarzSmoother(cn, o.RAS, 64).apply(rn))
    out["asm64_neumann"] = rel(gather(S.SchwarzSmoother(spn, S.ASM, 64).apply(rn[sl.local_slice()])),
                               o.SchwarzSmoother(cn, o.ASM, 64).apply(rn))
    # ProjectionBasis (krylov.cpp:131-152) with rank-local owned-range reductions
    X = np.random.default_rng(3).standard_normal((3, c.n))
    pbg, pbo = S.ProjectionBasis(2), o.ProjectionBasis(2)
    for x in X:
        pbg.insert(sp.to_device(x[sl.local_slice()]), sp.as_linop())
        pbo.insert(x, c.apply_A)
    bb = np.random.default_rng(4).standard_normal(c.n)
    out["proj"] = rel(gather(pbg.initial_guess(sp.to_device(bb[sl.local_slice()]))), pbo.initial_guess(bb))

    pm = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 64, S.COARSE_DIRECT)
    pmo = o.Pmg(o.generate_kershaw(eps, E), (7, 3, 1), "ras", 2, 0.1, 1.1, "direct", 64)
    out["lam"] = [abs(pm.lam(l) - pmo.levels[l]["lam"]) / pmo.levels[l]["lam"] for l in range(2)]
    bo = o.build_rhs(c, 1)
    b_loc = pm.spaces[0].build_rhs(1)
    out["rhs"] = rel(gather(b_loc), bo)
    # transfers (level 0 <-> 1 and 1 <-> 2) on slabs
    for lvl in range(2):
        slf, slc = Slab(pm.orders[lvl], E, E, E, rank, world), Slab(pm.orders[lvl + 1], E, E, E, rank, world)
        T = pmo.transfers[lvl]
        uc = np.random.default_rng(5 + lvl).standard_normal(pmo.spaces[lvl + 1].n)
        vf = np.random.default_rng(7 + lvl).standard_normal(pmo.spaces[lvl].n)
        Pu = pm.prolong(lvl, pm.spaces[lvl + 1].to_device(uc[slc.local_slice()]))
        PTv = pm.restrict(lvl, pm.spaces[lvl].to_device(vf[slf.local_slice()]))
        slf_g = lambda v, s=slf: np.concatenate(_allg(v.cpu().numpy()[s.owned_slice_local()], world))
        slc_g = lambda v, s=slc: np.concatenate(_allg(v.cpu().numpy()[s.owned_slice_local()], world))
        out[f"prolong{lvl}"] = rel(slf_g(Pu), T.prolong(uc))
        out[f"restrict{lvl}"] = rel(slc_g(PTv), T.restrict(vf))
    pmj = S.Pmg(mesh, (3, 1), S.JACOBI_SMOOTHER, 2, 0.1, 1.1, 64, S.COARSE_DIRECT)
    pmjo = o.Pmg(o.generate_kershaw(eps, E), (3, 1), "jacobi", 2, 0.1, 1.1, "direct", 64)
    s3 = Slab(3, E, E, E, rank, world)
    b3 = o.build_rhs(pmjo.spaces[0], 1)
    z3 = pmj.vcycle(pmj.spaces[0].to_device(b3[s3.local_slice()]))
    out["vcycle_jac_31"] = rel(np.concatenate(_allg(z3.cpu().numpy()[s3.owned_slice_local()], world)), pmjo.vcycle(b3))
    out["vcycle"] = rel(gather(pm.vcycle(b_loc)), pmo.vcycle(bo))

    # Chebyshev-ASM hierarchy on slabs (generic Chebyshev path with the ASM exchange)
    pma = S.Pmg(mesh, (7, 3, 1), S.ASM_SMOOTHER, 2, 0.1, 1.1, 64, S.COARSE_DIRECT)
    pmao = o.Pmg(o.generate_kershaw(eps, E), (7, 3, 1), "asm", 2, 0.1, 1.1, "direct", 64)
    out["vcycle_asm"] = rel(gather(pma.vcycle(b_loc)), pmao.vcycle(bo))
    del pma

    x = torch.zeros_like(b_loc)
    st = S.gmres_solve(pm.spaces[0].as_linop(), pm.as_linop(), b_loc, x, S.GmresConfig())
    xo = np.zeros(c.n)
    sto = o.gmres_solve(c.apply_A, pmo.vcycle, bo, xo, o.GmresConfig())
    out["gmres_iters"] = [st.iterations, sto.iterations]
    out["gmres_conv"] = bool(st.converged)
    out["gmres_x"] = rel(gather(x), xo)
    # the NVLink peer-memory exchanges and NCCL send/recv give bitwise the same results
    if os.environ.get("DIST_EXCHANGE", "peer") == "peer":
        w_peer = sp.apply_A(u[sl.local_slice()])
        z_peer = pm.vcycle(b_loc).clone()
        ctx.set_exchange(False)
        w_nccl = sp.apply_A(u[sl.local_slice()])
        pm_n = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 64, S.COARSE_DIRECT)
        z_nccl = pm_n.vcycle(b_loc)
        ctx.set_exchange(True)
        out["peer_vs_nccl_bitwise"] = bool(torch.equal(w_peer, w_nccl) and torch.equal(z_peer, z_nccl))
    # the bench setting on slabs: FP32 smoother (fused slab Chebyshev-RAS, FP32-factor Ax), FP64 GMRES
    pm32 = S.Pmg(mesh, (7, 3, 1), S.RAS_SMOOTHER, 2, 0.1, 1.1, 32, S.COARSE_AMG)
    pmo_amg = o.Pmg(o.generate_kershaw(eps, E), (7, 3, 1), "ras", 2, 0.1, 1.1, "amg", 64)
    x32 = torch.zeros_like(b_loc)
    st32 = S.gmres_solve(pm32.spaces[0].as_linop(), pm32.as_linop(), b_loc, x32, S.GmresConfig())
    xa = np.zeros(c.n)
    sta = o.gmres_solve(c.apply_A, pmo_amg.vcycle, bo, xa, o.GmresConfig())
    out["gmres32_iters"] = [st32.iterations, sta.iterations]
    out["gmres32_conv"] = bool(st32.converged)
    out["gmres32_x"] = rel(gather(x32), xa)
    if rank == 0:
        print("DIST_RESULT " + json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
