"""Benchmark of the SE pressure-Poisson solve (BASELINE.json metric) — one JSON line on rank 0.

Workload (configs[3], the config the 1/2/4/8-GPU metric is quoted on): Kershaw-deformed box
eps=0.3, E=32^3, p=7, GMRES(20) to 1e-8 preconditioned by a Chebyshev(2)-RAS p-multigrid V-cycle
(7,3,1) with FP32 FDM smoother, FP64 Krylov and one AMG V-cycle as the p=1 coarse solve.
A step = one full solve from x0 = 0 (time-to-1e-8). value = n * iterations / t (GDOF*iter/s).

  python bench.py [--gpus N --steps K --warmup W]        # our sm_100a path (torchrun for N>1)
  python bench.py --impl reference ...                    # the reference's CPU path on host cores
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Poisson solve GDOF*iter/s (time-to-1e-8)"
UNIT = "GDOF*iter/s"
CONFIGS = {
    "c4": dict(eps=0.3, E=32, p=7, orders=(7, 3, 1), smoother="ras", eta=2, precision=32, coarse="amg",
               krylov="gmres"),
    "c1": dict(eps=1.0, E=8, p=7, orders=(7,), smoother="jacobi", eta=0, precision=64, coarse="direct",
               krylov="pcg"),
    "c2": dict(eps=1.0, E=16, p=7, orders=(7, 3, 1), smoother="jacobi", eta=2, precision=64, coarse="direct",
               krylov="pcg"),
    "c3": dict(eps=1.0, E=16, p=7, orders=(7, 3, 1), smoother="ras", eta=2, precision=32, coarse="direct",
               krylov="gmres"),
    "c5": dict(eps=0.3, E=96, p=7, orders=(7, 3, 1), smoother="ras", eta=2, precision=32, coarse="amg",
               krylov="gmres"),
}


def describe(name, c):
    return (f"{name}: Kershaw eps={c['eps']} E={c['E']}^3 p={c['p']}, {c['krylov'].upper()}"
            f"{'(20)' if c['krylov'] == 'gmres' else ''} tol 1e-8, Cheby({c['eta']})-{c['smoother'].upper()} "
            f"pMG{c['orders']} FP{c['precision']} smoother, coarse {c['coarse']}")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6 for i in range(4) if r[2 + i] == "Active"})
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------------------------- CPU baselines
def host_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


REF_BENCH = os.path.join(ROOT, "oracle", "_ref", "semlab_ref_bench")
# The reference costs ~35 s per Arnoldi iteration at E=32^3 on one core (plus ~135 s of setup): its
# K steps are sampled by the first min(K, 6) iterations so the arm ends within minutes.
REF_MAX_ITERS = 6


def ref_bench_cmd(cfg, iters, warm):
    return [REF_BENCH, "--eps", str(cfg["eps"]), "--elems", str(cfg["E"]), "--order", str(cfg["p"]),
            "--smoother", cfg["smoother"], "--coarse", cfg["coarse"], "--cheb-order", str(cfg["eta"]),
            "--krylov", cfg["krylov"], "--iters", str(iters), "--warmup-iters", str(warm),
            "--pmg", "1" if len(cfg["orders"]) > 1 else "0"]


def ref_sample_desc(cfg, r, warm):
    return (f"reference semlab (own TUs, Eigen-API shim, g++ -O3 as the reference's Release build) + restated pMG/PCG/RHS on the "
            f"bench workload itself (eps={cfg['eps']} E={cfg['E']}^3 p={cfg['p']}, {cfg['krylov']}, FP64 smoother: "
            f"the reference has no FP32 path): setup {r['t_setup_s']:.0f}s, then the first {r['iters']} Arnoldi "
            f"iterations of the solve from x0=0 timed ({r['t_solve_s']:.1f}s, less {r.get('t_close_s', 0):.1f}s for "
            f"the cycle close M+A timed apart), 1 thread")


def start_cpu_reference(cfg, iters, warm):
    """The reference on the bench config as a child process pinned to the last host core (it runs
    beside the GPU measurement; single-threaded like the reference)."""
    if not os.path.exists(REF_BENCH):
        return None
    last = max(os.sched_getaffinity(0))

    def pin():
        try:
            os.sched_setaffinity(0, {last})
        except Exception:
            pass
    return subprocess.Popen(ref_bench_cmd(cfg, iters, warm), stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                            text=True, preexec_fn=pin)


def finish_cpu_reference(proc, cfg, warm, timeout=1800):
    if proc is None:
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref/semlab_ref_bench not built", **host_info()}
    out, err = proc.communicate(timeout=timeout)
    if proc.returncode != 0:
        raise RuntimeError(f"semlab_ref_bench failed: {err[-300:]}")
    r = json.loads(out.strip().splitlines()[-1])
    return {"value": r["gdof_iter_per_s"], "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": ref_sample_desc(cfg, r, warm), "ms_per_iteration": (r["t_solve_s"] - r.get("t_close_s", 0.0)) / max(1, r["iters"]) * 1e3,
            "setup_s": r["t_setup_s"], **host_info()}


def run_reference(args, cfg, name):
    """--impl reference: the reference's CPU path (oracle/_ref) on the bench workload itself. A step
    is one Krylov iteration of the bench's solve (A, the V-cycle, CGS2): the first min(K, 6)
    iterations of one solve from x0 = 0 are timed (the cycle close, one M + A, is timed apart and
    taken out). No warm-up iteration: on the CPU every iteration runs the same code and the Krylov
    buffers are allocated per solve anyway; one iteration of this single-threaded reference costs
    ~35 s at E=32^3."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    warm = 0
    proc = start_cpu_reference(cfg, min(args.steps, REF_MAX_ITERS), warm)
    if proc is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/semlab_ref_bench not built"}), flush=True)
        return
    cb = finish_cpu_reference(proc, cfg, warm, timeout=3600)
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_iteration"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": describe(name, cfg), "parallelism": "cpu, 1 thread (the reference is serial)",
                       "step": "one Krylov iteration of the bench solve (the first min(K, 6) from x0=0 timed)",
                       "warmup_iterations": warm, "setup_s": cb["setup_s"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "nproc", "cpu_model")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- byte model
def kernel_bytes(cfg, n, E, n3=None, E3=None):
    """Algorithmic HBM bytes per launch; n, E on the finest level."""
    nloc = (cfg["p"] + 1) ** 3
    P = cfg["p"] + 3
    F = 4 * E * (3 * P * P + 3 * P)  # FP32 FDM factors S (3 P^2) and lambda (3 P) per element
    return {
        "ax64": 48 * E * nloc + 16 * n,          # FP64 factors, u in, w out (Krylov operator)
        "ax32": 24 * E * nloc + 16 * n,          # FP32-rounded factors (smoother operator)
        "ras0": F + 16 * n,                      # plain RAS: r in, z out
        "ras1": F + 24 * n,                      # Chebyshev init: t in; r, d out
        "ras2": F + 56 * n,                      # Chebyshev step: t, d, r, x in; x, r, d out
        "ras3": F + 40 * n,                      # last step: t, d, r, x in; x out
        "F": F,
    }


def solve_bytes(cfg, n, E, n1, E1, iters, restart=20):
    """Algorithmic bytes of one bench solve (model, documented in DESIGN.md §6): per iteration the
    Krylov A, the V-cycle (level 0: 6 Ax with FP32 factors + 2x(init, step, last) fused RAS; the
    p=3 level likewise with FP64 factors; transfers; the small coarse solve omitted) and CGS2."""
    kb = kernel_bytes(cfg, n, E)
    P1 = 3 + 3
    F1 = 4 * E1 * (3 * P1 * P1 + 3 * P1)
    lvl0 = 6 * kb["ax32"] + 16 * n + 2 * (kb["ras1"] + kb["ras2"] + kb["ras3"])
    lvl1 = 6 * (48 * E1 * 64 + 16 * n1) + 16 * n1 + 2 * (3 * F1 + 120 * n1)
    transfers = 32 * n + 16 * n1
    vcyc = lvl0 + lvl1 + transfers
    total = 0
    for it in range(iters):
        j = it % restart
        total += kb["ax64"] + vcyc + 8 * n * (3 * j + 8) + 16 * n + 8 * n  # A, M, CGS2, normalise, store z
        if j == restart - 1 or it == iters - 1:
            total += 8 * n * (j + 3) + kb["ax64"] + 24 * n + 8 * n  # x += Z y, true residual, norm
    return total, vcyc


# ---------------------------------------------------------------------------------- our path
def run_ours(args, cfg, name):
    import torch
    import torch.distributed as dist
    from paper_2110_07663_b200 import semlab as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream(local)
    torch.cuda.set_stream(stream)
    if world > 1:
        # torch.distributed is plumbing only (NCCL id broadcast, barriers, max-over-ranks of the
        # event timings): gloo on the host. The data path (interface sums, halos, Krylov
        # allreduces) is the library's own NCCL communicator over NVLink; a second NCCL
        # communicator from torch would only compete with it.
        dist.init_process_group("gloo")
        uid = [S.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = S.Context(local, stream, rank, world, uid[0])
        ctx.set_exchange(args.exchange == "peer")
    else:
        ctx = S.Context(local, stream)

    # the reference on this same workload runs beside the GPU measurement (rank 0, N=1 only)
    cpu_proc = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_est = (cfg["E"] * cfg["p"] + 1) ** 3  # ~1 s of reference iterations at c1-c3, one at c4
        cpu_proc = start_cpu_reference(cfg, args.cpu_iters or max(1, min(100, int(2e7 / n_est))), 0)
    sm = {"ras": S.RAS_SMOOTHER, "jacobi": S.JACOBI_SMOOTHER, "asm": S.ASM_SMOOTHER}[cfg["smoother"]]
    cm = S.COARSE_AMG if cfg["coarse"] == "amg" else S.COARSE_DIRECT
    t0 = time.time()
    mesh = S.generate_kershaw(cfg["eps"], cfg["E"], ctx)
    if len(cfg["orders"]) == 1:  # c1: Jacobi-preconditioned CG, no multigrid
        pmg = None
        sp = S.SemSpace(mesh, cfg["p"])
        A, M = sp.as_linop(), sp.jacobi()
    else:
        pmg = S.Pmg(mesh, cfg["orders"], sm, cfg["eta"], 0.1, 1.1, cfg["precision"], cm)
        sp = pmg.spaces[0]
        A, M = sp.as_linop(), pmg.as_linop()
    solve = S.gmres_solve if cfg["krylov"] == "gmres" else S.pcg_solve
    gcfg = S.GmresConfig(restart=20, tol=1e-8, max_iters=500)
    b = sp.build_rhs(1)
    x = torch.zeros_like(b)
    setup_s = time.time() - t0
    n_global = sp.n_global

    def step():
        x.zero_()
        return solve(A, M, b, x, gcfg)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()
    barrier()
    launches0 = ctx.launch_count
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    conv = True
    rel = 0.0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        step_ms = []
        torch.cuda.nvtx.range_push("timed")  # lets `ncu --nvtx --nvtx-include timed/` list exactly these launches
        for _ in range(args.steps):
            ts = time.perf_counter()
            st = step()
            step_ms.append((time.perf_counter() - ts) * 1e3)
            iters += st.iterations
            conv = conv and st.converged
            rel = max(rel, st.rel_residual)
        torch.cuda.nvtx.range_pop()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = ctx.launch_count - launches0
    t = ev0.elapsed_time(ev1) * 1e-3
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = tt.item()
    value = n_global * iters / t / 1e9

    # end to end through the public API with HOST buffers (pinned): H2D of b, solve, D2H of x
    hb = b.cpu().pin_memory()
    hx = torch.empty_like(hb).pin_memory()
    xb = torch.empty_like(b)
    e2e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    barrier()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it2 = 0
    ev2.record(stream)
    for _ in range(e2e_steps):
        xb.copy_(hb, non_blocking=True)
        x.zero_()
        st = solve(A, M, xb, x, gcfg)
        it2 += st.iterations
        hx.copy_(x, non_blocking=True)
    ev3.record(stream)
    torch.cuda.synchronize()
    t2 = ev2.elapsed_time(ev3) * 1e-3
    if world > 1:
        tt = torch.tensor([t2], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t2 = tt.item()
    e2e = {"value": n_global * it2 / t2 / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * sp.n,
           "d2h_bytes_per_step": 8 * sp.n, "steps": e2e_steps}

    # ---- rooflines of the kernels that run in the solve, each timed live on the solve's stream
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in pk else "fallback (B200_PROFILING.md)"
    traffic_tab = {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "latest_ncu_summary.json")))
        if prof.get("workload") == name and world == 1:  # ncu --set full of this workload on one GPU
            traffic_tab = prof.get("dram_bytes_per_launch", {})
    except Exception:
        pass

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e4.record(stream)
        for _ in range(reps):
            fn()
        e5.record(stream)
        torch.cuda.synchronize()
        return e4.elapsed_time(e5) * 1e-3 / reps

    E_loc = sp.n_elements
    kb = kernel_bytes(cfg, sp.n, E_loc)
    u = torch.randn(sp.n, dtype=torch.float64, device="cuda")
    sp.mask_inplace(u)
    w = torch.empty_like(u)
    roofs = {}

    def guarded(fn):
        """A roofline probe that does not fit next to the solve (E = 96^3 on one GPU) is skipped."""
        try:
            fn()
        except (RuntimeError, MemoryError) as ex:
            skipped.append(f"{getattr(fn, '__name__', 'probe')}: {str(ex)[:120]}")
            torch.cuda.empty_cache()

    skipped = []

    def add(key, kernel, nbytes, t, launches=1, per_solve=None):
        ach = nbytes / t / 1e9
        roofs[key] = {"kernel": kernel, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                      "frac": ach / peak, "traffic": traffic_tab.get(key), "algorithmic_bytes_per_launch": nbytes,
                      "us_per_launch": t * 1e6 / launches, "launches": launches, "peak_source": peak_src}
        if per_solve is not None:  # share of the timed solve (launches per solve x time per launch)
            roofs[key]["per_solve"] = per_solve
            roofs[key]["share_of_solve"] = per_solve * t / launches / (t_solve_s)

    t_solve_s = t / args.steps
    its = iters / args.steps
    restarts = int(-(-its // 20))
    if world == 1:
        add("ax64", "k_axw<EWrite,double>: Krylov Ax, FP64 factors on DMMA, owner-ordered Q^T", kb["ax64"],
            timed(lambda: sp.apply_A(u, w)), per_solve=its + restarts + 1)
        if cfg["p"] == 7 and cfg["precision"] == 32:
            add("ax32", "k_axw<.,float>: smoother Ax, FP32-rounded factors, FP64 DMMA", kb["ax32"],
                timed(lambda: sp.apply_A_geom32(u, w)), per_solve=6 * its)
        def ras_probes():
            sch = S.SchwarzSmoother(sp, S.RAS, cfg["precision"])
            add("ras0", "k_rasw mode 0: RAS, FP32 FDM local solves, owner write", kb["ras0"],
                timed(lambda: sch.apply(u, w)), per_solve=6 * its)
            # the fused Chebyshev(eta)-RAS smoothing exactly as the V-cycle runs it on the fine level
            A32 = sp.as_linop_geom32() if (cfg["p"] == 7 and cfg["precision"] == 32) else sp.as_linop()
            cheb = S.ChebyshevSmoother(sch.as_linop(), A32, S.ChebyParams(cfg["eta"], 0.1, 1.1, pmg.lam(0)))
            xs = torch.zeros_like(u)
            bb = b.clone()

            def smooth():
                xs.copy_(u)
                cheb.smooth(bb, xs)
            ax_epi = kb["ax32"] if (cfg["p"] == 7 and cfg["precision"] == 32) else kb["ax64"]
            cheb_bytes = (cfg["eta"] + 1) * ax_epi + 8 * sp.n + kb["ras1"] + (cfg["eta"] - 1) * kb["ras2"] + kb["ras3"] \
                + 16 * sp.n  # + the x copy of this harness
            add("cheby_ras", f"Chebyshev({cfg['eta']})-RAS smoothing step, fine level: {cfg['eta'] + 1} Ax + "
                f"{cfg['eta'] + 1} fused RAS launches (init, step, last)", cheb_bytes, timed(smooth),
                launches=2 * (cfg["eta"] + 1) + 1, per_solve=2 * its * (2 * (cfg["eta"] + 1) + 1))
            del cheb, sch, xs

        if cfg["smoother"] == "ras":
            guarded(ras_probes)
        n1 = (cfg["E"] * 3 + 1) ** 3
        tot, vcyc = solve_bytes(cfg, sp.n, E_loc, n1, E_loc, int(round(its)))
        if pmg is not None and cfg["smoother"] == "ras" and cfg["orders"][1:2] == (3,):
            def vcycle_probe():
                vt = timed(lambda: pmg.vcycle(b, w), reps=10)
                add("vcycle", "one pMG V-cycle (all levels, CUDA graph)", vcyc, vt, per_solve=its)
            guarded(vcycle_probe)
    if world == 1 and pmg is not None and cfg["smoother"] == "ras" and cfg["orders"][1:2] == (3,):
        solver_roof = {"algorithmic_bytes_per_solve": tot, "t_solve_ms": t_solve_s * 1e3,
                       "achieved": tot / t_solve_s / 1e9, "peak": peak, "unit": "GB/s",
                       "frac": tot / t_solve_s / 1e9 / peak,
                       "model": "per iteration: Krylov Ax + V-cycle (6 fine Ax + 2x(init,step,last) fused RAS; p=3 "
                                "level likewise; transfers) + CGS2 8n(3j+8) + normalise; per restart: x += Z y, "
                                "true residual (DESIGN.md section 6)"}
    else:
        solver_roof = None
    # the dominant KERNEL: the single kernel with the largest share of the timed solve
    dominant = max((roofs[k] for k in ("ax64", "ax32", "ras0") if k in roofs),
                   key=lambda r: r["share_of_solve"], default=None)

    cpu = None
    if cpu_proc is not None:
        try:
            cpu = finish_cpu_reference(cpu_proc, cfg, 0)
            cpu.pop("ms_per_iteration", None)
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {ex}"}

    # like-for-like line: the same solve with the FP64 smoother (the reference's arithmetic)
    fp64 = None
    if cfg["precision"] == 32 and not args.no_fp64_line:
        del A, M, pmg, sp
        torch.cuda.empty_cache()
        pmg64 = S.Pmg(mesh, cfg["orders"], sm, cfg["eta"], 0.1, 1.1, 64, cm)
        sp64 = pmg64.spaces[0]
        A64, M64 = sp64.as_linop(), pmg64.as_linop()
        b64 = sp64.build_rhs(1)
        x64 = torch.zeros_like(b64)
        for _ in range(2):
            x64.zero_()
            solve(A64, M64, b64, x64, gcfg)
        k64 = max(1, min(args.steps, 5))
        torch.cuda.synchronize()
        barrier()
        e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it64 = 0
        e6.record(stream)
        for _ in range(k64):
            x64.zero_()
            st64 = solve(A64, M64, b64, x64, gcfg)
            it64 += st64.iterations
        e7.record(stream)
        torch.cuda.synchronize()
        t64 = e6.elapsed_time(e7) * 1e-3
        if world > 1:
            tt = torch.tensor([t64], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t64 = tt.item()
        fp64 = {"value": n_global * it64 / t64 / 1e9, "unit": UNIT, "ms_per_step": t64 / k64 * 1e3, "steps": k64,
                "iterations_per_solve": it64 / k64, "converged": bool(st64.converged),
                "smoother_precision": "fp64", "note": "same workload with the FP64 FDM smoother and FP64 smoother "
                                                      "operator: the reference's arithmetic (like-for-like line)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": describe(name, cfg), "n_dofs": n_global, "elements": cfg["E"] ** 3,
                           "order": cfg["p"], "iterations_per_solve": iters / args.steps, "converged": conv,
                           "max_rel_residual": rel, "smoother_precision": f"fp{cfg['precision']}",
                           "krylov_precision": "fp64", "parallelism": f"z-slab x{world}" + (f", {args.exchange} exchanges" if world > 1 else ""), "setup_s": setup_s,
                           "l2": "inputs larger than L2 (geometry 805 MB at E=32^3)",
                           "time_to_1e-8_ms": t / args.steps * 1e3, "step_wall_ms": [round(v, 1) for v in step_ms]},
                "e2e": e2e, "roofline": dominant, "rooflines": roofs, "rooflines_skipped": skipped or None,
                "solver_roofline": solver_roof,
                "fp64_smoother": fp64, "cpu_baseline": cpu, "clocks": clk.summary(),
                "gpu_launches": launches}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=0,
                    help="iterations of the reference timed for cpu_baseline after its setup (0: sized to the mesh)")
    ap.add_argument("--no-fp64-line", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["nccl", "peer"],
                    help="z-slab plane exchanges: NVLink peer-memory mail slots (default; falls back to "
                         "NCCL when a rank cannot map its neighbours) or NCCL send/recv")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("timing rules: --warmup must be >= 3")
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, args.config)
    else:
        run_ours(args, cfg, args.config)


if __name__ == "__main__":
    main()
