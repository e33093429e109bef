"""Python mirror of the reference semlab API (proj/core/include/semlab/*.hpp) over the C-ABI.

Names, argument meaning and error behaviour follow the reference: ValueError where the
reference throws std::invalid_argument, RuntimeError for std::runtime_error, non-convergence
reported in GmresStats.converged. Vectors are torch CUDA float64 tensors (device resident);
numpy arrays are accepted where a method returns a fresh vector and are copied to the device.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

DIRICHLET, NEUMANN = 0, 1          # BcMode, sem_space.hpp:12
ASM, RAS = 0, 1                    # SchwarzMode, schwarz.hpp:10
JACOBI_SMOOTHER, RAS_SMOOTHER, ASM_SMOOTHER, RAS_PLAIN_SMOOTHER, ASM_PLAIN_SMOOTHER = 0, 1, 2, 3, 4
STANDARD_CYCLE, ADDITIVE_CYCLE = 0, 1
COARSE_DIRECT, COARSE_AMG = 0, 1


def _ptr(t: torch.Tensor) -> int:
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous float64 CUDA tensor")
    return t.data_ptr()


def _own(obj, handle, destroy, *parents):
    """Record obj's native handle in a box its parents also list. A cycle of garbage is finalised
    in arbitrary order, so releasing a parent first releases every child box still live: handles
    are always destroyed child-before-parent (objects.hpp: smoother -> space -> mesh -> context).
    The box also holds a weak reference to obj: when a parent's release destroys the handle, obj's
    .handle is cleared, so a later call raises (NULL handle -> ValueError) instead of touching
    freed device memory."""
    box = [handle, destroy, [], weakref.ref(obj)]
    obj._box = box
    for par in parents:
        pb = getattr(par, "_box", None)
        if pb is not None:
            pb[2][:] = [c for c in pb[2] if c[0]]
            pb[2].append(box)


def _release(obj):
    box = getattr(obj, "_box", None)
    try:
        if box is not None and box[0]:
            for child in box[2]:
                _release_box(child)
            _release_box(box)
    except TypeError:  # interpreter shutdown: the ctypes library object is already gone
        pass
    obj.handle = None


def _release_box(box):
    if box[0]:
        for child in box[2]:
            _release_box(child)
        h, box[0] = box[0], None
        box[1](h)
        obj = box[3]() if len(box) > 3 else None
        if obj is not None:
            obj.handle = None


class Context:
    """Device + stream (+ NCCL communicator). One per process and GPU."""

    def __init__(self, device: int | None = None, stream=None, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None):
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = device
        torch.cuda.set_device(device)
        self.torch_device = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        h = C.c_void_p()
        if nranks == 1:
            check(lib.semlab_ctx_create(device, C.c_void_p(stream.cuda_stream), C.byref(h)))
        else:
            buf = C.create_string_buffer(nccl_id, 128)
            check(lib.semlab_ctx_create_dist(device, C.c_void_p(stream.cuda_stream), rank, nranks, buf, C.byref(h)))
        self.handle = h
        _own(self, h, lib.semlab_ctx_destroy)
        self.rank, self.nranks = rank, nranks

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.semlab_nccl_get_unique_id(buf))
        return buf.raw

    def synchronize(self):
        check(lib.semlab_ctx_synchronize(self.handle))

    def set_exchange(self, peer: bool) -> None:
        """z-slab exchanges over NVLink peer memory (True, when every rank can) or NCCL (default)."""
        check(lib.semlab_ctx_set_exchange(self.handle, 1 if peer else 0))

    @property
    def launch_count(self) -> int:
        return int(lib.semlab_ctx_launch_count(self.handle))

    def __del__(self):
        _release(self)


_DEFAULT: Context | None = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context()
    return _DEFAULT


class HexMesh:
    """HexMesh / generate_kershaw, mesh.hpp:44-108."""

    def __init__(self, handle, ctx: Context, dims, keep=None):
        self.handle, self.ctx, self.dims, self._keep = handle, ctx, tuple(dims), keep
        _own(self, handle, lib.semlab_mesh_destroy, ctx)

    @classmethod
    def kershaw(cls, eps: float, elements_per_axis: int, ctx: Context | None = None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib.semlab_mesh_kershaw(ctx.handle, float(eps), int(elements_per_axis), C.byref(h)))
        return cls(h, ctx, (elements_per_axis,) * 3)

    @classmethod
    def box(cls, dims, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0), ctx: Context | None = None):
        ctx = ctx or default_context()
        h = C.c_void_p()
        d = (C.c_int * 3)(*dims)
        check(lib.semlab_mesh_box(ctx.handle, d, (C.c_double * 3)(*lo), (C.c_double * 3)(*hi), C.byref(h)))
        return cls(h, ctx, dims)

    @classmethod
    def from_map(cls, dims, fn, ctx: Context | None = None):
        """fn(x, y, z) -> (X, Y, Z) on the unit cube, like HexMesh::from_map (mesh.cpp:91-93)."""
        ctx = ctx or default_context()

        def tramp(_user, x, y, z, out):
            X, Y, Z = fn(x, y, z)
            out[0], out[1], out[2] = X, Y, Z

        cb = _lib.MAP_FN(tramp)
        h = C.c_void_p()
        check(lib.semlab_mesh_from_map(ctx.handle, (C.c_int * 3)(*dims), cb, None, C.byref(h)))
        return cls(h, ctx, dims, keep=cb)

    def lattice_coords(self, order: int) -> np.ndarray:
        n = int(np.prod([d * order + 1 for d in self.dims]))
        out = np.empty(3 * n)
        check(lib.semlab_mesh_lattice_coords(self.handle, order, out.ctypes.data_as(_lib.pf64), out.size))
        return out.reshape(n, 3)

    def __del__(self):
        _release(self)


def generate_kershaw(eps: float, elements_per_axis: int, ctx: Context | None = None) -> HexMesh:
    """generate_kershaw(KershawParams{eps, E}), mesh.cpp:138-171."""
    return HexMesh.kershaw(eps, elements_per_axis, ctx)


class LinOp:
    """A device operator handle (types.hpp:13 LinOp)."""

    def __init__(self, handle, n: int, ctx: Context, keep=None):
        self.handle, self.n, self.ctx, self._keep = handle, n, ctx, keep
        _own(self, handle, lib.semlab_op_destroy, ctx, keep)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(x)
        check(lib.semlab_op_apply(self.handle, _ptr(x), _ptr(out)))
        return out

    @classmethod
    def from_callable(cls, fn, n: int, ctx: Context | None = None):
        """fn(in_tensor, out_tensor) on device vectors (views of the library's buffers)."""
        ctx = ctx or default_context()

        def tramp(_user, pin, pout):
            tin = _wrap_device(pin, n, ctx)
            tout = _wrap_device(pout, n, ctx)
            fn(tin, tout)

        cb = _lib.APPLY_FN(tramp)
        h = C.c_void_p()
        check(lib.semlab_op_callback(ctx.handle, n, cb, None, C.byref(h)))
        return cls(h, n, ctx, keep=cb)

    def __del__(self):
        _release(self)


def _wrap_device(ptr: int, n: int, ctx: Context) -> torch.Tensor:
    """Zero-copy torch view of a device buffer owned by the library."""
    class _Iface:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None, "stream": None}
    return torch.as_tensor(_Iface(), device=ctx.torch_device)


class SemSpace:
    """SemSpace(mesh, order, bc), sem_space.hpp:26-129; geometry built on the device."""

    def __init__(self, mesh: HexMesh, order: int, bc: int = DIRICHLET):
        self.mesh, self.order, self.bc, self.ctx = mesh, order, bc, mesh.ctx
        h = C.c_void_p()
        check(lib.semlab_space_create(mesh.handle, int(order), int(bc), C.byref(h)))
        self.handle = h
        _own(self, h, lib.semlab_space_destroy, mesh)
        s = (C.c_int64 * 11)()
        check(lib.semlab_space_sizes(h, s))
        (self.n, self.n_free, self.n_local_total, nx, ny, nz, self.n_global, self.n_elements,
         self.zlo, self.ez0, self.ez1) = (int(v) for v in s)
        self.npts = (nx, ny, nz)
        self.nodes_per_element = (order + 1) ** 3

    # -- vectors -------------------------------------------------------------------------------
    def zeros(self, n: int | None = None) -> torch.Tensor:
        return torch.zeros(self.n if n is None else n, dtype=torch.float64, device=self.ctx.torch_device)

    def to_device(self, v) -> torch.Tensor:
        if isinstance(v, torch.Tensor):
            return v.to(device=self.ctx.torch_device, dtype=torch.float64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(self.ctx.torch_device)

    # -- operator --------------------------------------------------------------------------------
    def apply_A(self, u, out: torch.Tensor | None = None) -> torch.Tensor:
        """sem_space.cpp:195-209 (returns a fresh vector like the reference unless out is given)."""
        u = self.to_device(u)
        out = self.zeros() if out is None else out
        check(lib.semlab_space_apply_A(self.handle, _ptr(u), _ptr(out)))
        return out

    def apply_A_geom32(self, u, out: torch.Tensor | None = None) -> torch.Tensor:
        """apply_A with FP32-rounded geometric factors (the FP32 smoother's operator; order 7 and
        orders <= 5)."""
        u = self.to_device(u)
        out = self.zeros() if out is None else out
        check(lib.semlab_space_apply_A_geom32(self.handle, _ptr(u), _ptr(out)))
        return out

    def apply_local_stiffness(self, local) -> torch.Tensor:
        local = self.to_device(local)
        out = self.zeros(self.n_local_total)
        check(lib.semlab_space_apply_local_stiffness(self.handle, _ptr(local), _ptr(out)))
        return out

    def gather(self, local) -> torch.Tensor:
        local = self.to_device(local)
        out = self.zeros()
        check(lib.semlab_space_gather(self.handle, _ptr(local), _ptr(out)))
        return out

    def scatter(self, glob) -> torch.Tensor:
        glob = self.to_device(glob)
        out = self.zeros(self.n_local_total)
        check(lib.semlab_space_scatter(self.handle, _ptr(glob), _ptr(out)))
        return out

    def gather_scatter(self, local) -> torch.Tensor:
        local = self.to_device(local)
        out = self.zeros(self.n_local_total)
        check(lib.semlab_space_gather_scatter(self.handle, _ptr(local), _ptr(out)))
        return out

    def mask_inplace(self, v: torch.Tensor) -> torch.Tensor:
        check(lib.semlab_space_mask(self.handle, _ptr(v)))
        return v

    def stiffness_diag(self) -> torch.Tensor:
        out = self.zeros()
        check(lib.semlab_space_stiffness_diag(self.handle, _ptr(out)))
        return out

    def mass_diag(self) -> torch.Tensor:
        out = self.zeros()
        check(lib.semlab_space_mass_diag(self.handle, _ptr(out)))
        return out

    def metric_at(self, e: int) -> np.ndarray:
        """(nloc, 6) geometric factors of element e (rr,rs,rt,ss,st,tt), sem_space.hpp:93-98."""
        out = np.empty(self.nodes_per_element * 6)
        check(lib.semlab_space_metric(self.handle, int(e), out.ctypes.data_as(_lib.pf64)))
        return out.reshape(-1, 6)

    def build_rhs(self, seed: int = 1) -> torch.Tensor:
        out = self.zeros()
        check(lib.semlab_space_build_rhs(self.handle, int(seed), _ptr(out)))
        return out

    def dot(self, a: torch.Tensor, b: torch.Tensor) -> float:
        r = C.c_double()
        check(lib.semlab_space_dot(self.handle, _ptr(a), _ptr(b), C.byref(r)))
        return r.value

    def as_linop(self) -> LinOp:
        h = C.c_void_p()
        check(lib.semlab_op_A(self.handle, C.byref(h)))
        return LinOp(h, self.n, self.ctx, keep=self)

    def as_linop_geom32(self) -> LinOp:
        """apply_A_geom32 as an operator: the FP32 smoother's A (order 7 and orders <= 5)."""
        h = C.c_void_p()
        check(lib.semlab_op_A_geom32(self.handle, C.byref(h)))
        return LinOp(h, self.n, self.ctx, keep=self)

    def jacobi(self) -> LinOp:
        """S = diag(A)^-1 (precond.cpp missing in the reference)."""
        h = C.c_void_p()
        check(lib.semlab_op_jacobi(self.handle, C.byref(h)))
        return LinOp(h, self.n, self.ctx, keep=self)

    def __del__(self):
        _release(self)


class SchwarzSmoother:
    """SchwarzSmoother(space, mode), schwarz.hpp:31-86. precision: 32 (paper) or 64."""

    def __init__(self, space: SemSpace, mode: int = RAS, precision: int = 32):
        self.space, self.mode, self.precision = space, mode, precision
        h = C.c_void_p()
        check(lib.semlab_schwarz_create(space.handle, int(mode), int(precision), C.byref(h)))
        self.handle = h
        _own(self, h, lib.semlab_schwarz_destroy, space)
        self.box = space.order + 3

    def apply(self, r, out: torch.Tensor | None = None) -> torch.Tensor:
        r = self.space.to_device(r)
        out = self.space.zeros() if out is None else out
        check(lib.semlab_schwarz_apply(self.handle, _ptr(r), _ptr(out)))
        return out

    def fdm_solve_all(self, boxes: torch.Tensor) -> torch.Tensor:
        boxes = self.space.to_device(boxes)
        out = torch.empty_like(boxes)
        check(lib.semlab_schwarz_fdm_solve_all(self.handle, _ptr(boxes), _ptr(out)))
        return out

    def element_info(self, e: int):
        L = (C.c_double * 3)()
        n = (C.c_int * 3)()
        lam = np.zeros(3 * self.box)
        check(lib.semlab_schwarz_element_info(self.handle, int(e), L, n, lam.ctypes.data_as(_lib.pf64)))
        return np.array(L[:]), np.array(n[:]), lam.reshape(3, self.box)

    def as_linop(self) -> LinOp:
        h = C.c_void_p()
        check(lib.semlab_op_schwarz(self.handle, C.byref(h)))
        return LinOp(h, self.space.n, self.space.ctx, keep=self)

    def __del__(self):
        _release(self)


@dataclass
class LambdaEstimate:
    value: float = 0.0
    breakdown: bool = False
    rounds_used: int = 0


def estimate_lambda_max(S: LinOp, A: LinOp, n: int, rounds: int = 10, seed: int = 0) -> LambdaEstimate:
    """chebyshev.cpp:9-56."""
    out = _lib.LambdaEstimateC()
    check(lib.semlab_estimate_lambda_max(S.handle, A.handle, int(n), int(rounds), int(seed), C.byref(out)))
    return LambdaEstimate(out.value, bool(out.breakdown), out.rounds_used)


@dataclass
class ChebyParams:
    order: int = 2
    lambda_min_mult: float = 0.1
    lambda_max_mult: float = 1.1
    lambda_max_est: float = 0.0


class ChebyshevSmoother:
    """ChebyshevSmoother(S, A, params), chebyshev.hpp:36-46."""

    def __init__(self, S: LinOp, A: LinOp, params: ChebyParams):
        self.S, self.A, self.params = S, A, params
        cp = _lib.ChebyParams(params.order, params.lambda_min_mult, params.lambda_max_mult, params.lambda_max_est)
        h = C.c_void_p()
        check(lib.semlab_cheby_create(S.handle, A.handle, C.byref(cp), C.byref(h)))
        self.handle = h
        _own(self, h, lib.semlab_cheby_destroy, S, A)

    def smooth(self, b: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        check(lib.semlab_cheby_smooth(self.handle, _ptr(b), _ptr(x)))
        return x

    def __del__(self):
        _release(self)


class Pmg:
    """p-multigrid V-cycle preconditioner (RESTATED: pmg.cpp missing)."""

    def __init__(self, mesh: HexMesh, orders=(7, 3, 1), smoother: int = JACOBI_SMOOTHER, cheb_order: int = 2,
                 lmin_mult: float = 0.1, lmax_mult: float = 1.1, precision: int = 32, coarse: int = COARSE_DIRECT,
                 bc: int = DIRICHLET, cycle: int = STANDARD_CYCLE):
        """smoother: Chebyshev-{Jacobi, RAS, ASM} or plain (un-accelerated) RAS / ASM; cycle: Alg. 1
        (standard) or additive (no post-smoothing); bc=NEUMANN builds every level in Neumann mode
        and solves the coarse problem on the zero-mean subspace (direct coarse solve)."""
        self.mesh, self.orders, self.bc = mesh, tuple(orders), bc
        arr = (C.c_int * len(orders))(*orders)
        h = C.c_void_p()
        opts = _lib.PmgOptionsC(int(smoother), int(cheb_order), float(lmin_mult), float(lmax_mult), int(precision),
                                int(coarse), int(bc), int(cycle))
        check(lib.semlab_pmg_create_ex(mesh.handle, len(orders), arr, C.byref(opts), C.byref(h)))
        self.handle = h
        _own(self, h, lib.semlab_pmg_destroy, mesh)
        self.spaces = []
        for lvl in range(len(orders)):
            sh = C.c_void_p()
            check(lib.semlab_pmg_space(h, lvl, C.byref(sh)))
            self.spaces.append(_BorrowedSpace(sh, mesh, orders[lvl], self, bc))
        self.n = self.spaces[0].n

    def lam(self, level: int) -> float:
        v = C.c_double()
        check(lib.semlab_pmg_lambda(self.handle, level, C.byref(v)))
        return v.value

    def coarse_levels(self) -> list:
        """Row counts of the coarse AMG hierarchy's levels (AmgHierarchy::level_size)."""
        nl = C.c_int()
        sizes = (C.c_int64 * 64)()
        check(lib.semlab_pmg_coarse_info(self.handle, C.byref(nl), sizes, 64))
        return [int(sizes[i]) for i in range(nl.value)]

    def vcycle(self, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        out = torch.empty_like(b) if out is None else out
        check(lib.semlab_pmg_vcycle(self.handle, _ptr(b), _ptr(out)))
        return out

    def prolong(self, level: int, coarse: torch.Tensor) -> torch.Tensor:
        out = self.spaces[level].zeros()
        check(lib.semlab_pmg_prolong(self.handle, level, _ptr(coarse), _ptr(out)))
        return out

    def restrict(self, level: int, fine: torch.Tensor) -> torch.Tensor:
        out = self.spaces[level + 1].zeros()
        check(lib.semlab_pmg_restrict(self.handle, level, _ptr(fine), _ptr(out)))
        return out

    def as_linop(self) -> LinOp:
        h = C.c_void_p()
        check(lib.semlab_op_pmg(self.handle, C.byref(h)))
        return LinOp(h, self.n, self.mesh.ctx, keep=self)

    def __del__(self):
        _release(self)


class _BorrowedSpace(SemSpace):
    """A SemSpace owned by a Pmg hierarchy (destroyed with it, never from Python). It keeps its
    Pmg alive (self._owner), and objects built on it (smoothers, operators) register as children
    of the Pmg's box, so they are released before the hierarchy frees the space."""

    def __init__(self, handle, mesh, order, owner, bc=DIRICHLET):
        self.mesh, self.order, self.bc, self.ctx = mesh, order, bc, mesh.ctx
        self._owner = owner
        self._box = owner._box
        self.handle = None
        s = (C.c_int64 * 11)()
        check(lib.semlab_space_sizes(handle, s))
        (self.n, self.n_free, self.n_local_total, nx, ny, nz, self.n_global, self.n_elements,
         self.zlo, self.ez0, self.ez1) = (int(v) for v in s)
        self.npts = (nx, ny, nz)
        self.nodes_per_element = (order + 1) ** 3
        self.handle = handle

    def __del__(self):
        pass


class SemfemPreconditioner:
    """SemfemPreconditioner(space, SemfemInner::Amg), semfem.hpp:36-54: the linear-tetrahedral
    stiffness matrix on the space's GLL lattice with one AMG V-cycle as the inner solve."""

    def __init__(self, space: SemSpace):
        self.space = space
        h = C.c_void_p()
        check(lib.semlab_semfem_create(space.handle, C.byref(h)))
        self.handle = h
        _own(self, h, lib.semlab_semfem_destroy, space)

    def apply(self, r, out: torch.Tensor | None = None) -> torch.Tensor:
        r = self.space.to_device(r)
        out = self.space.zeros() if out is None else out
        check(lib.semlab_semfem_apply(self.handle, _ptr(r), _ptr(out)))
        return out

    def levels(self) -> list:
        nl = C.c_int()
        sizes = (C.c_int64 * 64)()
        check(lib.semlab_semfem_levels(self.handle, C.byref(nl), sizes, 64))
        return [int(sizes[i]) for i in range(nl.value)]

    def as_linop(self) -> LinOp:
        h = C.c_void_p()
        check(lib.semlab_op_semfem(self.handle, C.byref(h)))
        return LinOp(h, self.space.n, self.space.ctx, keep=self)

    def __del__(self):
        _release(self)


@dataclass
class GmresConfig:
    restart: int = 20
    tol: float = 1e-8
    max_iters: int = 500
    use_abs_tol: bool = False
    abs_tol: float = 0.0


@dataclass
class GmresStats:
    iterations: int = 0
    converged: bool = False
    breakdown: bool = False
    initial_residual: float = 0.0
    abs_residual: float = 0.0
    rel_residual: float = 0.0
    history: list = field(default_factory=list)


def _solve(fn, A: LinOp, M: LinOp | None, b: torch.Tensor, x: torch.Tensor, config: GmresConfig) -> GmresStats:
    cfg = _lib.GmresConfigC(config.restart, config.tol, config.max_iters, int(config.use_abs_tol), config.abs_tol)
    hist = np.zeros(max(config.max_iters, 1))
    st = _lib.GmresStatsC()
    st.history = hist.ctypes.data_as(_lib.pf64)
    st.history_capacity = hist.size
    check(fn(A.handle, M.handle if M is not None else None, _ptr(b), _ptr(x), C.byref(cfg), C.byref(st)))
    return GmresStats(st.iterations, bool(st.converged), bool(st.breakdown), st.initial_residual,
                      st.abs_residual, st.rel_residual, hist[:st.history_len].tolist())


def gmres_solve(A: LinOp, M: LinOp | None, b: torch.Tensor, x: torch.Tensor, config: GmresConfig | None = None) -> GmresStats:
    """krylov.cpp:20-129 (x updated in place)."""
    return _solve(lib.semlab_gmres_solve, A, M, b, x, config or GmresConfig())


def pcg_solve(A: LinOp, M: LinOp | None, b: torch.Tensor, x: torch.Tensor, config: GmresConfig | None = None) -> GmresStats:
    """RESTATED PCG (not in the reference)."""
    return _solve(lib.semlab_pcg_solve, A, M, b, x, config or GmresConfig())


# ---- host-only helpers --------------------------------------------------------------------------
class ProjectionBasis:
    """ProjectionBasis(capacity), krylov.hpp:39-59: A-orthonormal prior solutions on the device.
    n is the vector length of the operator's space (fixed at the first use)."""

    def __init__(self, capacity: int = 10, n: int | None = None, ctx: Context | None = None):
        self.capacity, self.n, self.ctx = int(capacity), n, ctx
        self.handle = None
        if n is not None:
            self._create(n, ctx)

    def _create(self, n: int, ctx: Context | None):
        self.ctx = ctx or self.ctx or default_context()
        self.n = int(n)
        h = C.c_void_p()
        check(lib.semlab_proj_create(self.ctx.handle, self.n, self.capacity, C.byref(h)))
        self.handle = h
        _own(self, h, lib.semlab_proj_destroy, self.ctx)

    def initial_guess(self, b: torch.Tensor) -> torch.Tensor:
        u = torch.zeros_like(b)
        if self.handle is None:
            return u
        check(lib.semlab_proj_initial_guess(self.handle, _ptr(b), _ptr(u)))
        return u

    def insert(self, x: torch.Tensor, A: LinOp) -> None:
        if A is None:
            raise ValueError("ProjectionBasis: missing operator")
        if self.handle is None:
            self._create(A.n, A.ctx)
        check(lib.semlab_proj_insert(self.handle, _ptr(x), A.handle))

    def size(self) -> int:
        if self.handle is None:
            return 0
        v = C.c_int()
        check(lib.semlab_proj_size(self.handle, C.byref(v)))
        return v.value

    def vectors(self) -> list:
        out = []
        for i in range(self.size()):
            v = torch.empty(self.n, dtype=torch.float64, device=self.ctx.torch_device)
            check(lib.semlab_proj_vector(self.handle, i, _ptr(v)))
            out.append(v)
        return out

    def clear(self) -> None:
        if self.handle is not None:
            check(lib.semlab_proj_clear(self.handle))

    def __del__(self):
        _release(self)


def debug_set_grid_cap(max_ctas: int) -> None:
    """Cap the persistent kernels' grids (0 = occupancy-sized): forces many elements per warp."""
    check(lib.semlab_debug_set_grid_cap(int(max_ctas)))


def debug_set_gmres_form(flexible: bool) -> None:
    """False: GMRES always uses the reference's x += M (V y) (as when Z does not fit in memory)."""
    check(lib.semlab_debug_set_gmres_form(1 if flexible else 0))


def host_gll(order: int):
    n = order + 1
    nodes, w, d = np.zeros(n), np.zeros(n), np.zeros(n * n)
    check(lib.semlab_host_gll(order, nodes.ctypes.data_as(_lib.pf64), w.ctypes.data_as(_lib.pf64),
                              d.ctypes.data_as(_lib.pf64)))
    return nodes, w, d.reshape(n, n, order="F")


def host_kershaw_map(eps, x, y, z):
    out = (C.c_double * 3)()
    check(lib.semlab_host_kershaw_map(eps, x, y, z, out))
    return tuple(out)


def host_uniform_pm1(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    check(lib.semlab_host_uniform_pm1(seed, n, out.ctypes.data_as(_lib.pf64)))
    return out


def host_gen_eig(A: np.ndarray, B: np.ndarray):
    n = A.shape[0]
    Af = np.asfortranarray(A, dtype=np.float64)
    Bf = np.asfortranarray(B, dtype=np.float64)
    lam = np.zeros(n)
    S = np.zeros((n, n), order="F")
    check(lib.semlab_host_gen_eig(n, Af.ctypes.data_as(_lib.pf64), Bf.ctypes.data_as(_lib.pf64),
                                  lam.ctypes.data_as(_lib.pf64), S.ctypes.data_as(_lib.pf64)))
    return lam, S


def host_max_abs_eig(H: np.ndarray) -> float:
    Hf = np.asfortranarray(H, dtype=np.float64)
    out = C.c_double()
    check(lib.semlab_host_max_abs_eig(H.shape[0], Hf.ctypes.data_as(_lib.pf64), C.byref(out)))
    return out.value
