"""CPU ORACLE — test infrastructure only, never the product.

numpy/scipy restatement of the reference semlab hot path (/root/reference/proj/core).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this
module, and only as the checker. Every function cites the reference file:line it follows
(paths relative to proj/core/src unless stated).

Pieces the reference does NOT ship (pmg.cpp, precond.cpp, bench.cpp are listed in
core/CMakeLists.txt:12-15 but absent; there is no CG anywhere) are restated from
SPEC.md / PAPER.md and marked "RESTATED (no reference code)": their parity is pinned only
by SPEC invariants (adjointness, linearity, polynomial exactness), not by reference output.

Pinning: tests/test_oracle_pin.py checks this module against golden vectors produced by
the reference's own translation units compiled against oracle/eigen_shim (oracle/_ref,
recipe oracle/Makefile, fixtures tests/golden/ with generator tests/golden/make_golden.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------- gll.cpp


def legendre(p: int, x: float):
    """P_p(x), P_p'(x) by the Bonnet recurrences — gll.cpp:12-25."""
    if p == 0:
        return 1.0, 0.0
    pm1, pn = 1.0, x
    dpm1, dpn = 0.0, 1.0
    for n in range(2, p + 1):
        pnext = ((2.0 * n - 1.0) * x * pn - (n - 1.0) * pm1) / n
        dpnext = dpm1 + (2.0 * n - 1.0) * pn
        pm1, dpm1, pn, dpn = pn, dpn, pnext, dpnext
    return pn, dpn


def barycentric_weights(nodes):
    """gll.cpp:27-34."""
    n = len(nodes)
    w = np.ones(n)
    for j in range(n):
        for k in range(n):
            if k != j:
                w[j] /= nodes[j] - nodes[k]
    return w


def lagrange_diff_matrix(nodes):
    """d(i,j) = (w_j/w_i)/(x_i-x_j), diagonal = -row sum — gll.cpp:120-134."""
    n = len(nodes)
    w = barycentric_weights(nodes)
    d = np.zeros((n, n))
    for i in range(n):
        diag = 0.0
        for j in range(n):
            if j == i:
                continue
            d[i, j] = (w[j] / w[i]) / (nodes[i] - nodes[j])
            diag -= d[i, j]
        d[i, i] = diag
    return d


def lagrange_interpolation_matrix(from_nodes, to_points):
    """out(i,j) = l_j(to_points[i]), barycentric, exact delta on node hits — gll.cpp:93-118."""
    from_nodes = np.asarray(from_nodes, dtype=np.float64)
    n, m = len(from_nodes), len(to_points)
    w = barycentric_weights(from_nodes)
    out = np.zeros((m, n))
    for i in range(m):
        x = to_points[i]
        hit = -1
        for j in range(n):
            if x == from_nodes[j]:
                hit = j
                break
        if hit >= 0:
            out[i, hit] = 1.0
            continue
        denom = 0.0
        for j in range(n):
            denom += w[j] / (x - from_nodes[j])
        for j in range(n):
            out[i, j] = (w[j] / (x - from_nodes[j])) / denom
    return out


@dataclass
class Gll1D:
    order: int
    nodes: np.ndarray
    weights: np.ndarray
    diff: np.ndarray  # diff[i, j] = h_j'(x_i)


_GLL_CACHE: dict[int, Gll1D] = {}


def gll(p: int) -> Gll1D:
    """Newton on P_p' from -cos(pi j/p), forced symmetry, symmetrised weights — gll.cpp:36-91."""
    if p < 1 or p > 16:
        raise ValueError(f"gll: order must be in [1,16], got {p}")
    if p in _GLL_CACHE:
        return _GLL_CACHE[p]
    nodes = np.zeros(p + 1)
    weights = np.zeros(p + 1)
    nodes[0], nodes[p] = -1.0, 1.0
    eps = np.finfo(np.float64).eps
    for j in range(1, p):
        x = -math.cos(math.pi * j / p)
        for _ in range(100):
            pp, dp = legendre(p, x)
            d2p = (2.0 * x * dp - p * (p + 1.0) * pp) / (1.0 - x * x)
            dx = dp / d2p
            x -= dx
            if abs(dx) < 4.0 * eps:
                break
        nodes[j] = x
    j = 1
    while j < p - j:
        t = 0.5 * (nodes[p - j] - nodes[j])
        nodes[j], nodes[p - j] = -t, t
        j += 1
    if p % 2 == 0:
        nodes[p // 2] = 0.0
    for j in range(p + 1):
        pp = legendre(p, nodes[j])[0]
        weights[j] = 2.0 / (p * (p + 1.0) * pp * pp)
    j = 0
    while j < p + 1 - j:
        t = 0.5 * (weights[j] + weights[p - j])
        weights[j] = weights[p - j] = t
        j += 1
    g = Gll1D(p, nodes, weights, lagrange_diff_matrix(nodes))
    _GLL_CACHE[p] = g
    return g


# ----------------------------------------------------------------------------- mesh.cpp


def _profile_right(eps, x):
    """mesh.cpp:18-20."""
    return np.where(x <= 0.5, (2.0 - eps) * x, 1.0 + eps * (x - 1.0))


def _profile_left(eps, x):
    """mesh.cpp:22-24."""
    return 1.0 - _profile_right(eps, 1.0 - x)


def _blend(a, b, t):
    """mesh.cpp:27-31."""
    return np.where(t <= 0.0, a, np.where(t >= 1.0, b, a + (b - a) * t * t * (3.0 - 2.0 * t)))


def _kershaw_profile(eps, x, s):
    """Six x-layers with smoothstep blends — mesh.cpp:33-48."""
    x = np.asarray(x, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    layer = np.minimum((x * 6.0).astype(np.int64), 5)
    lam = x * 6.0 - layer
    l = _profile_left(eps, s)
    r = _profile_right(eps, s)
    out = np.select(
        [layer == 0, layer == 1, layer == 2, layer == 3, layer == 4],
        [l, _blend(l, r, lam), _blend(r, l, lam / 2.0), _blend(r, l, (1.0 + lam) / 2.0), _blend(l, r, lam)],
        default=r,
    )
    return out


def kershaw_map(eps, x, y, z):
    """Unit cube -> [-1/2,1/2]^3 — mesh.cpp:52-55."""
    return (np.asarray(x, dtype=np.float64) - 0.5,
            _kershaw_profile(eps, x, y) - 0.5,
            _kershaw_profile(eps, x, z) - 0.5)


class HexMesh:
    """Structured nx*ny*nz element grid pushed through a coordinate map — mesh.hpp:44-108."""

    def __init__(self, dims, map_fn):
        if min(dims) < 1:
            raise ValueError("HexMesh: element counts must be positive")
        self.dims = tuple(int(d) for d in dims)
        self.map_fn = map_fn  # vectorised: (x, y, z) unit coordinates -> (X, Y, Z)

    @property
    def n_elements(self):
        return self.dims[0] * self.dims[1] * self.dims[2]

    def element_ijk(self):
        """element id e = i + nx (j + ny k) — mesh.hpp:58-60."""
        nx, ny, nz = self.dims
        e = np.arange(self.n_elements)
        return e % nx, (e // nx) % ny, e // (nx * ny)

    def neighbor(self, e, face):
        """Faces 0..5 = -x,+x,-y,+y,-z,+z; -1 across the boundary — mesh.cpp:95-102."""
        ijk = [int(v[e]) for v in self.element_ijk()]
        axis = face // 2
        ijk[axis] += -1 if face % 2 == 0 else 1
        if ijk[axis] < 0 or ijk[axis] >= self.dims[axis]:
            return -1
        return ijk[0] + self.dims[0] * (ijk[1] + self.dims[1] * ijk[2])

    def lattice_axes(self, order):
        """1-D unit coordinates of the global GLL lattice — mesh.cpp:104-123."""
        g = gll(order)
        axes = []
        for d in range(3):
            npts = self.dims[d] * order + 1
            gidx = np.arange(npts)
            e = gidx // order
            i = gidx % order
            last = e == self.dims[d]
            e = np.where(last, e - 1, e)
            i = np.where(last, order, i)
            axes.append((e.astype(np.float64) + 0.5 * (g.nodes[i] + 1.0)) / self.dims[d])
        return axes

    def lattice_coords(self, order):
        """(n,3) physical coordinates, x lattice index fastest — mesh.cpp:104-136."""
        ax, ay, az = self.lattice_axes(order)
        Z, Y, X = np.meshgrid(az, ay, ax, indexing="ij")
        px, py, pz = self.map_fn(X.ravel(), Y.ravel(), Z.ravel())
        return np.stack([np.broadcast_to(px, X.size), np.broadcast_to(py, X.size),
                         np.broadcast_to(pz, X.size)], axis=1).astype(np.float64)


def box_mesh(dims, lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
    """HexMesh::box — mesh.cpp:82-89."""
    def fn(x, y, z):
        return (lo[0] + (hi[0] - lo[0]) * x, lo[1] + (hi[1] - lo[1]) * y, lo[2] + (hi[2] - lo[2]) * z)
    return HexMesh(dims, fn)


def generate_kershaw(eps: float, elements_per_axis: int, p: int = 1) -> HexMesh:
    """Parameter checks of generate_kershaw — mesh.cpp:138-171 (the Jacobian validity
    check at :169 is implied by SemSpace, which throws on det <= 0, sem_space.cpp:82-84)."""
    if not (eps > 0.0) or eps > 1.0:
        raise ValueError("generate_kershaw: eps must lie in (0,1]")
    n = elements_per_axis
    if n < 2 or n % 2 != 0:
        raise ValueError("generate_kershaw: elements_per_axis must be even and >= 2")
    return HexMesh((n, n, n), lambda x, y, z: kershaw_map(eps, x, y, z))


# ----------------------------------------------------------------------------- sem_space.cpp

DIRICHLET, NEUMANN = 0, 1


def _d_r(D, u):  # sum_m D(i,m) u(m,j,k); u indexed [e,k,j,i]
    return np.einsum("im,ekjm->ekji", D, u, optimize=True)


def _d_s(D, u):
    return np.einsum("jm,ekmi->ekji", D, u, optimize=True)


def _d_t(D, u):
    return np.einsum("km,emji->ekji", D, u, optimize=True)


class SemSpace:
    """Discrete SE space at one order — sem_space.hpp:26-129, sem_space.cpp:10-102."""

    def __init__(self, mesh: HexMesh, order: int, bc: int = DIRICHLET):
        self.mesh, self.order, self.bc = mesh, order, bc
        self.basis = gll(order)
        q, nd = order, order + 1
        self.nd, self.nloc = nd, nd ** 3
        self.npts = tuple(mesh.dims[d] * q + 1 for d in range(3))
        Nx, Ny, Nz = self.npts
        self.n = Nx * Ny * Nz
        self.coords = mesh.lattice_coords(q)
        # mask: every lattice boundary point (Dirichlet) — sem_space.cpp:20-28
        ii, jj, kk = np.meshgrid(np.arange(Nx), np.arange(Ny), np.arange(Nz), indexing="ij")
        m = (ii == 0) | (ii == Nx - 1) | (jj == 0) | (jj == Ny - 1) | (kk == 0) | (kk == Nz - 1)
        self.masked = np.transpose(m, (2, 1, 0)).ravel().astype(np.uint8)
        if bc != DIRICHLET:
            self.masked[:] = 0
        self.n_free = self.n - int(self.masked.sum())
        # local-to-global (element-major, i fastest) — sem_space.cpp:31-39, hpp:44-49
        ex, ey, ez = mesh.element_ijk()
        r = np.arange(nd)
        gx = ex[:, None, None, None] * q + r[None, None, None, :]
        gy = ey[:, None, None, None] * q + r[None, None, :, None]
        gz = ez[:, None, None, None] * q + r[None, :, None, None]
        self.l2g = (gx + Nx * (gy + Ny * gz)).reshape(-1).astype(np.int64)
        self.E = mesh.n_elements
        self.multiplicity = np.bincount(self.l2g, minlength=self.n).astype(np.int64)
        # geometric factors — sem_space.cpp:58-97
        X = self.coords[self.l2g].reshape(self.E, nd, nd, nd, 3)  # [e,k,j,i,c]
        D = self.basis.diff
        J = np.empty(X.shape + (3,))
        J[..., 0] = np.einsum("im,ekjmc->ekjic", D, X, optimize=True)
        J[..., 1] = np.einsum("jm,ekmic->ekjic", D, X, optimize=True)
        J[..., 2] = np.einsum("km,emjic->ekjic", D, X, optimize=True)
        det = np.linalg.det(J)
        if np.any(det <= 0.0):
            bad = int(np.argmax((det <= 0.0).reshape(self.E, -1).any(axis=1)))
            raise RuntimeError(f"SemSpace: non-positive Jacobian in element {bad}")
        w1 = self.basis.weights
        w = (w1[None, None, :] * w1[None, :, None] * w1[:, None, None])[None]  # [k,j,i]
        Jinv = np.linalg.inv(J)
        G = (w * det)[..., None, None] * np.einsum("...ab,...cb->...ac", Jinv, Jinv)
        self.geom = np.stack([G[..., 0, 0], G[..., 0, 1], G[..., 0, 2], G[..., 1, 1],
                              G[..., 1, 2], G[..., 2, 2]], axis=-1).reshape(self.E, self.nloc, 6)
        self.massw = (w * det).reshape(self.E, self.nloc)
        self.mass_diag = self.gather(self.massw.ravel())

    # -- gather / scatter ------------------------------------------------------------------
    def gather(self, local):
        """Q^T in ascending local index per dof (bincount accumulates in input order) —
        sem_space.cpp:40-52, 110-119."""
        return np.bincount(self.l2g, weights=np.asarray(local, dtype=np.float64).ravel(),
                           minlength=self.n)

    def scatter(self, glob):
        """Q — sem_space.cpp:121-125."""
        return np.asarray(glob, dtype=np.float64)[self.l2g]

    def gather_scatter(self, local):
        """QQ^T — sem_space.hpp:86-88."""
        return self.scatter(self.gather(local))

    def mask_inplace(self, v):
        """sem_space.cpp:104-108."""
        if self.bc == DIRICHLET:
            v[self.masked.astype(bool)] = 0.0
        return v

    # -- operator ------------------------------------------------------------------------------
    def apply_local_stiffness(self, local):
        """A^e u^e for all elements: D-contractions, G, D^T-contractions — sem_space.cpp:127-175."""
        nd = self.nd
        u = np.asarray(local, dtype=np.float64).reshape(self.E, nd, nd, nd)
        D = self.basis.diff
        ur, us, ut = _d_r(D, u), _d_s(D, u), _d_t(D, u)
        g = self.geom.reshape(self.E, nd, nd, nd, 6)
        vr = g[..., 0] * ur + g[..., 1] * us + g[..., 2] * ut
        vs = g[..., 1] * ur + g[..., 3] * us + g[..., 4] * ut
        vt = g[..., 2] * ur + g[..., 4] * us + g[..., 5] * ut
        DT = D.T
        out = _d_r(DT, vr) + _d_s(DT, vs) + _d_t(DT, vt)
        return out.reshape(-1)

    def with_geom32(self):
        """A view of this space whose geometric factors are rounded to FP32 (arithmetic stays
        FP64): the operator the B200 product's FP32 smoother applies at orders 7 and <= 5 (its pMG
        levels' smoother A, lambda estimate and V-cycle residual). Not a reference function: the reference
        has no FP32 smoother; this pins that product variant to FP64-arithmetic ground truth."""
        import copy
        c = copy.copy(self)
        c.geom = self.geom.astype(np.float32).astype(np.float64)
        return c

    def apply_A(self, u):
        """mask o Q^T A_L Q o mask (Neumann: minus the mean) — sem_space.cpp:195-209."""
        v = self.mask_inplace(np.array(u, dtype=np.float64))
        r = self.gather(self.apply_local_stiffness(self.scatter(v)))
        self.mask_inplace(r)
        if self.bc == NEUMANN:
            r -= r.mean()
        return r

    def stiffness_diag(self):
        """Assembled, masked diagonal — sem_space.cpp:211-236."""
        nd = self.nd
        D = self.basis.diff
        D2 = D * D
        g = self.geom.reshape(self.E, nd, nd, nd, 6)
        acc = (np.einsum("mi,ekjm->ekji", D2, g[..., 0], optimize=True)
               + np.einsum("mj,ekmi->ekji", D2, g[..., 3], optimize=True)
               + np.einsum("mk,emji->ekji", D2, g[..., 5], optimize=True))
        dd = np.diag(D)
        Di = dd[None, None, None, :]
        Dj = dd[None, None, :, None]
        Dk = dd[None, :, None, None]
        acc = acc + 2.0 * (Di * Dj * g[..., 1] + Di * Dk * g[..., 2] + Dj * Dk * g[..., 4])
        d = self.gather(acc.ravel())
        return self.mask_inplace(d)

    def apply_mass(self, u):
        """sem_space.hpp:73."""
        return self.mass_diag * u

    def local_stiffness_mults(self):
        """sem_space.cpp:182-185."""
        nd = self.nd
        return 6 * nd ** 4 + 9 * nd ** 3


# ----------------------------------------------------------------------------- RNG (libstdc++)

_MT_N, _MT_M = 312, 156
_MT_A = np.uint64(0xB5026F5AA96619E9)
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)


def mt19937_64(seed: int, count: int) -> np.ndarray:
    """std::mt19937_64 output stream (C++11 [rand.predef]), vectorised twist."""
    mt = np.zeros(_MT_N, dtype=np.uint64)
    mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    f = 6364136223846793005
    prev = int(mt[0])
    for i in range(1, _MT_N):
        prev = (f * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        mt[i] = np.uint64(prev)
    out = np.empty(count, dtype=np.uint64)
    pos = 0
    one = np.uint64(1)
    with np.errstate(over="ignore"):
        while pos < count:
            # twist in three dependency-respecting chunks
            i = np.arange(0, _MT_N - _MT_M)
            x = (mt[i] & _UPPER) | (mt[i + 1] & _LOWER)
            mt[i] = mt[i + _MT_M] ^ (x >> one) ^ np.where((x & one) != 0, _MT_A, np.uint64(0))
            i = np.arange(_MT_N - _MT_M, _MT_N - 1)
            x = (mt[i] & _UPPER) | (mt[i + 1] & _LOWER)
            mt[i] = mt[i - (_MT_N - _MT_M)] ^ (x >> one) ^ np.where((x & one) != 0, _MT_A, np.uint64(0))
            x = (mt[_MT_N - 1] & _UPPER) | (mt[0] & _LOWER)
            mt[_MT_N - 1] = mt[_MT_M - 1] ^ (x >> one) ^ (_MT_A if (int(x) & 1) else np.uint64(0))
            y = mt.copy()
            y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
            y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
            y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
            y ^= y >> np.uint64(43)
            take = min(_MT_N, count - pos)
            out[pos:pos + take] = y[:take]
            pos += take
    return out


def uniform_pm1(seed: int, count: int) -> np.ndarray:
    """std::uniform_real_distribution<double>(-1,1) over mt19937_64 (libstdc++
    generate_canonical with one 64-bit draw) — the start vector of chebyshev.cpp:12-15."""
    u = mt19937_64(seed, count).astype(np.float64) / 18446744073709551616.0
    u = np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)
    return 2.0 * u + (-1.0)


# ----------------------------------------------------------------------------- schwarz.cpp

INTERIOR, DIRICHLET_FACE, NEUMANN_FACE = 0, 1, 2
ASM, RAS = 0, 1


class SchwarzSmoother:
    """Overlapping Schwarz with FDM box solves — schwarz.hpp:31-86, schwarz.cpp:46-289.

    precision=32 restates the FP32 smoother variant used by the B200 path (S, inv_D and the
    extended residual cast to float32; contractions in float32)."""

    def __init__(self, space: SemSpace, mode: int = RAS, precision: int = 64):
        self.space, self.mode, self.precision = space, mode, precision
        mesh = space.mesh
        q, g = space.order, space.basis
        E = mesh.n_elements
        ex, ey, ez = mesh.element_ijk()
        self.ijk = np.stack([ex, ey, ez], axis=1)
        # box lengths: mean of 4 edge arc lengths by the level's GLL rule — schwarz.cpp:53-86
        Nx, Ny, _ = space.npts
        lengths = np.zeros((E, 3))
        for d in range(3):
            total = np.zeros(E)
            for ca in (0, 1):
                for cb in (0, 1):
                    m = np.arange(q + 1)
                    ijk = [None, None, None]
                    ijk[d] = m[None, :]
                    ijk[(d + 1) % 3] = np.full((1, q + 1), ca * q)
                    ijk[(d + 2) % 3] = np.full((1, q + 1), cb * q)
                    gx = self.ijk[:, 0:1] * q + ijk[0]
                    gy = self.ijk[:, 1:2] * q + ijk[1]
                    gz = self.ijk[:, 2:3] * q + ijk[2]
                    edge = space.coords[gx + Nx * (gy + Ny * gz)]  # (E, q+1, 3)
                    tangent = np.einsum("ml,elc->emc", g.diff, edge)
                    total = total + np.sum(g.weights[None, :] * np.linalg.norm(tangent, axis=2), axis=1)
            lengths[:, d] = total / 4.0
        if not np.all(lengths > 0.0):
            raise RuntimeError("SchwarzSmoother: degenerate element")
        self.lengths = lengths
        # per element/direction 1-D extended operators — schwarz.cpp:133-214
        from scipy.linalg import eigh
        gap01 = 0.5 * (g.nodes[1] - g.nodes[0])
        khat = np.einsum("m,mi,mj->ij", g.weights, g.diff, g.diff)
        P = q + 3
        self.P = P
        self.n = np.zeros((E, 3), dtype=np.int64)
        self.lo = np.zeros((E, 3), dtype=np.int64)
        self.ghost_left = np.zeros((E, 3), dtype=bool)
        self.ghost_right = np.zeros((E, 3), dtype=bool)
        self.S = np.zeros((E, 3, P, P))
        self.lam = np.zeros((E, 3, P))
        for e in range(E):
            for d in range(3):
                L = lengths[e, d]

                def classify(face):
                    nb = mesh.neighbor(e, face)
                    if nb >= 0:
                        return INTERIOR, lengths[nb, d] * gap01
                    return (DIRICHLET_FACE if space.bc == DIRICHLET else NEUMANN_FACE), 0.0

                lk, lgap = classify(2 * d)
                rk, rgap = classify(2 * d + 1)
                i0 = 1 if lk == DIRICHLET_FACE else 0
                i1 = q - 1 if rk == DIRICHLET_FACE else q
                gl = 1 if lk == INTERIOR else 0
                gr = 1 if rk == INTERIOR else 0
                n = (i1 - i0 + 1) + gl + gr
                if n < 1:
                    raise RuntimeError(f"SchwarzSmoother: element {e} has no local dofs")
                lo = int(self.ijk[e, d]) * q + i0 - gl
                A = np.zeros((n, n))
                B = np.zeros((n, n))
                for i in range(i0, i1 + 1):
                    a = i - i0 + gl
                    B[a, a] += 0.5 * L * g.weights[i]
                    for j in range(i0, i1 + 1):
                        b = j - i0 + gl
                        A[a, b] += (2.0 / L) * khat[i, j]
                if gl:
                    h = lgap
                    A[0, 0] += 2.0 / h
                    A[0, 1] += -1.0 / h
                    A[1, 0] += -1.0 / h
                    A[1, 1] += 1.0 / h
                    B[0, 0] += h
                    B[1, 1] += 0.5 * h
                if gr:
                    h = rgap
                    last = n - 1
                    A[last, last] += 2.0 / h
                    A[last, last - 1] += -1.0 / h
                    A[last - 1, last] += -1.0 / h
                    A[last - 1, last - 1] += 1.0 / h
                    B[last, last] += h
                    B[last - 1, last - 1] += 0.5 * h
                lam, S = eigh(A, B)  # S^T B S = I, ascending — schwarz.cpp:207-212
                self.n[e, d], self.lo[e, d] = n, lo
                self.ghost_left[e, d], self.ghost_right[e, d] = bool(gl), bool(gr)
                self.S[e, d, :n, :n] = S
                self.lam[e, d, :n] = lam
        # inverse diagonal (padded entries 0) — schwarz.cpp:92-108
        lx = self.lam[:, 0][:, None, None, :]
        ly = self.lam[:, 1][:, None, :, None]
        lz = self.lam[:, 2][:, :, None, None]
        s = lx + ly + lz
        ar = np.arange(P)
        valid = ((ar[None, None, None, :] < self.n[:, 0, None, None, None])
                 & (ar[None, None, :, None] < self.n[:, 1, None, None, None])
                 & (ar[None, :, None, None] < self.n[:, 2, None, None, None]))
        if np.any(valid & ~(s > 0.0)):
            raise RuntimeError("SchwarzSmoother: non-positive diagonal entry")
        self.inv_D = np.where(valid, 1.0 / np.where(valid, s, 1.0), 0.0)
        # extended-box global indices + participation (outside <= 1) — schwarz.cpp:110-127, 216-221
        gidx = []
        ghost = []
        for d in range(3):
            a = ar[None, :]
            gd = self.lo[:, d:d + 1] + a
            gh = (self.ghost_left[:, d:d + 1] & (a == 0)) | (self.ghost_right[:, d:d + 1] & (a == self.n[:, d:d + 1] - 1))
            inside = a < self.n[:, d:d + 1]
            gidx.append(np.where(inside, gd, 0))
            ghost.append(gh.astype(np.int64))
        Nx, Ny, _ = space.npts
        G = (gidx[0][:, None, None, :] + Nx * (gidx[1][:, None, :, None] + Ny * gidx[2][:, :, None, None]))
        outside = ghost[0][:, None, None, :] + ghost[1][:, None, :, None] + ghost[2][:, :, None, None]
        self.box_g = G
        self.box_part = valid & (outside <= 1)
        self.box_core = valid & (outside == 0)
        self.counts = np.bincount(G[self.box_part], minlength=space.n).astype(np.int64)
        owners = np.full(space.n, -1, dtype=np.int64)
        eid = np.broadcast_to(np.arange(E)[:, None, None, None], G.shape)
        core_g = G[self.box_core]
        core_e = eid[self.box_core]
        order = np.lexsort((core_e, core_g))
        cg, ce = core_g[order], core_e[order]
        first = np.ones(len(cg), dtype=bool)
        first[1:] = cg[1:] != cg[:-1]
        owners[cg[first]] = ce[first]  # lowest element id whose core holds g
        self.owners = owners
        self.weights = np.where(self.counts > 0, 1.0 / np.maximum(self.counts, 1), 0.0)

    def fdm_solve_all(self, rloc):
        """Batched fdm_solve on padded boxes (x fastest) — schwarz.cpp:228-240."""
        dt = np.float32 if self.precision == 32 else np.float64
        S = self.S.astype(dt)
        r = np.asarray(rloc).astype(dt)
        t = np.einsum("eia,ekji->ekja", S[:, 0], r, optimize=True)
        t = np.einsum("ejb,ekja->ekba", S[:, 1], t, optimize=True)
        t = np.einsum("ekc,ekba->ecba", S[:, 2], t, optimize=True)
        t = t * self.inv_D.astype(dt)
        t = np.einsum("eia,ekja->ekji", S[:, 0], t, optimize=True)
        t = np.einsum("ejb,ekbi->ekji", S[:, 1], t, optimize=True)
        t = np.einsum("ekc,ecji->ekji", S[:, 2], t, optimize=True)
        return t.astype(np.float64)

    def extract(self, r):
        """Extended-box residual, sites outside in >1 direction zero-filled — schwarz.cpp:255-265."""
        return np.where(self.box_part, np.asarray(r)[self.box_g], 0.0)

    def apply(self, r):
        """RAS owner-write / ASM weighted sum — schwarz.cpp:242-289."""
        eloc = self.fdm_solve_all(self.extract(r))
        n = self.space.n
        if self.mode == RAS:
            out = np.zeros(n)
            E = eloc.shape[0]
            eid = np.broadcast_to(np.arange(E)[:, None, None, None], eloc.shape)
            sel = self.box_part & (self.owners[self.box_g] == eid)
            out[self.box_g[sel]] = eloc[sel]
            return out
        out = np.bincount(self.box_g[self.box_part], weights=eloc[self.box_part], minlength=n)
        return out * self.weights

    def box_matrix(self, e):
        """Dense extended-box operator Abar = B(x)B(x)A + B(x)A(x)B + A(x)B(x)B rebuilt from the
        FDM factors (S^-T diag(lam) S^-1 per direction) — for the SPEC.md:611 exactness test."""
        mats = []
        for d in range(3):
            n = self.n[e, d]
            S = self.S[e, d, :n, :n]
            Si = np.linalg.inv(S)
            Bm = Si.T @ Si
            Am = Si.T @ np.diag(self.lam[e, d, :n]) @ Si
            mats.append((Am, Bm))
        (Ax, Bx), (Ay, By), (Az, Bz) = mats
        return np.kron(Bz, np.kron(By, Ax)) + np.kron(Bz, np.kron(Ay, Bx)) + np.kron(Az, np.kron(By, Bx))


# ----------------------------------------------------------------------------- chebyshev.cpp


@dataclass
class LambdaEstimate:
    value: float = 0.0
    breakdown: bool = False
    rounds_used: int = 0


def estimate_lambda_max(S, A, n, rounds=10, seed=0):
    """10-round CGS2 Arnoldi on S*A from a seeded U(-1,1) start — chebyshev.cpp:9-56."""
    if rounds < 1:
        raise ValueError("estimate_lambda_max: rounds >= 1")
    v = uniform_pm1(seed, n)
    est = LambdaEstimate()
    V = np.zeros((n, rounds + 1))
    H = np.zeros((rounds + 1, rounds))
    w = S(A(v))
    nrm = np.linalg.norm(w)
    if not nrm > 0.0:
        est.breakdown = True
        return est
    V[:, 0] = w / nrm
    m = 0
    for j in range(rounds):
        w = S(A(V[:, j]))
        h = V[:, :j + 1].T @ w
        w = w - V[:, :j + 1] @ h
        h2 = V[:, :j + 1].T @ w
        w = w - V[:, :j + 1] @ h2
        h = h + h2
        H[:j + 1, j] = h
        hnext = np.linalg.norm(w)
        H[j + 1, j] = hnext
        m = j + 1
        if hnext <= 1e-12 * np.max(np.abs(h)):
            est.breakdown = True
            break
        V[:, j + 1] = w / hnext
    est.rounds_used = m
    est.value = float(np.max(np.abs(np.linalg.eigvals(H[:m, :m]))))
    return est


@dataclass
class ChebyParams:
    order: int = 2
    lambda_min_mult: float = 0.1
    lambda_max_mult: float = 1.1
    lambda_max_est: float = 0.0


class ChebyshevSmoother:
    """Paper Alg. 2 — chebyshev.hpp:36-46, chebyshev.cpp:58-96."""

    def __init__(self, S, A, params: ChebyParams):
        if params.order < 1:
            raise ValueError("ChebyshevSmoother: order must be >= 1")
        if not (params.lambda_min_mult > 0.0) or not (params.lambda_max_mult > params.lambda_min_mult):
            raise ValueError("ChebyshevSmoother: need 0 < lambda_min_mult < lambda_max_mult")
        if not params.lambda_max_est > 0.0:
            raise ValueError("ChebyshevSmoother: lambda_max_est not set")
        self.S, self.A, self.params = S, A, params
        lmin = params.lambda_min_mult * params.lambda_max_est
        lmax = params.lambda_max_mult * params.lambda_max_est
        self.theta = 0.5 * (lmax + lmin)
        self.delta = 0.5 * (lmax - lmin)
        self.sigma = self.theta / self.delta

    def smooth(self, b, x):
        """In-place on x; returns x."""
        t = b - self.A(x)
        r = self.S(t)
        d = r / self.theta
        rho = 1.0 / self.sigma
        for _ in range(self.params.order):
            x += d
            sad = self.S(self.A(d))
            r = r - sad
            rho_next = 1.0 / (2.0 * self.sigma - rho)
            d = rho_next * rho * d + (2.0 * rho_next / self.delta) * r
            rho = rho_next
        x += d
        return x


# ----------------------------------------------------------------------------- krylov.cpp


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


def gmres_solve(A, M, b, x, config: GmresConfig) -> GmresStats:
    """Restarted right-preconditioned GMRES(m), CGS2, Givens — krylov.cpp:20-129. x in place."""
    if config.restart < 1:
        raise ValueError("gmres: restart must be >= 1")
    if not config.tol > 0.0:
        raise ValueError("gmres: tol must be positive")
    Mop = M if M is not None else (lambda v: v.copy())
    n, m = b.size, config.restart
    st = GmresStats()
    r = b - A(x)
    st.initial_residual = float(np.linalg.norm(r))
    target = config.abs_tol if config.use_abs_tol else config.tol * st.initial_residual
    V = np.zeros((n, m + 1))
    H = np.zeros((m + 1, m))
    g = np.zeros(m + 1)
    cs, sn = np.zeros(m), np.zeros(m)

    def finish(res):
        st.abs_residual = float(res)
        st.rel_residual = float(res / st.initial_residual) if st.initial_residual > 0 else 0.0

    beta = st.initial_residual
    if beta <= target:
        st.converged = True
        finish(beta)
        return st
    while st.iterations < config.max_iters:
        V[:, 0] = r / beta
        g[:] = 0.0
        g[0] = beta
        H[:] = 0.0
        j = 0
        lucky = False
        while j < m and st.iterations < config.max_iters:
            z = Mop(V[:, j])
            w = A(z)
            h = V[:, :j + 1].T @ w
            w = w - V[:, :j + 1] @ h
            h2 = V[:, :j + 1].T @ w
            w = w - V[:, :j + 1] @ h2
            h = h + h2
            H[:j + 1, j] = h
            hnext = float(np.linalg.norm(w))
            H[j + 1, j] = hnext
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = math.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / denom if denom > 0.0 else 1.0
            sn[j] = H[j + 1, j] / denom if denom > 0.0 else 0.0
            H[j, j] = denom
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] *= cs[j]
            st.iterations += 1
            res_est = abs(g[j + 1])
            st.history.append(res_est)
            if hnext <= 1e-14 * beta:
                st.breakdown = True
                lucky = True
                j += 1
                break
            V[:, j + 1] = w / hnext
            if res_est <= target:
                j += 1
                break
            j += 1
        if j > 0:
            from scipy.linalg import solve_triangular
            y = solve_triangular(H[:j, :j], g[:j], lower=False)
            x += Mop(V[:, :j] @ y)
        r = b - A(x)
        beta = float(np.linalg.norm(r))
        if beta <= target or lucky:
            st.converged = True
            finish(beta)
            return st
    finish(beta)
    st.converged = beta <= target
    return st


class ProjectionBasis:
    """krylov.hpp:39-59 / krylov.cpp:131-152: A-orthonormal prior solutions, oldest first."""

    def __init__(self, capacity=10):
        self.capacity, self.basis = capacity, []

    def initial_guess(self, b):
        u = np.zeros_like(b)
        for v in self.basis:  # krylov.cpp:134-137
            u += v.dot(b) * v
        return u

    def insert(self, x, A):
        if A is None:
            raise ValueError("ProjectionBasis: missing operator")
        w = x.copy()
        aw = A(w)
        norm0 = np.sqrt(max(0.0, w.dot(aw)))
        for _ in range(2):  # krylov.cpp:144-147: coefficients from the same A w within a pass
            for v in self.basis:
                w -= v.dot(aw) * v
            aw = A(w)
        norm = np.sqrt(max(0.0, w.dot(aw)))
        if not norm > 1e-12 * max(norm0, 1e-300):
            return
        self.basis.append(w / norm)
        if len(self.basis) > self.capacity:
            self.basis.pop(0)


@dataclass
class PcgStats:
    iterations: int = 0
    converged: bool = False
    initial_residual: float = 0.0
    abs_residual: float = 0.0
    rel_residual: float = 0.0
    history: list = field(default_factory=list)


def pcg_solve(A, M, b, x, tol=1e-8, max_iters=500) -> PcgStats:
    """RESTATED (no reference code; the reference has only GMRES):
    textbook preconditioned CG, stopping on the unpreconditioned recurrence residual
    ||r_k|| <= tol ||b - A x0|| like gmres_solve's relative test (krylov.cpp:33-36), then
    recomputing the true residual for the stats (krylov.cpp:116-118)."""
    Mop = M if M is not None else (lambda v: v.copy())
    st = PcgStats()
    r = b - A(x)
    r0 = float(np.linalg.norm(r))
    st.initial_residual = r0
    target = tol * r0
    if r0 <= target or r0 == 0.0:
        st.converged = True
        return st
    z = Mop(r)
    p = z.copy()
    rz = float(r @ z)
    while st.iterations < max_iters:
        w = A(p)
        alpha = rz / float(p @ w)
        x += alpha * p
        r -= alpha * w
        st.iterations += 1
        rn = float(np.linalg.norm(r))
        st.history.append(rn)
        if rn <= target:
            break
        z = Mop(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    res = float(np.linalg.norm(b - A(x)))
    st.abs_residual = res
    st.rel_residual = res / r0
    st.converged = st.history[-1] <= target
    return st


# ----------------------------------------------------------------------------- amg.cpp


@dataclass
class AmgOptions:
    strength_threshold: float = 0.25
    jacobi_damping: float = 0.9
    pre_sweeps: int = 1
    post_sweeps: int = 1
    max_levels: int = 25
    max_coarse_size: int = 200
    coarse_direct: bool = True
    coarse_sweeps: int = 8


def amg_aggregate(A, theta):
    """Greedy 3-pass aggregation over the strength graph — amg.cpp:12-65."""
    A = A.tocsr()
    n = A.shape[0]
    indptr, indices, data = A.indptr, A.indices, A.data
    strong = []
    for i in range(n):
        cols = indices[indptr[i]:indptr[i + 1]]
        vals = data[indptr[i]:indptr[i + 1]]
        off = cols != i
        row_max = float(np.max(np.abs(vals[off]))) if np.any(off) else 0.0
        if row_max == 0.0:
            strong.append(np.zeros(0, dtype=np.int64))
            continue
        cutoff = theta * row_max
        sel = off & (np.abs(vals) >= cutoff)
        strong.append(cols[sel].astype(np.int64))
    agg = np.full(n, -1, dtype=np.int64)
    n_agg = 0
    for i in range(n):
        if agg[i] >= 0:
            continue
        s = strong[i]
        if len(s) == 0 or np.any(agg[s] >= 0):
            continue
        agg[i] = n_agg
        agg[s] = n_agg
        n_agg += 1
    for i in range(n):
        if agg[i] >= 0:
            continue
        best, best_agg = 0.0, -1
        for j in strong[i]:
            if agg[j] < 0:
                continue
            w = abs(A[i, j])
            if w > best:
                best, best_agg = w, agg[j]
        if best_agg >= 0:
            agg[i] = best_agg
    for i in range(n):
        if agg[i] < 0:
            agg[i] = n_agg
            n_agg += 1
    return agg, n_agg


class AmgHierarchy:
    """Aggregation AMG, Galerkin coarse ops, damped-Jacobi V-cycle — amg.hpp:34-61, amg.cpp:69-165."""

    def __init__(self, A, opts: AmgOptions | None = None):
        import scipy.sparse as sp
        opts = opts or AmgOptions()
        self.opts = opts
        self.levels = []  # dicts: A, inv_diag, P (None on the coarsest), agg
        current = sp.csr_matrix(A)
        while len(self.levels) < opts.max_levels - 1 and current.shape[0] > opts.max_coarse_size:
            d = current.diagonal()
            if np.any(d == 0.0):
                raise RuntimeError("AmgHierarchy: zero diagonal")
            agg, n_agg = amg_aggregate(current, opts.strength_threshold)
            lvl = {"A": current, "inv_diag": 1.0 / d, "agg": agg, "P": None}
            if n_agg >= current.shape[0]:
                self.levels.append(lvl)
                break
            P = sp.csr_matrix((np.ones(len(agg)), (np.arange(len(agg)), agg)), shape=(len(agg), n_agg))
            lvl["P"] = P
            coarse = (P.T.tocsr() @ current @ P).tocsr()
            self.levels.append(lvl)
            current = coarse
        if not self.levels or self.levels[-1]["P"] is not None:
            d = current.diagonal()
            self.levels.append({"A": current, "inv_diag": 1.0 / d, "agg": None, "P": None})
        self.coarse_dense = self.levels[-1]["A"].toarray()

    def _relax(self, lvl, b, x, sweeps):
        for _ in range(sweeps):
            r = b - lvl["A"] @ x
            x += self.opts.jacobi_damping * lvl["inv_diag"] * r
        return x

    def _cycle(self, l, r):
        lvl = self.levels[l]
        if l == len(self.levels) - 1:
            if self.opts.coarse_direct:
                return np.linalg.solve(self.coarse_dense, r)
            return self._relax(lvl, r, np.zeros_like(r), self.opts.coarse_sweeps)
        z = self._relax(lvl, r, np.zeros_like(r), self.opts.pre_sweeps)
        res = r - lvl["A"] @ z
        rc = lvl["P"].T @ res
        z += lvl["P"] @ self._cycle(l + 1, rc)
        return self._relax(lvl, r, z, self.opts.post_sweeps)

    def vcycle(self, r):
        return self._cycle(0, np.asarray(r, dtype=np.float64))


# ----------------------------------------------------------------------------- RESTATED: rhs, jacobi, pmg


def build_rhs(space: SemSpace, seed: int = 1):
    """RESTATED (bench.cpp is missing, Eq. 11): f = 3 pi^2 prod
    sin(pi (x_d + 1/2)) (the product-sine on the shifted domain, vanishing on the boundary of
    [-1/2,1/2]^3) + g, g = U(-1,1) nodal noise from mt19937_64(seed) (one draw per lattice dof
    in index order) times the bubble 64 prod(1/4 - x_d^2); b = mask(mass_diag * f)."""
    X = space.coords
    f = 3.0 * math.pi ** 2 * np.prod(np.sin(math.pi * (X + 0.5)), axis=1)
    bubble = 64.0 * np.prod(0.25 - X * X, axis=1)
    f = f + uniform_pm1(seed, space.n) * bubble
    return space.mask_inplace(space.mass_diag * f)


def jacobi_inverse_diag(space: SemSpace):
    """RESTATED (precond.cpp missing): S = diag(A)^-1, masked entries 0."""
    d = space.stiffness_diag()
    return np.where(d != 0.0, 1.0 / np.where(d != 0.0, d, 1.0), 0.0)


def interpolation_1d(q_coarse, q_fine):
    """Element 1-D transfer J (q_f+1 x q_c+1) — gll.cpp:93-118 on the two GLL node sets."""
    return lagrange_interpolation_matrix(gll(q_coarse).nodes, gll(q_fine).nodes)


class Transfer:
    """RESTATED (pmg.cpp missing): P = mask_f o (assembled average of the
    element-local tensor interpolation J(x)J(x)J) o mask_c, P^T its exact transpose."""

    def __init__(self, fine: SemSpace, coarse: SemSpace):
        self.fine, self.coarse = fine, coarse
        self.J = interpolation_1d(coarse.order, fine.order)

    def _local(self, J, u, E, n_in):
        u = u.reshape(E, n_in, n_in, n_in)
        t = np.einsum("ia,ekja->ekji", J, u, optimize=True)
        t = np.einsum("jb,ekbi->ekji", J, t, optimize=True)
        return np.einsum("kc,ecji->ekji", J, t, optimize=True).reshape(-1)

    def prolong(self, uc):
        f, c = self.fine, self.coarse
        uc = c.mask_inplace(np.array(uc, dtype=np.float64))
        loc = self._local(self.J, c.scatter(uc), c.E, c.nd)
        uf = f.gather(loc) / f.multiplicity
        return f.mask_inplace(uf)

    def restrict(self, rf):
        f, c = self.fine, self.coarse
        rf = f.mask_inplace(np.array(rf, dtype=np.float64)) / f.multiplicity
        loc = self._local(self.J.T, f.scatter(rf), f.E, f.nd)
        return c.mask_inplace(c.gather(loc))


def assemble_p1(space: SemSpace):
    """Sparse assembled operator at the coarse order (element matrices from
    apply_local_stiffness columns), restricted to the free (unmasked) dofs — the coarse
    system of SPEC.md:326,341 (masked rows would be identity; they are dropped)."""
    import scipy.sparse as sp
    nl = space.nloc
    E = space.E
    Ae = np.zeros((E, nl, nl))
    for c in range(nl):
        u = np.zeros((E, nl))
        u[:, c] = 1.0
        Ae[:, :, c] = space.apply_local_stiffness(u.ravel()).reshape(E, nl)
    l2g = space.l2g.reshape(E, nl)
    rows = np.broadcast_to(l2g[:, :, None], Ae.shape).ravel()
    cols = np.broadcast_to(l2g[:, None, :], Ae.shape).ravel()
    A = sp.coo_matrix((Ae.ravel(), (rows, cols)), shape=(space.n, space.n)).tocsr()
    free = np.flatnonzero(space.masked == 0) if space.bc == DIRICHLET else np.arange(space.n)
    return A[free][:, free].tocsr(), free


class CoarseSolve:
    """RESTATED coarse solve: 'direct' exact sparse factorisation of the
    free-dof coarse matrix, or 'amg' = one AmgHierarchy V-cycle (amg.cpp:140-165)."""

    def __init__(self, space: SemSpace, mode="direct", amg_opts=None):
        self.space, self.mode = space, mode
        self.A, self.free = assemble_p1(space)
        self.neumann = space.bc == NEUMANN
        if self.neumann and mode != "direct":
            raise ValueError("pmg: the Neumann coarse problem is singular; it needs the direct coarse solve")
        if mode == "direct":
            from scipy.sparse.linalg import splu
            A = self.A
            if self.neumann:  # constants span the nullspace: A + 1 1^T / n is SPD
                n = A.shape[0]
                A = A.toarray() + 1.0 / n
                from scipy.sparse import csc_matrix
                A = csc_matrix(A)
            self.lu = splu(A.tocsc())
        else:
            self.amg = AmgHierarchy(self.A, amg_opts)

    def solve(self, r):
        z = np.zeros(self.space.n)
        rf = np.asarray(r)[self.free]
        if self.neumann:  # zero-mean right-hand side and solution (nullspace projection)
            rf = rf - rf.mean()
        zf = self.lu.solve(rf) if self.mode == "direct" else self.amg.vcycle(rf)
        if self.neumann:
            zf = zf - zf.mean()
        z[self.free] = zf
        return z


class Pmg:
    """RESTATED p-multigrid V-cycle (pmg.cpp missing, Alg. 1):
    x0 = 0, Chebyshev pre-smooth, residual, r_C = P^T r, recurse / coarse solve,
    x += P e_C, Chebyshev post-smooth with the same eta."""

    def __init__(self, mesh, orders=(7, 3, 1), smoother="jacobi", cheb_order=2,
                 lmin_mult=0.1, lmax_mult=1.1, coarse="direct", precision=64, seed=0, bc=DIRICHLET,
                 cycle="standard"):
        """smoother: "jacobi" | "ras" | "asm" (Chebyshev) | "ras_plain" | "asm_plain" (one plain
        application per smoothing step); cycle: "standard" (Alg. 1) | "additive"."""
        if list(orders) != sorted(orders, reverse=True) or orders[-1] != 1 or len(set(orders)) != len(orders):
            raise ValueError("pmg: schedule must be strictly decreasing and end at 1")
        self.orders = tuple(orders)
        self.plain = smoother.endswith("_plain")
        self.additive = cycle == "additive"
        smoother = smoother[:3] if self.plain else smoother
        self.spaces = [SemSpace(mesh, q, bc) for q in orders]
        self.levels = []
        for sp_ in self.spaces[:-1]:
            # precision 32: every smoothed level's operator uses FP32-rounded factors, like the
            # product (pmg.cpp build(): L.A->geom32, orders 7 and <= 5); the Krylov operator is
            # not part of Pmg
            A = sp_.with_geom32().apply_A if (precision == 32 and (sp_.order == 7 or sp_.order <= 5)) \
                else sp_.apply_A
            if smoother == "jacobi":
                inv = jacobi_inverse_diag(sp_)
                S = (lambda inv: (lambda v: inv * v))(inv)
            else:
                sch = SchwarzSmoother(sp_, RAS if smoother == "ras" else ASM, precision)
                S = sch.apply
            if self.plain:
                lam, cheb = 0.0, None
            else:
                lam = estimate_lambda_max(S, A, sp_.n, 10, seed).value
                cheb = ChebyshevSmoother(S, A, ChebyParams(cheb_order, lmin_mult, lmax_mult, lam))
            self.levels.append({"space": sp_, "A": A, "S": S, "lam": lam, "cheb": cheb})
        self.transfers = [Transfer(self.spaces[l], self.spaces[l + 1]) for l in range(len(orders) - 1)]
        self.coarse = CoarseSolve(self.spaces[-1], coarse)

    def _smooth(self, l, b, x):
        lvl = self.levels[l]
        if not self.plain:
            lvl["cheb"].smooth(b, x)
        elif not x.any():
            x[:] = lvl["S"](b)
        else:
            x += lvl["S"](b - lvl["A"](x))
        return x

    def vcycle(self, b, l=0):
        if self.additive:
            return self._additive(b, l)
        if l == len(self.levels):
            return self.coarse.solve(b)
        lvl = self.levels[l]
        x = self._smooth(l, b, np.zeros_like(b))
        r = b - lvl["A"](x)
        ec = self.vcycle(self.transfers[l].restrict(r), l + 1)
        x += self.transfers[l].prolong(ec)
        return self._smooth(l, b, x)

    def _additive(self, b, l=0):
        """Additive V-cycle: every level smooths its restricted right-hand side from
        zero, the coarsest is solved, the prolongated corrections are summed; no post-smoothing."""
        if l == len(self.levels):
            return self.coarse.solve(b)
        x = self._smooth(l, b, np.zeros_like(b))
        x += self.transfers[l].prolong(self._additive(self.transfers[l].restrict(b), l + 1))
        return x


def assemble_semfem(space: SemSpace):
    """Linear-tetrahedral stiffness on the GLL lattice — semfem.cpp:12-98: every hex sub-cell is
    covered by its 8 corner tetrahedra with an overall 1/2; masked dofs eliminated (unit
    diagonal); exact zeros pruned. Vectorised over sub-cells (numpy rounding, not bitwise)."""
    import scipy.sparse as sps
    p, E = space.order, space.E
    X = space.coords
    Nx, Ny, Nz = space.npts
    ex, ey, ez = space.mesh.element_ijk()
    r = np.arange(p)
    # sub-cell origin lattice indices, element-major then (k, j, i)
    gx = (ex[:, None, None, None] * p + r[None, None, None, :])
    gy = (ey[:, None, None, None] * p + r[None, None, :, None])
    gz = (ez[:, None, None, None] * p + r[None, :, None, None])
    gx, gy, gz = np.broadcast_arrays(gx, gy, gz)
    gx, gy, gz = gx.ravel(), gy.ravel(), gz.ravel()
    cell = np.stack([(gx + cx) + Nx * ((gy + cy) + Ny * (gz + cz))
                     for cz in (0, 1) for cy in (0, 1) for cx in (0, 1)], axis=1)
    tets = []
    for cz in (0, 1):
        for cy in (0, 1):
            for cx in (0, 1):
                c = lambda x, y, z: x + 2 * y + 4 * z  # noqa: E731
                t = [c(cx, cy, cz), c(1 - cx, cy, cz), c(cx, 1 - cy, cz), c(cx, cy, 1 - cz)]
                if (cx + cy + cz) % 2:
                    t[1], t[2] = t[2], t[1]
                tets.append(t)
    masked = space.masked.astype(bool)
    rows, cols, vals = [], [], []
    for t in tets:
        v = cell[:, t]
        P0 = X[v[:, 0]]
        T = np.stack([X[v[:, 1]] - P0, X[v[:, 2]] - P0, X[v[:, 3]] - P0], axis=2)
        det = np.linalg.det(T)
        if np.any(det <= 0.0):
            raise RuntimeError("assemble_semfem: inverted tetrahedron")
        Ti = np.linalg.inv(T)
        grad = np.stack([-Ti.sum(axis=1), Ti[:, 0, :], Ti[:, 1, :], Ti[:, 2, :]], axis=1)
        K = 0.5 * (det / 6.0)[:, None, None] * np.einsum("nad,nbd->nab", grad, grad)
        ga = np.broadcast_to(v[:, :, None], K.shape)
        gb = np.broadcast_to(v[:, None, :], K.shape)
        keep = ~(masked[ga] | masked[gb])
        rows.append(ga[keep])
        cols.append(gb[keep])
        vals.append(K[keep])
    mi = np.flatnonzero(masked)
    rows.append(mi)
    cols.append(mi)
    vals.append(np.ones(mi.size))
    A = sps.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                       shape=(space.n, space.n)).tocsr()
    A.eliminate_zeros()
    return A


class SemfemPreconditioner:
    """semfem.cpp:112-134 with the AMG inner solve: z = mask(AmgHierarchy(A_F).vcycle(r))."""

    def __init__(self, space: SemSpace, amg_opts=None):
        self.space = space
        self.A = assemble_semfem(space)
        self.amg = AmgHierarchy(self.A, amg_opts)

    def apply(self, r):
        return self.space.mask_inplace(self.amg.vcycle(np.asarray(r, dtype=np.float64)))
