"""BASELINE.json configs c1-c4 at their own sizes: the case table and the deterministic inputs and
sample sets shared by the fixture generator (make_golden_scale.py, runs the reference here) and the
GPU tests (tests/test_scale_gpu.py, run on the B200 box without /root/reference).

Vectors at these sizes (up to 11.4M doubles) are too large to commit, so a fixture keeps, per
output vector: the values on one full element-interface z-plane plus 8192 seeded random lattice
sites, the 2-norm, the max-norm and the dot product with a seeded random weight vector (a
checksum over every entry).
"""
import numpy as np

# name: (eps, E, orders, precond, coarse, krylov 0=GMRES(20) / 1=PCG, chebyshev order)
CASES = {
    "c1": (1.0, 8, (7,), "jacobi", "direct", 1, 2),           # Jacobi-PCG, box E=8^3
    "c2": (1.0, 16, (7, 3, 1), "jacobi", "direct", 1, 2),     # pMG Cheby-Jacobi, PCG, box E=16^3
    "c3": (1.0, 16, (7, 3, 1), "ras", "direct", 0, 2),        # pMG Cheby-RAS, GMRES, box E=16^3
    "c4": (0.3, 32, (7, 3, 1), "ras", "amg", 0, 2),           # pMG Cheby-RAS, GMRES, Kershaw E=32^3
}


def n_of(E, p):
    return (E * p + 1) ** 3


def sample_index(E, p):
    """Lattice sites kept in a fixture: the z-plane at the element interface z = p*E/2 (every x-,
    y- and z-face of the Q^T sum meets it) and 8192 seeded random sites."""
    N = E * p + 1
    z = p * (E // 2)
    plane = z * N * N + np.arange(N * N, dtype=np.int64)
    rnd = np.random.default_rng(99).integers(0, N ** 3, 8192, dtype=np.int64)
    return np.unique(np.concatenate([plane, rnd]))


def boundary_mask(E, p):
    """True on the lattice boundary (the Dirichlet mask, sem_space.cpp:20-28)."""
    N = E * p + 1
    a = np.zeros(N, dtype=bool)
    a[0] = a[-1] = True
    return (a[None, None, :] | a[None, :, None] | a[:, None, None]).reshape(-1)


def input_u(E, p):
    return np.random.default_rng(2000 + E).standard_normal(n_of(E, p))


def input_r(E, p):
    r = np.random.default_rng(3000 + E).standard_normal(n_of(E, p))
    r[boundary_mask(E, p)] = 0.0
    return r


def weights(n):
    return np.random.default_rng(777).standard_normal(n)


def summarize(v, idx, w):
    """(samples, [2-norm, max-norm, w.v])"""
    return v[idx].copy(), np.array([np.linalg.norm(v), np.abs(v).max(), float(w @ v)])
