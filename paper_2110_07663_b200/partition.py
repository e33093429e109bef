"""Host-side mirror of the z-slab partition used by the distributed path (csrc/common.hpp Slab).

Rank r of R owns element layers [ez0, ez1) with ez0 = r*Ez//R; its local lattice vectors hold
global planes [zlo, zlo+nzl) = the slab's planes [ez0 q, ez1 q] plus one ghost plane across each
internal boundary. Reductions count the planes [ez0 q, ez1 q) (+ the global top plane on the
last rank), so every interface plane is counted exactly once.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Slab:
    q: int
    Ex: int
    Ey: int
    Ez: int
    rank: int
    nranks: int

    @property
    def ez0(self) -> int:
        return (self.rank * self.Ez) // self.nranks

    @property
    def ez1(self) -> int:
        return ((self.rank + 1) * self.Ez) // self.nranks

    @property
    def Nx(self) -> int:
        return self.Ex * self.q + 1

    @property
    def Ny(self) -> int:
        return self.Ey * self.q + 1

    @property
    def Nz(self) -> int:
        return self.Ez * self.q + 1

    @property
    def below(self) -> bool:
        return self.ez0 > 0

    @property
    def above(self) -> bool:
        return self.ez1 < self.Ez

    @property
    def zlo(self) -> int:
        return self.ez0 * self.q - (1 if self.below else 0)

    @property
    def nzl(self) -> int:
        return self.ez1 * self.q + (1 if self.above else 0) - self.zlo + 1

    @property
    def plane(self) -> int:
        return self.Nx * self.Ny

    @property
    def n_local(self) -> int:
        return self.plane * self.nzl

    @property
    def own_z0(self) -> int:
        return self.ez0 * self.q

    @property
    def own_z1(self) -> int:
        return self.ez1 * self.q + (1 if self.ez1 == self.Ez else 0)

    def local_slice(self):
        """Global-vector slice of this rank's local planes (ghosts included)."""
        return slice(self.zlo * self.plane, (self.zlo + self.nzl) * self.plane)

    def owned_slice_global(self):
        return slice(self.own_z0 * self.plane, self.own_z1 * self.plane)

    def owned_slice_local(self):
        a = (self.own_z0 - self.zlo) * self.plane
        return slice(a, a + (self.own_z1 - self.own_z0) * self.plane)

    def element_range(self):
        """Global element ids on this rank (contiguous: e = ex + Ex (ey + Ey ez))."""
        return range(self.ez0 * self.Ex * self.Ey, self.ez1 * self.Ex * self.Ey)
