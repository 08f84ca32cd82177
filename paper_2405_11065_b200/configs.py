"""BASELINE.json configs C1-C5 as synthetic inputs (SURVEY 8d input table).

The paper states neither the polynomial order nor the mesh of its runs (R2);
these seeded box meshes stand in for Nekbone's generated box runs (P:559,
P:642).  No dataset or benchmark suite is involved.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    ex: int
    ey: int
    ez: int            # per GPU for the weak-scaling configs (global ez = ez * P)
    N: int
    jitter: float
    seed_geom: int
    seed_rhs: int
    niter: int
    weak: bool = False
    note: str = ""

    def mesh_args(self, nranks: int = 1):
        ez = self.ez * nranks if self.weak else self.ez
        return dict(ex=self.ex, ey=self.ey, ez=ez, N=self.N, jitter=self.jitter,
                    seed_geom=self.seed_geom, seed_rhs=self.seed_rhs)


CONFIGS = {
    "C1": Config("C1", 2, 2, 2, 8, 0.0, 0, 1001, 100,
                 note="tiny oracle case: undeformed 2x2x2, p=7"),
    "C2": Config("C2", 16, 16, 16, 8, 0.0, 0, 1002, 100, weak=True,
                 note="undeformed 16^3 (per GPU), p=7, 100 CG iterations"),
    "C3": Config("C3", 32, 32, 32, 12, 0.1, 2003, 1003, 100, weak=True,
                 note="deformed 32^3 (per GPU), p=11, +-10% vertex jitter"),
    "C4": Config("C4", 64, 64, 32, 8, 0.0, 0, 1004, 100, weak=True,
                 note="weak scaling 64x64x32 per GPU, p=7"),
    "C5": Config("C5", 64, 64, 64, 10, 0.1, 2005, 1005, 200,
                 note="strong scaling 64^3, p=9, deformed, 200 iterations"),
}
