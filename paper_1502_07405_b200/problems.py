"""BASELINE.json configurations and the shared seeded right-hand side.

x_true[i] ~ U(-1, 1) from splitmix64(seed, i) with 53-bit mantissas; both the
product harness and the oracle harness consume exactly these bytes, and
b = A x_true is computed once on the host with a deterministic CSR matvec
("shared RHS rule"). BASELINE's configs use no public data
set: every input is this seeded synthetic data.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (np.arange(n, dtype=np.uint64) + np.uint64(1) + (np.uint64(seed) << np.uint64(32)))
        z = z * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def x_true(n: int, seed: int = 1) -> np.ndarray:
    z = splitmix64(seed, n)
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def csr_matvec(ptr, ind, val, x) -> np.ndarray:
    """row-sequential y = A x (same summation order as SparseMatrix::matvec)"""
    prod = val * x[ind]
    y = np.zeros(len(ptr) - 1)
    # np.add.reduceat sums left to right within each row
    nz = ptr[1:] > ptr[:-1]
    y[nz] = np.add.reduceat(prod, ptr[:-1][nz])
    return y


@dataclass(frozen=True)
class Config:
    name: str
    kind: str        # p2d | p3d | cd3d | dense
    k: int           # grid size (or N for dense)
    nd_leaf: int
    ls: int
    min_hss: int
    eps: float
    leaf: int
    mode: str = "auto"
    d0: int = 128
    dd: int = 128
    p: int = 10

    def solver_options(self):
        from .api import SolverOptions
        return SolverOptions(nd_leaf=self.nd_leaf, ls=self.ls, eps=self.eps, leaf=self.leaf,
                             d0=self.d0, dd=self.dd, p=self.p, min_hss=self.min_hss,
                             mode=self.mode)


# BASELINE.json "configs", mapped as in SURVEY.md §8d
CONFIGS = {
    "c1": Config("c1_p2d256_hss", "p2d", 256, 64, 64, 256, 1e-6, 64),
    "c1_mf": Config("c1_p2d256_mf", "p2d", 256, 64, 0, 256, 1e-6, 64, mode="mf"),
    "c2": Config("c2_dense16384", "dense", 16384, 0, 0, 0, 1e-8, 128),
    "c3": Config("c3_p3d64_hss", "p3d", 64, 32, 64, 1000, 1e-4, 128),
    "c4": Config("c4_cd3d96_hss", "cd3d", 96, 32, 64, 2000, 1e-5, 128),
    "c5": Config("c5_p3d128_hss", "p3d", 128, 32, 64, 4000, 1e-4, 256),
    "c5_mf": Config("c5_p3d128_mf", "p3d", 128, 32, 0, 4000, 1e-4, 256, mode="mf"),
    # config 5's options on smaller grids (reference runs that fit in time and
    # memory; the validation of the reference arm's sample scaling)
    "c5_96": Config("p3d96_c5opts", "p3d", 96, 32, 64, 4000, 1e-4, 256),
    "c5_112": Config("p3d112_c5opts", "p3d", 112, 32, 64, 4000, 1e-4, 256),
}


def dense_c2(n: int) -> np.ndarray:
    """A_ij = 1/(1+|i-j|) + 4 delta_ij (BASELINE config 2), column-major"""
    i = np.arange(n)
    A = 1.0 / (1.0 + np.abs(i[:, None] - i[None, :]).astype(np.float64))
    A[i, i] += 4.0
    return np.asfortranarray(A)
