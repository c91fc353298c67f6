"""Seeded synthetic workload generators shared by the oracle tests, the GPU
parity tests and bench.py.

This module holds NO arithmetic of the AFN method: it only draws the points X
and the right-hand side b of (K + mu I) a = b (eq:Problem) with
the shapes and distributions of the paper's synthetic experiments (uniform
points in a d-cube whose edge is scaled by n^(1/d) to keep the density
constant) and of BASELINE.json's configs C1..C5.

Recipe: rng = numpy.random.default_rng(seed);
X = rng.uniform(0, edge, (n, d)) (or rng.standard_normal((n, d)) for the
regression-shaped C4), then b = rng.standard_normal(n) from the same generator.
BASELINE.json fixes b ~ N(0,1) (the paper used U[-0.5,0.5]).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    data: str                 # "cube" or "normal"
    ls: tuple                 # length-scales l (a sweep for C2, C4)
    mu: float
    k_cap: int
    k_adaptive: bool
    w: int                    # FSAI nnz per row, including the diagonal
    tol: float = 1e-4
    maxit: int = 500

    @property
    def edge(self) -> float:
        # constant density: edge 10 at n=1000, scaled by (n/1000)^(1/d)
        return 10.0 * (self.n / 1000.0) ** (1.0 / self.d)


CONFIGS = {
    "C1": Config("C1", 1000, 3, "cube", (1.0,), 1e-4, 100, False, 50),
    "C2": Config("C2", 16384, 3, "cube", (0.1, 0.5, 1.0, 2.0, 5.0, 10.0), 1e-4, 2000, True, 100),
    "C3": Config("C3", 131072, 3, "cube", (1.0,), 1e-4, 4000, True, 100),
    "C4": Config("C4", 262144, 8, "normal", (1.0, 3.0), 1e-2, 4000, True, 64),
    "C5": Config("C5", 1048576, 3, "cube", (1.0,), 1e-4, 8000, True, 100),
}


def gen_points(n: int, d: int, data: str = "cube", seed: int = 0, edge: float | None = None):
    """Return (X, rng) with X an (n, d) C-contiguous float64 array."""
    rng = np.random.default_rng(seed)
    if data == "cube":
        if edge is None:
            edge = 10.0 * (n / 1000.0) ** (1.0 / d)
        X = rng.uniform(0.0, edge, size=(n, d))
    elif data == "normal":
        X = rng.standard_normal((n, d))
    else:
        raise ValueError(f"unknown data kind {data!r}")
    return np.ascontiguousarray(X, dtype=np.float64), rng


def gen_problem(cfg: Config | str, seed: int = 0):
    """X then b from one generator."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    X, rng = gen_points(cfg.n, cfg.d, cfg.data, seed, cfg.edge if cfg.data == "cube" else None)
    b = np.ascontiguousarray(rng.standard_normal(cfg.n), dtype=np.float64)
    return X, b


def gen_small(n: int, d: int, seed: int = 0, edge: float | None = None):
    """Small uniform-cube problem of constant density (tests)."""
    X, rng = gen_points(n, d, "cube", seed, edge)
    b = rng.standard_normal(n)
    return X, np.ascontiguousarray(b)
