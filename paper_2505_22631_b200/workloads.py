"""Synthetic graphs of the BASELINE.json config shapes.

The GSET / SATLIB instance files are not shipped with the reference
(/root/reference/pkg/README.md:99-103) and there is no network, so every benchmark and
parity workload is a seeded synthetic graph of the stated shape.
All generators return canonical edge arrays (u < v, lexicographically sorted, int64) plus
float64 weights, i.e. exactly what `Graph(n, u, v, w)` stores.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

EdgeArrays = Tuple[np.ndarray, np.ndarray, np.ndarray]

# name -> (n, m) of the shapes named in BASELINE.json "configs"
SHAPES = {
    "G1": (800, 19176),
    "G22": (2000, 19990),
    "flat200": (200, 479),
    "G81": (20000, 40000),
    "SK16384": (16384, 16384 * 16383 // 2),
}


def _unrank_pairs(k: np.ndarray, n: int) -> Tuple[np.ndarray, np.ndarray]:
    """Map ranks 0..n(n-1)/2-1 to pairs (u < v) in lexicographic order."""
    k = k.astype(np.int64)
    # row u starts at offset u*n - u*(u+1)/2 ; solve with a float guess then fix up
    b = 2 * n - 1
    u = np.floor((b - np.sqrt(np.maximum(b * b - 8.0 * k, 0.0))) / 2.0).astype(np.int64)
    start = u * n - u * (u + 1) // 2
    u = np.where(start > k, u - 1, u)
    start = u * n - u * (u + 1) // 2
    nxt = (u + 1) * n - (u + 1) * (u + 2) // 2
    u = np.where(k >= nxt, u + 1, u)
    start = u * n - u * (u + 1) // 2
    v = k - start + u + 1
    return u, v


def random_gnm(n: int, m: int, seed: int, weights=(1.0,)) -> EdgeArrays:
    """Uniform random simple graph G(n, m); weights drawn i.i.d. from `weights`."""
    total = n * (n - 1) // 2
    if m > total:
        raise ValueError("too many edges")
    rng = np.random.default_rng(seed)
    ranks = np.sort(rng.choice(total, size=m, replace=False))
    u, v = _unrank_pairs(ranks, n)
    w = rng.choice(np.asarray(weights, dtype=np.float64), size=m) if len(weights) > 1 else np.full(m, float(weights[0]))
    return u, v, w


def gset_like(name: str) -> EdgeArrays:
    """G1 / G22 shapes: G(n, m) with unit weights; graph seed = the GSET number."""
    n, m = SHAPES[name]
    return random_gnm(n, m, seed=int(name[1:]))


def torus_pm1(rows: int = 100, cols: int = 200, seed: int = 81) -> EdgeArrays:
    """G81 shape: rows x cols periodic grid (4-regular), weights +-1 i.i.d."""
    n = rows * cols
    idx = np.arange(n, dtype=np.int64).reshape(rows, cols)
    right = np.roll(idx, -1, axis=1)
    down = np.roll(idx, -1, axis=0)
    a = np.concatenate([idx.ravel(), idx.ravel()])
    b = np.concatenate([right.ravel(), down.ravel()])
    u, v = np.minimum(a, b), np.maximum(a, b)
    order = np.lexsort((v, u))
    u, v = u[order], v[order]
    keep = np.ones(len(u), dtype=bool)
    keep[1:] = (u[1:] != u[:-1]) | (v[1:] != v[:-1])
    keep &= u != v
    u, v = u[keep], v[keep]
    w = np.random.default_rng(seed).choice(np.array([-1.0, 1.0]), size=len(u))
    return u, v, w


def planted_coloring(n: int = 200, m: int = 479, n_colors: int = 3, seed: int = 0) -> EdgeArrays:
    """flat200-479 shape: m unit edges drawn uniformly from the cross-group pairs of the
    planted colouring `i mod n_colors` (same construction as the reference's
    generate_colorable_graph, problems.py:255-276)."""
    if n_colors < 2 or n < n_colors:
        raise ValueError("bad colouring shape")
    total = n * (n - 1) // 2
    u, v = _unrank_pairs(np.arange(total, dtype=np.int64), n)
    cross = (u % n_colors) != (v % n_colors)
    u, v = u[cross], v[cross]
    if m > len(u):
        raise ValueError("m exceeds the available cross-group pairs")
    pick = np.sort(np.random.default_rng(seed).choice(len(u), size=m, replace=False))
    return u[pick], v[pick], np.ones(m)


def sk_dense(n: int, seed: int | None = None) -> np.ndarray:
    """Dense symmetric +-1 Sherrington-Kirkpatrick couplings, zero diagonal, as int8 [n, n]."""
    rng = np.random.default_rng(n if seed is None else seed)
    J = np.zeros((n, n), dtype=np.int8)
    block = 2048
    for r0 in range(0, n, block):
        r1 = min(n, r0 + block)
        bits = rng.integers(0, 2, size=(r1 - r0, n), dtype=np.int8)
        J[r0:r1] = 2 * bits - 1
    J = np.triu(J, 1)
    J = J + J.T
    return J


def shape_graph(name: str) -> Tuple[int, EdgeArrays, int, str]:
    """(n, edges, n_states, objective) for a BASELINE.json config name."""
    if name in ("G1", "G22"):
        return SHAPES[name][0], gset_like(name), 2, "maxcut"
    if name == "G81":
        return SHAPES[name][0], torus_pm1(), 2, "maxcut"
    if name == "flat200":
        return SHAPES[name][0], planted_coloring(), 3, "coloring"
    raise KeyError(name)
