"""Seeded synthetic workloads C1..C5 (BASELINE.json ``configs``) and small variants.

This module is INPUT SYNTHESIS ONLY.  It is shared by the CPU oracle (``oracle/``)
and the CUDA product path (``paper_1705_04531_b200``) and therefore holds none of
the method's arithmetic: no basis evaluation, no assembly, no multigrid, no
IETI-DP algebra.  It emits, per patch, what the C-ABI ``ieti_setup`` takes
(Sec. 2): degree, open knot vector per direction and the
physical control points P_i on the lexicographic dof lattice (direction 1
fastest), plus the problem data of Eq. (1): the right-hand side
function f as a closed form of the physical coordinates.

Geometry recipes:
  * identity maps (C1, C4): patch (a,b[,c]) -> [a/N, (a+1)/N] x ...
  * jitter (C2, C5): interior patch-grid vertices moved by U(-0.1,0.1)*H_delta
    (numpy default_rng(seed), vertices lexicographic x fastest, components in
    order), multilinear patch maps from the 2^d corners
  * quarter annulus (C3): r in [1,2], theta in [0, pi/2]; patch (a,b):
    xi -> r in [1+a/Nr.., ], eta -> theta
Control points are the map sampled at the Greville abscissae of the patch's
knot vector (exact for affine/multilinear maps; variation-diminishing for the
polar map).  Greville points are a property of the *input* parametrisation,
not of the solver.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

PRIMAL_VERTEX = 1
PRIMAL_EDGE = 2
PRIMAL_FACE = 4

LOCAL_VCYCLES = 0
LOCAL_PCG = 1
LOCAL_EXACT = 2


@dataclasses.dataclass
class Patch:
    degree: Tuple[int, ...]            # p_delta per direction
    knots: Tuple[np.ndarray, ...]      # open knot vector per direction
    ctrl: np.ndarray                   # [prod M_delta, dim], lexicographic, direction 1 fastest

    @property
    def dim(self) -> int:
        return len(self.degree)

    @property
    def n_basis(self) -> Tuple[int, ...]:
        return tuple(len(t) - p - 1 for t, p in zip(self.knots, self.degree))


@dataclasses.dataclass
class Workload:
    name: str
    dim: int
    grid: Tuple[int, ...]              # patches per direction
    p: int
    m: int                             # elements per patch per direction
    patches: List[Patch]
    primal: int                        # bitmask PRIMAL_*
    local_mode: int                    # LOCAL_VCYCLES / LOCAL_PCG / LOCAL_EXACT (Neumann solves)
    cycles: int                        # V-cycles per fixed-cycle local solve (Neumann)
    dirichlet_cycles: int              # V-cycles in the scaled Dirichlet preconditioner
    inner_tol: float                   # C2 inner PCG tolerance (R19)
    inner_maxit: int
    pcg_tol: float                     # outer dual PCG tolerance
    pcg_maxit: int
    alpha_reg: float                   # K + alpha*Mhat on floating patches
    f: Callable[[np.ndarray], np.ndarray]   # f(x) with x [..., dim] physical coordinates
    f_name: str
    u_exact: Optional[Callable[[np.ndarray], np.ndarray]] = None
    nu_pre: int = 1                    # forward / backward colour sweeps per level (R5)
    nu_post: int = 1

    @property
    def n_patches(self) -> int:
        return len(self.patches)


# ----------------------------------------------------------------------------------------
# knot vectors / Greville abscissae (input parametrisation only)
# ----------------------------------------------------------------------------------------

def open_uniform_knots(p: int, m: int) -> np.ndarray:
    """Open uniform knot vector of degree p with m elements on [0, 1]."""
    interior = [i / m for i in range(1, m)]
    return np.array([0.0] * (p + 1) + interior + [1.0] * (p + 1), dtype=np.float64)


def greville(t: np.ndarray, p: int) -> np.ndarray:
    n = len(t) - p - 1
    return np.array([t[i + 1:i + p + 1].mean() for i in range(n)], dtype=np.float64)


def _lattice_params(knots: Sequence[np.ndarray], degree: Sequence[int]) -> np.ndarray:
    """Greville parameter points on the lexicographic lattice (direction 1 fastest)."""
    g = [greville(t, p) for t, p in zip(knots, degree)]
    mesh = np.meshgrid(*g, indexing="ij")                 # mesh[d][i0, i1, ...]
    # lexicographic with direction 1 (index 0) fastest -> transpose to [i_{d-1}, ..., i_0]
    pts = np.stack([mm.transpose(tuple(range(len(g) - 1, -1, -1))).ravel() for mm in mesh], axis=-1)
    return pts


# ----------------------------------------------------------------------------------------
# right-hand sides (R16)
# ----------------------------------------------------------------------------------------

def f_sin2(x: np.ndarray) -> np.ndarray:
    return 2.0 * math.pi ** 2 * np.sin(math.pi * x[..., 0]) * np.sin(math.pi * x[..., 1])


def u_sin2(x: np.ndarray) -> np.ndarray:
    return np.sin(math.pi * x[..., 0]) * np.sin(math.pi * x[..., 1])


def f_sin3(x: np.ndarray) -> np.ndarray:
    return (3.0 * math.pi ** 2 * np.sin(math.pi * x[..., 0]) * np.sin(math.pi * x[..., 1])
            * np.sin(math.pi * x[..., 2]))


def u_sin3(x: np.ndarray) -> np.ndarray:
    return np.sin(math.pi * x[..., 0]) * np.sin(math.pi * x[..., 1]) * np.sin(math.pi * x[..., 2])


def f_one(x: np.ndarray) -> np.ndarray:
    return np.ones(x.shape[:-1])


# ----------------------------------------------------------------------------------------
# geometry builders
# ----------------------------------------------------------------------------------------

def _patch_ids(grid: Sequence[int]):
    """Patch multi-indices in patch-id order (direction 1 fastest)."""
    if len(grid) == 2:
        for b in range(grid[1]):
            for a in range(grid[0]):
                yield (a, b)
    else:
        for c in range(grid[2]):
            for b in range(grid[1]):
                for a in range(grid[0]):
                    yield (a, b, c)


def _box_patches(grid, p, m, box_map) -> List[Patch]:
    dim = len(grid)
    t = open_uniform_knots(p, m)
    knots = tuple(t.copy() for _ in range(dim))
    degree = (p,) * dim
    xi = _lattice_params(knots, degree)                   # [n, dim] in [0,1]^dim
    patches = []
    for idx in _patch_ids(grid):
        patches.append(Patch(degree=degree, knots=knots, ctrl=box_map(idx, xi)))
    return patches


def identity_patches(grid, p, m, extent=None) -> List[Patch]:
    """Affine patches of the unit square/cube (R18)."""
    dim = len(grid)
    extent = extent or (1.0,) * dim

    def box_map(idx, xi):
        out = np.empty_like(xi)
        for d in range(dim):
            h = extent[d] / grid[d]
            out[:, d] = (idx[d] + xi[:, d]) * h
        return out

    return _box_patches(grid, p, m, box_map)


def jitter_vertices(grid, seed, amp=0.1) -> np.ndarray:
    """Patch-grid vertices of the unit square/cube; interior ones jittered (R17).

    Returns V with shape (grid[0]+1, grid[1]+1[, grid[2]+1], dim) indexed [i, j(, l)].
    Vertices are visited lexicographically (x fastest), components in order.
    """
    dim = len(grid)
    rng = np.random.default_rng(seed)
    H = [1.0 / g for g in grid]
    shape = tuple(g + 1 for g in grid)
    V = np.zeros(shape + (dim,))
    ranges = [range(s) for s in shape]
    if dim == 2:
        order = [(i, j) for j in ranges[1] for i in ranges[0]]
    else:
        order = [(i, j, l) for l in ranges[2] for j in ranges[1] for i in ranges[0]]
    for v in order:
        for d in range(dim):
            V[v + (d,)] = v[d] * H[d]
        interior = all(0 < v[d] < grid[d] for d in range(dim))
        if interior:
            for d in range(dim):
                V[v + (d,)] += rng.uniform(-amp, amp) * H[d]
    return V


def jitter_patches(grid, p, m, seed, amp=0.1) -> List[Patch]:
    dim = len(grid)
    V = jitter_vertices(grid, seed, amp)

    def box_map(idx, xi):
        out = np.zeros_like(xi)
        # multilinear interpolation of the 2^dim patch corners
        for corner in range(1 << dim):
            bits = [(corner >> d) & 1 for d in range(dim)]
            w = np.ones(xi.shape[0])
            for d in range(dim):
                w = w * (xi[:, d] if bits[d] else (1.0 - xi[:, d]))
            vtx = V[tuple(idx[d] + bits[d] for d in range(dim))]
            out += w[:, None] * vtx[None, :]
        return out

    return _box_patches(grid, p, m, box_map)


def annulus_patches(grid, p, m, r0=1.0, r1=2.0) -> List[Patch]:
    """Quarter annulus (R15): patch (a,b): xi -> r, eta -> theta; polar map at Greville points."""
    nr, nth = grid

    def box_map(idx, xi):
        a, b = idx
        r = r0 + (r1 - r0) * (a + xi[:, 0]) / nr
        th = 0.5 * math.pi * (b + xi[:, 1]) / nth
        return np.stack([r * np.cos(th), r * np.sin(th)], axis=-1)

    return _box_patches(grid, p, m, box_map)


def annulus3d_patches(grid, p, m, r0=1.0, r1=2.0, height=1.0) -> List[Patch]:
    """Extruded quarter annulus (SURVEY NEXT-4 stand-in for the paper's twisted 3D domain, whose
    twist is undefined, E2): patch (a,b,c): xi -> r, eta -> theta, zeta -> z; polar map sampled at
    the Greville points as in R15."""
    nr, nth, nz = grid

    def box_map(idx, xi):
        a, b, c = idx
        r = r0 + (r1 - r0) * (a + xi[:, 0]) / nr
        th = 0.5 * math.pi * (b + xi[:, 1]) / nth
        z = height * (c + xi[:, 2]) / nz
        return np.stack([r * np.cos(th), r * np.sin(th), z], axis=-1)

    return _box_patches(grid, p, m, box_map)


# ----------------------------------------------------------------------------------------
# named configurations
# ----------------------------------------------------------------------------------------

def make_workload(name: str, m: Optional[int] = None, grid: Optional[Tuple[int, ...]] = None,
                  p: Optional[int] = None, **overrides) -> Workload:
    """Return one of C1..C5 (BASELINE.json configs[0..4]) or a named small variant.

    ``m``, ``grid`` and ``p`` override the config's elements per patch, patch grid and
    degree (used for oracle-sized parity cases with the same geometry recipe).
    """
    name = name.upper()
    common = dict(inner_tol=1e-6, inner_maxit=200, pcg_tol=1e-8, pcg_maxit=500, alpha_reg=1e-2)
    if name == "C1":
        g, pp, mm = grid or (2, 2), p or 2, m or 4
        w = Workload(name, 2, g, pp, mm, identity_patches(g, pp, mm), PRIMAL_VERTEX,
                     LOCAL_VCYCLES, 2, 2, f=f_sin2, f_name="2pi^2 sin sin", u_exact=u_sin2, **common)
    elif name == "C2":
        g, pp, mm = grid or (4, 4), p or 3, m or 64
        w = Workload(name, 2, g, pp, mm, jitter_patches(g, pp, mm, seed=2), PRIMAL_VERTEX,
                     LOCAL_PCG, 1, 2, f=f_sin2, f_name="2pi^2 sin sin", u_exact=u_sin2, **common)
    elif name == "C3":
        g, pp, mm = grid or (8, 8), p or 4, m or 128
        w = Workload(name, 2, g, pp, mm, annulus_patches(g, pp, mm), PRIMAL_VERTEX | PRIMAL_EDGE,
                     LOCAL_VCYCLES, 1, 1, f=f_sin2, f_name="2pi^2 sin sin", u_exact=None, **common)
    elif name == "C4":
        g, pp, mm = grid or (4, 4, 4), p or 2, m or 16
        w = Workload(name, 3, g, pp, mm, identity_patches(g, pp, mm), PRIMAL_VERTEX | PRIMAL_EDGE,
                     LOCAL_VCYCLES, 2, 2, f=f_sin3, f_name="3pi^2 sin sin sin", u_exact=u_sin3, **common)
    elif name == "C5":
        g, pp, mm = grid or (8, 8, 4), p or 3, m or 32
        w = Workload(name, 3, g, pp, mm, jitter_patches(g, pp, mm, seed=5),
                     PRIMAL_VERTEX | PRIMAL_EDGE | PRIMAL_FACE,
                     LOCAL_VCYCLES, 2, 2, f=f_sin3, f_name="3pi^2 sin sin sin", u_exact=u_sin3, **common)
    elif name == "E1":          # paper replica: Table 1's 8x4 quarter annulus, MG-MG
        # 4 radial x 8 angular patches: with this orientation the GPU reproduces Table 1's MG-MG
        # iteration counts (9, 10, 11 for m = 64, 128, 256; profiles/r01/paper_replica_E1_4x8.jsonl)
        g, pp, mm = grid or (4, 8), p or 2, m or 64
        w = Workload(name, 2, g, pp, mm, annulus_patches(g, pp, mm), PRIMAL_VERTEX | PRIMAL_EDGE,
                     LOCAL_PCG, 1, 2, f=f_sin2, f_name="2pi^2 sin sin", u_exact=None,
                     **dict(common, pcg_tol=1e-6, inner_tol=1e-10))
    elif name == "E2":          # 3D counterpart of Table 2 (4x4x8 patches, p = 2, edge averages only,
        g, pp, mm = grid or (4, 8, 4), p or 2, m or 8          # MG-MG), untwisted (twist undefined)
        w = Workload(name, 3, g, pp, mm, annulus3d_patches(g, pp, mm), PRIMAL_EDGE,
                     LOCAL_PCG, 1, 2, f=f_sin3, f_name="3pi^2 sin sin sin", u_exact=None,
                     **dict(common, pcg_tol=1e-6, inner_tol=1e-10))
    elif name == "STRIP":       # 1x2 strip: no interior vertex -> n_Pi = 0 (pure FETI)
        g, pp, mm = grid or (2, 1), p or 2, m or 4
        w = Workload(name, 2, g, pp, mm, identity_patches(g, pp, mm, extent=(1.0, 0.5)), PRIMAL_VERTEX,
                     LOCAL_VCYCLES, 2, 2, f=f_one, f_name="1", **common)
    elif name == "SINGLE":      # single all-Dirichlet patch
        g, pp, mm = grid or (1, 1), p or 2, m or 4
        w = Workload(name, 2, g, pp, mm, identity_patches(g, pp, mm), PRIMAL_VERTEX,
                     LOCAL_VCYCLES, 2, 2, f=f_sin2, f_name="2pi^2 sin sin", u_exact=u_sin2, **common)
    else:
        raise ValueError(f"unknown workload {name}")
    for k, v in overrides.items():
        setattr(w, k, v)
    return w


CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5")
