"""Multipatch topology, primal constraints and jump operators -- oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Interfaces / Dirichlet sides: a patch side is an interface
  side if every control point on it coincides (to 1e-10*diam) with a control
  point of one other patch; otherwise it lies on the boundary and carries the
  homogeneous Dirichlet condition of Eq. (1) (V_0 = H^1_0), its dofs are
  eliminated.
* Dof groups: active boundary dofs that coincide geometrically; multiplicity =
  group size.  Entities (vertex / edge / face) by the codimension of the dof's
  position in its patch (reading R13, O2/O4 of SURVEY Sec. 8(c)).
* Primal constraints C^(k): vertex values
  (unit row) and open-entity averages with weights w_a ~ prod int N_a
  = prod (t_{a+p+1}-t_a)/(p+1), normalised to sum 1 (R13).
* Multipliers / jump operator B: non-redundant chain per dual
  dof group, rows x_{k_i} - x_{k_{i+1}} over ascending patch ids, primal vertex
  dofs excluded, rows sorted by (k_1, flat index in k_1, i)  (R12).
* Scaled jump operator B_D ("a scaled version of the jump operator"):
  per group (B_g B_g^T)^{-1} B_g  (R12; App. A.4).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Tuple

import numpy as np
import scipy.sparse as sp
from scipy.spatial import cKDTree

from . import bspline

VERTEX, EDGE, FACE = "vertex", "edge", "face"
PRIMAL_VERTEX, PRIMAL_EDGE, PRIMAL_FACE = 1, 2, 4


def unravel(flat, M):
    """Full-lattice multi-index of a flat index (direction 1 fastest)."""
    out = []
    for Md in M:
        out.append(flat % Md)
        flat //= Md
    return tuple(out)


def ravel(idx, M):
    flat, s = 0, 1
    for i, Md in zip(idx, M):
        flat += i * s
        s *= Md
    return flat


@dataclasses.dataclass
class PatchTopo:
    M: Tuple[int, ...]
    n_full: int
    dirichlet_sides: List[Tuple[int, int]]        # (direction, 0|1)
    active: np.ndarray                            # bool [n_full]
    act_idx: np.ndarray                           # full indices of active dofs (ascending)
    full_to_act: np.ndarray                       # int [n_full], -1 if eliminated
    floating: bool
    gamma: np.ndarray                             # active-numbering indices of Gamma^(k)
    interior: np.ndarray                          # active-numbering indices of I^(k) = [1,M-2]^d


@dataclasses.dataclass
class Entity:
    kind: str
    members: Dict[int, np.ndarray]                # patch -> full indices of the open entity (sorted)
    weights: Dict[int, np.ndarray]                # patch -> constraint weights (sum 1)
    key: Tuple[int, int]                          # (k1, min flat index in k1)


class Topology:
    def __init__(self, patches, primal_mask):
        self.dim = patches[0].dim
        self.n_patches = len(patches)
        self.patches = patches
        self.primal_mask = primal_mask
        self._find_groups()
        self._sides_and_activity()
        self._entities()
        self._constraints()
        self._multipliers()

    # -- geometric identification of boundary dofs ---------------------------------------
    def _find_groups(self):
        pts, owner = [], []
        self.M = []
        for k, pa in enumerate(self.patches):
            M = pa.n_basis
            self.M.append(M)
            n = int(np.prod(M))
            for flat in range(n):
                idx = unravel(flat, M)
                if any(i == 0 or i == Md - 1 for i, Md in zip(idx, M)):
                    pts.append(pa.ctrl[flat])
                    owner.append((k, flat))
        pts = np.asarray(pts)
        diam = float(np.max(np.ptp(pts, axis=0)))
        tree = cKDTree(pts)
        pairs = tree.query_pairs(r=1e-10 * diam, output_type="ndarray")
        parent = list(range(len(pts)))

        def find(a):
            while parent[a] != a:
                parent[a] = parent[parent[a]]
                a = parent[a]
            return a

        for a, b in pairs:
            ra, rb = find(int(a)), find(int(b))
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
        groups: Dict[int, List[Tuple[int, int]]] = {}
        for i, o in enumerate(owner):
            groups.setdefault(find(i), []).append(o)
        self.geo_group_of: Dict[Tuple[int, int], Tuple] = {}
        for g in groups.values():
            g = tuple(sorted(g))
            ks = [k for k, _ in g]
            if len(set(ks)) != len(ks):
                raise ValueError("two dofs of one patch coincide geometrically")
            for o in g:
                self.geo_group_of[o] = g

    def _side_dofs(self, k, d, s):
        M = self.M[k]
        n = int(np.prod(M))
        out = []
        for flat in range(n):
            idx = unravel(flat, M)
            if idx[d] == (0 if s == 0 else M[d] - 1):
                out.append(flat)
        return out

    def _sides_and_activity(self):
        self.ptopo: List[PatchTopo] = []
        self.side_partner: Dict[Tuple[int, int, int], int] = {}
        for k in range(self.n_patches):
            M = self.M[k]
            n = int(np.prod(M))
            dsides = []
            for d in range(self.dim):
                for s in (0, 1):
                    dofs = self._side_dofs(k, d, s)
                    partners = None
                    for flat in dofs:
                        mates = {kk for kk, _ in self.geo_group_of[(k, flat)] if kk != k}
                        partners = mates if partners is None else partners & mates
                    if partners:
                        l = min(partners)
                        ldofs = [ff for kk, ff in self.geo_group_of[(k, dofs[0])] if kk == l]
                        del ldofs
                        self.side_partner[(k, d, s)] = l
                    else:
                        dsides.append((d, s))
            active = np.ones(n, dtype=bool)
            for (d, s) in dsides:
                active[self._side_dofs(k, d, s)] = False
            act_idx = np.nonzero(active)[0]
            f2a = -np.ones(n, dtype=np.int64)
            f2a[act_idx] = np.arange(len(act_idx))
            gamma, interior = [], []
            for a, flat in enumerate(act_idx):
                idx = unravel(int(flat), M)
                if any(i == 0 or i == Md - 1 for i, Md in zip(idx, M)):
                    gamma.append(a)
                else:
                    interior.append(a)
            self.ptopo.append(PatchTopo(tuple(M), n, dsides, active, act_idx, f2a, len(dsides) == 0,
                                        np.array(gamma, dtype=np.int64), np.array(interior, dtype=np.int64)))
        for k in range(self.n_patches):
            if len(self.ptopo[k].dirichlet_sides) == 2 * self.dim and self.n_patches > 1:
                raise ValueError("patch has neither interface nor ... (isolated patch)")
        # interface groups among active dofs
        seen = set()
        self.groups: List[Tuple[Tuple[int, int], ...]] = []
        for (k, flat), g in self.geo_group_of.items():
            if g in seen:
                continue
            seen.add(g)
            act = [self.ptopo[kk].active[ff] for kk, ff in g]
            if any(act) and not all(act):
                raise ValueError("non-conforming Dirichlet elimination at an interface dof")
            if all(act) and len(g) >= 2:
                self.groups.append(g)
        self.groups.sort(key=lambda g: (g[0][0], g[0][1]))

    # -- entities -------------------------------------------------------------------------
    def _subentity(self, k, flat):
        M = self.M[k]
        idx = unravel(flat, M)
        return tuple(0 if i == 0 else (1 if i == Md - 1 else -1) for i, Md in zip(idx, M))

    def _entities(self):
        ents: Dict[frozenset, List] = {}
        self.group_entity = {}
        for g in self.groups:
            subs = [(k, self._subentity(k, f)) for k, f in g]
            codims = {sum(1 for s in se if s >= 0) for _, se in subs}
            if len(codims) != 1:
                raise ValueError("non-conforming junction (entity codimension differs across patches)")
            key = frozenset(subs)
            ents.setdefault(key, []).append(g)
            self.group_entity[g] = key
        self.entities: Dict[frozenset, Entity] = {}
        for key, glist in ents.items():
            codim = sum(1 for s in next(iter(key))[1] if s >= 0)
            if self.dim == 2:
                kind = {2: VERTEX, 1: EDGE}[codim]
            else:
                kind = {3: VERTEX, 2: EDGE, 1: FACE}[codim]
            members = {}
            for g in glist:
                for k, f in g:
                    members.setdefault(k, []).append(f)
            members = {k: np.array(sorted(v), dtype=np.int64) for k, v in members.items()}
            k1 = min(members)
            weights = {k: self._avg_weights(k, members[k], key) for k in members}
            self.entities[key] = Entity(kind, members, weights, (k1, int(members[k1][0])))

    def _avg_weights(self, k, flats, key):
        """R13: w_a ~ prod over free directions of int N_a = (t_{a+p+1} - t_a)/(p+1)."""
        pa = self.patches[k]
        M = self.M[k]
        w = np.ones(len(flats))
        for j, flat in enumerate(flats):
            idx = unravel(int(flat), M)
            se = self._subentity(k, int(flat))
            for d in range(self.dim):
                if se[d] < 0:
                    t = np.asarray(pa.knots[d], dtype=np.float64)
                    p = pa.degree[d]
                    w[j] *= (t[idx[d] + p + 1] - t[idx[d]]) / (p + 1)
        return w / w.sum()

    def _is_primal(self, ent):
        return ((ent.kind == VERTEX and self.primal_mask & PRIMAL_VERTEX)
                or (ent.kind == EDGE and self.primal_mask & PRIMAL_EDGE)
                or (ent.kind == FACE and self.primal_mask & PRIMAL_FACE))

    # -- primal constraints C^(k) ---------------------------------------------
    def _constraints(self):
        prim = [e for e in self.entities.values() if self._is_primal(e)]
        prim.sort(key=lambda e: e.key)
        self.primal = prim
        self.n_pi = len(prim)
        self.C: List[sp.csr_matrix] = []
        self.R: List[np.ndarray] = []                 # local row j -> global primal id
        for k in range(self.n_patches):
            pt = self.ptopo[k]
            rows, cols, vals, gids = [], [], [], []
            for gid, e in enumerate(prim):
                if k not in e.members:
                    continue
                j = len(gids)
                gids.append(gid)
                for f, w in zip(e.members[k], e.weights[k]):
                    rows.append(j)
                    cols.append(pt.full_to_act[f])
                    vals.append(w)
            self.C.append(sp.csr_matrix((vals, (rows, cols)), shape=(len(gids), len(pt.act_idx))))
            self.R.append(np.array(gids, dtype=np.int64))

    # -- multipliers, B, B_D (R12) --------------------------------------------------------
    def _multipliers(self):
        primal_vertex_groups = set()
        for e in self.primal:
            if e.kind == VERTEX:
                for k, fl in e.members.items():
                    primal_vertex_groups.add(self.geo_group_of[(k, int(fl[0]))])
        rows = []          # (sortkey, [(k, full, coeff)], group, i)
        self.dual_groups = []
        for g in self.groups:
            if g in primal_vertex_groups:
                continue
            mem = sorted(g)                             # ascending patch ids
            self.dual_groups.append(mem)
            for i in range(len(mem) - 1):
                rows.append(((mem[0][0], mem[0][1], i), mem[i], mem[i + 1], len(self.dual_groups) - 1, i))
        rows.sort(key=lambda r: r[0])
        self.n_lambda = len(rows)
        self.mult = [(r[1][0], r[1][1], r[2][0], r[2][1]) for r in rows]   # (k+, full+, k-, full-)
        row_of = {(r[3], r[4]): idx for idx, r in enumerate(rows)}
        # B^(k) and B_D^(k), n_lambda x n_act^(k)
        Bt = [([], [], []) for _ in range(self.n_patches)]
        BDt = [([], [], []) for _ in range(self.n_patches)]
        for gi, mem in enumerate(self.dual_groups):
            m = len(mem)
            Bg = np.zeros((m - 1, m))
            for i in range(m - 1):
                Bg[i, i], Bg[i, i + 1] = 1.0, -1.0
            BDg = np.linalg.solve(Bg @ Bg.T, Bg)
            for i in range(m - 1):
                r = row_of[(gi, i)]
                for c, (k, fl) in enumerate(mem):
                    a = self.ptopo[k].full_to_act[fl]
                    if Bg[i, c] != 0.0:
                        Bt[k][0].append(r); Bt[k][1].append(a); Bt[k][2].append(Bg[i, c])
                    BDt[k][0].append(r); BDt[k][1].append(a); BDt[k][2].append(BDg[i, c])
        self.B, self.BD = [], []
        for k in range(self.n_patches):
            na = len(self.ptopo[k].act_idx)
            self.B.append(sp.csr_matrix((Bt[k][2], (Bt[k][0], Bt[k][1])), shape=(self.n_lambda, na)))
            self.BD.append(sp.csr_matrix((BDt[k][2], (BDt[k][0], BDt[k][1])), shape=(self.n_lambda, na)))

    # -- helpers --------------------------------------------------------------------------
    def n_pi_local(self, k):
        return len(self.R[k])
