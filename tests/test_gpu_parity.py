"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerances: building blocks (stencils, V-cycles, F^, M_sD, Phibar)
1e-11 relative (fp64 with different summation order, O(1e-14) per operation, amplified
mildly by the V-cycle); end-to-end u and lambda after a fixed iteration count <= 1e-9
relative l2 (north star); converged iteration counts +-1 at tol 1e-8 (north star).
"""
import numpy as np
import pytest

from oracle.ieti import IetiOracle
from tests.conftest import parity_log
from workloads import make_workload

pytestmark = pytest.mark.gpu

CASES = {
    "C1": dict(),
    "C4s": dict(m=4, grid=(3, 2, 2)),            # 3D p=2 V+E, identity, 2 levels
    "C3s": dict(m=8, grid=(4, 3)),               # annulus p=4 V+E
    "C5s": dict(m=4, grid=(3, 2, 2)),            # 3D p=3 jitter V+E+F
    "C2v": dict(m=8, grid=(3, 3)),               # 2D p=3 jitter, fixed-cycle variant (R2 alt.)
    "C2s": dict(m=16, grid=(3, 3)),              # 2D p=3 jitter, inner MG-PCG local solves (R19)
}
# C4's full per-patch size (18^3 dofs, 216 rows per colour = a full 128-row block + a ragged tail)
LARGE = ("C4", dict(m=16, grid=(3, 2, 2)))


def base(name):
    return {"C4s": "C4", "C3s": "C3", "C5s": "C5", "C2v": "C2", "C2s": "C2"}.get(name, name)


_cache = {}


def systems(name):
    if name in _cache:
        return _cache[name]
    import paper_1705_04531_b200 as lib
    kw = CASES[name]
    wl = make_workload(base(name), **kw)
    if name == "C2v":
        wl.local_mode, wl.cycles, wl.dirichlet_cycles = 0, 2, 2
    orc = IetiOracle(wl)
    gpu = lib.Ieti.from_workload(wl)
    _cache[name] = (wl, orc, gpu)
    return _cache[name]


def lat_offsets(orc):
    offs = [0]
    for pt in orc.topo.ptopo:
        offs.append(offs[-1] + pt.n_full)
    return offs


def act_to_lat(orc, vecs):
    out = np.zeros(lat_offsets(orc)[-1])
    offs = lat_offsets(orc)
    for k, v in enumerate(vecs):
        out[offs[k] + orc.topo.ptopo[k].act_idx] = v
    return out


def lat_to_act(orc, lat):
    offs = lat_offsets(orc)
    return [lat[offs[k] + pt.act_idx] for k, pt in enumerate(orc.topo.ptopo)]


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def column_mask(M, mask, p, dim):
    """[rows][(2p+1)^d] True where the column a+o is an active dof of the grid."""
    act = np.nonzero(mask)[0]
    W1 = 2 * p + 1
    offs = np.array([(o0, o1, o2) for o2 in (range(-p, p + 1) if dim == 3 else [0])
                     for o1 in range(-p, p + 1) for o0 in range(-p, p + 1)])
    i0, i1 = act % M[0], (act // M[0]) % M[1]
    i2 = act // (M[0] * M[1]) if dim == 3 else np.zeros_like(act)
    j0, j1, j2 = i0[:, None] + offs[None, :, 0], i1[:, None] + offs[None, :, 1], i2[:, None] + offs[None, :, 2]
    inb = (j0 >= 0) & (j0 < M[0]) & (j1 >= 0) & (j1 < M[1])
    if dim == 3:
        inb &= (j2 >= 0) & (j2 < M[2])
    flat = np.where(inb, j0 + M[0] * (j1 + (M[1] * j2 if dim == 3 else 0)), 0)
    return inb & mask[flat]


def oracle_stencil(A, M, mask, p, dim):
    """Active-row stencil [rows][(2p+1)^d] of a per-patch level matrix (oracle CSR over active dofs)."""
    act = np.nonzero(mask)[0]
    pos = -np.ones(len(mask), dtype=np.int64)
    pos[act] = np.arange(len(act))
    W1 = 2 * p + 1
    S = W1 ** dim
    out = np.zeros((len(act), S))
    A = A.tocsr()
    strides = [1, M[0], M[0] * (M[1] if dim > 1 else 1)]
    for r, flat in enumerate(act):
        i = [flat % M[0], (flat // M[0]) % M[1], flat // (M[0] * M[1]) if dim == 3 else 0]
        for idx in range(A.indptr[r], A.indptr[r + 1]):
            cflat = act[A.indices[idx]]
            j = [cflat % M[0], (cflat // M[0]) % M[1], cflat // (M[0] * M[1]) if dim == 3 else 0]
            o = [j[d] - i[d] + p for d in range(dim)]
            oi = o[0] + W1 * o[1] + (W1 * W1 * o[2] if dim == 3 else 0)
            out[r, oi] = A.data[idx]
    return out


@pytest.mark.parametrize("name", list(CASES))
def test_counts_match(name):
    wl, orc, gpu = systems(name)
    assert gpu.n_lambda == orc.topo.n_lambda
    assert gpu.n_pi == orc.topo.n_pi
    assert gpu.levels == orc.L
    kp, ap, km, am = gpu.multiplier_map()
    ref = np.array(orc.topo.mult)
    assert np.array_equal(kp, ref[:, 0]) and np.array_equal(ap, ref[:, 1])
    assert np.array_equal(km, ref[:, 2]) and np.array_equal(am, ref[:, 3])


@pytest.mark.parametrize("name", list(CASES))
def test_stencils_all_levels(name):
    wl, orc, gpu = systems(name)
    for hier, H, levs in ((0, orc.HN, orc.levN), (1, orc.HD, orc.levD)):
        for l in range(orc.L):
            sizes = [int(lv.mask[l].sum()) for lv in levs]
            off = np.cumsum([0] + sizes)
            for k in range(orc.topo.n_patches):
                blk = H.A[l][off[k]:off[k + 1]][:, off[k]:off[k + 1]]
                ref = oracle_stencil(blk, levs[k].M[l], levs[k].mask[l], wl.p, wl.dim)
                got = gpu.stencil(hier, l, k)
                if hier == 1 and l == orc.L - 1:
                    # Dirichlet fine rows keep the true-K Gamma columns (used for K_IG v): compare the
                    # K_II part only
                    got = np.where(column_mask(levs[k].M[l], levs[k].mask[l], wl.p, wl.dim), got, 0.0)
                scale = np.abs(ref).max()
                assert np.abs(got - ref).max() <= 1e-12 * scale, (hier, l, k)


@pytest.mark.parametrize("name", list(CASES))
def test_vcycle_and_local_solves(name):
    wl, orc, gpu = systems(name)
    import paper_1705_04531_b200 as lib
    rng = np.random.default_rng(7)
    q = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
    if wl.local_mode == 1:
        # inner PCG on the singular K of floating patches needs a consistent rhs (1^T q = 0)
        q = [v - v.mean() if pt.floating else v for v, pt in zip(q, orc.topo.ptopo)]
    got = lat_to_act(orc, gpu.apply(lib.OP_VCYCLE_N, act_to_lat(orc, q)))
    ref = orc._split(orc.HN.apply_cycles(orc._stack(q), 1), orc.offN)
    assert rel(np.concatenate(got), np.concatenate(ref)) <= 1e-11
    got = lat_to_act(orc, gpu.apply(lib.OP_NEUMANN, act_to_lat(orc, q)))
    ref = orc.local_neumann(q)
    # c V-cycles: 1e-11; C2's inner PCG (R19, ~13 Krylov steps on the singular floating K) amplifies
    # the summation-order differences further: 1e-10
    assert rel(np.concatenate(got), np.concatenate(ref)) <= (1e-10 if wl.local_mode == 1 else 1e-11)
    # Dirichlet hierarchy: interior vectors
    s = [rng.standard_normal(len(pt.interior)) for pt in orc.topo.ptopo]
    full = []
    for k, pt in enumerate(orc.topo.ptopo):
        v = np.zeros(len(pt.act_idx))
        v[pt.interior] = s[k]
        full.append(v)
    gl = lat_to_act(orc, gpu.apply(lib.OP_DIRICHLET, act_to_lat(orc, full)))
    got = [g[pt.interior] for g, pt in zip(gl, orc.topo.ptopo)]
    ref = orc.local_dirichlet(s)
    assert rel(np.concatenate(got), np.concatenate(ref)) <= 1e-11


@pytest.mark.parametrize("name", list(CASES))
def test_primal_basis(name):
    wl, orc, gpu = systems(name)
    for k, pt in enumerate(orc.topo.ptopo):
        Phi = gpu.primal_basis(k, pt.n_full)
        if Phi.shape[0] == 0:
            continue
        got = Phi[:, pt.act_idx].T
        assert rel(got, orc.Phi[k]) <= 1e-10, k


@pytest.mark.parametrize("name", list(CASES))
def test_operators_F_MsD_d(name):
    wl, orc, gpu = systems(name)
    import paper_1705_04531_b200 as lib
    rng = np.random.default_rng(3)
    lam = rng.standard_normal(orc.topo.n_lambda)
    assert rel(gpu.apply(lib.OP_F, lam), orc.apply_F(lam)) <= 1e-11
    assert rel(gpu.apply(lib.OP_MSD, lam), orc.apply_MsD(lam)) <= 1e-11
    # d^ and Ktilde^-1 read the FULL primal basis, which the product iterates to the paper's
    # primal-basis tolerance 1e-12 (the oracle's is exact): they inherit Phibar's 1e-10 bar
    # (test_primal_basis), while F^ touches only Phibar_Gamma and stays at 1e-11
    rhs = act_to_lat(orc, orc.f)
    assert rel(gpu.apply(lib.OP_D, rhs), orc.rhs_d()) <= 1e-10
    r = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
    got = lat_to_act(orc, gpu.apply(lib.OP_KTINV, act_to_lat(orc, r)))
    assert rel(np.concatenate(got), np.concatenate(orc.ktilde_inv(r))) <= 1e-10


@pytest.mark.parametrize("name", list(CASES))
def test_load_vector(name):
    wl, orc, gpu = systems(name)
    import paper_1705_04531_b200 as lib
    fid = {2: lib.F_SIN2, 3: lib.F_SIN3}[wl.dim]
    got = lat_to_act(orc, gpu.load_builtin(fid))
    assert rel(np.concatenate(got), np.concatenate(orc.f)) <= 1e-12


def kernel_basis(orc):
    """Orthonormal basis of ker F when averages are primal (App. A.3 of SURVEY.md; R14):
    for every averaged entity e and chain link (k_i, k_{i+1}) of its patches, lambda_r = w_a on the
    rows r = (k_i, a) - (k_{i+1}, a), a in e."""
    T = orc.topo
    row_of = {(kp, fp, km): r for r, (kp, fp, km, fm) in enumerate(T.mult)}
    vecs = []
    for e in T.primal:
        if e.kind == "vertex":
            continue
        ks = sorted(e.members)
        for k1, k2 in zip(ks[:-1], ks[1:]):
            v = np.zeros(T.n_lambda)
            for a, w in zip(e.members[k1], e.weights[k1]):
                v[row_of[(k1, int(a), k2)]] = w
            vecs.append(v)
    if not vecs:
        return np.zeros((T.n_lambda, 0))
    Q, _ = np.linalg.qr(np.column_stack(vecs))
    return Q


def oracle_self_sensitivity(orc, kfix, proj):
    """R26: the oracle's own spread in lambda (on range F) after kfix iterations when (a) its load is
    perturbed by 1e-14 or (b) the output of every d^ / F^ / M_sD application by 1e-14 (seeded; a
    rounding-level change of summation order in each application, as in tools/oracle_dump.py)."""
    f0 = [f.copy() for f in orc.f]
    base = orc.solve(fixed_iters=kfix).lam
    spread = 0.0
    for seed in (11, 12):
        rng = np.random.default_rng(seed)
        orc.f = [f * (1.0 + 1e-14 * rng.standard_normal(f.shape)) for f in f0]
        spread = max(spread, rel(proj(orc.solve(fixed_iters=kfix).lam), proj(base)))
    orc.f = f0
    ops = {nm: getattr(orc, nm) for nm in ("apply_F", "apply_MsD", "rhs_d")}
    for seed in (31, 32):
        rng = np.random.default_rng(seed)
        for nm, fn in ops.items():
            setattr(orc, nm, (lambda fn: lambda *a: (lambda v: v * (1.0 + 1e-14 * rng.standard_normal(v.shape)))(fn(*a)))(fn))
        spread = max(spread, rel(proj(orc.solve(fixed_iters=kfix).lam), proj(base)))
    for nm in ops:
        delattr(orc, nm)
    return spread


@pytest.mark.parametrize("name", list(CASES))
def test_kernel_of_F(name):
    """The predicted kernel (App. A.3) is a kernel of the GPU's inexact F^ (validity of the non-unique part)."""
    wl, orc, gpu = systems(name)
    import paper_1705_04531_b200 as lib
    Q = kernel_basis(orc)
    if Q.shape[1] == 0:
        pytest.skip("no averaged primal entities")
    lam = np.random.default_rng(5).standard_normal(orc.topo.n_lambda)
    scale = np.linalg.norm(gpu.apply(lib.OP_F, lam))
    for j in range(Q.shape[1]):
        assert np.linalg.norm(gpu.apply(lib.OP_F, Q[:, j])) <= 1e-10 * scale


@pytest.mark.parametrize("name", list(CASES))
def test_solve_parity(name):
    """North star: +-1 iteration at tol 1e-8; <= 1e-9 relative l2 in u and lambda after k_fix iterations (R20)."""
    wl, orc, gpu = systems(name)
    rhs = act_to_lat(orc, orc.f)
    ref = orc.solve(tol=1e-8)
    u, lam, its, rr, rc = gpu.solve(rhs)
    assert abs(its - ref.iters) <= 1, (its, ref.iters)
    kfix = ref.iters
    ref_fix = orc.solve(fixed_iters=kfix)
    uf, lf, _ = gpu.solve_fixed(rhs, kfix)
    uref = np.concatenate(ref_fix.u)
    assert rel(uf, uref) <= 1e-9
    # lambda is unique only modulo ker F when averages are primal (R14): compare the part on range F
    # at the north star's 1e-9 -- unless the oracle itself is not reproducible to that level: when
    # its own lambda moves by more than 1e-9/8 under a 1e-14 (relative, seeded) load perturbation,
    # no implementation with a different summation order can meet 1e-9, and the bar becomes 8x that
    # measured spread (R26; only C3s needs it: p = 4, one V-cycle, ~1e5 rounding amplification).
    Q = kernel_basis(orc)
    proj = lambda v: v - Q @ (Q.T @ v)
    err_u, err_lam = rel(uf, uref), rel(proj(lf), proj(ref_fix.lam))
    sens = oracle_self_sensitivity(orc, kfix, proj)
    tol_lam = max(1e-9, 8 * sens)
    parity_log(test="solve_parity", case=name, iters_gpu=its, iters_oracle=ref.iters, err_u=err_u,
               err_lam_range=err_lam, err_lam_raw=rel(lf, ref_fix.lam), oracle_self_sensitivity=sens,
               tol_lam=tol_lam, r26_used=bool(tol_lam > 1e-9))
    assert err_lam <= tol_lam
    # u is continuous up to the PCG tolerance
    assert orc.continuity_residual([uf[a:b] for a, b in zip(lat_offsets(orc)[:-1], lat_offsets(orc)[1:])]) <= 1e-6


def test_inner_pcg_counts_match_oracle():
    """C2 (R19): the per-patch inner PCG iteration counts of every local solve call match the oracle's."""
    wl, orc, gpu = systems("C2s")
    rhs = act_to_lat(orc, orc.f)
    kfix = 4
    ref = orc.solve(fixed_iters=kfix)
    gpu.solve_fixed(rhs, kfix)
    got = gpu.inner_log()
    want = np.array(ref.inner_iters)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.array_equal(got, want), np.argwhere(got != want)[:10]
    assert want.max() >= 3          # the inner solves really iterate


@pytest.mark.parametrize("name", ["C4s", "C2v"])
def test_fused_vcycle_option(name, monkeypatch):
    """The opt-in fused small-level V-cycle (IETI_FUSE=1, one cluster launch per V-cycle) computes
    the same N_c, D_c and end-to-end solution as the oracle."""
    import paper_1705_04531_b200 as lib
    wl, orc, _ = systems(name)
    monkeypatch.setenv("IETI_FUSE", "1")
    gpu = lib.Ieti.from_workload(wl)
    rng = np.random.default_rng(7)
    q = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
    got = lat_to_act(orc, gpu.apply(lib.OP_NEUMANN, act_to_lat(orc, q)))
    assert rel(np.concatenate(got), np.concatenate(orc.local_neumann(q))) <= 1e-11
    rhs = act_to_lat(orc, orc.f)
    ref = orc.solve(tol=1e-8)
    u, lam, its, rr, rc = gpu.solve(rhs)
    assert abs(its - ref.iters) <= 1
    fix = orc.solve(fixed_iters=ref.iters)
    uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
    assert rel(uf, np.concatenate(fix.u)) <= 1e-9
    gpu.close()


def test_user_load_matches_oracle_assembly():
    """ieti_quadrature_points + ieti_assemble_load (Eq. (1) load for a user f) against the oracle's
    element-by-element load, on a jittered 3D case (curved Jacobians) and the annulus."""
    import paper_1705_04531_b200 as lib
    from oracle import assembly
    f = lambda x: 1.0 + x[..., 0] ** 2 - 0.5 * x[..., 1] * (x[..., 2] if x.shape[-1] == 3 else 1.0)
    for name in ("C5s", "C3s"):
        wl, orc, gpu = systems(name)
        got = gpu.load(f)
        offs = lat_offsets(orc)
        for k, pa in enumerate(wl.patches):
            _, ref = assembly.assemble_patch(pa, f)
            ref = ref.copy()
            ref[~orc.topo.ptopo[k].active] = 0.0
            g = got[offs[k]:offs[k + 1]]
            assert np.abs(g - ref).max() <= 1e-12 * np.abs(ref).max(), (name, k)
        # the workload's own f through the user path equals the oracle's load (and the built-in path)
        fb = wl.f
        got_f = lat_to_act(orc, gpu.load(fb))
        assert rel(np.concatenate(got_f), np.concatenate(orc.f)) <= 1e-12, name
        fid = lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3
        assert rel(np.concatenate(got_f), np.concatenate(lat_to_act(orc, gpu.load_builtin(fid)))) <= 1e-12, name


def test_accurate_local_solves_next1():
    """SURVEY NEXT-1 (the paper's MG-MG): Neumann solves by MG-PCG to 1e-10 inside F^, d^
    and the recovery. Parity with the oracle's inner-PCG mode, and the outer iteration count stays
    within one of the oracle's exact (direct local solves) count."""
    import paper_1705_04531_b200 as lib
    wl = make_workload("C4", m=8, grid=(3, 2, 2))   # (2,2,2) is degenerate: d^ = 0 by symmetry
    wl.local_mode, wl.inner_tol = 1, 1e-10
    orc = IetiOracle(wl)
    gpu = lib.Ieti.from_workload(wl)
    rhs = act_to_lat(orc, orc.f)
    ref = orc.solve(tol=1e-8)
    u, lam, its, rr, rc = gpu.solve(rhs)
    assert abs(its - ref.iters) <= 1
    exact = IetiOracle(wl, neumann="exact", dirichlet="vcycle").solve(tol=1e-8)
    assert abs(its - exact.iters) <= 1, (its, exact.iters)
    fix = orc.solve(fixed_iters=ref.iters)
    uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
    assert rel(uf, np.concatenate(fix.u)) <= 1e-9
    gpu.close()


@pytest.mark.parametrize("tpr", ["default", "1"])
def test_cycle_boundary_modes_match_full_sweeps(tpr, monkeypatch):
    """Modes 6/7 (the backward sweep records the higher-colour sums U, the next cycle's forward
    sweep streams only lower-colour coefficients) equal the plain full sweeps (IETI_USWEEP=0) up
    to summation order, on both stencil layouts, for N_c and D_c (c = 2) and the whole solve."""
    import paper_1705_04531_b200 as lib
    wl, orc, _ = systems("C4s")
    if tpr != "default":
        monkeypatch.setenv("IETI_TPR", tpr)
    res = {}
    rng = np.random.default_rng(5)
    q = rng.standard_normal(sum(pt.n_full for pt in orc.topo.ptopo))
    for sw in ("1", "0"):
        monkeypatch.setenv("IETI_USWEEP", sw)
        gpu = lib.Ieti.from_workload(wl)
        res[sw] = (gpu.apply(lib.OP_NEUMANN, q), gpu.apply(lib.OP_DIRICHLET, q),
                   gpu.solve_fixed(act_to_lat(orc, orc.f), 10)[0])
        gpu.close()
    for a, b in zip(res["1"], res["0"]):
        assert rel(a, b) <= 1e-12


@pytest.mark.parametrize("name,kw", [("C4", dict(m=8, grid=(3, 2, 2))), ("C3", dict(m=16, grid=(3, 2)))])
def test_exact_variants_next3(name, kw):
    """SURVEY NEXT-3 (the paper's D-D and MG-D): local solves to machine accuracy by MG-PCG
    (R27: LOCAL_PCG and DIRICHLET_PCG at 1e-12 stand in for the paper's direct solvers).
    (a) the Dirichlet PCG equals K_II^{-1} (oracle sparse LU) to 1e-10;
    (b) D-D and MG-D solve parity with the oracle's exact modes: iterations +-1, u and lambda after a
        fixed iteration count to 1e-8 (the inner tolerance 1e-12, amplified by the outer Krylov steps);
    (c) the variants agree on the solution (1e-5 at outer tolerance 1e-8).  The paper's
        iteration agreement MG-D = D-D +-1 needs its p-robust smoother and large m; with our
        Gauss-Seidel smoother it holds on the E1 / E2 replicas, not on these tiny
        p = 2 / p = 4 cases (D-D 7 vs MG-D 9 / 16 iterations)."""
    import paper_1705_04531_b200 as lib
    wl = make_workload(name, **kw)
    wl.local_mode, wl.inner_tol, wl.inner_maxit = 1, 1e-12, 500
    rng = np.random.default_rng(7)
    gpus = {}
    gpus["DD"] = lib.Ieti.from_workload(wl, dirichlet_mode=lib.DIRICHLET_PCG, dirichlet_tol=1e-12)
    gpus["MGD"] = lib.Ieti.from_workload(wl)
    orcs = {"DD": IetiOracle(wl, neumann="exact", dirichlet="exact"),
            "MGD": IetiOracle(wl, neumann="exact", dirichlet="vcycle")}
    # (a) Dirichlet solve
    orc, gpu = orcs["DD"], gpus["DD"]
    s = [rng.standard_normal(len(pt.interior)) for pt in orc.topo.ptopo]
    full = []
    for k, pt in enumerate(orc.topo.ptopo):
        v = np.zeros(len(pt.act_idx))
        v[pt.interior] = s[k]
        full.append(v)
    gl = lat_to_act(orc, gpu.apply(lib.OP_DIRICHLET, act_to_lat(orc, full)))
    got = [g[pt.interior] for g, pt in zip(gl, orc.topo.ptopo)]
    assert rel(np.concatenate(got), np.concatenate(orc.local_dirichlet(s))) <= 1e-10
    r = rng.standard_normal(orc.topo.n_lambda)
    assert rel(gpu.apply(lib.OP_MSD, r), orc.apply_MsD(r)) <= 1e-10
    # (b) solve parity per variant
    rhs = act_to_lat(orc, orc.f)
    its, us = {}, {}
    for v in ("DD", "MGD"):
        ref = orcs[v].solve(tol=1e-8)
        us[v], lam, its[v], rr, rc = gpus[v].solve(rhs)
        assert rc == lib.OK and abs(its[v] - ref.iters) <= 1, (v, its[v], ref.iters)
        fix = orcs[v].solve(fixed_iters=ref.iters)
        uf, lf, _ = gpus[v].solve_fixed(rhs, ref.iters)
        assert rel(uf, np.concatenate(fix.u)) <= 1e-8, v
        assert rel(lf, fix.lam) <= 1e-8, v
    # (c) variant agreement on the GPU (MG-MG = inner PCG 1e-10, 2 Dirichlet V-cycles)
    wl.inner_tol = 1e-10
    mgmg = lib.Ieti.from_workload(wl)
    u_mgmg = mgmg.solve(rhs)[0]
    assert rel(us["MGD"], us["DD"]) <= 1e-5 and rel(u_mgmg, us["DD"]) <= 1e-5
    for g in list(gpus.values()) + [mgmg]:
        g.close()


_large = {}


def large_system():
    if "orc" not in _large:
        wl = make_workload(LARGE[0], **LARGE[1])
        _large["wl"], _large["orc"] = wl, IetiOracle(wl)
    return _large["wl"], _large["orc"]


@pytest.mark.parametrize("tpr", ["default", "1", "1split1", "1split2"])
def test_large_patches_both_kernel_paths(tpr, monkeypatch):
    """Full C4 patch size, several blocks per colour with a ragged tail, on both stencil paths:
    row-major rows with 4 threads per row (default for this size) and the offset-major
    one-thread-per-row path used on C5's finest level (IETI_TPR=1)."""
    import paper_1705_04531_b200 as lib
    wl, orc = large_system()
    if tpr != "default":
        monkeypatch.setenv("IETI_TPR", tpr[0])
    if "split" in tpr:                   # two warps per row group (k_stencil_split, 8- / 4-deep batches)
        monkeypatch.setenv("IETI_SPLIT", tpr[-1])
    gpu = lib.Ieti.from_workload(wl)
    rng = np.random.default_rng(9)
    q = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
    got = lat_to_act(orc, gpu.apply(lib.OP_NEUMANN, act_to_lat(orc, q)))
    assert rel(np.concatenate(got), np.concatenate(orc.local_neumann(q))) <= 1e-11
    lam = rng.standard_normal(orc.topo.n_lambda)
    assert rel(gpu.apply(lib.OP_F, lam), orc.apply_F(lam)) <= 1e-11
    assert rel(gpu.apply(lib.OP_MSD, lam), orc.apply_MsD(lam)) <= 1e-11
    rhs = act_to_lat(orc, orc.f)
    ref = orc.solve(tol=1e-8)
    u, lm, its, rr, rc = gpu.solve(rhs)
    assert abs(its - ref.iters) <= 1
    fix = orc.solve(fixed_iters=ref.iters)
    uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
    assert rel(uf, np.concatenate(fix.u)) <= 1e-9
    gpu.close()


def test_nccl_path_one_rank(monkeypatch):
    """IETI_NCCL_SELFTEST=1: the reductions of the multi-GPU path (dot-product allgathers, the
    coarse right-hand-side allgather, the S_PiPi allreduce) run through a 1-rank NCCL
    communicator captured into the PCG graphs; results equal the oracle's."""
    import paper_1705_04531_b200 as lib
    wl, orc, _ = systems("C4s")
    monkeypatch.setenv("IETI_NCCL_SELFTEST", "1")
    gpu = lib.Ieti.from_workload(wl)
    rhs = act_to_lat(orc, orc.f)
    ref = orc.solve(tol=1e-8)
    u, lam, its, rr, rc = gpu.solve(rhs)
    assert abs(its - ref.iters) <= 1
    fix = orc.solve(fixed_iters=ref.iters)
    uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
    assert rel(uf, np.concatenate(fix.u)) <= 1e-9
    gpu.close()


def test_tma_stencil_variant(monkeypatch):
    """The opt-in TMA-fed finest-level stencil kernel (IETI_STENCIL=tma: cp.async.bulk coefficient
    slabs into an mbarrier ring) computes the same N_c, F^ and solution as the oracle."""
    import paper_1705_04531_b200 as lib
    wl, orc = large_system()
    monkeypatch.setenv("IETI_TPR", "1")
    monkeypatch.setenv("IETI_STENCIL", "tma")
    gpu = lib.Ieti.from_workload(wl)
    rng = np.random.default_rng(10)
    q = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
    got = lat_to_act(orc, gpu.apply(lib.OP_NEUMANN, act_to_lat(orc, q)))
    assert rel(np.concatenate(got), np.concatenate(orc.local_neumann(q))) <= 1e-11
    lam = rng.standard_normal(orc.topo.n_lambda)
    assert rel(gpu.apply(lib.OP_F, lam), orc.apply_F(lam)) <= 1e-11
    gpu.close()


@pytest.mark.parametrize("name", ["C4s", "C5s"])
def test_multirank_loopback_matches_one_rank(name, monkeypatch):
    """The multi-GPU device path on one GPU: two ranks in one process (IETI_LOOPBACK=1, one host
    thread each) run the partitioned operators -- localized topology, pack / unpack / ordered
    reverse sums of the exchange plan, the coarse right-hand-side allgather, the global S_PiPi --
    with device copies ordered by a host barrier in place of NCCL (no kernel waits on another
    rank). F^, M_sD and d^ on the owned multipliers equal the one-rank results."""
    import threading
    import paper_1705_04531_b200 as lib
    wl, orc, one = systems(name)
    n = wl.n_patches
    owner = [k % 2 for k in range(n)]                # non-contiguous ownership, cut m=4 edges
    rng = np.random.default_rng(21)
    lam = rng.standard_normal(orc.topo.n_lambda)
    rhs = act_to_lat(orc, orc.f)
    offs = lat_offsets(orc)
    ref = {lib.OP_F: one.apply(lib.OP_F, lam), lib.OP_MSD: one.apply(lib.OP_MSD, lam), lib.OP_D: one.apply(lib.OP_D, rhs)}
    monkeypatch.setenv("IETI_LOOPBACK", "1")
    uid = lib.nccl_unique_id()
    out, err = {}, {}

    def worker(r):
        try:
            ie = lib.Ieti.from_workload(wl, rank=r, world=2, nccl_unique_id=uid, patch_owner=owner)
            ids, pts = ie.local_multipliers()
            rl = np.concatenate([rhs[offs[k]:offs[k + 1]] for k in pts])
            res = {op: ie.apply(op, lam[ids] if op != lib.OP_D else rl) for op in (lib.OP_F, lib.OP_MSD, lib.OP_D)}
            out[r] = (ids, ie.n_own, res)
            ie.close()
        except Exception as e:  # pragma: no cover - surfaced below
            err[r] = repr(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    seen = np.zeros(orc.topo.n_lambda, dtype=int)
    for r in range(2):
        ids, n_own, res = out[r]
        seen[ids[:n_own]] += 1
        for op, v in res.items():
            assert rel(v[:n_own], ref[op][ids[:n_own]]) <= 1e-12, (r, op)
    assert np.all(seen == 1)


def test_fault_injection():
    """Reported states, not crashes: a NaN in the rhs is a breakdown; a
    patch with negative Jacobian is E_GEOMETRY; a partially matching interface is E_TOPOLOGY."""
    import copy
    import paper_1705_04531_b200 as lib
    wl, orc, gpu = systems("C1")
    f_bad = [v.copy() for v in orc.f]
    f_bad[0][orc.topo.ptopo[0].interior[0]] = np.nan            # an active interior dof
    rhs = act_to_lat(orc, f_bad)
    with pytest.raises(lib.IetiError) as e:
        gpu.solve(rhs)
    assert e.value.code == -5
    # the context stays usable afterwards
    u, lam, its, rr, rc = gpu.solve(act_to_lat(orc, orc.f))
    assert its == orc.solve(tol=1e-8).iters
    # mirrored patch: det J < 0 at every quadrature point
    bad = copy.deepcopy(wl)
    bad.patches[0].ctrl = bad.patches[0].ctrl.copy()
    bad.patches[0].ctrl[:, 0] = -bad.patches[0].ctrl[:, 0]
    with pytest.raises(lib.IetiError) as e:
        lib.Ieti.from_workload(bad)
    assert e.value.code in (-2, -3)
    # one control point of a shared side moved: the side matches only partially
    nc = copy.deepcopy(wl)
    pa = nc.patches[0]
    pa.ctrl = pa.ctrl.copy()
    M0 = len(pa.knots[0]) - pa.degree[0] - 1
    pa.ctrl[M0 * 2 + (M0 - 1), 1] += 1e-3         # (i0 = M0-1, i1 = 2): on the side shared with patch 1
    with pytest.raises(lib.IetiError) as e:
        lib.Ieti.from_workload(nc)
    assert e.value.code == -3


def test_full_size_C5_sampled_and_properties():
    """BASELINE.json's full C5 (256 patches, p = 3, m = 32, 11 M dofs) in bench.py's launch
    configuration (default context: offset-major finest level, x-resident sweep groups, fused
    cluster V-cycle on level 1).  Sampled outputs the oracle computes one by one: the local
    Neumann solve N_c (K + alpha Mhat, R4) and the Dirichlet solve D_c of an interior floating
    patch, element by element at 1e-11.  Properties that hold at any size: F^ and M_sD symmetric,
    and the recovered u satisfies B u = d^ - F^ lambda (the final dual residual)."""
    import paper_1705_04531_b200 as lib
    from oracle import assembly, mg
    wl = make_workload("C5")
    gpu = lib.Ieti.from_workload(wl)
    n_full = int(np.prod([len(t) - wl.p - 1 for t in wl.patches[0].knots]))
    mid = tuple(g // 2 for g in wl.grid)
    k = mid[0] + wl.grid[0] * (mid[1] + wl.grid[1] * mid[2])
    pa = wl.patches[k]
    K, _ = assembly.assemble_patch(pa)
    L = mg.num_levels(wl.m)
    lvN = mg.PatchLevels(pa.knots, wl.p, L, [False] * 3, [False] * 3)
    lvD = mg.PatchLevels(pa.knots, wl.p, L, [True] * 3, [True] * 3)
    HN = mg.Hierarchy([(K + wl.alpha_reg * assembly.parameter_mass(pa)).tocsr()], [lvN])
    mI = lvD.mask[-1]
    HD = mg.Hierarchy([K[mI][:, mI].tocsr()], [lvD])
    rng = np.random.default_rng(21)
    q = rng.standard_normal(gpu.ndofs)
    sl = slice(k * n_full, (k + 1) * n_full)
    got = gpu.apply(lib.OP_NEUMANN, q)[sl]
    assert rel(got, HN.apply_cycles(q[sl], wl.cycles)) <= 1e-11
    got = gpu.apply(lib.OP_DIRICHLET, q)[sl][mI]
    assert rel(got, HD.apply_cycles(q[sl][mI], wl.dirichlet_cycles)) <= 1e-11
    # properties at full size
    x, y = rng.standard_normal(gpu.n_lambda), rng.standard_normal(gpu.n_lambda)
    for op in (lib.OP_F, lib.OP_MSD):
        Fx, Fy = gpu.apply(op, x), gpu.apply(op, y)
        # relative to |y| |F x| (the dot products cancel ~600-fold here)
        assert abs(y @ Fx - x @ Fy) <= 1e-10 * np.linalg.norm(y) * np.linalg.norm(Fx)
    rhs = gpu.load_builtin(lib.F_SIN3)
    u, lam, its, rr, rc = gpu.solve(rhs)
    assert rc == lib.OK and rr <= wl.pcg_tol
    kp, ap, km, am = gpu.multiplier_map()
    jump = u[kp.astype(np.int64) * n_full + ap] - u[km.astype(np.int64) * n_full + am]
    d = gpu.apply(lib.OP_D, rhs)
    r_final = d - gpu.apply(lib.OP_F, lam)
    assert np.linalg.norm(jump - r_final) <= 1e-10 * np.linalg.norm(d)
    assert np.linalg.norm(r_final) <= 1.5 * wl.pcg_tol * np.linalg.norm(d)
    gpu.close()


def test_setup_and_solve_bitwise_reproducible():
    """Two independent setups of the full C3 (64 patches, p = 4, m = 128) give bitwise identical
    stencils of both hierarchies and a bitwise identical solve (no atomics in reductions, R23;
    every host->device upload ordered on the library stream: a pageable legacy-stream copy could
    land after the kernels that read it)."""
    import paper_1705_04531_b200 as lib
    wl = make_workload("C3")
    outs = []
    for _ in range(2):
        ie = lib.Ieti.from_workload(wl)
        L = ie.levels - 1
        st = [np.concatenate([ie.stencil(h, L, k).ravel() for k in range(ie.n_patches)]) for h in (0, 1)]
        u, lam, its, rr, rc = ie.solve(ie.load_builtin(lib.F_SIN2))
        outs.append((st, u, its))
        ie.close()
    (s0, u0, i0), (s1, u1, i1) = outs
    assert np.array_equal(s0[0], s1[0]) and np.array_equal(s0[1], s1[1])
    assert i0 == i1 and np.array_equal(u0, u1)


EDGE = {
    "STRIP": ("STRIP", dict()),                         # 1x2 strip: n_Pi = 0 (pure FETI)
    "SINGLE": ("SINGLE", dict()),                       # one all-Dirichlet patch: n_lambda = 0
    "E1s": ("E1", dict(m=8, grid=(2, 4))),              # Table-1 shape (annulus, p=2, V+E, MG-MG, tol 1e-6)
    "E2s": ("E2", dict(m=4, grid=(2, 2, 2))),           # Table-2 shape: edge averages only, multiplicity-8 vertex
    # Table 1's p = 7 shape, MG-MG: the Gauss-Seidel MG-PCG needs more than the default 200
    # inner steps at p = 7 (up to 351 here; the paper's p-robust smoother is out of scope)
    "E1p7": ("E1", dict(m=16, grid=(2, 4), p=7, inner_maxit=1000)),
    "C1p5": ("C1", dict(m=8, p=5)),                     # 2D p = 5, fixed V-cycles
}


@pytest.mark.parametrize("case", list(EDGE))
def test_edge_cases_and_paper_shapes(case):
    """Degenerate cases of the method and the paper's experiment shapes (reduced) against the oracle:
    STRIP (no primal constraints, n_Pi = 0), SINGLE (no multipliers: the solve is one local
    Dirichlet problem, k = 0), E1 (MG-MG: inner MG-PCG to 1e-10, outer tol 1e-6) and E2
    (edge averages only, so the interior vertex is dual with multiplicity 8)."""
    import paper_1705_04531_b200 as lib
    name, kw = EDGE[case]
    wl = make_workload(name, **kw)
    orc = IetiOracle(wl)
    gpu = lib.Ieti.from_workload(wl)
    try:
        assert gpu.n_lambda == orc.topo.n_lambda and gpu.n_pi == orc.topo.n_pi
        rhs = act_to_lat(orc, orc.f)
        ref = orc.solve(tol=wl.pcg_tol)
        u, lam, its, rr, rc = gpu.solve(rhs)
        assert rc == lib.OK and abs(its - ref.iters) <= 1, (its, ref.iters)
        uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
        err_u = rel(uf, np.concatenate(orc.solve(fixed_iters=ref.iters).u))
        parity_log(test="edge_cases", case=case, iters_gpu=its, iters_oracle=ref.iters, err_u=err_u,
                   n_pi=int(gpu.n_pi), n_lambda=int(gpu.n_lambda))
        assert err_u <= 1e-9
        if case == "SINGLE":
            assert gpu.n_lambda == 0 and its == 0
        if case == "STRIP":
            assert gpu.n_pi == 0
    finally:
        gpu.close()


@pytest.mark.parametrize("name", ["C1", "C4s"])
def test_zero_rhs(name):
    """d^ = 0: zero iterations, u = 0, lambda = 0 (O10: k = 0 if d = 0)."""
    import paper_1705_04531_b200 as lib
    wl, orc, gpu = systems(name)
    rhs = np.zeros(lat_offsets(orc)[-1])
    u, lam, its, rr, rc = gpu.solve(rhs)
    assert rc == lib.OK and its == 0
    assert not np.any(u) and not np.any(lam)
    assert orc.solve(tol=1e-8).iters > 0       # the context still solves the real load afterwards
    u, lam, its, rr, rc = gpu.solve(act_to_lat(orc, orc.f))
    assert its == orc.solve(tol=1e-8).iters


def _loopback_solve(wl, world, owner, kw, fixed=None):
    """world ranks as threads of this process (IETI_LOOPBACK=1): every rank runs the whole solve --
    d^, the dual PCG (or BPCG) with its dot-product allgathers, halo exchanges and the coarse
    right-hand-side allgather, the recovery -- eagerly, collectives through device copies ordered by
    a host barrier (no kernel waits on another rank)."""
    import threading
    import paper_1705_04531_b200 as lib
    uid = lib.nccl_unique_id()
    out, err = {}, {}

    def worker(r):
        try:
            ie = lib.Ieti.from_workload(wl, rank=r, world=world, nccl_unique_id=uid, patch_owner=owner, **kw)
            ids, pts = ie.local_multipliers()
            rhs = ie.load_builtin(lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3)
            if fixed is None:
                u, lam, its, rr, rc = ie.solve(rhs)
            else:
                u, lam, rr = ie.solve_fixed(rhs, fixed)
                its = fixed
            out[r] = (ids[:ie.n_own], pts, u, lam, its)
            ie.close()
        except Exception as e:  # pragma: no cover - surfaced below
            err[r] = repr(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not err, err
    return out


@pytest.mark.parametrize("case,world,outer", [("C4s", 2, "dual"), ("C4s", 4, "dual"), ("C5s", 2, "dual"),
                                              ("C5s", 4, "dual"), ("C2s", 2, "dual"), ("C4s", 2, "bpcg"),
                                              ("C5s", 4, "owned"), ("C2v", 3, "owned")])
def test_multirank_loopback_whole_solve(case, world, outer, monkeypatch):
    """The multi-GPU solve path end to end on one GPU (verdict: 'extend loopback mode to the whole
    ieti_solve'): 2 / 4 ranks with non-contiguous (modulo) patch ownership give exactly the one-rank
    iteration count, and u (owned patches) and lambda (owned multipliers) equal the one-rank
    solution to 1e-11: the rank-ordered sums of the PCG dots and of g_Pi only change summation order
    (O(1e-16) per dot), which the PCG amplifies by up to the condition number of M_sD F (~1e4 here);
    every realized deviation is logged (IETI_PARITY_LOG).
    'owned': every rank passes only its own patches' geometry; the library all-gathers it."""
    import paper_1705_04531_b200 as lib
    wl, orc, _ = systems(case)
    kw = {}
    if case == "C2v":
        wl = make_workload("C2", **CASES[case])
        wl.local_mode, wl.cycles, wl.dirichlet_cycles = 0, 2, 2
    if outer == "bpcg":
        wl = make_workload(base(case), **CASES[case])
        wl.local_mode = 0
        kw = dict(cycles=3, outer_mode=lib.OUTER_BPCG)
    one = lib.Ieti.from_workload(wl, **kw)
    rhs = one.load_builtin(lib.F_SIN2 if wl.dim == 2 else lib.F_SIN3)
    u1, lam1, its1, rr1, rc1 = one.solve(rhs)
    one.close()
    owner = [k % world for k in range(wl.n_patches)]
    rkw = dict(kw, geometry_scope=lib.GEOMETRY_OWNED) if outer == "owned" else kw
    offs = np.cumsum([0] + [int(np.prod([len(t) - wl.p - 1 for t in pa.knots])) for pa in wl.patches])
    monkeypatch.setenv("IETI_LOOPBACK", "1")
    res = _loopback_solve(wl, world, owner, rkw)
    seen = np.zeros(len(lam1), dtype=int)
    du = dl = 0.0
    for r, (ids, pts, u, lam, its) in res.items():
        assert its == its1, (r, its, its1)
        ref_u = np.concatenate([u1[offs[k]:offs[k + 1]] for k in pts])
        du, dl = max(du, rel(u, ref_u)), max(dl, rel(lam, lam1[ids]))
        seen[ids] += 1
    parity_log(test="loopback_whole_solve", case=case, world=world, outer=outer, iters=its1, rel_u=du, rel_lam=dl)
    assert du <= 1e-11 and dl <= 1e-11, (du, dl)
    assert np.all(seen == 1)


@pytest.mark.parametrize("name,tpr", [("C4s", "default"), ("C5s", "1"), ("C3s", "default"), ("C2s", "default")])
def test_persistent_sweep(name, tpr, monkeypatch):
    """IETI_PSWEEP=1: every colour sweep is ONE cooperative launch (k_sweep, grid barrier between the
    colour phases, x read through L2) -- the same N_c, F^ and solution as the oracle, on the
    row-major small-level path and (IETI_TPR=1) the offset-major big-level path."""
    import paper_1705_04531_b200 as lib
    wl, orc, _ = systems(name)
    monkeypatch.setenv("IETI_PSWEEP", "1")
    if tpr != "default":
        monkeypatch.setenv("IETI_TPR", tpr)
    gpu = lib.Ieti.from_workload(wl)
    try:
        rng = np.random.default_rng(12)
        q = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
        if wl.local_mode == 1:
            q = [v - v.mean() if pt.floating else v for v, pt in zip(q, orc.topo.ptopo)]
        got = lat_to_act(orc, gpu.apply(lib.OP_NEUMANN, act_to_lat(orc, q)))
        assert rel(np.concatenate(got), np.concatenate(orc.local_neumann(q))) <= (1e-10 if wl.local_mode == 1 else 1e-11)
        lam = rng.standard_normal(orc.topo.n_lambda)
        assert rel(gpu.apply(lib.OP_F, lam), orc.apply_F(lam)) <= (1e-10 if wl.local_mode == 1 else 1e-11)
        assert rel(gpu.apply(lib.OP_MSD, lam), orc.apply_MsD(lam)) <= 1e-11
        rhs = act_to_lat(orc, orc.f)
        ref = orc.solve(tol=1e-8)
        u, lm, its, rr, rc = gpu.solve(rhs)
        assert abs(its - ref.iters) <= 1
        uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
        assert rel(uf, np.concatenate(orc.solve(fixed_iters=ref.iters).u)) <= 1e-9
    finally:
        gpu.close()


DIRECT_CASES = [("C3", dict(m=8, grid=(3, 2))), ("C2", dict(m=8, grid=(3, 3))), ("C4", dict(m=4, grid=(3, 2, 2))),
                ("E1", dict(m=8, grid=(2, 4))), ("C5", dict(m=4, grid=(3, 2, 2)))]


@pytest.mark.parametrize("name,kw", DIRECT_CASES)
def test_direct_local_solvers_dd(name, kw):
    """SURVEY NEXT-3 as the paper scopes it: D-D with direct local solvers. IETI_LOCAL_DIRECT /
    IETI_DIRICHLET_DIRECT factor K (one dof pinned on floating patches) and K_II per patch as bands
    (batched banded Cholesky) at setup.  (a) the Dirichlet solve equals K_II^-1 (oracle sparse LU)
    to 1e-12; (b) Ktilde^-1 with exact local solves equals the oracle's exact-mode App. A.1 form to
    1e-10 (its full primal basis is iterated to P:309's 1e-12); (c) the D-D solve: iterations +-1,
    u and lambda (range F) within 1e-9 of the oracle's exact modes after its count; (d) at tol
    1e-12 u equals the global conforming direct solve (brute force) to 1e-9."""
    import paper_1705_04531_b200 as lib
    from oracle import brute
    wl = make_workload(name, **kw)
    wl.local_mode = 0
    orc = IetiOracle(wl, neumann="exact", dirichlet="exact")
    gpu = lib.Ieti.from_workload(wl, local_mode=lib.LOCAL_DIRECT, dirichlet_mode=lib.DIRICHLET_DIRECT)
    try:
        rng = np.random.default_rng(17)
        s = [rng.standard_normal(len(pt.interior)) for pt in orc.topo.ptopo]
        full = []
        for k, pt in enumerate(orc.topo.ptopo):
            v = np.zeros(len(pt.act_idx))
            v[pt.interior] = s[k]
            full.append(v)
        gl = lat_to_act(orc, gpu.apply(lib.OP_DIRICHLET, act_to_lat(orc, full)))
        got = [g[pt.interior] for g, pt in zip(gl, orc.topo.ptopo)]
        assert rel(np.concatenate(got), np.concatenate(orc.local_dirichlet(s))) <= 1e-12
        r = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
        got = lat_to_act(orc, gpu.apply(lib.OP_KTINV, act_to_lat(orc, r)))
        assert rel(np.concatenate(got), np.concatenate(orc.ktilde_inv(r))) <= 1e-10
        rhs = act_to_lat(orc, orc.f)
        ref = orc.solve(tol=wl.pcg_tol)
        u, lam, its, rr, rc = gpu.solve(rhs)
        assert rc == lib.OK and abs(its - ref.iters) <= 1, (its, ref.iters)
        fix = orc.solve(fixed_iters=ref.iters)
        uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
        Q = kernel_basis(orc)
        proj = lambda v: v - Q @ (Q.T @ v)
        err_u, err_l = rel(uf, np.concatenate(fix.u)), rel(proj(lf), proj(fix.lam))
        parity_log(test="direct_dd", case=name, iters_gpu=its, iters_oracle=ref.iters, err_u=err_u, err_lam_range=err_l)
        assert err_u <= 1e-9 and err_l <= 1e-9, (err_u, err_l)
        tight = lib.Ieti.from_workload(wl, local_mode=lib.LOCAL_DIRECT, dirichlet_mode=lib.DIRICHLET_DIRECT,
                                       pcg_tol=1e-12)
        try:
            ut = tight.solve(rhs)[0]
        finally:
            tight.close()
        ub, _ = brute.solve_global(orc)
        assert rel(ut, np.concatenate(ub)) <= 1e-9
    finally:
        gpu.close()


@pytest.mark.parametrize("name,kw", [("C4", dict(m=4, grid=(3, 2, 2))), ("C5", dict(m=8, grid=(2, 2, 2))),
                                     ("C2", dict(m=8, grid=(3, 3)))])
def test_smoothing_steps_nu(name, kw):
    """R5 through the boundary (ieti_setup_args.nu_pre / nu_post = 2): N_c, D_c, F^ and the solve equal
    the oracle's with two forward / two backward colour sweeps per level (the fused small-level
    kernel is bypassed, the half-stream residual uses the last forward sweep's increments)."""
    import paper_1705_04531_b200 as lib
    wl = make_workload(name, **kw)
    wl.local_mode, wl.cycles, wl.dirichlet_cycles = 0, 2, 2
    wl.nu_pre, wl.nu_post = 2, 2
    orc = IetiOracle(wl)
    gpu = lib.Ieti.from_workload(wl)
    try:
        rng = np.random.default_rng(23)
        q = [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo]
        got = lat_to_act(orc, gpu.apply(lib.OP_NEUMANN, act_to_lat(orc, q)))
        assert rel(np.concatenate(got), np.concatenate(orc.local_neumann(q))) <= 1e-11
        lam = rng.standard_normal(orc.topo.n_lambda)
        assert rel(gpu.apply(lib.OP_F, lam), orc.apply_F(lam)) <= 1e-11
        assert rel(gpu.apply(lib.OP_MSD, lam), orc.apply_MsD(lam)) <= 1e-11
        rhs = act_to_lat(orc, orc.f)
        ref = orc.solve(tol=1e-8)
        u, lm, its, rr, rc = gpu.solve(rhs)
        assert abs(its - ref.iters) <= 1
        uf, lf, _ = gpu.solve_fixed(rhs, ref.iters)
        assert rel(uf, np.concatenate(orc.solve(fixed_iters=ref.iters).u)) <= 1e-9
        parity_log(test="nu2", case=name, iters_gpu=its, iters_oracle=ref.iters)
    finally:
        gpu.close()


def test_inner_pcg_cap_is_reported():
    """an inner local MG-PCG that stops at its iteration cap is no longer silent -- the
    solve returns IETI_NOT_CONVERGED (outputs written) instead of IETI_OK."""
    import paper_1705_04531_b200 as lib
    wl = make_workload("C2", m=8, grid=(3, 3))
    gpu = lib.Ieti.from_workload(wl, inner_maxit=2)           # C2's inner solves need ~10 steps
    try:
        u, lam, its, rr, rc = gpu.solve(gpu.load_builtin(lib.F_SIN2))
        assert rc == lib.NOT_CONVERGED
    finally:
        gpu.close()
    ok = lib.Ieti.from_workload(wl)
    try:
        assert ok.solve(ok.load_builtin(lib.F_SIN2))[4] == lib.OK
    finally:
        ok.close()


def test_msd_with_dirichlet_pcg_is_a_fixed_operator():
    """with DIRICHLET_PCG the Dirichlet rhs box doubles as the inner preconditioner's input;
    it is cleared before every M_sD, so M_sD does not depend on the previous call (two applications
    with a loose dirichlet_tol are bitwise identical)."""
    import paper_1705_04531_b200 as lib
    wl = make_workload("C4", m=4, grid=(3, 2, 2))
    gpu = lib.Ieti.from_workload(wl, dirichlet_mode=lib.DIRICHLET_PCG, dirichlet_tol=1e-3)
    try:
        rng = np.random.default_rng(2)
        x, y = rng.standard_normal(gpu.n_lambda), rng.standard_normal(gpu.n_lambda)
        a = gpu.apply(lib.OP_MSD, x)
        gpu.apply(lib.OP_MSD, y)
        b = gpu.apply(lib.OP_MSD, x)
        assert np.array_equal(a, b)
    finally:
        gpu.close()


@pytest.mark.parametrize("name,cs", [("C4s", "0"), ("C5s", "0"), ("C3s", "0"), ("C2s", "0"), ("C2v", "0"),
                                     ("LARGE", "0"), ("LARGE", "4"), ("LARGE", "16"), ("C4s", "16"), ("C4s", "g"),
                                     ("LARGE", "g"), ("C4s", "rep"), ("C3s", "rep"), ("LARGE", "rep")])
def test_cluster_sweep_bitwise(name, cs, monkeypatch):
    """k_sweep_cl (kernels_sweep.cu: one cluster launch per colour sweep on the row-major levels, the
    next phase's coefficient slab staged by TMA, cluster barriers between the phases) computes the
    same arithmetic in the same order as the one-launch-per-phase path: N_c, F^, M_sD and the whole
    solve must be BITWISE equal to IETI_CLSWEEP=0.  cs forces the CTAs per problem (IETI_CLCS; 4 =
    two row passes per CTA on C4's full per-patch size, 16 = non-portable cluster size; g = coefficients
    read from global memory instead of TMA-staged slabs, IETI_CLGLOBAL; rep = x replicated in every
    CTA's shared memory with the updates broadcast through DSMEM, IETI_CLREP).  C4's finest level runs the
    cycle-boundary modes 6 / 7 (U recorded by the backward sweep) through the same kernel."""
    import paper_1705_04531_b200 as lib
    if name == "LARGE":
        wl = make_workload(LARGE[0], **LARGE[1])
        orc = IetiOracle(wl)
    else:
        wl, orc, _ = systems(name)
    if cs == "g":
        monkeypatch.setenv("IETI_CLGLOBAL", "1")
    elif cs == "rep":
        monkeypatch.setenv("IETI_CLREP", "1")
    elif cs != "0":
        monkeypatch.setenv("IETI_CLCS", cs)
    outs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("IETI_CLSWEEP", flag)
        gpu = lib.Ieti.from_workload(wl)
        try:
            rng = np.random.default_rng(5)
            q = act_to_lat(orc, [rng.standard_normal(len(pt.act_idx)) for pt in orc.topo.ptopo])
            lam = rng.standard_normal(orc.topo.n_lambda)
            u, lm, its, rr, rc = gpu.solve(act_to_lat(orc, orc.f))
            outs[flag] = (gpu.apply(lib.OP_NEUMANN, q), gpu.apply(lib.OP_F, lam), gpu.apply(lib.OP_MSD, lam), u, lm, its)
        finally:
            gpu.close()
    for a, b in zip(outs["0"][:5], outs["1"][:5]):
        assert np.array_equal(a, b)
    assert outs["0"][5] == outs["1"][5]
    parity_log(test="cluster_sweep_bitwise", case=name, cs=cs, iters=outs["1"][5])
