"""paper_1705_04531_b200 -- B200-native inexact IETI-DP (arXiv:1705.04531).

Thin ctypes binding of the C ABI in ``include/ieti.h`` (argument marshalling only; every
step of the method runs in the sm_100a kernels of ``libieti.so``).  Importing this
package fails loudly if the in-tree library has not been built: there is no CPU
fallback.  PyTorch is used only by callers for device memory and streams
(``solve_device`` takes raw device pointers, e.g. ``tensor.data_ptr()``).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libieti.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libieti.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = ctypes.CDLL(LIB_PATH)
_lib.ieti_build_info.restype = ctypes.c_char_p
BUILD_INFO = _lib.ieti_build_info().decode()


def _check_provenance():
    """The library must have been built from the sources next to it (fails loudly on a stale .so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_ieti_build_hash", os.path.join(_HERE, "build.py"))
    mod = importlib.util.module_from_spec(spec)
    try:
        spec.loader.exec_module(mod)
        want = mod.source_hash()
    except (OSError, RuntimeError):      # sources not shipped (binary-only install): nothing to compare
        return
    if ("src=" + want) not in BUILD_INFO:
        raise ImportError(f"libieti.so is stale: built from {BUILD_INFO}, sources are src={want}; rebuild with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")


if os.environ.get("IETI_ALLOW_STALE") != "1":
    _check_provenance()

PRIMAL_VERTEX, PRIMAL_EDGE, PRIMAL_FACE = 1, 2, 4
LOCAL_VCYCLES, LOCAL_PCG, LOCAL_DIRECT = 0, 1, 2
DIRICHLET_VCYCLES, DIRICHLET_PCG, DIRICHLET_DIRECT = 0, 1, 2
OUTER_DUAL_PCG, OUTER_BPCG = 0, 1
GEOMETRY_GLOBAL, GEOMETRY_OWNED = 0, 1
F_ZERO, F_SIN2, F_SIN3, F_ONE = 0, 1, 2, 3
OP_F, OP_MSD, OP_D, OP_NEUMANN, OP_DIRICHLET, OP_KTINV, OP_VCYCLE_N, OP_KT, OP_CAN, OP_KHAT = range(10)
OK, NOT_CONVERGED = 0, 1
ERRORS = {-1: "E_ARG", -2: "E_GEOMETRY", -3: "E_TOPOLOGY", -4: "E_NOT_SPD", -5: "E_BREAKDOWN",
          -6: "E_CUDA", -7: "E_NCCL", -8: "E_NOMEM", -9: "E_UNSUPPORTED"}

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_llp = ctypes.POINTER(ctypes.c_longlong)


class SetupArgs(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n_patches", ctypes.c_int),
                ("degree", _ip), ("n_knots", _ip), ("knots", _dp), ("ctrl", _dp),
                ("primal", ctypes.c_uint), ("local_mode", ctypes.c_int), ("cycles", ctypes.c_int),
                ("dirichlet_cycles", ctypes.c_int), ("mg_levels", ctypes.c_int),
                ("alpha_reg", ctypes.c_double), ("inner_tol", ctypes.c_double), ("inner_maxit", ctypes.c_int),
                ("pcg_tol", ctypes.c_double), ("pcg_maxit", ctypes.c_int), ("basis_tol", ctypes.c_double),
                ("rank", ctypes.c_int), ("world", ctypes.c_int), ("device", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("patch_owner", _ip),
                ("dirichlet_mode", ctypes.c_int), ("dirichlet_tol", ctypes.c_double),
                ("dirichlet_maxit", ctypes.c_int), ("outer_mode", ctypes.c_int), ("lanczos_steps", ctypes.c_int),
                ("khat_margin", ctypes.c_double), ("geometry_scope", ctypes.c_int), ("nu_pre", ctypes.c_int),
                ("nu_post", ctypes.c_int)]


_lib.ieti_setup.argtypes = [ctypes.POINTER(SetupArgs), ctypes.POINTER(ctypes.c_void_p)]
_lib.ieti_setup.restype = ctypes.c_int
_lib.ieti_assemble_load_builtin.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp]
_lib.ieti_solve.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _ip, _dp]
_lib.ieti_solve_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _ip, _dp,
                                   ctypes.c_void_p]
_lib.ieti_solve_fixed.argtypes = [ctypes.c_void_p, _dp, ctypes.c_int, _dp, _dp, _dp]
_lib.ieti_info.argtypes = [ctypes.c_void_p, _llp]
_lib.ieti_multiplier_map.argtypes = [ctypes.c_void_p, _ip, _ip, _ip, _ip]
_lib.ieti_apply.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
_lib.ieti_get_stencil.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _ip]
_lib.ieti_get_primal_basis.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _ip]
_lib.ieti_timing.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _dp, _llp, _dp]
_lib.ieti_quadrature_points.argtypes = [ctypes.c_void_p, _dp, _llp]
_lib.ieti_assemble_load.argtypes = [ctypes.c_void_p, _dp, _dp]
_lib.ieti_nccl_unique_id.argtypes = [ctypes.c_void_p]
_lib.ieti_local_multipliers.argtypes = [ctypes.c_void_p, _ip, _ip]
_lib.ieti_plan_info.argtypes = [ctypes.POINTER(SetupArgs), ctypes.c_int, ctypes.c_int, _llp]
_lib.ieti_plan_get.argtypes = [ctypes.POINTER(SetupArgs), ctypes.c_int, ctypes.c_int] + [_ip] * 7
_lib.ieti_inner_log.argtypes = [ctypes.c_void_p, _ip, ctypes.c_int, _ip]
_lib.ieti_last_error.argtypes = [ctypes.c_void_p]
_lib.ieti_last_error.restype = ctypes.c_char_p
_lib.ieti_bpcg_info.argtypes = [ctypes.c_void_p, _dp]
_lib.ieti_phase_times.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp]
_lib.ieti_destroy.argtypes = [ctypes.c_void_p]
_lib.ieti_destroy.restype = None

EXPORTS = ("ieti_build_info", "ieti_setup", "ieti_assemble_load_builtin", "ieti_solve", "ieti_solve_device", "ieti_solve_fixed",
           "ieti_info", "ieti_multiplier_map", "ieti_apply", "ieti_get_stencil", "ieti_get_primal_basis",
           "ieti_timing", "ieti_inner_log", "ieti_nccl_unique_id", "ieti_local_multipliers", "ieti_plan_info",
           "ieti_plan_get", "ieti_quadrature_points", "ieti_assemble_load", "ieti_last_error",
           "ieti_bpcg_info", "ieti_phase_times", "ieti_destroy")


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to be broadcast to every rank before ``Ieti(..., world>1)``."""
    buf = ctypes.create_string_buffer(128)
    rc = _lib.ieti_nccl_unique_id(buf)
    if rc != OK:
        raise IetiError(rc, _lib.ieti_last_error(None).decode())
    return buf.raw


class IetiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


def _p(a, ct=_dp):
    return a.ctypes.data_as(ct)


def make_setup_args(keep: list, dim, degree, knots, ctrl, primal, local_mode=LOCAL_VCYCLES, cycles=2,
                    dirichlet_cycles=2, mg_levels=0, alpha_reg=1e-2, inner_tol=1e-6, inner_maxit=200,
                    pcg_tol=1e-8, pcg_maxit=500, basis_tol=1e-12, device=0, rank=0, world=1,
                    nccl_unique_id=None, patch_owner=None, dirichlet_mode=DIRICHLET_VCYCLES,
                    dirichlet_tol=1e-12, dirichlet_maxit=500, outer_mode=OUTER_DUAL_PCG, lanczos_steps=40,
                    khat_margin=0.05, geometry_scope=GEOMETRY_GLOBAL, n_patches=None, nu_pre=1,
                    nu_post=1) -> SetupArgs:
    """Marshal the geometry and options into ``ieti_setup_args`` (arrays kept alive in ``keep``).
    geometry_scope OWNED: degree / knots / ctrl hold only this rank's patches; n_patches = global count."""
    n_patches = len(ctrl) if n_patches is None else n_patches
    deg = np.ascontiguousarray(np.repeat(np.asarray(degree, dtype=np.int32)[:, None], dim, axis=1)
                               if np.ndim(degree) == 1 else np.asarray(degree, dtype=np.int32)).ravel()
    nk = np.array([len(t) for kv in knots for t in kv], dtype=np.int32)
    kn = np.ascontiguousarray(np.concatenate([np.asarray(t, dtype=np.float64) for kv in knots for t in kv]))
    ct = np.ascontiguousarray(np.concatenate([np.asarray(c, dtype=np.float64).reshape(-1) for c in ctrl]))
    keep += [deg, nk, kn, ct]
    uid = None
    if nccl_unique_id is not None:
        uid = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        keep.append(uid)
    own = None
    if patch_owner is not None:
        own = np.ascontiguousarray(np.asarray(patch_owner, dtype=np.int32))
        keep.append(own)
    return SetupArgs(dim=dim, n_patches=n_patches, degree=_p(deg, _ip), n_knots=_p(nk, _ip), knots=_p(kn),
                     ctrl=_p(ct), primal=primal, local_mode=local_mode, cycles=cycles,
                     dirichlet_cycles=dirichlet_cycles, mg_levels=mg_levels, alpha_reg=alpha_reg,
                     inner_tol=inner_tol, inner_maxit=inner_maxit, pcg_tol=pcg_tol, pcg_maxit=pcg_maxit,
                     basis_tol=basis_tol, rank=rank, world=world, device=device,
                     nccl_unique_id=ctypes.cast(uid, ctypes.c_void_p) if uid is not None else None,
                     patch_owner=_p(own, _ip) if own is not None else None, dirichlet_mode=dirichlet_mode,
                     dirichlet_tol=dirichlet_tol, dirichlet_maxit=dirichlet_maxit, outer_mode=outer_mode,
                     lanczos_steps=lanczos_steps, khat_margin=khat_margin, geometry_scope=geometry_scope,
                     nu_pre=nu_pre, nu_post=nu_post)


def partition_plan(wl, rank: int, world: int, patch_owner=None) -> dict:
    """Host-only multi-GPU partition plan of a workload for (rank, world) (ieti_plan_info/_get)."""
    keep = []
    a = make_setup_args(keep, wl.dim, [pa.degree for pa in wl.patches], [pa.knots for pa in wl.patches],
                        [pa.ctrl for pa in wl.patches], wl.primal, rank=rank, world=world, patch_owner=patch_owner)
    info = np.zeros(6, dtype=np.int64)
    rc = _lib.ieti_plan_info(ctypes.byref(a), rank, world, _p(info, _llp))
    if rc != OK:
        raise IetiError(rc, _lib.ieti_last_error(None).decode())
    npat, nloc, nown, npeer, nsend, nrecv = (int(v) for v in info)
    arr = [np.zeros(max(1, n), dtype=np.int32) for n in (npat, nloc, npeer, npeer + 1, nsend, npeer + 1, nrecv)]
    rc = _lib.ieti_plan_get(ctypes.byref(a), rank, world, *[_p(x, _ip) for x in arr])
    if rc != OK:
        raise IetiError(rc, _lib.ieti_last_error(None).decode())
    return dict(local_patches=arr[0][:npat], local_mult=arr[1][:nloc], n_own=nown, peers=arr[2][:npeer],
                send_ptr=arr[3][:npeer + 1], send_idx=arr[4][:nsend], recv_ptr=arr[5][:npeer + 1],
                recv_idx=arr[6][:nrecv])


class Ieti:
    """One ``ieti_ctx``: setup from patch knots/degree/control points; solve rhs -> u, lambda."""

    def __init__(self, dim: int, degree: Sequence[int], knots: Sequence[Sequence[np.ndarray]],
                 ctrl: Sequence[np.ndarray], primal: int, local_mode: int = LOCAL_VCYCLES, cycles: int = 2,
                 dirichlet_cycles: int = 2, mg_levels: int = 0, alpha_reg: float = 1e-2, inner_tol: float = 1e-6,
                 inner_maxit: int = 200, pcg_tol: float = 1e-8, pcg_maxit: int = 500, basis_tol: float = 1e-12,
                 device: int = 0, rank: int = 0, world: int = 1, nccl_unique_id: Optional[bytes] = None,
                 patch_owner: Optional[Sequence[int]] = None, dirichlet_mode: int = DIRICHLET_VCYCLES,
                 dirichlet_tol: float = 1e-12, dirichlet_maxit: int = 500, outer_mode: int = OUTER_DUAL_PCG,
                 lanczos_steps: int = 40, khat_margin: float = 0.05, geometry_scope: int = GEOMETRY_GLOBAL,
                 n_patches: Optional[int] = None, nu_pre: int = 1, nu_post: int = 1):
        self._keep = []
        a = make_setup_args(self._keep, dim, degree, knots, ctrl, primal, local_mode=local_mode, cycles=cycles,
                            dirichlet_cycles=dirichlet_cycles, mg_levels=mg_levels, alpha_reg=alpha_reg,
                            inner_tol=inner_tol, inner_maxit=inner_maxit, pcg_tol=pcg_tol, pcg_maxit=pcg_maxit,
                            basis_tol=basis_tol, device=device, rank=rank, world=world,
                            nccl_unique_id=nccl_unique_id, patch_owner=patch_owner,
                            dirichlet_mode=dirichlet_mode, dirichlet_tol=dirichlet_tol,
                            dirichlet_maxit=dirichlet_maxit, outer_mode=outer_mode, lanczos_steps=lanczos_steps,
                            khat_margin=khat_margin, geometry_scope=geometry_scope, n_patches=n_patches,
                            nu_pre=nu_pre, nu_post=nu_post)
        h = ctypes.c_void_p()
        rc = _lib.ieti_setup(ctypes.byref(a), ctypes.byref(h))
        if rc != OK:
            raise IetiError(rc, _lib.ieti_last_error(None).decode())
        self._h = h
        info = self.info()
        self.dim, self.p, self.n_patches, self.ndofs = info[0], info[1], info[2], info[3]
        self.n_lambda, self.n_pi, self.levels = info[4], info[5], info[6]
        self.n_own, self.world = int(info[14]), int(info[15])

    @classmethod
    def from_workload(cls, wl, **kw):
        args = dict(local_mode=wl.local_mode, cycles=wl.cycles, dirichlet_cycles=wl.dirichlet_cycles,
                    alpha_reg=wl.alpha_reg, inner_tol=wl.inner_tol, inner_maxit=wl.inner_maxit,
                    pcg_tol=wl.pcg_tol, pcg_maxit=wl.pcg_maxit, nu_pre=getattr(wl, "nu_pre", 1),
                    nu_post=getattr(wl, "nu_post", 1))
        args.update(kw)
        pats = wl.patches
        if args.get("geometry_scope") == GEOMETRY_OWNED:
            # each rank passes only its own patches (the library all-gathers the geometry)
            owner = args["patch_owner"]
            pats = [pa for pa, o in zip(wl.patches, owner) if o == args.get("rank", 0)]
            args["n_patches"] = wl.n_patches
        return cls(wl.dim, [pa.degree for pa in pats], [pa.knots for pa in pats],
                   [pa.ctrl for pa in pats], wl.primal, **args)

    def _check(self, rc, ok=(OK,)):
        if rc not in ok:
            raise IetiError(rc, _lib.ieti_last_error(self._h).decode())
        return rc

    def info(self):
        out = np.zeros(16, dtype=np.int64)
        self._check(_lib.ieti_info(self._h, _p(out, _llp)))
        return out

    def load_builtin(self, f_id: int) -> np.ndarray:
        rhs = np.zeros(self.ndofs)
        self._check(_lib.ieti_assemble_load_builtin(self._h, f_id, _p(rhs)))
        return rhs

    def quadrature_points(self) -> np.ndarray:
        """Physical Gauss points of the owned patches, [n_points][dim]."""
        n = ctypes.c_longlong(0)
        self._check(_lib.ieti_quadrature_points(self._h, None, ctypes.byref(n)))
        out = np.zeros((n.value, self.dim))
        self._check(_lib.ieti_quadrature_points(self._h, _p(out), ctypes.byref(n)))
        return out

    def load(self, f) -> np.ndarray:
        """Torn patch loads for a user f: a callable on [n][dim] points, or values at quadrature_points()."""
        fq = f(self.quadrature_points()) if callable(f) else np.asarray(f, dtype=np.float64)
        fq = np.ascontiguousarray(fq, dtype=np.float64)
        rhs = np.zeros(self.ndofs)
        self._check(_lib.ieti_assemble_load(self._h, _p(fq), _p(rhs)))
        return rhs

    def solve(self, rhs: np.ndarray):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        u = np.zeros(self.ndofs)
        lam = np.zeros(max(1, self.n_own))
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0)
        rc = self._check(_lib.ieti_solve(self._h, _p(rhs), _p(u), _p(lam), ctypes.byref(it), ctypes.byref(rr)),
                         ok=(OK, NOT_CONVERGED))
        return u, lam[:self.n_own], it.value, rr.value, rc

    def solve_fixed(self, rhs: np.ndarray, iters: int):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        u = np.zeros(self.ndofs)
        lam = np.zeros(max(1, self.n_own))
        rr = ctypes.c_double(0)
        self._check(_lib.ieti_solve_fixed(self._h, _p(rhs), iters, _p(u), _p(lam), ctypes.byref(rr)),
                    ok=(OK, NOT_CONVERGED))
        return u, lam[:self.n_own], rr.value

    def solve_device(self, rhs_ptr: int, u_ptr: int, lam_ptr: Optional[int] = None, stream: int = 0):
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0)
        rc = self._check(_lib.ieti_solve_device(self._h, ctypes.c_void_p(rhs_ptr), ctypes.c_void_p(u_ptr),
                                                ctypes.c_void_p(lam_ptr or 0), ctypes.byref(it), ctypes.byref(rr),
                                                ctypes.c_void_p(stream)), ok=(OK, NOT_CONVERGED))
        return it.value, rr.value, rc

    def apply(self, op: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n_out = self.n_lambda if op in (OP_F, OP_MSD, OP_D) else self.ndofs
        out = np.zeros(max(1, n_out))
        self._check(_lib.ieti_apply(self._h, op, _p(x), _p(out)))
        return out[:n_out]

    def stencil(self, hier: int, level: int, patch: int) -> np.ndarray:
        n = ctypes.c_int(0)
        self._check(_lib.ieti_get_stencil(self._h, hier, level, patch, None, ctypes.byref(n)))
        s = (2 * self.p + 1) ** self.dim
        out = np.zeros((n.value, s))
        self._check(_lib.ieti_get_stencil(self._h, hier, level, patch, _p(out), ctypes.byref(n)))
        return out

    def primal_basis(self, patch: int, n_full: int) -> np.ndarray:
        """Phibar^(k) as [n_pi_k][n_full] (full lattice of patch k)."""
        n = ctypes.c_int(0)
        self._check(_lib.ieti_get_primal_basis(self._h, patch, None, ctypes.byref(n)))
        out = np.zeros((n.value, n_full))
        if n.value:
            self._check(_lib.ieti_get_primal_basis(self._h, patch, _p(out), ctypes.byref(n)))
        return out

    def bpcg_info(self):
        """outer_mode BPCG (R30): (s, theta_min, theta_max, Lanczos steps)."""
        out = np.zeros(4)
        self._check(_lib.ieti_bpcg_info(self._h, _p(out)))
        return float(out[0]), float(out[1]), float(out[2]), int(out[3])

    def phase_times(self, reset=False):
        """Accumulated solve-phase / V-cycle timing (ieti_phase_times): dict of ms and bytes."""
        out = np.zeros(16)
        self._check(_lib.ieti_phase_times(self._h, 1 if reset else 0, _p(out)))
        return dict(d_ms=out[0], loop_ms=out[1], recovery_ms=out[2], solves=int(out[3]),
                    vN_ms=out[4], vN_bytes=out[5], vN_bytes3=out[6], vN_sets=int(out[7]),
                    vD_ms=out[8], vD_bytes=out[9], vD_bytes3=out[10], vD_sets=int(out[11]))

    def inner_log(self):
        """LOCAL_PCG: per local-solve call of the last solve, per patch inner PCG counts [calls][patches]."""
        n = ctypes.c_int(0)
        self._check(_lib.ieti_inner_log(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros((max(1, n.value), self.n_patches), dtype=np.int32)
        self._check(_lib.ieti_inner_log(self._h, _p(out, _ip), n.value, ctypes.byref(n)))
        return out[:n.value]

    def local_multipliers(self):
        """(global ids of the local multipliers: owned first, then ghosts; global ids of owned patches)"""
        ids = np.zeros(max(1, self.n_lambda), dtype=np.int32)
        pt = np.zeros(max(1, self.n_patches), dtype=np.int32)
        self._check(_lib.ieti_local_multipliers(self._h, _p(ids, _ip), _p(pt, _ip)))
        return ids[:self.n_lambda], pt[:self.n_patches]

    def multiplier_map(self):
        n = self.n_lambda
        kp, ap, km, am = (np.zeros(max(1, n), dtype=np.int32) for _ in range(4))
        self._check(_lib.ieti_multiplier_map(self._h, _p(kp, _ip), _p(ap, _ip), _p(km, _ip), _p(am, _ip)))
        return kp[:n], ap[:n], km[:n], am[:n]

    def close(self):
        if getattr(self, "_h", None):
            _lib.ieti_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
