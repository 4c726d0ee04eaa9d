/* ieti.h -- C ABI of libieti: the B200 (sm_100a) hot path of inexact IETI-DP.
 *
 * Method: Hofer, Langer, Takacs, "Inexact Dual-Primal Isogeometric Tearing and
 * Interconnecting Methods" (arXiv:1705.04531), PAPER.md.  Citations below are
 * PAPER.md line numbers (P:nnn) and the readings R1..R25 listed in DESIGN.md.
 *
 * What the library computes (north star, K-level form, reading R1):
 *   Poisson problem of Eq. (1) on a multipatch B-spline domain
 *   (P:93-112), torn into patches; the dual problem F lambda = d of Eq. (4)
 *    with F = B Ktilde^{-1} B^T is solved by CG with the scaled
 *   Dirichlet preconditioner M_sD = B_D S B_D^T.  Every local solve
 *   inside F, d, the recovery and M_sD is a fixed number of geometric multigrid
 *   V-cycles or, for LOCAL_PCG, an MG-preconditioned CG
 *   (P:229-231).  The primal basis is the energy-minimising basis of Eq. (6)
 *   (P:186-201); the coarse problem S_PiPi is solved directly.
 *
 * Conventions
 *   - All arithmetic is IEEE fp64.  Index work is int32/int64.
 *   - Dof order: per patch the FULL tensor lattice prod_d M_d (M_d = #knots - p - 1),
 *     lexicographic with direction 1 fastest; patches concatenated by patch id.
 *   - Multipliers: canonical non-redundant chain order (R12): for a dual dof group
 *     with copies on ascending patch ids k1 < ... < km, rows x_{k_i} - x_{k_{i+1}},
 *     sorted by (k1, flat index in k1, i); primal vertex dofs carry none.
 *   - Pointers are HOST pointers unless the function name ends in _device.
 *   - The caller owns every buffer.  ieti_setup deep-copies what it needs and keeps
 *     no caller pointer.  The context owns all device memory, streams and graphs
 *     until ieti_destroy.
 *   - Return codes: IETI_OK (0) or IETI_NOT_CONVERGED (1, outputs written);
 *     negative codes mean nothing was written; ieti_last_error() explains.
 *   - Multi-GPU: rank/world select the patch partition (contiguous blocks of
 *     patch ids); with world > 1 every call is collective (NCCL unique id passed in).
 */
#ifndef IETI_H
#define IETI_H

#ifdef __cplusplus
extern "C" {
#endif

enum { IETI_PRIMAL_VERTEX = 1, IETI_PRIMAL_EDGE = 2, IETI_PRIMAL_FACE = 4 };
enum { IETI_LOCAL_VCYCLES = 0, IETI_LOCAL_PCG = 1, IETI_LOCAL_DIRECT = 2 };     /* R2, R19 */
enum { IETI_DIRICHLET_VCYCLES = 0, IETI_DIRICHLET_PCG = 1, IETI_DIRICHLET_DIRECT = 2 };  /* P:243-248, R27 */
enum { IETI_F_ZERO = 0, IETI_F_SIN2 = 1, IETI_F_SIN3 = 2, IETI_F_ONE = 3 };   /* built-in loads, R16 */
enum { IETI_OUTER_DUAL_PCG = 0, IETI_OUTER_BPCG = 1 };                          /* P:260-262, R28-R31 */
enum { IETI_GEOMETRY_GLOBAL = 0, IETI_GEOMETRY_OWNED = 1 };                     /* who passes which patches */

enum {
  IETI_OK = 0, IETI_NOT_CONVERGED = 1,
  IETI_E_ARG = -1, IETI_E_GEOMETRY = -2, IETI_E_TOPOLOGY = -3, IETI_E_NOT_SPD = -4,
  IETI_E_BREAKDOWN = -5, IETI_E_CUDA = -6, IETI_E_NCCL = -7, IETI_E_NOMEM = -8,
  IETI_E_UNSUPPORTED = -9
};

typedef struct ieti_ctx ieti_ctx;   /* opaque */

typedef struct {
  int dim;                 /* d in {2,3} */
  int n_patches;           /* global patch count N */
  const int *degree;       /* [n_patches*dim] p per patch and direction; must all be equal, 1..4 */
  const int *n_knots;      /* [n_patches*dim] knot-vector lengths */
  const double *knots;     /* concatenated open knot vectors, per patch, per direction;
                              interior knots simple, uniform dyadic nesting down to the coarsest level */
  const double *ctrl;      /* [sum_k prod_d M_kd][dim] control points P_i, lexicographic */
  unsigned primal;         /* bitmask of IETI_PRIMAL_* */
  int local_mode;          /* IETI_LOCAL_VCYCLES (c V-cycles, R2), IETI_LOCAL_PCG (R19: per-patch PCG on K,
                              preconditioner one Neumann V-cycle, x0 = 0, stop at ||r|| <= inner_tol ||q||) or
                              IETI_LOCAL_DIRECT (the paper's direct solver: batched banded Cholesky of K,
                              one dof pinned on floating patches -- exact on the consistent P^T r, App. A.1;
                              IETI_E_NOMEM when the bands do not fit, as 3D C5 patches) */
  int cycles;              /* V-cycles per Neumann local solve (R2, R10) */
  int dirichlet_cycles;    /* V-cycles per Dirichlet solve in M_sD */
  int mg_levels;           /* <= 0: rule R7 */
  double alpha_reg;        /* regularisation K + alpha*Mhat on floating patches (R4) */
  double inner_tol;        /* LOCAL_PCG relative tolerance (R19) */
  int inner_maxit;
  double pcg_tol;          /* outer dual PCG relative tolerance (R11) */
  int pcg_maxit;
  double basis_tol;        /* primal-basis solver tolerance (1e-12) */
  int rank, world, device; /* partition and CUDA device; world > 1 needs nccl_unique_id */
  const void *nccl_unique_id;  /* 128 bytes from ieti_nccl_unique_id() on rank 0, broadcast by the caller
                                  (torch.distributed); NULL when world == 1 */
  const int *patch_owner;  /* [n_patches] rank owning each patch, or NULL = contiguous blocks of patch ids.
                              Every rank passes the SAME partition; the geometry is global or per rank
                              (geometry_scope).  Every rank must own at least one patch (checked on every rank
                              before the first collective). */
  int dirichlet_mode;      /* local Dirichlet solve D in M_sD: IETI_DIRICHLET_VCYCLES = dirichlet_cycles
                              V-cycles (MG in the preconditioner); IETI_DIRICHLET_PCG = per-patch PCG on
                              K_II, preconditioner one Dirichlet V-cycle, x0 = 0, stop at ||r|| <= dirichlet_tol ||q||
                              (R27: the paper's direct Dirichlet solver of D-D, to dirichlet_tol);
                              IETI_DIRICHLET_DIRECT = batched banded Cholesky of K_II */
  double dirichlet_tol;    /* DIRICHLET_PCG relative tolerance (<= 0: 1e-12) */
  int dirichlet_maxit;     /* DIRICHLET_PCG iteration cap (<= 0: 500) */
  int outer_mode;          /* IETI_OUTER_DUAL_PCG: CG on F lambda = d (Eq. (4), the paper's D-D / MG-D / MG-MG);
                              IETI_OUTER_BPCG: MG-MG-S -- Bramble-Pasciak CG on the saddle point
                              Eq. (2) with K^~^-1 = the App. A.1 form of Ktilde^-1 with `cycles` V-cycles
                              (3), scaled below K~ (R29, R30), and F^ = M_sD.
                              Requires local_mode = IETI_LOCAL_VCYCLES. */
  int lanczos_steps;       /* BPCG calibration: Lanczos steps on K^~_1^-1 K~ (R30; <= 0: 40) */
  double khat_margin;      /* BPCG calibration: s = (1 - margin) theta_min (R30; <= 0: 0.05) */
  int geometry_scope;      /* IETI_GEOMETRY_GLOBAL: degree / n_knots / knots / ctrl describe all n_patches patches
                              (every rank the same); IETI_GEOMETRY_OWNED (world > 1): each rank passes ONLY the
                              patches it owns (patch_owner[k] == rank, ascending id; patch_owner stays the
                              global, replicated [n_patches] array) and ieti_setup all-gathers the geometry
                              (collective) before the topology is built */
  int nu_pre, nu_post;     /* colour Gauss-Seidel sweeps per level before / after the coarse correction (R5;
                              P:287 "standard GS", count unstated; <= 0: 1 / 1) */
} ieti_setup_args;

/* Multi-GPU (world > 1, one process per GPU; every call below is then collective):
 *   - each rank owns the patches with patch_owner[k] == rank; rhs / u of ieti_solve* cover the
 *     OWNED patches' full lattices, concatenated in ascending patch id;
 *   - a multiplier is owned by the rank owning its k+ patch (R12); lambda outputs hold the owned
 *     multipliers in canonical order (ieti_local_multipliers gives their global ids);
 *   - per PCG iteration: halo exchanges of interface lambda / partial jumps (grouped ncclSend /
 *     ncclRecv), an allgather of the per-rank coarse right-hand sides (summed in rank order) and
 *     allgathers of the per-rank dot-product partials (summed in rank order).
 * NCCL is loaded at run time only when world > 1. */

/* Validate, build topology, assemble (Eq. (1)), build MG hierarchies,
 * constraints, multipliers, the primal basis (Eq. (6)) and S_PiPi; capture graphs.
 * Errors: IETI_E_ARG (bad sizes/knots), IETI_E_GEOMETRY (det J <= 0), IETI_E_TOPOLOGY
 * (non-conforming interface), IETI_E_NOT_SPD (coarse factorisation), IETI_E_CUDA. */
int ieti_setup(const ieti_setup_args *a, ieti_ctx **out);

/* Patch loads f^(k)_a = int f N_a (Eq. (1)) with a built-in f (IETI_F_*), written to
 * rhs [sum_k prod_d M_kd] (host).  Dirichlet entries are 0. */
int ieti_assemble_load_builtin(ieti_ctx *c, int f_id, double *rhs);

/* Physical quadrature points of the owned patches (Eq. (1) quadrature, (p+1) Gauss points per
 * element and direction, q_1 fastest within a patch, patches in ascending id): xq [n][dim] (host,
 * nullable: then only *n_points is written). */
int ieti_quadrature_points(ieti_ctx *c, double *xq, long long *n_points);

/* Patch loads f_a = sum_q f(x_q) w_q |det J(x_q)| N_a(x_q) (Eq. (1)) from user values
 * f_at_qp [n_points] at the points of ieti_quadrature_points; rhs as in ieti_assemble_load_builtin. */
int ieti_assemble_load(ieti_ctx *c, const double *f_at_qp, double *rhs);

/* Solve with host buffers: rhs = torn patch loads on the full lattices (Dirichlet entries
 * ignored); u = full-lattice coefficients (Dirichlet entries 0); lambda (nullable) = the
 * multipliers in canonical order; iters = PCG iterations (F applications); rel_res =
 * ||r_k||/||r_0|| (R11).  In outer_mode BPCG: iters = BPCG iterations on Eq. (2), rel_res = the
 * relative unpreconditioned residual of Eq. (2) (R31); breakdown = negative curvature.  Returns IETI_OK, IETI_NOT_CONVERGED (outputs valid) or
 * IETI_E_BREAKDOWN (p.Fp <= 0 or non-finite; last iterate written). */
int ieti_solve(ieti_ctx *c, const double *rhs, double *u, double *lambda, int *iters, double *rel_res);

/* Same with device buffers (sizes as above), ordered on cuda_stream (cudaStream_t, NULL=legacy). */
int ieti_solve_device(ieti_ctx *c, const double *d_rhs, double *d_u, double *d_lambda,
                      int *iters, double *rel_res, void *cuda_stream);

/* Fixed-iteration solve (R20): tolerance disabled, exactly `iters` PCG iterations. */
int ieti_solve_fixed(ieti_ctx *c, const double *rhs, int iters, double *u, double *lambda, double *rel_res);

/* info[0..15]: dim, p, n_patches (owned), full dofs (owned patches), n_lambda (local set: owned +
 * ghosts; = global count on one rank), n_pi (global), levels, n_floating, stencil bytes (all
 * levels, both hierarchies), colours, setup ms, basis PCG its (max), kernel launches per PCG
 * iteration, device bytes allocated, n_lambda owned, world size. */
int ieti_info(const ieti_ctx *c, long long info[16]);

/* Canonical multiplier map: for row i, (kp[i], ap[i]) has +1, (km[i], am[i]) has -1
 * (a = full-lattice flat index). */
int ieti_multiplier_map(const ieti_ctx *c, int *kp, int *ap, int *km, int *am);

/* ---- diagnostics (parity tests; host buffers) ------------------------------------- */
enum {
  IETI_OP_F = 0,          /* lambda -> F^ lambda                          (n_lambda -> n_lambda) */
  IETI_OP_MSD = 1,        /* r -> M_sD r                                  (n_lambda -> n_lambda) */
  IETI_OP_D = 2,          /* rhs (full lattices) -> d^ = B K^~^{-1} f     (ndofs -> n_lambda) */
  IETI_OP_NEUMANN = 3,    /* per patch q (full lattices) -> N(q)          (ndofs -> ndofs) */
  IETI_OP_DIRICHLET = 4,  /* per patch s (full lattices, interior used) -> D_c(s) (ndofs -> ndofs) */
  IETI_OP_KTINV = 5,      /* r (full lattices) -> K^~^{-1} r              (ndofs -> ndofs) */
  IETI_OP_VCYCLE_N = 6,   /* one Neumann V-cycle from x=0 (N_1)           (ndofs -> ndofs) */
  IETI_OP_KT = 7,         /* u -> (K^(k) u^(k))_k, the true K (R28)      (ndofs -> ndofs) */
  IETI_OP_CAN = 8,        /* r -> null-part-free representative (R31)     (ndofs -> ndofs) */
  IETI_OP_KHAT = 9        /* r -> K^~^-1 r = Ktilde^-1_{N_c} r / s (R29)   (ndofs -> ndofs; outer_mode BPCG) */
};
int ieti_apply(ieti_ctx *c, int op, const double *in, double *out);

/* Stencil of one grid: hier 0 = Neumann, 1 = Dirichlet; level 0 = coarsest.  out =
 * [rows][ (2p+1)^d ] over the ACTIVE rows in lexicographic order; offsets o = (o_1..o_d)
 * in [-p,p]^d, o_1 fastest.  n_rows returns the active row count (out may be NULL). */
int ieti_get_stencil(ieti_ctx *c, int hier, int level, int patch, double *out, int *n_rows);

/* Primal basis Phibar^(k) of Eq. (6): out [n_pi_k][full lattice] (column j contiguous). */
int ieti_get_primal_basis(ieti_ctx *c, int patch, double *out, int *n_pi_k);

/* Device timing of the dominant kernel class, measured with CUDA events recorded inside the
 * per-iteration graphs (on the library's stream) while timing is enabled:
 *   class 0 = finest-level Neumann colour-SGS sweeps, class 1 = finest-level Dirichlet sweeps;
 *   t_ms[i] = accumulated sweep time, n[i] = colour-phase kernel launches, bytes[i] = their
 *   accumulated algorithmic bytes.
 *   n[7] = kernel launches of the last solve; t_ms[7] = kernel launches per PCG iteration.
 * enable switches accumulation on/off for subsequent solves; reset zeroes the accumulators
 * before the values are returned.  Any pointer may be NULL. */
int ieti_timing(ieti_ctx *c, int enable, int reset, double t_ms[8], long long n[8], double bytes[8]);

/* Rank 0 creates the NCCL unique id (128 bytes into out128) that every rank passes in
 * ieti_setup_args.nccl_unique_id.  Returns IETI_E_NCCL if NCCL cannot be loaded. */
int ieti_nccl_unique_id(void *out128);

/* Local multiplier set of this rank: global_ids [ieti_info[4]] = owned multipliers (the first
 * ieti_info[14]) then ghosts, each in canonical order; local_patches [ieti_info[2]] = global ids
 * of the owned patches.  Either pointer may be NULL. */
int ieti_local_multipliers(const ieti_ctx *c, int *global_ids, int *local_patches);

/* Host-only partition plan (no GPU; used by the multi-rank CPU tests).  For (rank, world) and the
 * args' geometry / patch_owner: out = {owned patches, local multipliers, owned multipliers, peers,
 * forward-send entries, forward-recv entries}.  ieti_plan_get fills (nullable) local_patches
 * [out0], local_mult [out1] (global ids, owned first), peers [out3], send_ptr/recv_ptr [out3+1],
 * send_idx [out4] (local indices of my owned rows each peer holds as ghosts) and recv_idx [out5]
 * (local indices of my ghost rows, per owning peer).  The reverse exchange uses the same lists
 * with roles swapped; owners add received partials in ascending peer order. */
int ieti_plan_info(const ieti_setup_args *a, int rank, int world, long long out[6]);
int ieti_plan_get(const ieti_setup_args *a, int rank, int world, int *local_patches, int *local_mult, int *peers,
                  int *send_ptr, int *send_idx, int *recv_ptr, int *recv_idx);

/* Inner-iteration log of the last solve in LOCAL_PCG mode (C2, reading R19): for every local
 * Neumann solve call (d^, each F^ application, the recovery, in call order) the per-patch inner
 * PCG iteration counts.  counts [max_calls][n_patches] (nullable); n_calls = calls logged.
 * Empty (n_calls = 0) in LOCAL_VCYCLES mode. */
int ieti_inner_log(const ieti_ctx *c, int *counts, int max_calls, int *n_calls);

const char *ieti_last_error(const ieti_ctx *c);
void ieti_destroy(ieti_ctx *c);

/* Solve-phase and V-cycle timing, accumulated while ieti_timing(enable=1) is on (CUDA events on the
 * library stream; DESIGN.md 9 "Measurement"): out[0] = ms of d^ + PCG start (BPCG: start), out[1] = ms
 * of the outer loop, out[2] = ms of the recovery, out[3] = solves; out[4..7] = Neumann c-V-cycle
 * sets (all levels): ms, algorithmic bytes, the survey's 3-stream reference bytes
 * 8 n_l (3S + 12) per level + 8 n_0^2, count; out[8..11] the same for the Dirichlet
 * V-cycles of M_sD.  reset zeroes these accumulators after reading. */
int ieti_phase_times(ieti_ctx *c, int reset, double out[16]);

/* BPCG calibration (outer_mode = IETI_OUTER_BPCG, R30): out[0] = s, out[1] = theta_min,
 * out[2] = theta_max (Ritz values of K^~_1^-1 K~), out[3] = Lanczos steps taken.  IETI_E_ARG in
 * the dual-PCG mode. */
int ieti_bpcg_info(const ieti_ctx *c, double out[4]);

/* Build provenance (no paper passage: engineering): a static string
 * "src=<sha256[:16] of the library sources> arch=sm_100a nvcc_flags=..." compiled into the library by
 * paper_1705_04531_b200/build.py.  The Python binding refuses a library whose hash differs from the
 * sources next to it, and bench.py records it, so every run names the sources it executed.
 * Never NULL; owned by the library. */
const char *ieti_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* IETI_H */
