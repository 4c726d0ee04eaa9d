// internal.h -- shared host/device declarations of libieti (not part of the C ABI).
//
// Data layout in HBM:
//  * A "grid" is one MG level of one hierarchy (Neumann or Dirichlet) of one patch.
//    Its vectors live on a zero-padded box of (M_d + 2p) points per direction (halo p),
//    so a stencil read a+o never leaves the box and never needs a bounds check.
//  * Stencil coefficients of a grid: padded full rows, (2p+1)^d per ACTIVE row (R24),
//    rows in colour-major order (R6 colours, then lexicographic inside the colour's
//    sub-lattice), stored offset-major: coef[coef_off + o*ld + r].  A colour phase
//    therefore streams one contiguous, coalesced range per offset.
//  * A "problem" is one right-hand side on one grid; a batch of problems (all patches,
//    or (patch, column) pairs in the primal-basis setup) is one kernel launch.
#pragma once
#include <cstdint>
#include <cstddef>
#include <stdexcept>
#include <string>
#include <vector>
#include <memory>
#include <array>
#include <cuda_runtime.h>

#define IETI_MAXD 3

struct GridDesc {
  int M[3];          // full lattice dims at this level (unused dims = 1)
  int lo[3], hi[3];  // active box [lo, hi)
  int ns[3];         // sub-lattice box dims ceil(M/(p+1)) + 2 (unused dims = 1); layout.cuh
  int sb;            // ns[0]*ns[1]*ns[2]
  int nrows;         // active rows
  int ld;            // coefficient leading dimension (>= nrows, multiple of 32)
  int tg;            // coefficient interleave of the layout (always 1: offset-major rows)
  int col_off;       // first ColourInfo of this grid
  int box;           // (p+1)^d * sb
  long long coef_off;// offset (doubles) of the coefficient block in the level pool
  double mass_beta;  // on-the-fly parameter-mass coefficient used by spmv_mass (0 = none)
  int mass_off;      // offset (doubles) of the 1D mass tables [d][M_d][2p+1]
  int patch;         // owning patch (local index)
  int tpr;           // threads per stencil row in the kernels (1 on bandwidth-bound levels, 4/8 on small ones)
  int ent_off;       // offset (int2 units) of the grid's offset tables in the level pool: per colour c,
                     // [c][0][o] = (o, box delta) in natural order, [c][1][i] = (o, delta) for the
                     // lower-colour offsets then the higher-colour ones (diagonal excluded)
  int pad2_;
};

struct ColourInfo {  // rows of colour c: lattice i_d = first_d + (p+1) j_d, j_d < n_d
  int start;         // first colour-major row
  int n[3];
  int first[3];
  int pad_;
};

struct ProbDesc {
  int grid;          // index into the level's GridDesc array
  int pad_;
  long long vec_off; // offset (doubles) of this problem's box vector in the level vector pools
};

struct BlockEntry {  // one thread block of a batched launch
  int prob;
  int colour;        // colour (stencil kernels) or -1 (point kernels)
  int row0;          // first row of the colour (or first active point) handled by the block
  int nrow;          // rows in this block
};

struct BandDesc {     // one banded SPD system of the direct local solvers (kernels_direct.cu)
  int n;             // unknowns
  int bw;            // half bandwidth
  long long off;     // first entry of its n * (bw + 1) lower band (and of its transposed band)
};

struct TransDesc {   // 1D knot-insertion tables of P (level l-1 -> l) of one grid pair
  int rc_off[3];     // restriction: per coarse index a: first fine index (int pool) ...
  int rw_off[3];     //   ... and (p+2) weights (double pool)
  int pf_off[3];     // prolongation: per fine index i: first coarse index ...
  int pw_off[3];     //   ... and W weights
  int W;             // max coarse contributors per fine index
  int pad_;
};

// ---- host-side topology (host_topology.cpp) --------------------------------------------
struct HostPatch {
  int p;
  int M[3];
  int melem[3];
  std::vector<double> knots[3];
  std::vector<double> ctrl;      // [n][dim]
};

struct Topo {
  int dim = 0, p = 0, n_patches = 0;
  std::vector<HostPatch> patch;
  // per patch
  std::vector<int> floating;
  std::vector<std::array<int, 6>> dir_side;        // [d*2+s] = 1 if Dirichlet
  std::vector<std::vector<int>> gamma;             // full flat indices of Gamma^(k) (ascending)
  // multipliers (canonical, R12)
  int n_lambda = 0;
  std::vector<int> mkp, map_, mkm, mam;             // (k+, a+, k-, a-)
  // B_D per multiplier: list of (patch, flat, weight); B_D^T per (patch, flat): (mult, weight)
  std::vector<int> bd_ptr; std::vector<int> bd_k, bd_a; std::vector<double> bd_w;
  // primal constraints
  int n_pi = 0;
  std::vector<std::vector<int>> R;                 // per patch: local row -> global primal id
  std::vector<std::vector<int>> c_row;             // per patch, per Gamma entry: local row or -1
  std::vector<std::vector<double>> c_w;            // per patch, per Gamma entry: weight
  // per patch per Gamma entry: Bt lists (mult, weight=+-1) and BDt lists (mult, weight)
  std::vector<std::vector<int>> bt_ptr, bt_m; std::vector<std::vector<double>> bt_w;
  std::vector<std::vector<int>> bdt_ptr, bdt_m; std::vector<std::vector<double>> bdt_w;
  std::string err;
};

int build_topology(int dim, int n_patches, const int *degree, const int *n_knots, const double *knots,
                   const double *ctrl, unsigned primal, Topo &T);

// ---- multi-GPU partition and exchange plan (partition.cpp) -------------------------------
struct Plan {
  int rank = 0, world = 1;
  std::vector<int> local_patches;   // global ids, ascending
  std::vector<int> local_mult;      // global multiplier ids: owned (canonical) then ghosts (canonical)
  int n_own = 0;
  std::vector<int> peers;           // ranks exchanged with, ascending
  std::vector<int> send_ptr, send_idx;   // per peer: my owned rows in the peer's set (local idx)
  std::vector<int> recv_ptr, recv_idx;   // per peer: my ghost rows owned by the peer (local idx)
  std::vector<int> rsum_ptr, rsum_src;   // owned row -> positions of received partials (reverse)
  std::vector<int> gkp, gkm;             // global patch ids (k+, k-) of the local multipliers
};
std::vector<int> default_owner(int n_patches, int world);
int build_partition(const Topo &G, const std::vector<int> &owner, int rank, int world, Topo &L, Plan &P);

// ---- NCCL (comm.cpp; loaded with dlopen only when world > 1) -----------------------------
struct CommError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct LoopGroup;
struct Comm {
  int rank = 0, world = 1;
  void *comm = nullptr;
  std::shared_ptr<LoopGroup> loop;      // in-process loopback group (tests): eager calls only
  void init(const void *uid128, int rank, int world, bool force = false);   // force: NCCL even for 1 rank
  void destroy();
  void allgather(const double *send, double *recv, size_t count, cudaStream_t s);
  void allreduce_sum(double *buf, size_t count, cudaStream_t s);
  void exchange(const std::vector<int> &peers, const double *send, const std::vector<int> &send_ptr, double *recv,
                const std::vector<int> &recv_ptr, cudaStream_t s);
};
int comm_unique_id(void *out128, std::string &err);

// host B-spline utilities (independent C++ implementation; host_topology.cpp)
void bspline_basis_ders(const std::vector<double> &t, int p, double x, int nder, int &span, double *out);
void gauss_legendre01(int n, double *x, double *w);
std::vector<double> knot_insertion_dense(const std::vector<double> &tc, int p, const std::vector<double> &tf,
                                         int &Mf, int &Mc);
std::vector<double> coarsen_knots(const std::vector<double> &t, int p);
std::vector<double> mass_1d(const std::vector<double> &t, int p);   // dense M x M

// ---- kernel launchers (kernels_*.cu) ------------------------------------------------------
struct LevelView {             // what the stencil kernels need for one batched launch
  const GridDesc *grids;
  const ColourInfo *cinfo;
  const ProbDesc *probs;
  const double *coef;
  const double *mass;          // 1D mass pool (may be null)
  const int2 *ent;             // per-grid offset tables (GridDesc::ent_off)
  long long nvec = 0;          // length of the level's vector pool (bounds checks, IETI_DEBUG_BOUNDS builds)
};

struct PatchIface {            // per patch interface descriptor (device array)
  int g_off;                   // first global Gamma index
  int ng;                      // |Gamma_k|
  int npi;                     // n_Pi^(k)
  int pi_off;                  // first entry in the per-patch t / R arrays
  long long phi_off;           // Phibar_G (column-major [npi][ng]) offset
  long long phif_off;          // full Phibar (column-major [npi][box]) offset
  long long box_off;           // fine-level box offset of the patch (vector pools)
  int box;                     // fine-level box size
  int floating;                // 1 if the patch has no Dirichlet side (K singular, kernel = constants)
};

// fused V-cycle over the small levels 0..ltop of a batch: one thread-block cluster per problem
// (kernels_mg.cu, k_vcycle_fused)
#define IETI_MAXL 10
struct FusedLevel {
  const GridDesc *grids;
  const ColourInfo *cinfo;
  const int2 *ent;
  const ProbDesc *probs;
  const double *coef;
  double *x, *b, *r, *d;       // level vectors of the batch (d: forward increments, may be null)
  const TransDesc *td;         // P from level l-1 to l (l >= 1)
  const int *ip;
  const double *wp;
};
struct FusedArgs {
  FusedLevel lev[IETI_MAXL];
  const long long *inv_off;    // coarsest explicit inverse
  const double *inv;
  const short *olist, *nlow;
  int ltop, zero_top, ncol, max_coarse_rows;
  int slab;                    // doubles per coefficient buffer (max rows per CTA slice x S + 2)
  int tprf;                    // threads per row (power of two <= 32)
};
void launch_vcycle_fused(int dim, int p, const FusedArgs &a, int nprob, int cs, cudaStream_t s);

// kernels_mg.cu
// stencil kernels: tpr = threads per row (1 on large grids, 4 on small ones); olist / nlow = the
// per-colour offset lists (lower-colour offsets first, then higher-colour ones; see kernels_mg.cu)
// pcol: colour of the next phase of the sweep (its coefficients are prefetched into L2 on the
// small row-major levels), -1 for none
void launch_sgs_phase(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks, double *x,
                      const double *b, double *dx, int pcol, cudaStream_t s);
void launch_sgs_phase_zero(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                           double *x, const double *b, const short *olist, const short *nlow, int pcol, cudaStream_t s);
void launch_residual(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                     const double *x, const double *b, double *y, cudaStream_t s);
void launch_residual_upper(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                           const double *dsrc, double *y, const short *olist, const short *nlow, cudaStream_t s);
void launch_apply(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                  const double *x, double *y, double scale, cudaStream_t s);
void launch_mass_add(int dim, int p, const LevelView &lv, const BlockEntry *blocks, int nblocks, int nthr,
                     const double *x, double *y, cudaStream_t s);
void launch_sgs_phase_u(int dim, int p, int tpr, int mode, const LevelView &lv, const BlockEntry *blocks,
                        int nblocks, double *x, const double *b, double *u, double *dx, const short *olist,
                        const short *nlow, int pcol, cudaStream_t s);
// one whole colour sweep (all phases) of a row-major level, one thread-block cluster of cs CTAs per
// problem (kernels_sweep.cu; mode 0 / 4 / 6 / 7 as k_stencil; slab 0: coefficients read from global
// memory; rep > 0: x replicated per CTA in shared memory, rep >= box + 2 guard doubles); query = true
// returns the co-resident cluster count instead (<= 0: the configuration cannot run), else 1 on
// success / -1 on a launch error
int launch_sweep_cluster(int dim, int p, int tpr, int mode, const LevelView &lv, int nprob, int cs, int nthr, int slab,
                         int rmax, int rep, int guard, int ncol, bool fwd, double *x, const double *b, double *dx,
                         double *U, const short *nlow, cudaStream_t s, bool query);
bool launch_sweep(int dim, int p, int tpr, int mode, const LevelView &lv, const BlockEntry *blocks, const int2 *ptab,
                  int nphase, int maxent, unsigned *bar, double *x, const double *b, double *u, double *dx,
                  const short *olist, const short *nlow, cudaStream_t s);
void launch_rowlist(int dim, int p, const GridDesc *grids, const ProbDesc *probs, const BlockEntry *blocks, int nblocks,
                    const double *coef, long long ld, const int *rpos, const int *rout, const double *x,
                    const double *x2, double *y, int out_mode, cudaStream_t s);
void launch_restrict(int dim, int p, const GridDesc *gc, const GridDesc *gf, const TransDesc *td,
                     const ProbDesc *pc, const ProbDesc *pf, const int *ipool, const double *wpool,
                     const BlockEntry *blocks, int nblocks, int nthr, const double *rf, double *bc, double *xc,
                     cudaStream_t s);
void launch_prolong(int dim, int p, const GridDesc *gc, const GridDesc *gf, const TransDesc *td,
                    const ProbDesc *pc, const ProbDesc *pf, const int *ipool, const double *wpool,
                    const BlockEntry *blocks, int nblocks, int nthr, const double *xc, double *xf,
                    cudaStream_t s);
void launch_coarse_solve(const GridDesc *g, const ProbDesc *pr, const long long *inv_off, const double *inv,
                         int nprob, int dim, int p, const double *b, double *x, int max_rows, cudaStream_t s);
void launch_galerkin_stages(int dim, int p, const GridDesc &gf, const ColourInfo *cif, const GridDesc &gc,
                            const ColourInfo *cic, const TransDesc &td, int CW, const int *cwin, const int *ipool,
                            const double *wpool, const double *coef_f, double *coef_c, double *B, int ncol,
                            cudaStream_t s);
void launch_dense_from_stencil(int dim, int p, const GridDesc *g, const ColourInfo *ci, const double *coef,
                               int ngrid, double *dense, const long long *dense_off, cudaStream_t s, int max_rows);
void launch_spd_inverse2(double *dense, const long long *dense_off, const int *n, int ngrid, double *scratch,
                         const long long *scratch_off, int *fail, cudaStream_t s);

// kernels_asm.cu
void launch_geometry2(int dim, int p, const int *nq, const int *M, const double *val, const double *der,
                      const int *toff, const double *wq, const int *woff, const double *ctrl, double *G, double *X,
                      double *detw, int *bad, cudaStream_t s);
long long sf_scratch_doubles(int dim, int p, const int *M, const int *melem);
void launch_stencil_sf(int dim, int p, const GridDesc &g, const ColourInfo *ci, int ncol, const int *melem,
                       const double *val, const double *der, const int *toff_host, const double *G, double alpha,
                       const double *mass, double *coef, double *scratch, cudaStream_t s);
void launch_mul(long long n, const double *f, const double *detw, double *fw, cudaStream_t s);
void launch_eval_f2(int dim, int f_id, const double *X, const double *detw, long long n, double *fw, cudaStream_t s);
void launch_load2(int dim, int p, const int *M, const int *melem, const int *lo, const int *hi, const double *val,
                  const int *toff, const double *fw, double *rhs, cudaStream_t s);

// kernels_ieti.cu
void ik_iface_t(int npatch, const void *pif, const int *gbox, const int *bt_ptr, const int *bt_m, const double *bt_w,
                const double *phiG, const int *crow, const double *cw, const double *lam, double *t_all, double *bN,
                double *rG, cudaStream_t s);
void ik_full_t(int npatch, const void *pif, const int *gbox, const int *bt_ptr, const int *bt_m, const double *bt_w,
               const double *phiF, const int *crow, const double *cw, const double *lam, const double *fbox,
               double *t_all, double *bN, cudaStream_t s, int ngamma = 0, int max_npi = 0, double *rG = nullptr);
void ik_gather_pi(int n_pi, const int *ptr, const int *src, const double *t_all, double *g, cudaStream_t s);
void ik_gemv(int n, const double *A, const double *x, double *y, cudaStream_t s);
void ik_iface_w(int npatch, const void *pif, const int *gbox, const double *phiG, const int *c_ptr, const int *c_idx,
                const double *cw, const int *Rg, const double *uPi, const double *xN, double *cvec, double *wG,
                cudaStream_t s);
void ik_full_u(int npatch, int maxbox, const void *pif, const double *phiF, const double *cvec, const double *xN,
               double *ubox, cudaStream_t s);
void ik_jump(int n, const int *gp, const int *gm, const double *wG, double *q, cudaStream_t s);
void ik_bdt(int ngamma, const long long *gabs, const int *ptr, const int *m, const double *w, const double *r,
            double *vbox, cudaStream_t s);
void ik_bd_gather(int n, const int *ptr, const int *gi, const double *w, const long long *gabs, const double *y,
                  double *z, cudaStream_t s);
void ik_dot_partial(long long n, const double *a, const double *b, double *partial, int nb, cudaStream_t s);
void ik_pcg_alpha(const double *partial, int nb, double *sc, cudaStream_t s);
void ik_pcg_update(long long n, const double *sc, const double *p, const double *q, double *lam, double *r,
                   double *partial, int nb, cudaStream_t s);
void ik_store_scalar(const double *partial, int nb, double *sc, int slot, int take_sqrt, cudaStream_t s);
void ik_pcg_beta(const double *partial, int nb, double *sc, cudaStream_t s);
void ik_pcg_p(long long n, const double *sc, const double *z, double *p, int nb, cudaStream_t s);
void ik_copy(long long n, const double *a, double *b, cudaStream_t s);
void ik_scale_copy(long long n, double sc, const double *a, double *b, cudaStream_t s);
void ik_lattice_to_box(int dim, int p, int npatch, long long maxn, const GridDesc *g, const ProbDesc *pr,
                       const long long *loff, const double *lat, double *box, int only_interior, cudaStream_t s);
void ik_box_to_lattice(int dim, int p, int npatch, long long maxn, const GridDesc *g, const ProbDesc *pr,
                       const long long *loff, const double *box, double *lat, cudaStream_t s);
void ik_mask_box(int dim, int p, int nprob, int maxbox, const GridDesc *g, const ProbDesc *pr, double *v, cudaStream_t s);
// multi-GPU exchange helpers
void ik_pack(int n, const int *idx, const double *src, double *dst, cudaStream_t s);
void ik_unpack(int n, const int *idx, const double *src, double *dst, cudaStream_t s);
void ik_rsum(int n_own, const int *ptr, const int *srcpos, const double *recv, double *v, cudaStream_t s);
void ik_sum_ranks(int n, int world, const double *all, double *out, cudaStream_t s);
void ik_reduce_to(const double *partial, int nb, double *out, cudaStream_t s);
// direct local solvers (banded Cholesky; D-D / MG-D)
void ik_band_factor(int nprob, const BandDesc *bd, double *band, double *up, long long max_len, int *info,
                    cudaStream_t s);
void ik_band_solve(int nprob, int max_bw, const BandDesc *bd, const double *band, const double *up,
                   const long long *voff, double *v, cudaStream_t s);
void ik_gather_pos(long long n, const long long *pos, const double *box, double *v, cudaStream_t s);
void ik_scatter_pos(long long n, const long long *pos, const double *v, double *box, cudaStream_t s);
// MG-MG-S (BPCG on Eq. (2), R28-R31)
void ik_can_add(int npatch, const void *pif, const int *gbox, const int *crow, const double *cw, const int *R,
                const double *g, const double *invmult, const double *bN, double *out, cudaStream_t s);
void ik_bt_add(int ngamma, const long long *gabs, const int *ptr, const int *m, const double *w, const double *lam,
               double *box, cudaStream_t s);
void ik_jump_box(int n, const int *gp, const int *gm, const long long *gabs, const double *box, double *q,
                 cudaStream_t s);
void ik_axpy_s(long long n, const double *sc, int slot, double sign, const double *x, double *y, cudaStream_t s);
void ik_xpby_s(long long n, const double *sc, int slot, const double *x, double *y, cudaStream_t s);
void ik_sub(long long n, const double *a, const double *b, double *out, cudaStream_t s);
void ik_bp_scalar(int op, double *sc, cudaStream_t s);
// C2 inner PCG (R19), one block per patch
void ik_inner_init(int nprob, const ProbDesc *pr, const GridDesc *g, const double *q, double *r, double *x, double *qn,
                   int *active, int *its, int *ctr, cudaStream_t s);
void ik_inner_dir(int nprob, const ProbDesc *pr, const GridDesc *g, const double *r, const double *z, double *p,
                  double *rho, const int *active, int first, cudaStream_t s);
void ik_inner_begin(int *ctr, cudaStream_t s);
void ik_inner_step(int nprob, const ProbDesc *pr, const GridDesc *g, const double *p, const double *Ap, double *x,
                   double *r, const double *rho, const double *qn, int *active, int *its, int *ctr, double tol,
                   const int *proj, int pdeg, int dim, cudaStream_t s);

// kernels_basis.cu (primal-basis setup: per-problem segmented operations)
void bk_rhs_ct(int nprob, const int *prob_patch, const int *prob_col, const ProbDesc *pr, const void *pif,
               const int *gbox, const int *crow, const double *cw, double *b, cudaStream_t s);
void bk_seg_dot(int nprob, const ProbDesc *pr, const GridDesc *g, const double *a, const double *b, double *out,
                cudaStream_t s);
void bk_seg_axpy(int nprob, const ProbDesc *pr, const GridDesc *g, const double *coef, double sign, const double *x,
                 double *y, const int *active, cudaStream_t s);
void bk_seg_xpby(int nprob, const ProbDesc *pr, const GridDesc *g, const double *z, const double *beta, double *p,
                 const int *active, cudaStream_t s);
void bk_cx(int nprob, const int *prob_patch, const ProbDesc *pr, const void *pif, const int *gbox, const int *crow,
           const double *cw, const double *x, double *out, int out_stride, cudaStream_t s);
void bk_combine(int npatch, int maxbox, const void *pif, const long long *hoff, const double *Hinv,
                const double *cconst, const GridDesc *g, int p, int dim, const double *src, double *dst,
                cudaStream_t s);
void bk_phi_dots(int nprob, const int *prob_patch, const ProbDesc *pr, const void *pif, const double *phif,
                 const double *y, double *out, int stride, cudaStream_t s);
void bk_extract_gamma(int npatch, int maxng, const void *pif, const int *gbox, const double *phif, double *phiG,
                      cudaStream_t s);
void bk_prob_cols(int nprob, int maxbox, const int *prob_patch, const int *prob_col, const ProbDesc *pr,
                  const void *pif, const double *x, double *cols, int to_cols, cudaStream_t s);
// dst[o * ostride + row * rstride] = coef of source row rrow[row] (+ mass_beta * Mhat): (ld, 1) for
// offset-major targets, (1, S) for row-major ones
void launch_extract_rows(int dim, int p, const GridDesc *g, const double *coef, const double *mass, const int *rgrid,
                         const int *rrow, const int *rflat, long long nrows, double *dst, long long ostride,
                         long long rstride, cudaStream_t s);
