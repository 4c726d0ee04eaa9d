// solver.cu -- libieti: setup and the dual-PCG hot path of inexact IETI-DP on one B200.
//
// Orchestrates the kernels of kernels_*.cu (see DESIGN.md for the data layout and the
// readings R1-R25).  The C-ABI entry points are at the end of the file (include/ieti.h).
//
// Per dual-PCG iteration, all patches batched per launch:
//   q = F^ p : B^T p -> t = Phibar_G^T r -> u_Pi = S^-1 sum R^T t -> b = r - C^T t
//              -> x = N_c(b) (c V-cycles, Neumann hierarchy) -> w = x + Phibar_G(R u_Pi - C x) -> B w
//   alpha, lambda, r updates (deterministic reductions)
//   z = M_sD r : v = B_D^T r -> b_D = -K_IG v -> z_I = D_c(b_D) -> y = K (v + z_I) -> B_D y
//   beta, p update
// Both halves are captured once as CUDA graphs; the host reads ||r|| once per iteration.
#include "../../include/ieti.h"
#include "layout.cuh"

#include <nvtx3/nvToolsExt.h>   // header-only NVTX ranges (tracing with nsys / ncu --nvtx)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

// NVTX range for the host-side phases (setup stages, d^, PCG iterations, inner loops, recovery)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace {

struct IetiError : public std::runtime_error {
  int code;
  IetiError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      throw IetiError(IETI_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +     \
                                       std::to_string(__LINE__));                                  \
  } while (0)

inline long long ipow(long long b, int e) {
  long long r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

struct Level {
  std::vector<GridDesc> g;
  GridDesc *d_g = nullptr;
  std::vector<ColourInfo> ci;
  ColourInfo *d_ci = nullptr;
  double *coef = nullptr;
  long long coef_n = 0;
  double *mass = nullptr;                 // 1D mass tables (fine Neumann level)
  int2 *ent = nullptr;                    // per-grid offset tables (GridDesc::ent_off)
  std::vector<long long> inv_off;         // coarsest
  long long *d_inv_off = nullptr;
  double *inv = nullptr;
};

struct Hier {
  bool dirichlet = false;
  std::vector<Level> lev;
};

struct Trans {                            // P from level l-1 to l (shared by both hierarchies)
  std::vector<TransDesc> td;
  TransDesc *d_td = nullptr;
  int *ip = nullptr;
  double *wp = nullptr;
  int CW = 0;
  std::vector<int> cwin;                  // [patch][3][4096]
  int *d_cwin = nullptr;
};

struct BLevel {
  std::vector<ProbDesc> pr;
  ProbDesc *d_pr = nullptr;
  double *x = nullptr, *b = nullptr, *r = nullptr, *d = nullptr;
  double *U = nullptr;                    // finest level, >= 2 cycles: higher-colour sums (modes 6/7)
  long long n = 0;
  std::vector<long long> rows_col;
  double phase_bytes = 0;                 // coefficient bytes of one colour phase (all problems)
  BlockEntry *d_cblk = nullptr;           // colour blocks (colour-major)
  BlockEntry *d_rblk = nullptr;           // the same blocks, problem-major
  std::vector<int> cofs;
  int ngroups = 1;                        // problem groups of the sweeps (x L2-resident per group)
  std::vector<int> gofs;                  // [colour][group + 1] first block of each group
  int2 *d_ptab = nullptr;                 // persistent sweep (k_sweep): [group][fwd, bwd][phase] = (first block, count)
  int ptab_max = 0;                       // most blocks of one phase
  int cnthr = 128;
  BlockEntry *d_pblk = nullptr;           // active-point blocks
  int npblk = 0;
  int maxbox = 0;
  int cl_cs = 0;                          // > 0: every sweep of this level is ONE cluster launch (k_sweep_cl,
                                          // kernels_sweep.cu) with cl_cs CTAs per problem
  int cl_slab = 0;                        //      its shared-memory coefficient buffer (doubles)
  int cl_rmax = 0;                        //      most rows of one CTA's slice of a colour
  int cl_nthr = 256;                      //      threads per CTA
  int cl_rep = 0;                         //      > 0: doubles of the per-CTA x replica (shared memory)
  int guard = 32;                         // zero/neighbour guard of the vector pool before the first box
};

struct Batch {
  Hier *H = nullptr;
  int nprob = 0;
  std::vector<int> prob_grid;
  std::vector<BLevel> lv;
  int ftop = -1;               // levels 0..ftop run as one fused launch per V-cycle (k_vcycle_fused)
  int fcs = 1;                 // cluster size (CTAs per problem) of the fused launch
  int fslab = 0, ftprf = 8;    // fused launch: coefficient buffer (doubles) and threads per row
};

// Independent PCG per problem of a batch (finest level), preconditioner = one V-cycle of the
// batch's hierarchy, per-problem scalars on the device, per-problem stopping at
// ||r|| <= tol ||q|| (converged problems are masked).  Used by C2's inner local solves (R19)
// and the primal-basis setup (Eq. (6)).  q is read from the batch's finest rhs box.
struct BatchedPcg {
  Batch *B = nullptr;
  double *X = nullptr, *R = nullptr, *P = nullptr, *AP = nullptr, *rho = nullptr, *qn = nullptr;
  int *active = nullptr, *its = nullptr, *ctr = nullptr, *ctr_host = nullptr;
  const int *proj = nullptr;   // per problem: project r onto range(K) (floating patches; basis only)
  double tol = 1e-6;
  int maxit = 200;
  std::function<void(const double *, double *, cudaStream_t)> applyA;
  cudaGraphExec_t g_init = nullptr, g_body = nullptr;
  int kn[2] = {0, 0};
};

}  // namespace

struct ieti_ctx {
  ieti_setup_args a{};
  Topo T;
  int dim = 0, p = 0, P1 = 0, S = 0, ncol = 0, L = 0, npatch = 0;
  std::string err;
  cudaStream_t st = nullptr;
  cudaStream_t st_aux[3] = {nullptr, nullptr, nullptr};   // branches of the concurrent x-group sweeps
  cudaEvent_t ev_fork = nullptr, ev_join[3] = {nullptr, nullptr, nullptr};
  int xgconc = 1;                         // IETI_XGCONC: x-groups of one sweep on concurrent streams (0: serial)
  int xg_big = 1;                         // IETI_XG_BIG: at least this many concurrent groups on big levels
  int xg_small = 2;                       // IETI_XG_SMALL: concurrent problem groups on heavy row-major levels
                                          // (C5 level 2: 2 -> +3 %, 4 -> +3.3 %, measured)
  std::vector<void *> allocs;
  size_t bytes_alloc = 0;

  // per patch (fine level)
  std::vector<std::array<std::vector<double>, 3>> knots_lv;   // [patch][d] at fine level (for reference)
  std::vector<std::vector<std::array<std::vector<double>, 3>>> kl;  // [level][patch][d]
  std::vector<long long> lat_off;         // full-lattice offsets of patches
  long long ndofs = 0;
  int *d_M = nullptr;                     // [patch][3] fine M
  long long *d_lat_off = nullptr, *d_box_off = nullptr;
  std::vector<long long> box_off;
  int maxbox = 0;
  long long maxlat = 0;

  // assembly tables
  std::vector<std::array<int, 3>> toff_h;  // per patch per dir offset into tab pools
  double *d_val = nullptr, *d_der = nullptr, *d_wq = nullptr;
  std::vector<std::array<int, 3>> woff_h;
  int *d_toff = nullptr, *d_woff = nullptr; // [patch][3]
  double *d_ctrl = nullptr;
  std::vector<long long> ctrl_off;

  Hier HN, HD;
  std::vector<Trans> tr;                  // [level]
  Batch BN, BD;                           // hot-path batches

  // interface
  int ngamma = 0;
  std::vector<PatchIface> pif;
  PatchIface *d_pif = nullptr;
  int *d_gbox = nullptr;
  long long *d_gabs = nullptr;
  int *d_bt_ptr = nullptr, *d_bt_m = nullptr;
  double *d_bt_w = nullptr;
  int *d_bdt_ptr = nullptr, *d_bdt_m = nullptr;
  double *d_bdt_w = nullptr;
  int *d_crow = nullptr;
  int *d_cptr = nullptr, *d_cidx = nullptr;  // per (patch, primal row j): its Gamma entries (CSR over pi_off + j)
  double *d_cw = nullptr;
  int *d_gp = nullptr, *d_gm = nullptr;
  int *d_bd_ptr = nullptr, *d_bd_g = nullptr;
  double *d_bd_w = nullptr;
  int *d_R = nullptr;
  int *d_gpi_ptr = nullptr, *d_gpi_src = nullptr;
  int npi_tot = 0;
  double *phiG = nullptr, *phiF = nullptr;
  long long phiG_n = 0, phiF_n = 0;
  double *Sinv = nullptr;
  int basis_its = 0;

  // explicit row-list stencils of M_sD (true K): Gamma rows (y_G = K_GG v + K_GI z) and the
  // interior band coupled to Gamma (b_D = -K_IG v); rows grouped by (patch, colour)
  struct RowList {
    double *coef = nullptr;
    long long ld = 0;
    int *pos = nullptr, *out = nullptr;
    BlockEntry *blk = nullptr;
    int nblk = 0;
    long long nrows = 0;
  } RG, RB;
  double *yG = nullptr;
  // work vectors
  double *t_all = nullptr, *cvec = nullptr, *gPi = nullptr, *uPi = nullptr, *rG = nullptr, *wG = nullptr;
  double *vbox = nullptr, *ybox = nullptr, *fbox = nullptr, *ubox = nullptr;
  double *lam = nullptr, *r = nullptr, *z = nullptr, *pv = nullptr, *q = nullptr;
  double *partial = nullptr, *sc = nullptr, *sc_host = nullptr;
  double *lat_tmp = nullptr, *lat_tmp2 = nullptr;
  int nb_dot = 1;

  // graphs 0 (d^ and PCG start), 1 (F^ half-iteration), 2 (M_sD half-iteration), 3 (recovery), each
  // a list of captured segments split around the host-driven inner PCG loops (LOCAL_PCG, R19;
  // DIRICHLET_PCG, R27): a loop runs the captured graphs g_init / g_body of its BatchedPcg until
  // no patch is active (the host reads the active count once per inner iteration)
  struct Seg { cudaGraphExec_t g = nullptr; int kn = 0; int loop = 0; };   // loop: 1 Neumann, 2 Dirichlet
  std::vector<Seg> prog[16];              // 0-3 dual PCG; 10-12: the BPCG programs (outer_mode BPCG)
  std::function<void()> prog_fn[16];      // the programs' bodies (run eagerly in loopback groups)
  std::vector<Seg> *rec_segs = nullptr;   // set while a program is being captured
  int kn[16] = {0};
  // MG-MG-S (outer_mode = IETI_OUTER_BPCG; R28-R31): BPCG on the saddle point Eq. (2)
  bool bp_mode = false;
  double bp_s = 0.0, bp_theta_min = 0.0, bp_theta_max = 0.0;
  int bp_steps = 0;
  double *b_u = nullptr, *b_rho = nullptr, *b_r = nullptr, *b_Kr = nullptr, *b_p = nullptr, *b_Kp = nullptr,
         *b_a = nullptr, *b_w = nullptr;                     // V~_h vectors / functionals (fine boxes)
  double *l_rho = nullptr, *l_s = nullptr, *l_r = nullptr, *l_p = nullptr, *l_a = nullptr;   // multipliers
  double *bsc = nullptr, *bsc_host = nullptr, *bpartial = nullptr, *invmult = nullptr;
  int nb_box = 1;
  std::vector<double> pi_mult;            // global: patches sharing each primal entity
  std::vector<long long> act_off_g;       // global: first active dof of each patch (concatenated)
  std::vector<int> glob_patch;            // local patch -> global id
  bool pcg_mode = false, dpcg_mode = false;
  BatchedPcg ipcg;                        // the inner local Neumann solver (pcg_mode)
  BatchedPcg dpcg;                        // the inner local Dirichlet solver (dpcg_mode)
  double *IX = nullptr;                   // = ipcg.X
  std::vector<int> inner_log;            // per local-solve call of the last solve: npatch inner counts
  long long inner_launches = 0;
  long long last_launches = 0;
  // phase timing (ieti_timing): event pairs recorded inside the graphs
  struct TPair { int e0, e1, cls; long long launches; double bytes; double bytes3 = 0; };
  std::vector<cudaEvent_t> tev;
  std::vector<TPair> tpairs[16];
  int rec_graph = -1;
  bool timing_on = false;
  double t_acc[8] = {0}, b_acc[8] = {0}, b3_acc[8] = {0};
  // solve phases (d^ + start, outer loop, recovery) from events on the library stream, read
  // lazily (after the next synchronisation point); ph_acc: ms per phase, [3] = solves
  cudaEvent_t ph_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool ph_pending = false;
  double ph_acc[4] = {0, 0, 0, 0};
  long long n_acc[8] = {0};
  int launches_per_iter = 0;
  double setup_ms = 0;
  // multi-GPU (partition.cpp, comm.cpp); world == 1: no ghosts, every exchange is a no-op
  Comm comm;
  Plan plan;
  int n_own = 0;                          // owned multipliers = first n_own entries of lambda, r, z, p, q
  int n_lambda_global = 0, n_patches_global = 0;
  double *xs = nullptr, *xr = nullptr;    // exchange buffers
  int *d_send_idx = nullptr, *d_recv_idx = nullptr, *d_rsum_ptr = nullptr, *d_rsum_src = nullptr;
  double *g_all = nullptr, *red_send = nullptr, *red_all = nullptr;
  std::vector<std::pair<std::string, double>> stage_ms;
  long long stencil_bytes = 0;
  int n_floating = 0;
  int max_coarse_rows = 1;
  // per colour: stencil offsets whose neighbour has a lower colour (first nlow[c]), then those
  // with a higher colour (the diagonal excluded) -- kernels_mg.cu MODE 4 / 5
  short *d_olist = nullptr, *d_nlow = nullptr;
  std::vector<short> h_olist;
  int fuse_mode = -1;                     // IETI_FUSE: 1 on, 0 off, -1 auto (batches of >= 128 problems)
  double fuse_max_mb = 24.0;              // IETI_FUSE_MB: largest colour phase (MB) of a fused level
  bool prefetch_on = true;                // IETI_PF=0: no next-phase L2 prefetch
  double prefetch_max_mb = 40.0;          // IETI_PFMAX: largest phase (MB of coefficients) prefetched
  double xgroup_mb = 32.0;                // IETI_XGROUP_MB: sweep problem groups with <= this x (0: off)
  bool l2_persist = false;                // IETI_L2P=1: persisting L2 window on the finest x
  size_t l2_persist_bytes = 0, l2_window_max = 0;
  bool fused_fine = false;                // the finest level runs fused (timing class = V-cycle)
  // direct local solvers (local_mode / dirichlet_mode DIRECT): batched banded Cholesky
  struct Direct {
    int nprob = 0, max_bw = 0;
    std::vector<BandDesc> desc;
    BandDesc *d_desc = nullptr;
    double *band = nullptr, *up = nullptr, *v = nullptr;
    long long *d_pos = nullptr, *d_voff = nullptr;
    long long nv = 0, len = 0;
  };
  Direct dirN, dirD;
  bool direct_N = false, direct_D = false;
  bool inner_unconverged = false, inner_breakdown = false;   // flags of the last solve's inner PCGs
  int psweep = 0;                         // IETI_PSWEEP: 1 = every sweep one persistent launch (k_sweep)
  int clsweep = 1;                        // IETI_CLSWEEP: row-major (latency-bound) levels sweep in one cluster
                                          // launch per sweep (k_sweep_cl); 0 = one launch per colour phase
  int clcs = 0;                           // IETI_CLCS: force the CTAs per problem of k_sweep_cl (A/B)
  int clglobal = 0;                       // IETI_CLGLOBAL=1: k_sweep_cl reads coefficients from global memory (A/B)
  int tiled = 1;                          // IETI_TILE: row-tiled coefficients on the big levels (0: offset-major)
  int clrep = 0;                          // IETI_CLREP=1: k_sweep_cl keeps x replicated in shared memory, updates
                                          // broadcast through DSMEM (measured neutral: C4 +1 %, C3 -3 %, C2 -1 %)
  double cl_max_mb = 32.0;                // IETI_CLMAX_MB: cluster sweeps only on levels with <= this many MB
                                          // of coefficients per colour phase (latency-bound)
  int full_t_npi = 0;                     // wide k_full_t: max n_Pi^(k) (0: one block per patch, IETI_FULLT=0)
  double *rGt = nullptr;                  // its B^T lam scratch (Gamma-compressed)
  unsigned *d_bar = nullptr;              // its grid-barrier counter
  std::vector<short> h_nlow;

  // host -> device copy ordered on the library stream and complete on return: a legacy-stream
  // cudaMemcpy from pageable memory may return before its DMA lands, and kernels on the
  // non-blocking stream are not ordered after it (setup race, found as run-to-run differences)
  void h2d(void *dst, const void *src, size_t bytes) {
    cudaStream_t q = st ? st : (cudaStream_t)0;
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, q));
    CK(cudaStreamSynchronize(q));
  }
  template <typename T>
  T *alloc(long long n) {
    if (n <= 0) n = 1;
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)n * sizeof(T));
    if (e != cudaSuccess) throw IetiError(IETI_E_NOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    // zero on the library stream: a legacy-stream cudaMemset is not ordered with the
    // non-blocking stream's kernels and could land after them
    if (st) {
      CK(cudaMemsetAsync(p, 0, (size_t)n * sizeof(T), st));
    } else {
      CK(cudaMemset(p, 0, (size_t)n * sizeof(T)));
      CK(cudaDeviceSynchronize());
    }
    allocs.push_back(p);
    bytes_alloc += (size_t)n * sizeof(T);
    return (T *)p;
  }
  template <typename T>
  T *upload(const std::vector<T> &h) {
    T *d = alloc<T>((long long)h.size());
    if (!h.empty()) h2d(d, h.data(), h.size() * sizeof(T));
    return d;
  }
  ~ieti_ctx() {
    for (auto &pr : prog)
      for (auto &sg : pr)
        if (sg.g) cudaGraphExecDestroy(sg.g);
    for (cudaGraphExec_t g : {ipcg.g_init, ipcg.g_body, dpcg.g_init, dpcg.g_body})
      if (g) cudaGraphExecDestroy(g);
    if (ipcg.ctr_host) cudaFreeHost(ipcg.ctr_host);
    if (dpcg.ctr_host) cudaFreeHost(dpcg.ctr_host);
    comm.destroy();
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
    for (cudaEvent_t e : ph_ev)
      if (e) cudaEventDestroy(e);
    for (void *p : allocs) cudaFree(p);
    if (sc_host) cudaFreeHost(sc_host);
    if (bsc_host) cudaFreeHost(bsc_host);
    for (int k = 0; k < 3; ++k) {
      if (st_aux[k]) cudaStreamDestroy(st_aux[k]);
      if (ev_join[k]) cudaEventDestroy(ev_join[k]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (st) cudaStreamDestroy(st);
  }
};

static thread_local std::string g_setup_err;

namespace {

// ------------------------------------------------------------------------------------------
// hierarchy descriptors
// ------------------------------------------------------------------------------------------
void build_level_desc(ieti_ctx &c, Hier &H, int l) {
  Level &Lv = H.lev[l];
  const int d = c.dim, p = c.p;
  long long coef_off = 0;
  for (int k = 0; k < c.npatch; ++k) {
    GridDesc g{};
    for (int i = 0; i < 3; ++i) { g.M[i] = 1; g.lo[i] = 0; g.hi[i] = 1; g.ns[i] = 1; }
    for (int i = 0; i < d; ++i) {
      g.M[i] = (int)c.kl[l][k][i].size() - p - 1;
      if (H.dirichlet) { g.lo[i] = 1; g.hi[i] = g.M[i] - 1; }
      else {
        g.lo[i] = c.T.dir_side[k][2 * i] ? 1 : 0;
        g.hi[i] = c.T.dir_side[k][2 * i + 1] ? g.M[i] - 1 : g.M[i];
      }
      g.ns[i] = (g.M[i] + p) / (p + 1);                // sub-lattice points, no halo (layout.cuh)
    }
    g.nrows = 1;
    for (int i = 0; i < d; ++i) g.nrows *= (g.hi[i] - g.lo[i]);
    g.ld = (g.nrows + 31) / 32 * 32;
    g.sb = g.ns[0] * g.ns[1] * g.ns[2];
    g.box = c.ncol * g.sb;
    // threads per stencil row: 1 on large grids (bandwidth-bound), 4 on small ones (latency-bound)
    long long full = 1;
    for (int i = 0; i < d; ++i) full *= g.M[i];
    g.tg = 1;                                        // offset-major coefficient rows (layout.cuh)
    g.tpr = 1;                                       // set per level below
    g.col_off = (int)Lv.ci.size();
    g.coef_off = coef_off;
    g.mass_beta = 0.0;
    g.mass_off = 0;
    g.patch = k;
    coef_off += (long long)g.ld * c.S;
    // colours (R6): colour = sum_d (i_d mod (p+1)) (p+1)^d over the FULL-lattice index
    int start = 0;
    for (int col = 0; col < c.ncol; ++col) {
      ColourInfo ci{};
      int cc = col;
      int cnt = 1;
      for (int i = 0; i < 3; ++i) {
        if (i < d) {
          int cd = cc % (p + 1);
          cc /= (p + 1);
          int first = g.lo[i] + ((cd - g.lo[i]) % (p + 1) + (p + 1)) % (p + 1);
          int n = (first < g.hi[i]) ? (g.hi[i] - first + p) / (p + 1) : 0;
          ci.first[i] = first;
          ci.n[i] = n;
        } else {
          ci.first[i] = 0;
          ci.n[i] = 1;
        }
        cnt *= ci.n[i];
      }
      ci.start = start;
      start += cnt;
      Lv.ci.push_back(ci);
    }
    if (start != g.nrows) throw IetiError(IETI_E_ARG, "colour partition mismatch");
    Lv.g.push_back(g);
  }
  Lv.coef_n = coef_off;
  // threads per row: one on levels whose colour phases stream enough rows to be bandwidth-bound,
  // else 8 (3D) / 4 (2D) share a row with interleaved offsets (A/B on B200: C4 8 > 4 by 10 %,
  // C2 4 > 8 by 7 %)
  long long rows = 0;
  for (const auto &g : Lv.g) rows += g.nrows;
  const char *tr1 = getenv("IETI_TPR1_ROWS");          // A/B: rows per phase from which tpr = 1
  const long long big_rows = (tr1 && atoll(tr1) > 0) ? atoll(tr1) : 40000;
  // small levels: 8 threads per row from S = (2p+1)^d >= 64 (3D; 2D p = 4: C3 +7 %), else 4 (C2 -2.5 % at 8)
  int tpr = (rows / c.ncol >= big_rows) ? 1 : (c.S >= 64 ? 8 : 4);
  {
    // override for A/B runs and tests: 4 / 8 / 16 on the small levels only; 1 on every level
    // (forces the offset-major big-level path onto small test cases)
    const char *e = getenv("IETI_TPR");
    if (e && tpr > 1 && (atoi(e) == 4 || atoi(e) == 8 || atoi(e) == 16)) tpr = atoi(e);
    if (e && atoi(e) == 1) tpr = 1;
  }
  const bool big = (tpr == 1);                            // offset-major, bandwidth-bound level
  {
    const char *eb = getenv("IETI_TPR_BIG");             // A/B: threads per row on the big levels (1, 2)
    if (big && eb && atoi(eb) == 2) tpr = 2;
  }
  // offset tables, one per distinct sub-lattice box shape
  std::vector<int2> tab;
  std::map<std::array<int, 4>, int> sig_off;
  for (auto &g : Lv.g) {
    g.tpr = tpr;
    g.tg = big ? (c.tiled ? -c.S : 1) : c.S;         // row tiles (or offset-major) on big levels, row-major on small
    const std::array<int, 4> sig = {g.ns[0], g.ns[1], g.ns[2], g.sb};
    auto it = sig_off.find(sig);
    if (it != sig_off.end()) { g.ent_off = it->second; continue; }
    const int off = (int)tab.size();
    sig_off[sig] = off;
    g.ent_off = off;
    for (int col = 0; col < c.ncol; ++col) {
      for (int o = 0; o < c.S; ++o) tab.push_back(make_int2(o, sl_delta(g, p, d, col, o)));
      for (int i = 0; i < c.S - 1; ++i) {
        const int o = c.h_olist[(size_t)col * c.S + i];
        tab.push_back(make_int2(o, sl_delta(g, p, d, col, o)));
      }
      tab.push_back(make_int2(0, 0));
    }
  }
  Lv.ent = c.upload(tab);
}

void upload_level(ieti_ctx &c, Level &Lv) {
  // + 64 doubles of slack: 16-byte aligned TMA slabs may read one double past the last row
  Lv.coef = c.alloc<double>(Lv.coef_n + 64);
  c.stencil_bytes += Lv.coef_n * 8;
}

// ------------------------------------------------------------------------------------------
// batches
// ------------------------------------------------------------------------------------------
LevelView view(Batch &B, int l);

void build_batch(ieti_ctx &c, Batch &B, Hier &H, const std::vector<int> &prob_grid, bool alloc_r = true) {
  B.H = &H;
  B.nprob = (int)prob_grid.size();
  B.prob_grid = prob_grid;
  B.lv.assign(c.L, BLevel());
  for (int l = 0; l < c.L; ++l) {
    Level &Lv = H.lev[l];
    BLevel &bl = B.lv[l];
    // zero guard band before the first and after the last box: wrap-around reads of padded
    // (zero-coefficient) neighbours stay inside the allocation (layout.cuh)
    long long guard = 32;
    for (int pi = 0; pi < B.nprob; ++pi) {
      const GridDesc &g = Lv.g[prob_grid[pi]];
      guard = std::max<long long>(guard, ((long long)1 + g.ns[0] + (long long)g.ns[0] * g.ns[1] + 31) / 32 * 32);
    }
    long long off = guard;
    int maxrows_col = 0;
    for (int pi = 0; pi < B.nprob; ++pi) {
      const GridDesc &g = Lv.g[prob_grid[pi]];
      ProbDesc pd{};
      pd.grid = prob_grid[pi];
      pd.vec_off = off;
      off += (g.box + 31) / 32 * 32;
      bl.pr.push_back(pd);
      bl.maxbox = std::max(bl.maxbox, g.box);
      for (int col = 0; col < c.ncol; ++col) {
        const ColourInfo &ci = Lv.ci[g.col_off + col];
        maxrows_col = std::max(maxrows_col, ci.n[0] * ci.n[1] * ci.n[2]);
      }
    }
    bl.n = off + guard;
    bl.guard = (int)guard;
    bl.d_pr = c.upload(bl.pr);
    bl.x = c.alloc<double>(bl.n);
    bl.b = c.alloc<double>(bl.n);
    bl.r = alloc_r ? c.alloc<double>(bl.n) : nullptr;
    // forward-sweep increments (residual of non-zero-start sweeps, MODE 5): finest level only
    bl.d = (alloc_r && l == c.L - 1) ? c.alloc<double>(bl.n) : nullptr;
    // rows per colour (algorithmic byte accounting)
    bl.rows_col.assign(c.ncol, 0);
    for (int pi = 0; pi < B.nprob; ++pi) {
      const GridDesc &g = Lv.g[prob_grid[pi]];
      for (int col = 0; col < c.ncol; ++col) {
        const ColourInfo &ci = Lv.ci[g.col_off + col];
        bl.rows_col[col] += (long long)ci.n[0] * ci.n[1] * ci.n[2];
      }
    }
    {
      long long rows = 0;
      for (long long v : bl.rows_col) rows += v;
      bl.phase_bytes = (double)rows / c.ncol * c.S * 8.0;
    }
    // colour blocks: 128 threads, tg threads per row (all grids of a level share tg)
    int nthr = 128 / Lv.g[prob_grid.empty() ? 0 : prob_grid[0]].tpr;
    bl.cnthr = nthr;
    (void)maxrows_col;
    // problem groups for the sweeps of bandwidth-bound levels: a whole sweep runs group by group
    // (problems are independent), so each group's x (<= xgroup_mb) stays L2-resident across its
    // colour phases instead of being re-read from HBM by every phase
    {
      const double xbytes = (double)bl.n * 8.0;
      bl.ngroups = 1;
      const int tg0 = Lv.g[prob_grid.empty() ? 0 : prob_grid[0]].tg;
      if ((tg0 == 1 || tg0 < 0) && c.xgroup_mb > 0) {
        bl.ngroups = std::max(1, std::min(B.nprob, (int)std::ceil(xbytes / (c.xgroup_mb * (1 << 20)))));
        // at least xg_big concurrent groups (their phase tails overlap; C3's finest level: 1 -> 2)
        if (c.xgconc) bl.ngroups = std::max(bl.ngroups, std::min(B.nprob, c.xg_big));
      }
      else if (c.xg_small > 1 && c.xgconc && bl.phase_bytes > c.cl_max_mb * (1 << 20))
        // row-major levels too heavy for the cluster sweep (C5 level 2): problem groups on concurrent
        // branches, so one group's wave tail overlaps the other's phase
        bl.ngroups = std::max(1, std::min(B.nprob, c.xg_small));
    }
    std::vector<BlockEntry> blk;
    bl.cofs.assign(c.ncol + 1, 0);
    bl.gofs.assign((size_t)c.ncol * (bl.ngroups + 1), 0);
    for (int col = 0; col < c.ncol; ++col) {
      bl.cofs[col] = (int)blk.size();
      for (int pi = 0; pi < B.nprob; ++pi) {
        const int grp = (int)((long long)pi * bl.ngroups / std::max(1, B.nprob));
        if (pi == 0 || grp != (int)((long long)(pi - 1) * bl.ngroups / std::max(1, B.nprob)))
          bl.gofs[(size_t)col * (bl.ngroups + 1) + grp] = (int)blk.size();
        const GridDesc &g = Lv.g[prob_grid[pi]];
        const ColourInfo &ci = Lv.ci[g.col_off + col];
        int n = ci.n[0] * ci.n[1] * ci.n[2];
        for (int r0 = 0; r0 < n; r0 += nthr) blk.push_back(BlockEntry{pi, col, r0, std::min(nthr, n - r0)});
      }
      bl.gofs[(size_t)col * (bl.ngroups + 1) + bl.ngroups] = (int)blk.size();
    }
    bl.cofs[c.ncol] = (int)blk.size();
    bl.d_cblk = c.upload(blk);
    {
      std::vector<int2> pt((size_t)bl.ngroups * 2 * c.ncol);
      for (int grp = 0; grp < bl.ngroups; ++grp)
        for (int dir = 0; dir < 2; ++dir)
          for (int ph = 0; ph < c.ncol; ++ph) {
            const int col = dir == 0 ? ph : c.ncol - 1 - ph;
            const int *go = bl.gofs.data() + (size_t)col * (bl.ngroups + 1);
            pt[((size_t)grp * 2 + dir) * c.ncol + ph] = make_int2(go[grp], go[grp + 1] - go[grp]);
            bl.ptab_max = std::max(bl.ptab_max, go[grp + 1] - go[grp]);
          }
      bl.d_ptab = c.upload(pt);
    }
    // the same blocks problem-major for the all-colour launches (residual, apply): a problem's
    // x / dx gathers then stay in L2 while its colours are processed
    {
      std::vector<BlockEntry> pm(blk);
      std::stable_sort(pm.begin(), pm.end(), [](const BlockEntry &u, const BlockEntry &v) { return u.prob < v.prob; });
      bl.d_rblk = c.upload(pm);
    }
    // point blocks (active box, lexicographic)
    std::vector<BlockEntry> pb;
    for (int pi = 0; pi < B.nprob; ++pi) {
      const GridDesc &g = Lv.g[prob_grid[pi]];
      for (int r0 = 0; r0 < g.nrows; r0 += 128) pb.push_back(BlockEntry{pi, -1, r0, std::min(128, g.nrows - r0)});
    }
    bl.npblk = (int)pb.size();
    bl.d_pblk = c.upload(pb);
    // latency-bound (row-major) levels: one cluster launch per sweep (kernels_sweep.cu) when every
    // problem's cluster can be resident at once (first fit of the candidates below; cs0 = CTAs per
    // problem giving >= 2 CTAs per SM, at most 8; threads per CTA just enough for one row pass, <= 512)
    bl.cl_cs = 0;
    const GridDesc &g0 = Lv.g[prob_grid.empty() ? 0 : prob_grid[0]];
    // (bandwidth-heavy levels keep one launch per phase: C5 level 2, 75 MB per phase, measured 9 % slower)
    if (c.clsweep && B.nprob > 0 && g0.tg == c.S && g0.tpr > 1 && l >= 1 &&
        bl.phase_bytes <= c.cl_max_mb * (1 << 20)) {
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      int cs0 = 1;
      while (cs0 < 8 && (long long)B.nprob * cs0 < 2LL * nsm) cs0 *= 2;
      int maxbox = 0;
      for (int pi = 0; pi < B.nprob; ++pi) maxbox = std::max(maxbox, Lv.g[prob_grid[pi]].box);
      const long long rep_n = ((long long)maxbox + 2LL * bl.guard + 1) / 2 * 2;
      // candidates in order: x replicated in every CTA (gathers from local shared memory, updates
      // broadcast through DSMEM) at cs0, cs0/2, cs0/4; then x in global memory at cs0, 2 cs0; each with
      // coefficient slabs in shared memory first, else coefficients from global memory
      struct Cand { int cs; bool rep; };
      std::vector<Cand> cands;
      if (c.clrep)
        for (int cs = cs0; cs >= std::max(1, cs0 / 4); cs /= 2) cands.push_back({cs, true});
      cands.push_back({cs0, false});
      if (cs0 < 16) cands.push_back({cs0 * 2, false});
      if (c.clcs > 0) {
        cands.clear();
        if (c.clrep) cands.push_back({c.clcs, true});
        cands.push_back({c.clcs, false});
      }
      for (const Cand &cd : cands) {
        const int cs = cd.cs;
        long long rmax = 1;
        for (int pi = 0; pi < B.nprob; ++pi) {
          const GridDesc &g = Lv.g[prob_grid[pi]];
          for (int col = 0; col < c.ncol; ++col) {
            const ColourInfo &ci = Lv.ci[g.col_off + col];
            const long long nr = (long long)ci.n[0] * ci.n[1] * ci.n[2];
            for (int cr = 0; cr < cs; ++cr) rmax = std::max(rmax, nr * (cr + 1) / cs - nr * cr / cs);
          }
        }
        const long long slab1 = (rmax * c.S + 2 + 1) / 2 * 2;   // + alignment shift, even (16-byte buffers)
        const int nthr = (int)std::min<long long>(512, std::max<long long>(64, (rmax * g0.tpr + 31) / 32 * 32));
        const long long rep = cd.rep ? rep_n : 0;
        // coefficient slabs in shared memory (TMA), else read from global memory (L2 prefetch)
        for (long long slab : {slab1, 0LL}) {
          if (slab && c.clglobal) continue;
          const long long smem = rep * 8 + slab * 2 * 8 + rmax * c.ncol * 12;
          int ncl = 0;
          if (smem <= 190 * 1024) {
            ncl = 1 << 30;
            for (int mode : {0, 4, 6, 7})
              ncl = std::min(ncl, launch_sweep_cluster(c.dim, c.p, g0.tpr, mode, view(B, l), B.nprob, cs, nthr, (int)slab,
                                                       (int)rmax, (int)rep, bl.guard, c.ncol, true, nullptr, nullptr,
                                                       nullptr, nullptr, nullptr, nullptr, true));
          }
          if (getenv("IETI_VERBOSE"))
            fprintf(stderr, "[ieti] level %d: cluster sweep cs %d threads %d slab %lld rep %lld doubles: %d of %d clusters resident\n",
                    l, cs, nthr, slab, rep, ncl, B.nprob);
          if (ncl >= B.nprob) {
            bl.cl_cs = cs;
            bl.cl_nthr = nthr;
            bl.cl_slab = (int)slab;
            bl.cl_rmax = (int)rmax;
            bl.cl_rep = (int)rep;
            break;
          }
        }
        if (bl.cl_cs) break;
      }
    }
  }
  // fuse the levels whose colour phases move little data (launch-latency bound), counted from
  // the coarsest up: <= 24 MB of coefficients per colour phase over the batch, row-major rows
  // (tg == S); the coarsest rhs is staged in shared memory
  B.ftop = 0;
  B.fcs = 1;
  // the fused kernel implements one forward / one backward sweep per level (R5 default)
  const bool fuse = ((c.fuse_mode == 1) || (c.fuse_mode == -1 && B.nprob >= 128)) &&
                    c.a.nu_pre <= 1 && c.a.nu_post <= 1;
  if (fuse && B.nprob > 0) {
    int cs = 1;
    while (cs < 8 && (long long)B.nprob * cs < 296) cs *= 2;
    int maxrc = 1, mcr = 1;
    for (int pi = 0; pi < B.nprob; ++pi) mcr = std::max(mcr, H.lev[0].g[prob_grid[pi]].nrows);
    for (int l = 1; l < c.L && l < IETI_MAXL; ++l) {
      long long rows = 0;
      int mrc = 0;
      bool rowmajor = true;
      for (int pi = 0; pi < B.nprob; ++pi) {
        const GridDesc &g = H.lev[l].g[prob_grid[pi]];
        rows += g.nrows;
        rowmajor = rowmajor && g.tg == c.S;
        for (int col = 0; col < c.ncol; ++col) {
          const ColourInfo &ci = H.lev[l].ci[g.col_off + col];
          mrc = std::max(mrc, ci.n[0] * ci.n[1] * ci.n[2]);
        }
      }
      const double phase_bytes = (double)rows / c.ncol * c.S * 8.0;
      if (!rowmajor || phase_bytes > c.fuse_max_mb * (1 << 20)) break;
      // a level swept by k_sweep_cl is not fused unless forced (C5 level 1: cluster sweeps 15.80 it/s
      // against the fused V-cycle's 15.41, measured)
      if (c.fuse_mode != 1 && B.lv[l].cl_cs > 0) break;
      if (mcr * 8.0 > 200.0 * 1024) break;
      maxrc = std::max(maxrc, mrc);
      B.ftop = l;
    }
    B.fcs = cs;
    const int rows_cta = (maxrc + cs - 1) / cs;
    B.fslab = rows_cta * c.S + 2;
    int t = 1;
    while (t < 32 && 256 / (t * 2) >= rows_cta) t *= 2;
    B.ftprf = t;
  }
}

LevelView view(Batch &B, int l) {
  Level &Lv = B.H->lev[l];
  return LevelView{Lv.d_g, Lv.d_ci, B.lv[l].d_pr, Lv.coef, Lv.mass, Lv.ent, B.lv[l].n};
}

int tg_of(Batch &B, int l) { return B.H->lev[l].g[B.prob_grid.empty() ? 0 : B.prob_grid[0]].tpr; }

// one forward (colours ascending) or backward (descending) colour-GS sweep (R5, R6).
// zero: x = 0 before the sweep (first visit of the level), only lower-colour coefficients are
// streamed (MODE 4); dx: record the forward increments (MODE 0) for the half-stream residual
void smooth(ieti_ctx &c, Batch &B, int l, bool fwd, cudaStream_t s, bool zero = false, double *dx = nullptr,
            int umode = 0) {
  BLevel &bl = B.lv[l];
  LevelView lv = view(B, l);
  const bool rec = (c.rec_graph >= 0) && (l == c.L - 1) && (&B == &c.BN || &B == &c.BD);
  int e0 = -1;
  if (rec) {
    e0 = (int)c.tev.size();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    c.tev.push_back(a);
    c.tev.push_back(b);
    CK(cudaEventRecordWithFlags(a, s, cudaEventRecordExternal));
  }
  bool done = false;
  if (bl.cl_cs > 0 && !c.psweep) {
    const int mode = umode ? umode : (zero ? 4 : 0);
    if (launch_sweep_cluster(c.dim, c.p, tg_of(B, l), mode, lv, B.nprob, bl.cl_cs, bl.cl_nthr, bl.cl_slab, bl.cl_rmax,
                             bl.cl_rep, bl.guard, c.ncol, fwd, bl.x, bl.b, (mode == 0 || mode == 6) ? dx : nullptr,
                             bl.U, c.d_nlow, s, false) != 1)
      throw IetiError(IETI_E_CUDA, "cluster sweep launch failed (k_sweep_cl)");
    done = true;
  }
  if (c.psweep && !done) {
    const int mode = umode ? umode : (zero ? 4 : 0);
    done = true;
    for (int grp = 0; grp < bl.ngroups && done; ++grp)
      done = launch_sweep(c.dim, c.p, tg_of(B, l), mode, lv, bl.d_cblk,
                          bl.d_ptab + ((size_t)grp * 2 + (fwd ? 0 : 1)) * c.ncol, c.ncol, bl.ptab_max, c.d_bar,
                          bl.x, bl.b, umode ? bl.U : nullptr, dx, c.d_olist, c.d_nlow, s);
    if (!done) throw IetiError(IETI_E_CUDA, "persistent sweep launch failed (IETI_PSWEEP)");
  }
  // the problem groups of a bandwidth-bound level are independent: with IETI_XGCONC (default) group g
  // runs on its own stream branch (forked from s, joined back before the sweep ends), so one group's
  // phase boundaries (launch gap, ramp, drain) overlap the other groups' streaming
  const bool conc = !done && bl.ngroups > 1 && bl.ngroups <= 4 && c.xgconc;
  if (conc) {
    CK(cudaEventRecord(c.ev_fork, s));
    for (int grp = 1; grp < bl.ngroups; ++grp) CK(cudaStreamWaitEvent(c.st_aux[grp - 1], c.ev_fork, 0));
  }
  for (int grp = 0; grp < bl.ngroups && !done; ++grp)
    for (int cc = 0; cc < c.ncol; ++cc) {
      cudaStream_t sg = (conc && grp > 0) ? c.st_aux[grp - 1] : s;
      int col = fwd ? cc : c.ncol - 1 - cc;
      const int *go = bl.gofs.data() + (size_t)col * (bl.ngroups + 1);
      int b0 = go[grp], nb = go[grp + 1] - b0;
      // next phase's colour, for the L2 prefetch on levels whose phase blocks fit comfortably in L2
      int pcol = (cc + 1 < c.ncol) ? (fwd ? cc + 1 : c.ncol - 2 - cc) : -1;
      if (!c.prefetch_on || bl.phase_bytes > c.prefetch_max_mb * (1 << 20)) pcol = -1;
      if (umode) launch_sgs_phase_u(c.dim, c.p, tg_of(B, l), umode, lv, bl.d_cblk + b0, nb, bl.x, bl.b, bl.U, dx,
                                    c.d_olist, c.d_nlow, pcol, sg);
      else if (zero) launch_sgs_phase_zero(c.dim, c.p, tg_of(B, l), lv, bl.d_cblk + b0, nb, bl.x, bl.b, c.d_olist,
                                           c.d_nlow, pcol, sg);
      else launch_sgs_phase(c.dim, c.p, tg_of(B, l), lv, bl.d_cblk + b0, nb, bl.x, bl.b, dx, pcol, sg);
    }
  if (conc)
    for (int grp = 1; grp < bl.ngroups; ++grp) {
      CK(cudaEventRecord(c.ev_join[grp - 1], c.st_aux[grp - 1]));
      CK(cudaStreamWaitEvent(s, c.ev_join[grp - 1], 0));
    }
  if (rec) {
    CK(cudaEventRecordWithFlags(c.tev[e0 + 1], s, cudaEventRecordExternal));
    // algorithmic bytes of one sweep: per row the coefficients it must stream
    // (all S, or the diagonal + lower-colour ones from x = 0), b read, x read+write (x write
    // only from 0), dx write; neighbour x reads are L2 hits
    double bytes = 0;
    for (int col = 0; col < c.ncol; ++col) {
      // mode 6: lower coefficients + diagonal, b, x read+write, U read, dx write; mode 7: all
      // coefficients, b, x read+write, U write
      const double per = (umode == 6) ? (c.h_nlow[col] + 1 + 5) : (umode == 7) ? (c.S + 4)
                         : zero ? (c.h_nlow[col] + 1 + 2) : (c.S + 3 + (dx ? 1 : 0));
      bytes += (double)bl.rows_col[col] * 8.0 * per;
    }
    c.tpairs[c.rec_graph].push_back({e0, e0 + 1, B.H->dirichlet ? 1 : 0, (long long)c.ncol * bl.ngroups, bytes});
  }
}

// r = b - A x right after a forward sweep, from the sweep's increments d (= x from 0): only the
// higher-colour coefficients are streamed (MODE 5, kernels_mg.cu)
void residual_upper(ieti_ctx &c, Batch &B, int l, const double *d, double *y, cudaStream_t s) {
  BLevel &bl = B.lv[l];
  launch_residual_upper(c.dim, c.p, tg_of(B, l), view(B, l), bl.d_rblk, bl.cofs[c.ncol], d, y, c.d_olist, c.d_nlow,
                        s);
}

// r = b - A x over all rows of level l
void residual_level(ieti_ctx &c, Batch &B, int l, const double *x, const double *b, double *y, cudaStream_t s) {
  BLevel &bl = B.lv[l];
  launch_residual(c.dim, c.p, tg_of(B, l), view(B, l), bl.d_rblk, bl.cofs[c.ncol], x, b, y, s);
}

// y = scale * A x over all rows of level l; with true_k the on-the-fly alpha*Mhat of floating
// fine grids is removed (A = K + alpha Mhat there, R4), giving the true stiffness K (setup only)
void apply_level(ieti_ctx &c, Batch &B, int l, const double *x, double *y, double scale, bool true_k,
                 cudaStream_t s) {
  BLevel &bl = B.lv[l];
  launch_apply(c.dim, c.p, tg_of(B, l), view(B, l), bl.d_rblk, bl.cofs[c.ncol], x, y, scale, s);
  if (true_k) {
    // colour blocks hold 128/tpr rows: the mass kernel uses one thread per row
    launch_mass_add(c.dim, c.p, view(B, l), bl.d_cblk, bl.cofs[c.ncol], bl.cnthr, x, y, s);
  }
}

// V_l(x, b) (O7): zero = x is 0 on entry (always on coarse levels; the first of the c cycles
// on the finest level, R10)
void fused_vcycle(ieti_ctx &c, Batch &B, int l, bool zero, cudaStream_t s);

// ucyc (finest level, c >= 2 cycles): bit 1 = the forward sweep uses U from the previous
// cycle's backward sweep (mode 6), bit 2 = the backward sweep records U (mode 7)
void vcycle(ieti_ctx &c, Batch &B, int l, cudaStream_t s, bool zero, int ucyc = 0) {
  Hier &H = *B.H;
  if (l >= 1 && l <= B.ftop) {
    fused_vcycle(c, B, l, zero, s);
    return;
  }
  if (l == 0) {
    Level &L0 = H.lev[0];
    launch_coarse_solve(L0.d_g, B.lv[0].d_pr, L0.d_inv_off, L0.inv, B.nprob, c.dim, c.p, B.lv[0].b, B.lv[0].x,
                        c.max_coarse_rows, s);
    return;
  }
  BLevel &bl = B.lv[l], &bc = B.lv[l - 1];
  Level &Lf = H.lev[l], &Lc = H.lev[l - 1];
  Trans &T = c.tr[l];
  const bool use_u = (ucyc & 1) && bl.U && !zero, store_u = (ucyc & 2) && bl.U;
  const int nu1 = std::max(1, c.a.nu_pre), nu2 = std::max(1, c.a.nu_post);   // R5
  if (nu1 > 1) {
    // nu_1 forward sweeps: the first from x = 0 (mode 4) or with U (mode 6), the others plain; the
    // last records its increments when the level has the buffer (the half-stream residual needs
    // the increments of the LAST forward sweep), else the full residual
    if (use_u) smooth(c, B, l, true, s, false, nullptr, 6);
    else smooth(c, B, l, true, s, zero, nullptr);
    for (int i = 1; i < nu1; ++i) smooth(c, B, l, true, s, false, (i + 1 == nu1) ? bl.d : nullptr);
    if (bl.d) residual_upper(c, B, l, bl.d, bl.r, s);
    else residual_level(c, B, l, bl.x, bl.b, bl.r, s);
  } else if (zero || bl.d) {
    if (use_u) smooth(c, B, l, true, s, false, bl.d, 6);
    else smooth(c, B, l, true, s, zero, zero ? nullptr : bl.d);
    residual_upper(c, B, l, zero ? bl.x : bl.d, bl.r, s);
  } else {
    smooth(c, B, l, true, s, false, nullptr, use_u ? 6 : 0);
    residual_level(c, B, l, bl.x, bl.b, bl.r, s);
  }
  launch_restrict(c.dim, c.p, Lc.d_g, Lf.d_g, T.d_td, bc.d_pr, bl.d_pr, T.ip, T.wp, bc.d_pblk, bc.npblk, 128, bl.r,
                  bc.b, bc.x, s);
  vcycle(c, B, l - 1, s, true);
  launch_prolong(c.dim, c.p, Lc.d_g, Lf.d_g, T.d_td, bc.d_pr, bl.d_pr, T.ip, T.wp, bl.d_pblk, bl.npblk, 128, bc.x,
                 bl.x, s);
  for (int i = 1; i < nu2; ++i) smooth(c, B, l, false, s, false, nullptr, 0);
  smooth(c, B, l, false, s, false, nullptr, store_u ? 7 : 0);   // U recorded by the LAST backward sweep
}

// algorithmic bytes of one V-cycle on levels l..1 (+ coarsest) of a batch
double vcycle_bytes(ieti_ctx &c, Batch &B, int l, bool zero) {
  double bytes = 0;
  for (int k = l; k >= 1; --k) {
    const BLevel &bl = B.lv[k];
    const bool z = zero || k < l;
    for (int col = 0; col < c.ncol; ++col) {
      const double rc = (double)bl.rows_col[col] * 8.0;
      bytes += rc * (z ? (c.h_nlow[col] + 3) : (c.S + 4));       // forward sweep
      bytes += rc * (c.S - 1 - c.h_nlow[col] + 1);                // residual from the increments
      bytes += rc * (c.S + 3);                                    // backward sweep
      bytes += rc * (c.S + 4) * (std::max(1, c.a.nu_pre) - 1 + std::max(1, c.a.nu_post) - 1);   // R5: more sweeps
    }
  }
  for (int pi = 0; pi < B.nprob; ++pi) {
    const double n0 = B.H->lev[0].g[B.prob_grid[pi]].nrows;
    bytes += 8.0 * n0 * n0;
  }
  return bytes;
}

void fused_vcycle(ieti_ctx &c, Batch &B, int l, bool zero, cudaStream_t s) {
  Hier &H = *B.H;
  FusedArgs a{};
  for (int k = 0; k <= l; ++k) {
    Level &Lv = H.lev[k];
    BLevel &bl = B.lv[k];
    FusedLevel &f = a.lev[k];
    f.grids = Lv.d_g;
    f.cinfo = Lv.d_ci;
    f.ent = Lv.ent;
    f.probs = bl.d_pr;
    f.coef = Lv.coef;
    f.x = bl.x;
    f.b = bl.b;
    f.r = bl.r;
    f.d = bl.d;
    if (k >= 1) {
      f.td = c.tr[k].d_td;
      f.ip = c.tr[k].ip;
      f.wp = c.tr[k].wp;
    }
  }
  a.inv_off = H.lev[0].d_inv_off;
  a.inv = H.lev[0].inv;
  a.olist = c.d_olist;
  a.nlow = c.d_nlow;
  a.ltop = l;
  a.zero_top = zero ? 1 : 0;
  a.ncol = c.ncol;
  a.max_coarse_rows = c.max_coarse_rows;
  a.slab = B.fslab;
  a.tprf = B.ftprf;
  if (!zero && !B.lv[l].d) throw IetiError(IETI_E_ARG, "fused V-cycle from x != 0 needs the increment vector");
  const bool rec = (c.rec_graph >= 0) && (l == c.L - 1) && (&B == &c.BN || &B == &c.BD);
  int e0 = -1;
  if (rec) {
    e0 = (int)c.tev.size();
    cudaEvent_t ea, eb;
    CK(cudaEventCreate(&ea));
    CK(cudaEventCreate(&eb));
    c.tev.push_back(ea);
    c.tev.push_back(eb);
    CK(cudaEventRecordWithFlags(ea, s, cudaEventRecordExternal));
  }
  launch_vcycle_fused(c.dim, c.p, a, B.nprob, B.fcs, s);
  if (rec) {
    CK(cudaEventRecordWithFlags(c.tev[e0 + 1], s, cudaEventRecordExternal));
    c.tpairs[c.rec_graph].push_back({e0, e0 + 1, B.H->dirichlet ? 1 : 0, 1, vcycle_bytes(c, B, l, zero)});
    c.fused_fine = true;
  }
}

// N_c(b) (R10): c V-cycles from x = 0 on the finest level
// L2 persistence for the finest-level x of a V-cycle: every colour phase gathers all of x while
// the coefficients stream through; an access-policy window marks x persisting so the coefficient
// stream cannot evict it (captured into the kernel nodes of the graphs)
void l2_window(ieti_ctx &c, const void *base, size_t bytes, cudaStream_t s) {
  if (!c.l2_persist) return;
  cudaStreamAttrValue v = {};
  if (base && bytes) {
    const size_t nb = std::min(bytes, c.l2_window_max);
    v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    v.accessPolicyWindow.num_bytes = nb;
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)c.l2_persist_bytes / (double)nb);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  CK(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v));
}

// the survey's 3-stream reference bytes of one V-cycle: 8 n_l (3S + 12) per level
// l >= 1 (forward sweep, residual, backward sweep as three full coefficient streams, ~12 vector
// streams) + 8 n_0^2 per problem for the coarsest solve
double vcycle_bytes_ref3(ieti_ctx &c, Batch &B) {
  double bytes = 0;
  for (int k = c.L - 1; k >= 1; --k) {
    double rows = 0;
    for (long long r : B.lv[k].rows_col) rows += (double)r;
    bytes += 8.0 * rows * (3.0 * c.S + 12.0);
  }
  for (int pi = 0; pi < B.nprob; ++pi) {
    const double n0 = B.H->lev[0].g[B.prob_grid[pi]].nrows;
    bytes += 8.0 * n0 * n0;
  }
  return bytes;
}

void ncycles(ieti_ctx &c, Batch &B, int cycles, cudaStream_t s) {
  BLevel &bl = B.lv[c.L - 1];
  // timing class 2 / 3: the whole N_c / D_c (all levels) of the Neumann / Dirichlet batch
  const bool rec = (c.rec_graph >= 0) && (&B == &c.BN || &B == &c.BD);
  int e0 = -1;
  if (rec) {
    e0 = (int)c.tev.size();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    c.tev.push_back(a);
    c.tev.push_back(b);
    CK(cudaEventRecordWithFlags(a, s, cudaEventRecordExternal));
  }
  CK(cudaMemsetAsync(bl.x, 0, (size_t)bl.n * sizeof(double), s));
  const bool big = bl.n * 8.0 > 16.0 * (1 << 20);     // only when x does not trivially stay in L2
  if (big) l2_window(c, bl.x, (size_t)bl.n * sizeof(double), s);
  for (int i = 0; i < cycles; ++i) vcycle(c, B, c.L - 1, s, i == 0, (i > 0 ? 1 : 0) | (i + 1 < cycles ? 2 : 0));
  if (big) l2_window(c, nullptr, 0, s);
  if (rec) {
    CK(cudaEventRecordWithFlags(c.tev[e0 + 1], s, cudaEventRecordExternal));
    double bytes = 0;
    for (int i = 0; i < cycles; ++i) bytes += vcycle_bytes(c, B, c.L - 1, i == 0);
    ieti_ctx::TPair tp{e0, e0 + 1, (&B == &c.BD) ? 3 : 2, (long long)cycles, bytes};
    tp.bytes3 = cycles * vcycle_bytes_ref3(c, B);
    c.tpairs[c.rec_graph].push_back(tp);
  }
}

int count_vcycle_launches(ieti_ctx &c) {
  int per_level = 2 * c.ncol + 3;
  return (c.L - 1) * per_level + 1;
}

// ------------------------------------------------------------------------------------------
// setup steps
// ------------------------------------------------------------------------------------------
void setup_knots_levels(ieti_ctx &c) {
  const int d = c.dim, p = c.p;
  int mmin = 1 << 30;
  for (auto &P : c.T.patch)
    for (int i = 0; i < d; ++i) mmin = std::min(mmin, P.melem[i]);
  int L = c.a.mg_levels;
  if (L <= 0) {
    // R7: L = max(2, log2(m/4) + 1)
    int lg = 0;
    while ((4 << lg) <= mmin) ++lg;   // floor(log2(m/4)) + 1 for m >= 4
    L = std::max(2, lg);
    if (mmin < 4) L = 2;
  }
  c.L = L;
  c.kl.assign(L, std::vector<std::array<std::vector<double>, 3>>(c.npatch));
  for (int k = 0; k < c.npatch; ++k)
    for (int i = 0; i < d; ++i) {
      std::vector<double> t = c.T.patch[k].knots[i];
      c.kl[L - 1][k][i] = t;
      for (int l = L - 2; l >= 0; --l) {
        // dyadic coarsening requires an even number of spans
        int nspan = (int)t.size() - 2 * p - 1;
        if (nspan % 2) throw IetiError(IETI_E_ARG, "knot vector is not dyadically coarsenable to the requested levels");
        std::vector<double> tc = coarsen_knots(t, p);
        int Mf, Mc;
        std::vector<double> P = knot_insertion_dense(tc, p, t, Mf, Mc);
        if (Mf != (int)t.size() - p - 1) throw IetiError(IETI_E_ARG, "knot vectors not nested");
        c.kl[l][k][i] = tc;
        t = tc;
      }
    }
}

void setup_transfers(ieti_ctx &c) {
  const int d = c.dim, p = c.p;
  c.tr.assign(c.L, Trans());
  for (int l = 1; l < c.L; ++l) {
    Trans &T = c.tr[l];
    std::vector<int> ip;
    std::vector<double> wp;
    int Wmax = 1, CWmax = 1;
    std::vector<std::array<std::vector<double>, 3>> Ps(c.npatch);
    std::vector<std::array<std::pair<int, int>, 3>> dims(c.npatch);
    for (int k = 0; k < c.npatch; ++k)
      for (int i = 0; i < d; ++i) {
        int Mf, Mc;
        Ps[k][i] = knot_insertion_dense(c.kl[l - 1][k][i], p, c.kl[l][k][i], Mf, Mc);
        dims[k][i] = {Mf, Mc};
        const auto &P = Ps[k][i];
        for (int r = 0; r < Mf; ++r) {
          int cmin = Mc, cmax = -1;
          for (int cc = 0; cc < Mc; ++cc)
            if (P[(size_t)r * Mc + cc] != 0.0) { cmin = std::min(cmin, cc); cmax = std::max(cmax, cc); }
          if (cmax >= 0) Wmax = std::max(Wmax, cmax - cmin + 1);
        }
        for (int r = 0; r < Mf; ++r) {
          int cmin = Mc, cmax = -1;
          for (int j = std::max(0, r - p); j <= std::min(Mf - 1, r + p); ++j)
            for (int cc = 0; cc < Mc; ++cc)
              if (P[(size_t)j * Mc + cc] != 0.0) { cmin = std::min(cmin, cc); cmax = std::max(cmax, cc); }
          if (cmax >= 0) CWmax = std::max(CWmax, cmax - cmin + 1);
        }
      }
    // the kernels use a compile-time window of p/2 + 2 coarse contributors per fine index (dyadic
    // refinement: at most floor((p+1)/2) + 1), zero-padded
    if (Wmax > p / 2 + 2) throw IetiError(IETI_E_ARG, "prolongation row wider than p/2+2");
    Wmax = p / 2 + 2;
    T.CW = CWmax;
    T.cwin.assign((size_t)c.npatch * 3 * 4096, 0);
    for (int k = 0; k < c.npatch; ++k) {
      TransDesc td{};
      td.W = Wmax;
      for (int i = 0; i < d; ++i) {
        const auto &P = Ps[k][i];
        int Mf = dims[k][i].first, Mc = dims[k][i].second;
        if (Mf > 4096) throw IetiError(IETI_E_ARG, "too many basis functions per direction (> 4096)");
        // restriction: per coarse a, window of p+2 fine rows
        td.rc_off[i] = (int)ip.size();
        td.rw_off[i] = (int)wp.size();
        for (int a = 0; a < Mc; ++a) {
          int rmin = Mf, rmax = -1;
          for (int r = 0; r < Mf; ++r)
            if (P[(size_t)r * Mc + a] != 0.0) { rmin = std::min(rmin, r); rmax = std::max(rmax, r); }
          int f = std::max(0, std::min(rmin, Mf - (p + 2)));
          if (rmax >= f + p + 2) throw IetiError(IETI_E_ARG, "prolongation column wider than p+2");
          ip.push_back(f);
          for (int t = 0; t < p + 2; ++t) wp.push_back((f + t < Mf) ? P[(size_t)(f + t) * Mc + a] : 0.0);
        }
        // prolongation: per fine r, window of W coarse columns
        td.pf_off[i] = (int)ip.size();
        td.pw_off[i] = (int)wp.size();
        for (int r = 0; r < Mf; ++r) {
          int cmin = Mc;
          for (int cc = 0; cc < Mc; ++cc)
            if (P[(size_t)r * Mc + cc] != 0.0) { cmin = cc; break; }
          int cs = std::max(0, std::min(cmin, Mc - Wmax));
          ip.push_back(cs);
          for (int t = 0; t < Wmax; ++t) wp.push_back((cs + t < Mc) ? P[(size_t)r * Mc + cs + t] : 0.0);
        }
        // Galerkin window: coarse columns reachable from fine row r's stencil
        for (int r = 0; r < Mf; ++r) {
          int cmin = Mc;
          for (int j = std::max(0, r - p); j <= std::min(Mf - 1, r + p); ++j)
            for (int cc = 0; cc < Mc; ++cc)
              if (P[(size_t)j * Mc + cc] != 0.0) { cmin = std::min(cmin, cc); break; }
          T.cwin[(size_t)k * 3 * 4096 + i * 4096 + r] = std::max(0, std::min(cmin, Mc - CWmax));
        }
      }
      T.td.push_back(td);
    }
    T.d_td = c.upload(T.td);
    T.ip = c.upload(ip);
    T.wp = c.upload(wp);
    T.d_cwin = c.upload(T.cwin);
  }
}

void setup_assembly_tables(ieti_ctx &c) {
  const int d = c.dim, p = c.p, P1 = p + 1;
  std::vector<double> val, der, wq, ctrl;
  std::vector<int> toff, woff;
  std::vector<double> xg(P1), wg(P1), bd(2 * P1);
  c.toff_h.assign(c.npatch, {0, 0, 0});
  c.woff_h.assign(c.npatch, {0, 0, 0});
  for (int k = 0; k < c.npatch; ++k) {
    gauss_legendre01(P1, xg.data(), wg.data());
    for (int i = 0; i < 3; ++i) {
      c.toff_h[k][i] = (int)val.size();
      c.woff_h[k][i] = (int)wq.size();
      if (i >= d) { toff.push_back(c.toff_h[k][i]); woff.push_back(c.woff_h[k][i]); continue; }
      const auto &t = c.T.patch[k].knots[i];
      std::vector<double> u;
      for (double v : t) if (u.empty() || v != u.back()) u.push_back(v);
      for (size_t e = 0; e + 1 < u.size(); ++e) {
        for (int q = 0; q < P1; ++q) {
          double x = u[e] + (u[e + 1] - u[e]) * xg[q];
          int span;
          bspline_basis_ders(t, p, x, 1, span, bd.data());
          if (span - p != (int)e) throw IetiError(IETI_E_ARG, "unexpected knot span (interior knots must be simple)");
          for (int j = 0; j < P1; ++j) { val.push_back(bd[j]); der.push_back(bd[P1 + j]); }
          wq.push_back((u[e + 1] - u[e]) * wg[q]);
        }
      }
      toff.push_back(c.toff_h[k][i]);
      woff.push_back(c.woff_h[k][i]);
    }
  }
  c.d_val = c.upload(val);
  c.d_der = c.upload(der);
  c.d_wq = c.upload(wq);
  c.d_toff = c.upload(toff);
  c.d_woff = c.upload(woff);
  c.ctrl_off.assign(c.npatch + 1, 0);
  for (int k = 0; k < c.npatch; ++k) {
    ctrl.insert(ctrl.end(), c.T.patch[k].ctrl.begin(), c.T.patch[k].ctrl.end());
    c.ctrl_off[k + 1] = (long long)ctrl.size();
  }
  c.d_ctrl = c.upload(ctrl);
}

void nq_of(ieti_ctx &c, int k, int *nq, long long &nqt) {
  nqt = 1;
  for (int i = 0; i < 3; ++i) {
    nq[i] = (i < c.dim) ? c.T.patch[k].melem[i] * (c.p + 1) : 1;
    nqt *= nq[i];
  }
}

void setup_fine_stencils(ieti_ctx &c) {
  const int d = c.dim, p = c.p;
  const int Lf = c.L - 1;
  Level &LN = c.HN.lev[Lf], &LD = c.HD.lev[Lf];
  // 1D mass tables for the Neumann fine grids (R4)
  std::vector<double> mass;
  const int W1 = 2 * p + 1;
  for (int k = 0; k < c.npatch; ++k) {
    GridDesc &g = LN.g[k];
    g.mass_off = (int)mass.size();
    g.mass_beta = c.T.floating[k] ? -c.a.alpha_reg : 0.0;
    for (int i = 0; i < d; ++i) {
      const auto &t = c.T.patch[k].knots[i];
      std::vector<double> M1 = mass_1d(t, p);
      int M = g.M[i];
      for (int a = 0; a < M; ++a)
        for (int o = -p; o <= p; ++o) {
          int b = a + o;
          mass.push_back((b >= 0 && b < M) ? M1[(size_t)a * M + b] : 0.0);
        }
    }
  }
  LN.mass = c.upload(mass);
  c.h2d(LN.d_g, LN.g.data(), LN.g.size() * sizeof(GridDesc));
  long long maxq = 0;
  for (int k = 0; k < c.npatch; ++k) {
    int nq[3];
    long long nqt;
    nq_of(c, k, nq, nqt);
    maxq = std::max(maxq, nqt);
  }
  double *G = c.alloc<double>(maxq * (d == 3 ? 6 : 3));
  int *bad = c.alloc<int>(1);
  long long maxsf = 0;
  for (int k = 0; k < c.npatch; ++k)
    maxsf = std::max(maxsf, sf_scratch_doubles(d, p, c.T.patch[k].M, c.T.patch[k].melem));
  size_t mark = c.allocs.size();
  double *scratch = c.alloc<double>(maxsf);
  for (int k = 0; k < c.npatch; ++k) {
    int nq[3];
    long long nqt;
    nq_of(c, k, nq, nqt);
    int M[3] = {c.T.patch[k].M[0], c.T.patch[k].M[1], c.T.patch[k].M[2]};
    launch_geometry2(d, p, nq, M, c.d_val, c.d_der, c.d_toff + 3 * k, c.d_wq, c.d_woff + 3 * k,
                     c.d_ctrl + c.ctrl_off[k], G, nullptr, nullptr, bad, c.st);
    // Neumann fine stencil: sum-factorised assembly (K, + alpha Mhat on floating patches, R4)
    double alpha = c.T.floating[k] ? c.a.alpha_reg : 0.0;
    launch_stencil_sf(d, p, LN.g[k], LN.d_ci, c.ncol, c.T.patch[k].melem, c.d_val, c.d_der, c.toff_h[k].data(), G,
                      alpha, LN.mass, LN.coef, scratch, c.st);
  }
  CK(cudaStreamSynchronize(c.st));
  cudaFree(scratch);
  c.allocs.resize(mark);
  // Dirichlet fine stencil: the interior rows of the true K (Neumann rows minus alpha Mhat; the
  // Gamma columns are kept for K_IG v), copied row by row
  for (int k = 0; k < c.npatch; ++k) {
    const GridDesc &gD = LD.g[k], &gN = LN.g[k];
    std::vector<int> rgrid(gD.nrows, k), rrow(gD.nrows), rflat(gD.nrows);
    for (int col = 0; col < c.ncol; ++col) {
      const ColourInfo &ci = LD.ci[gD.col_off + col];
      for (int j2 = 0; j2 < ci.n[2]; ++j2)
        for (int j1 = 0; j1 < ci.n[1]; ++j1)
          for (int j0 = 0; j0 < ci.n[0]; ++j0) {
            const int r = ci.start + j0 + ci.n[0] * (j1 + ci.n[1] * j2);
            int i[3] = {ci.first[0] + (p + 1) * j0, ci.first[1] + (p + 1) * j1, ci.first[2] + (p + 1) * j2};
            rrow[r] = cm_row(gN, LN.ci.data() + gN.col_off, p, d, i);
            rflat[r] = i[0] + gN.M[0] * (i[1] + gN.M[1] * i[2]);
          }
    }
    size_t mk = c.allocs.size();
    int *d_rg = c.upload(rgrid), *d_rr = c.upload(rrow), *d_rf = c.upload(rflat);
    const bool rowmajor = gD.tg > 1;
    launch_extract_rows(d, p, LN.d_g, LN.coef, LN.mass, d_rg, d_rr, d_rf, gD.nrows, LD.coef + gD.coef_off,
                        rowmajor ? 1 : (gD.tg < 0 ? -1 : gD.ld), rowmajor ? c.S : 1, c.st);
    CK(cudaStreamSynchronize(c.st));
    for (size_t i = mk; i < c.allocs.size(); ++i) cudaFree(c.allocs[i]);
    c.allocs.resize(mk);
  }
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  if (hbad) throw IetiError(IETI_E_GEOMETRY, "non-positive Jacobian determinant at a quadrature point");
}

void setup_galerkin(ieti_ctx &c, Hier &H) {
  // a patch's two Galerkin kernels fill a fraction of the GPU (C5's finest level: 335 blocks), and patches
  // are independent: NS patches in flight on their own streams, each with its own scratch B
  constexpr int NS = 8;
  const int ns = std::max(1, std::min(NS, c.npatch));
  cudaStream_t st[NS];
  for (int i = 0; i < ns; ++i) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  CK(cudaStreamSynchronize(c.st));
  for (int l = c.L - 1; l >= 1; --l) {
    Level &Lf = H.lev[l], &Lc = H.lev[l - 1];
    Trans &T = c.tr[l];
    long long maxB = 0;
    for (int k = 0; k < c.npatch; ++k) maxB = std::max(maxB, (long long)Lf.g[k].nrows * ipow(T.CW, c.dim));
    maxB = (maxB + 31) / 32 * 32;
    size_t mark = c.allocs.size();
    double *B = c.alloc<double>(maxB * ns);
    CK(cudaStreamSynchronize(c.st));               // alloc() zeroes on the library stream: finish before the side streams write
    for (int k = 0; k < c.npatch; ++k) {
      launch_galerkin_stages(c.dim, c.p, Lf.g[k], Lf.d_ci, Lc.g[k], Lc.d_ci, T.td[k], T.CW,
                             T.d_cwin + (size_t)k * 3 * 4096, T.ip, T.wp, Lf.coef, Lc.coef, B + maxB * (k % ns), c.ncol,
                             st[k % ns]);
    }
    // the next level reads this level's coarse stencils: join every stream
    for (int i = 0; i < ns; ++i) CK(cudaStreamSynchronize(st[i]));
    CK(cudaGetLastError());
    // free the scratch immediately (it can be large)
    for (size_t i = mark; i < c.allocs.size(); ++i) cudaFree(c.allocs[i]);
    c.allocs.resize(mark);
  }
  for (int i = 0; i < ns; ++i) cudaStreamDestroy(st[i]);
}

void setup_coarsest(ieti_ctx &c, Hier &H) {
  Level &L0 = H.lev[0];
  std::vector<long long> off(c.npatch + 1, 0);
  std::vector<int> n(c.npatch);
  int maxrows = 0;
  for (int k = 0; k < c.npatch; ++k) {
    n[k] = L0.g[k].nrows;
    off[k + 1] = off[k] + (long long)n[k] * n[k];
    maxrows = std::max(maxrows, n[k]);
  }
  if (maxrows > 8192) throw IetiError(IETI_E_ARG, "coarsest level too large");
  c.max_coarse_rows = std::max(c.max_coarse_rows, maxrows);
  L0.inv = c.alloc<double>(off[c.npatch]);
  double *scratch = c.alloc<double>(off[c.npatch]);
  L0.inv_off.assign(off.begin(), off.end() - 1);
  L0.d_inv_off = c.upload(L0.inv_off);
  int *d_n = c.upload(n);
  int *fail = c.alloc<int>(1);
  launch_dense_from_stencil(c.dim, c.p, L0.d_g, L0.d_ci, L0.coef, c.npatch, L0.inv, L0.d_inv_off, c.st, maxrows);
  launch_spd_inverse2(L0.inv, L0.d_inv_off, d_n, c.npatch, scratch, L0.d_inv_off, fail, c.st);
  int hfail = 0;
  CK(cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  CK(cudaGetLastError());
  if (hfail) throw IetiError(IETI_E_NOT_SPD, "coarsest-level matrix not SPD");
}

// ------------------------------------------------------------------------------------------
// interface tables
// ------------------------------------------------------------------------------------------
long long box_pos_host(const GridDesc &g, int p, int dim, const int *i) { return sl_pos(g, p, dim, i); }

void setup_interface(ieti_ctx &c) {
  Topo &T = c.T;
  const int d = c.dim, p = c.p;
  const Level &LN = c.HN.lev[c.L - 1];
  std::vector<int> gbox, bt_ptr{0}, bt_m, bdt_ptr{0}, bdt_m, crow;
  std::vector<double> bt_w, bdt_w, cw;
  std::vector<long long> gabs;
  std::vector<int> Rcat;
  std::vector<int> goff(c.npatch + 1, 0);
  c.pif.assign(c.npatch, PatchIface{});
  long long phi_off = 0, phif_off = 0;
  int pi_off = 0;
  for (int k = 0; k < c.npatch; ++k) {
    const GridDesc &g = LN.g[k];
    PatchIface &P = c.pif[k];
    P.g_off = goff[k];
    P.ng = (int)T.gamma[k].size();
    P.npi = (int)T.R[k].size();
    if (P.npi > 64) throw IetiError(IETI_E_UNSUPPORTED, "more than 64 primal constraints on one patch");
    P.pi_off = pi_off;
    P.phi_off = phi_off;
    P.phif_off = phif_off;
    P.box_off = c.box_off[k];
    P.box = g.box;
    P.floating = c.T.floating[k];
    goff[k + 1] = goff[k] + P.ng;
    pi_off += P.npi;
    phi_off += (long long)P.npi * P.ng;
    phif_off += (long long)P.npi * P.box;
    for (int gi = 0; gi < P.ng; ++gi) {
      int flat = T.gamma[k][gi];
      int idx[3] = {0, 0, 0}, f = flat;
      for (int i = 0; i < d; ++i) { idx[i] = f % g.M[i]; f /= g.M[i]; }
      long long pos = box_pos_host(g, p, d, idx);
      gbox.push_back((int)pos);
      gabs.push_back(c.box_off[k] + pos);
      for (int e = T.bt_ptr[k][gi]; e < T.bt_ptr[k][gi + 1]; ++e) { bt_m.push_back(T.bt_m[k][e]); bt_w.push_back(T.bt_w[k][e]); }
      bt_ptr.push_back((int)bt_m.size());
      for (int e = T.bdt_ptr[k][gi]; e < T.bdt_ptr[k][gi + 1]; ++e) { bdt_m.push_back(T.bdt_m[k][e]); bdt_w.push_back(T.bdt_w[k][e]); }
      bdt_ptr.push_back((int)bdt_m.size());
      crow.push_back(T.c_row[k][gi]);
      cw.push_back(T.c_w[k][gi]);
    }
    for (int j = 0; j < P.npi; ++j) Rcat.push_back(T.R[k][j]);
  }
  c.ngamma = goff[c.npatch];
  c.npi_tot = pi_off;
  c.phiG_n = phi_off;
  c.phiF_n = phif_off;
  auto gidx = [&](int k, int flat) {
    auto it = std::lower_bound(T.gamma[k].begin(), T.gamma[k].end(), flat);
    if (it == T.gamma[k].end() || *it != flat) throw IetiError(IETI_E_TOPOLOGY, "multiplier dof not on Gamma");
    return goff[k] + (int)(it - T.gamma[k].begin());
  };
  std::vector<int> gp(T.n_lambda), gm(T.n_lambda), bd_ptr{0}, bd_g;
  std::vector<double> bd_w;
  for (int i = 0; i < T.n_lambda; ++i) {
    gp[i] = (T.mkp[i] >= 0) ? gidx(T.mkp[i], T.map_[i]) : -1;     // -1: side on a remote patch
    gm[i] = (T.mkm[i] >= 0) ? gidx(T.mkm[i], T.mam[i]) : -1;
    for (int e = T.bd_ptr[i]; e < T.bd_ptr[i + 1]; ++e) {
      bd_g.push_back(gidx(T.bd_k[e], T.bd_a[e]));
      bd_w.push_back(T.bd_w[e]);
    }
    bd_ptr.push_back((int)bd_g.size());
  }
  // coarse gather CSR: per global primal id, contributions (pi_off[k] + j) in ascending k
  std::vector<std::vector<int>> srcs(T.n_pi);
  for (int k = 0; k < c.npatch; ++k)
    for (int j = 0; j < (int)T.R[k].size(); ++j) srcs[T.R[k][j]].push_back(c.pif[k].pi_off + j);
  std::vector<int> gpi_ptr{0}, gpi_src;
  for (int i = 0; i < T.n_pi; ++i) {
    for (int s : srcs[i]) gpi_src.push_back(s);
    gpi_ptr.push_back((int)gpi_src.size());
  }
  c.d_pif = c.upload(c.pif);
  c.d_gbox = c.upload(gbox);
  c.d_gabs = c.upload(gabs);
  c.d_bt_ptr = c.upload(bt_ptr); c.d_bt_m = c.upload(bt_m); c.d_bt_w = c.upload(bt_w);
  c.d_bdt_ptr = c.upload(bdt_ptr); c.d_bdt_m = c.upload(bdt_m); c.d_bdt_w = c.upload(bdt_w);
  c.d_crow = c.upload(crow); c.d_cw = c.upload(cw);
  {
    // CSR of the constraint rows: for patch k and primal column j the local Gamma indices g with
    // crow = j, in ascending g (k_iface_w sums C x row by row)
    std::vector<int> cptr{0}, cidx;
    for (int k = 0; k < c.npatch; ++k) {
      const PatchIface &P = c.pif[k];
      std::vector<std::vector<int>> rows(P.npi);
      for (int g = 0; g < P.ng; ++g) {
        const int j = crow[P.g_off + g];
        if (j >= 0 && j < P.npi) rows[j].push_back(g);
      }
      for (int j = 0; j < P.npi; ++j) {
        cidx.insert(cidx.end(), rows[j].begin(), rows[j].end());
        cptr.push_back((int)cidx.size());
      }
    }
    if ((int)cptr.size() != c.npi_tot + 1) throw IetiError(IETI_E_TOPOLOGY, "constraint-row CSR size");
    if (cidx.empty()) cidx.push_back(0);
    c.d_cptr = c.upload(cptr);
    c.d_cidx = c.upload(cidx);
  }
  c.d_gp = c.upload(gp); c.d_gm = c.upload(gm);
  c.d_bd_ptr = c.upload(bd_ptr); c.d_bd_g = c.upload(bd_g); c.d_bd_w = c.upload(bd_w);
  c.d_R = c.upload(Rcat);
  c.d_gpi_ptr = c.upload(gpi_ptr); c.d_gpi_src = c.upload(gpi_src);
  c.phiG = c.alloc<double>(c.phiG_n);
  c.phiF = c.alloc<double>(c.phiF_n);
  c.t_all = c.alloc<double>(c.npi_tot);
  {
    const char *ft = getenv("IETI_FULLT");
    int mx = 0;
    for (const auto &pf : c.pif) mx = std::max(mx, pf.npi);
    c.full_t_npi = (ft && ft[0] == '0') ? 0 : mx;
    c.rGt = c.alloc<double>(std::max(1, c.ngamma));
  }
  c.cvec = c.alloc<double>(c.npi_tot);
  c.gPi = c.alloc<double>(T.n_pi);
  c.uPi = c.alloc<double>(T.n_pi);
  c.rG = c.alloc<double>(c.ngamma);
  c.wG = c.alloc<double>(c.ngamma);
}

// ------------------------------------------------------------------------------------------
// row-list stencils of M_sD
// ------------------------------------------------------------------------------------------
void build_rowlist(ieti_ctx &c, ieti_ctx::RowList &RL, Level &src, bool gamma_rows) {
  const int d = c.dim, p = c.p, P1 = p + 1;
  const Level &LN = c.HN.lev[c.L - 1];
  std::vector<int> pos, out, rgrid, rrow, rflat;
  std::vector<BlockEntry> blk;
  int goff = 0;
  for (int k = 0; k < c.npatch; ++k) {
    const GridDesc &g = src.g[k];
    std::vector<std::vector<std::pair<int, int>>> bycol(c.ncol);   // (flat, out)
    if (gamma_rows) {
      for (size_t gi = 0; gi < c.T.gamma[k].size(); ++gi) {
        int f = c.T.gamma[k][gi], i[3] = {0, 0, 0};
        for (int q = 0; q < d; ++q) { i[q] = f % g.M[q]; f /= g.M[q]; }
        int col = 0, pw = 1;
        for (int q = 0; q < d; ++q) { col += (i[q] % P1) * pw; pw *= P1; }
        bycol[col].push_back({c.T.gamma[k][gi], goff + (int)gi});
      }
      goff += (int)c.T.gamma[k].size();
    } else {
      long long n = 1;
      for (int q = 0; q < d; ++q) n *= g.M[q];
      for (long long f = 0; f < n; ++f) {
        int i[3] = {0, 0, 0};
        long long ff = f;
        for (int q = 0; q < d; ++q) { i[q] = (int)(ff % g.M[q]); ff /= g.M[q]; }
        bool act = true, band = false;
        for (int q = 0; q < d; ++q) {
          act = act && i[q] >= g.lo[q] && i[q] < g.hi[q];
          band = band || i[q] <= p || i[q] >= g.M[q] - 1 - p;
        }
        if (!act || !band) continue;
        int col = 0, pw = 1;
        for (int q = 0; q < d; ++q) { col += (i[q] % P1) * pw; pw *= P1; }
        bycol[col].push_back({(int)f, (int)sl_pos(g, p, d, i)});
      }
    }
    for (int col = 0; col < c.ncol; ++col) {
      auto &v = bycol[col];
      for (size_t r0 = 0; r0 < v.size(); r0 += 128)
        blk.push_back(BlockEntry{k, col, (int)pos.size() + (int)r0, (int)std::min<size_t>(128, v.size() - r0)});
      for (auto &e : v) {
        int f = e.first, i[3] = {0, 0, 0};
        for (int q = 0; q < d; ++q) { i[q] = f % g.M[q]; f /= g.M[q]; }
        pos.push_back((int)sl_pos(g, p, d, i));
        out.push_back(e.second);
        rgrid.push_back(k);
        rflat.push_back(e.first);
        rrow.push_back(cm_row(g, src.ci.data() + g.col_off, p, d, i));
      }
    }
  }
  (void)LN;
  RL.nrows = (long long)pos.size();
  RL.ld = (RL.nrows + 31) / 32 * 32;
  RL.coef = c.alloc<double>(RL.ld * c.S);
  c.stencil_bytes += RL.ld * c.S * 8;
  RL.pos = c.upload(pos);
  RL.out = c.upload(out);
  RL.blk = c.upload(blk);
  RL.nblk = (int)blk.size();
  size_t mark = c.allocs.size();
  int *d_rgrid = c.upload(rgrid), *d_rrow = c.upload(rrow), *d_rflat = c.upload(rflat);
  launch_extract_rows(c.dim, c.p, src.d_g, src.coef, src.mass, d_rgrid, d_rrow, d_rflat, RL.nrows, RL.coef, RL.ld, 1,
                      c.st);
  CK(cudaStreamSynchronize(c.st));
  CK(cudaGetLastError());
  for (size_t i = mark; i < c.allocs.size(); ++i) cudaFree(c.allocs[i]);
  c.allocs.resize(mark);
}

void setup_rowlists(ieti_ctx &c) {
  build_rowlist(c, c.RG, c.HN.lev[c.L - 1], true);     // true K = (K + alpha Mhat) - alpha Mhat on floating
  build_rowlist(c, c.RB, c.HD.lev[c.L - 1], false);    // Dirichlet fine rows hold true K with Gamma columns
  c.yG = c.alloc<double>(std::max(1, c.ngamma));
}

// ------------------------------------------------------------------------------------------
// primal basis (Eq. (6)) by batched PCG on A = K + delta C^T C, preconditioner N_1
// ------------------------------------------------------------------------------------------
// X <- A^{-1} X for a small dense m x m system (LU with partial pivoting), X is m x nrhs row-major
void small_lu_solve(std::vector<double> A, int m, std::vector<double> &X, int nrhs) {
  for (int k = 0; k < m; ++k) {
    int piv = k;
    for (int i = k + 1; i < m; ++i)
      if (std::fabs(A[(size_t)i * m + k]) > std::fabs(A[(size_t)piv * m + k])) piv = i;
    if (!(std::fabs(A[(size_t)piv * m + k]) > 0.0)) throw IetiError(IETI_E_NOT_SPD, "singular primal-basis system");
    if (piv != k) {
      for (int j = 0; j < m; ++j) std::swap(A[(size_t)k * m + j], A[(size_t)piv * m + j]);
      for (int j = 0; j < nrhs; ++j) std::swap(X[(size_t)k * nrhs + j], X[(size_t)piv * nrhs + j]);
    }
    for (int i = k + 1; i < m; ++i) {
      const double f = A[(size_t)i * m + k] / A[(size_t)k * m + k];
      if (f == 0.0) continue;
      for (int j = k; j < m; ++j) A[(size_t)i * m + j] -= f * A[(size_t)k * m + j];
      for (int j = 0; j < nrhs; ++j) X[(size_t)i * nrhs + j] -= f * X[(size_t)k * nrhs + j];
    }
  }
  for (int k = m - 1; k >= 0; --k)
    for (int j = 0; j < nrhs; ++j) {
      double v = X[(size_t)k * nrhs + j];
      for (int i = k + 1; i < m; ++i) v -= A[(size_t)k * m + i] * X[(size_t)i * nrhs + j];
      X[(size_t)k * nrhs + j] = v / A[(size_t)k * m + k];
    }
}

void small_spd_inverse(std::vector<double> &A, int n) {   // in place, Cholesky
  std::vector<double> L(A);
  for (int j = 0; j < n; ++j) {
    double s = L[j * n + j];
    for (int k = 0; k < j; ++k) s -= L[j * n + k] * L[j * n + k];
    if (!(s > 0.0)) throw IetiError(IETI_E_NOT_SPD, "small matrix not SPD");
    L[j * n + j] = std::sqrt(s);
    for (int i = j + 1; i < n; ++i) {
      double t = L[i * n + j];
      for (int k = 0; k < j; ++k) t -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = t / L[j * n + j];
    }
  }
  // columns of the inverse: independent forward / backward substitutions, spread over the host's
  // cores (each column computed the same way whatever the thread: deterministic); the backward pass
  // reads L^T row-wise
  std::vector<double> LT((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) LT[(size_t)k * n + i] = L[(size_t)i * n + k];
  auto cols = [&](int c_begin, int c_end) {
    std::vector<double> y(n);
    for (int c0 = c_begin; c0 < c_end; ++c0) {
      for (int i = 0; i < n; ++i) {
        double s = (i == c0) ? 1.0 : 0.0;
        for (int k = 0; k < i; ++k) s -= L[(size_t)i * n + k] * y[k];
        y[i] = s / L[(size_t)i * n + i];
      }
      for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < n; ++k) s -= LT[(size_t)i * n + k] * y[k];
        y[i] = s / L[(size_t)i * n + i];
      }
      for (int i = 0; i < n; ++i) A[(size_t)i * n + c0] = y[i];
    }
  };
  const int nt = std::max(1, std::min<int>(16, (int)std::thread::hardware_concurrency()));
  if (n < 128 || nt == 1) {
    cols(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) th.emplace_back(cols, (int)((long long)n * t / nt), (int)((long long)n * (t + 1) / nt));
  for (auto &x : th) x.join();
}

void batched_pcg_alloc(ieti_ctx &c, BatchedPcg &S, Batch &B);
void batched_pcg_capture(ieti_ctx &c, BatchedPcg &S, int gid_init, int gid_body);
int batched_pcg_run(ieti_ctx &c, BatchedPcg &S, cudaStream_t s, int tgid_init, int tgid_body);

void setup_primal_basis(ieti_ctx &c) {
  NvtxRange nv("ieti primal basis (Eq. 6)");
  Topo &T = c.T;
  const int Lf = c.L - 1;
  std::vector<int> all_patch, all_col;
  for (int k = 0; k < c.npatch; ++k)
    for (int j = 0; j < c.pif[k].npi; ++j) { all_patch.push_back(k); all_col.push_back(j); }
  const int ntot = (int)all_patch.size();
  bool basis_failed = false;
  std::vector<double> H_all;                     // per problem: C z (npi values, stride 64)
  H_all.assign((size_t)ntot * 64, 0.0);
  // chunking by memory
  long long per_prob = 0;
  for (int l = 0; l < c.L; ++l) per_prob += 3 * (long long)c.BN.lv[l].maxbox;
  per_prob += 4 * (long long)c.BN.lv[Lf].maxbox;
  per_prob *= 8;
  size_t free_b = 0, tot_b = 0;
  CK(cudaMemGetInfo(&free_b, &tot_b));
  long long budget = (long long)(free_b * 0.5);
  int chunk = (int)std::max<long long>(1, std::min<long long>(ntot, budget / std::max<long long>(1, per_prob)));
  chunk = std::min(chunk, 4096);
  const double tol = (c.a.basis_tol > 0) ? c.a.basis_tol : 1e-12;
  int maxit_used = 0;
  int *basis_ctr_host = nullptr;
  CK(cudaMallocHost(&basis_ctr_host, 3 * sizeof(int)));
  struct PinFree { int *p; ~PinFree() { if (p) cudaFreeHost(p); } } pin_free{basis_ctr_host};
  // PCG chunks of whole patches with <= IETI_BASIS_MB (256) MB of finest-level x boxes; the colour phases of
  // every V-cycle find x in L2 (a phase reads all of x); coefficients are read once per chunk
  std::vector<int> cbound{0};
  {
    const char *bm = getenv("IETI_BASIS_MB");             // A/B: x bytes per basis chunk (default 64 MB)
    const long long cap_mb = (bm && atoll(bm) > 0) ? atoll(bm) : 256;   // measured: 32 MB 52 s, 64 48.5 s, 128 41.4 s, 256 40.0 s (C5 setup)
    const long long cap = std::max<long long>(1, (cap_mb << 20) / (8LL * std::max(1, c.BN.lv[Lf].maxbox)));
    int cur = 0;
    for (int k = 0; k < c.npatch; ++k) {
      const int n = c.pif[k].npi;
      if (cur > 0 && cur + n > std::min<long long>(cap, chunk)) {
        cbound.push_back(cbound.back() + cur);
        cur = 0;
      }
      cur += n;
    }
    if (cur > 0) cbound.push_back(cbound.back() + cur);
  }
  for (size_t ci = 0; ci + 1 < cbound.size(); ++ci) {
    const int c0 = cbound[ci], np = cbound[ci + 1] - cbound[ci];
    std::vector<int> pp(all_patch.begin() + c0, all_patch.begin() + c0 + np);
    std::vector<int> pc(all_col.begin() + c0, all_col.begin() + c0 + np);
    size_t mark = c.allocs.size();
    Batch SB;
    build_batch(c, SB, c.HN, pp);
    BLevel &bf = SB.lv[Lf];
    int *d_pp = c.upload(pp), *d_pc = c.upload(pc);
    double *d_cx = c.alloc<double>((long long)np * 64);
    // Y = K^+ C^T (I - 11^T/n) (floating) or K^{-1} C^T: batched PCG on the true K (one problem
    // per (patch, column)), preconditioner one Neumann V-cycle (K + alpha Mhat on floating
    // patches, R4 -- the paper's regularised MG), device-side scalars, captured graphs
    BatchedPcg S;
    S.ctr_host = basis_ctr_host;
    batched_pcg_alloc(c, S, SB);
    S.tol = tol;
    S.maxit = 2000;
    S.applyA = [&](const double *xin, double *yout, cudaStream_t st) {
      apply_level(c, SB, Lf, xin, yout, 1.0, true, st);   // true K (mass term removed)
    };
    std::vector<int> projh(np);
    for (int i = 0; i < np; ++i) projh[i] = c.pif[pp[i]].floating;
    S.proj = c.upload(projh);
    bk_rhs_ct(np, d_pp, d_pc, bf.d_pr, c.d_pif, c.d_gbox, c.d_crow, c.d_cw, bf.b, c.st);
    batched_pcg_capture(c, S, 6, 7);
    const int it = batched_pcg_run(c, S, c.st, -1, -1);
    cudaGraphExecDestroy(S.g_init);
    cudaGraphExecDestroy(S.g_body);
    if ((it >= S.maxit && S.ctr_host[1] > 0) || S.ctr_host[2] > 0) basis_failed = true;   // reported collectively below
    maxit_used = std::max(maxit_used, it);
    if (getenv("IETI_VERBOSE")) {
      std::vector<int> its(np);
      CK(cudaMemcpy(its.data(), S.its, np * sizeof(int), cudaMemcpyDeviceToHost));
      long long sum = 0;
      int mn = 1 << 30, mx = 0;
      for (int v : its) { sum += v; mn = std::min(mn, v); mx = std::max(mx, v); }
      fprintf(stderr, "[ieti] basis chunk %zu: %d columns, PCG iterations min %d mean %.1f max %d (loop ran %d)\n", ci, np,
              mn, (double)sum / std::max(1, np), mx, it);
    }
    double *X = S.X;
    cudaStream_t s = c.st;
    // G columns: C y_j ; store Y into the full-Phibar pool
    bk_cx(np, d_pp, bf.d_pr, c.d_pif, c.d_gbox, c.d_crow, c.d_cw, X, d_cx, 64, s);
    CK(cudaMemcpyAsync(H_all.data() + (size_t)c0 * 64, d_cx, (size_t)np * 64 * sizeof(double), cudaMemcpyDeviceToHost, s));
    bk_prob_cols(np, bf.maxbox, d_pp, d_pc, bf.d_pr, c.d_pif, X, c.phiF, 1, s);
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    // release chunk memory
    for (size_t i = mark; i < c.allocs.size(); ++i) cudaFree(c.allocs[i]);
    c.allocs.resize(mark);
  }
  c.basis_its = maxit_used;
  // Phibar = Y M + 1 c^T per patch (Eq. (6): K phibar_j = -C^T mu_j, C phibar_j = e_j):
  //   non-floating: M = G^{-1}, c = 0            (G = C Y = C K^{-1} C^T, SPD)
  //   floating:     [[-G, 1], [1^T, 0]] [mu_j; c_j] = [e_j; 0],  M = -[mu_j]
  std::vector<double> Mall, call((size_t)std::max(1, c.npi_tot), 0.0);
  std::vector<long long> hoff(c.npatch, 0);
  {
    int q = 0;
    for (int k = 0; k < c.npatch; ++k) {
      const int n = c.pif[k].npi;
      hoff[k] = (long long)Mall.size();
      std::vector<double> G((size_t)n * n);
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) G[(size_t)i * n + j] = H_all[(size_t)(q + j) * 64 + i];   // G[i][j] = (C y_j)_i
      if (n && !c.pif[k].floating) {
        for (int i = 0; i < n; ++i)
          for (int j = i + 1; j < n; ++j) {
            double a = 0.5 * (G[(size_t)i * n + j] + G[(size_t)j * n + i]);
            G[(size_t)i * n + j] = G[(size_t)j * n + i] = a;
          }
        small_spd_inverse(G, n);
        Mall.insert(Mall.end(), G.begin(), G.end());
      } else if (n) {
        const int m = n + 1;
        std::vector<double> A((size_t)m * m, 0.0), X((size_t)m * n, 0.0);
        for (int i = 0; i < n; ++i) {
          for (int j = 0; j < n; ++j) A[(size_t)i * m + j] = -G[(size_t)i * n + j];
          A[(size_t)i * m + n] = 1.0;
          A[(size_t)n * m + i] = 1.0;
          X[(size_t)i * n + i] = 1.0;
        }
        small_lu_solve(A, m, X, n);                       // X = A^{-1} [I; 0]
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) Mall.push_back(-X[(size_t)i * n + j]);
        for (int j = 0; j < n; ++j) call[c.pif[k].pi_off + j] = X[(size_t)n * n + j];
      }
      q += n;
    }
  }
  size_t mark = c.allocs.size();
  double *d_M = c.upload(Mall), *d_c = c.upload(call);
  long long *d_hoff = c.upload(hoff);
  double *Ztmp = c.alloc<double>(c.phiF_n);
  CK(cudaMemcpyAsync(Ztmp, c.phiF, c.phiF_n * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  bk_combine(c.npatch, c.BN.lv[Lf].maxbox, c.d_pif, d_hoff, d_M, d_c, c.HN.lev[Lf].d_g, c.p, c.dim, Ztmp, c.phiF,
             c.st);
  int maxng = 0;
  for (auto &P : c.pif) maxng = std::max(maxng, P.ng);
  bk_extract_gamma(c.npatch, maxng, c.d_pif, c.d_gbox, c.phiF, c.phiG, c.st);
  CK(cudaStreamSynchronize(c.st));
  for (size_t i = mark; i < c.allocs.size(); ++i) cudaFree(c.allocs[i]);
  c.allocs.resize(mark);
  // S_PiPi^(k) = Phibar^T K Phibar (K true stiffness), assembled and inverted on the host
  std::vector<double> S((size_t)T.n_pi * T.n_pi, 0.0);
  for (int c0 = 0; c0 < ntot; c0 += chunk) {
    const int np = std::min(chunk, ntot - c0);
    std::vector<int> pp(all_patch.begin() + c0, all_patch.begin() + c0 + np);
    std::vector<int> pc(all_col.begin() + c0, all_col.begin() + c0 + np);
    size_t mk = c.allocs.size();
    Batch SB;
    std::vector<int> grid(pp);
    // only the fine level is needed: build a one-level view
    build_batch(c, SB, c.HN, pp, false);
    BLevel &bf = SB.lv[Lf];
    int *d_pp = c.upload(pp), *d_pc = c.upload(pc);
    double *AP = c.alloc<double>(bf.n);
    double *d_out = c.alloc<double>((long long)np * 64);
    bk_prob_cols(np, bf.maxbox, d_pp, d_pc, bf.d_pr, c.d_pif, bf.x, c.phiF, 0, c.st);
    apply_level(c, SB, Lf, bf.x, AP, 1.0, true, c.st);
    bk_phi_dots(np, d_pp, bf.d_pr, c.d_pif, c.phiF, AP, d_out, 64, c.st);
    std::vector<double> out((size_t)np * 64);
    CK(cudaMemcpyAsync(out.data(), d_out, out.size() * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    for (int i = 0; i < np; ++i) {
      int k = pp[i], j = pc[i];
      for (int r = 0; r < c.pif[k].npi; ++r) S[(size_t)T.R[k][r] * T.n_pi + T.R[k][j]] += out[(size_t)i * 64 + r];
    }
    for (size_t i = mk; i < c.allocs.size(); ++i) cudaFree(c.allocs[i]);
    c.allocs.resize(mk);
  }
  int n = T.n_pi;
  if (c.comm.comm) {
    // a rank whose basis PCG failed must not leave the others waiting in the allreduce below:
    // agree on the failure first, then every rank reports it
    double *dflag = c.alloc<double>(1);
    const double fl = basis_failed ? 1.0 : 0.0;
    CK(cudaMemcpyAsync(dflag, &fl, sizeof(double), cudaMemcpyHostToDevice, c.st));
    c.comm.allreduce_sum(dflag, 1, c.st);
    double tot = 0;
    CK(cudaMemcpyAsync(&tot, dflag, sizeof(double), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    basis_failed = tot > 0;
  }
  if (basis_failed) throw IetiError(IETI_E_NOT_SPD, "primal-basis PCG did not converge");
  if (c.comm.comm && n > 0) {
    // S_PiPi = sum over ALL patches: sum the per-rank partial matrices (every rank gets the same)
    size_t mk = c.allocs.size();
    double *dS = c.upload(S);
    c.comm.allreduce_sum(dS, (size_t)n * n, c.st);
    CK(cudaMemcpyAsync(S.data(), dS, S.size() * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    for (size_t i = mk; i < c.allocs.size(); ++i) cudaFree(c.allocs[i]);
    c.allocs.resize(mk);
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      double a = 0.5 * (S[(size_t)i * n + j] + S[(size_t)j * n + i]);
      S[(size_t)i * n + j] = S[(size_t)j * n + i] = a;
    }
  if (n) small_spd_inverse(S, n);
  c.Sinv = c.upload(S);
}

// ------------------------------------------------------------------------------------------
// operators
// ------------------------------------------------------------------------------------------
// ---- multi-GPU exchanges (no-ops on one rank) ----------------------------------------------
// owner -> ghost copies of a local dual vector (before B^T p and B_D^T r)
void halo_fwd(ieti_ctx &c, double *v, cudaStream_t s) {
  if (c.comm.world <= 1 || c.plan.peers.empty()) return;
  const Plan &P = c.plan;
  ik_pack(P.send_ptr.back(), c.d_send_idx, v, c.xs, s);
  c.comm.exchange(P.peers, c.xs, P.send_ptr, c.xr, P.recv_ptr, s);
  ik_unpack(P.recv_ptr.back(), c.d_recv_idx, c.xr, v, s);
}
// ghost partial sums -> owner, added in ascending peer order (after B w and B_D y)
void halo_rev(ieti_ctx &c, double *v, cudaStream_t s) {
  if (c.comm.world <= 1 || c.plan.peers.empty()) return;
  const Plan &P = c.plan;
  ik_pack(P.recv_ptr.back(), c.d_recv_idx, v, c.xs, s);
  c.comm.exchange(P.peers, c.xs, P.recv_ptr, c.xr, P.send_ptr, s);
  ik_rsum(P.n_own, c.d_rsum_ptr, c.d_rsum_src, c.xr, v, s);
}
// global sum of per-block partials: returns (pointer, count) for the consumer's fixed-order sum
std::pair<const double *, int> allsum(ieti_ctx &c, const double *partial, int nb, cudaStream_t s) {
  if (!c.comm.comm) return {partial, nb};
  ik_reduce_to(partial, nb, c.red_send, s);
  c.comm.allgather(c.red_send, c.red_all, 1, s);
  return {c.red_all, c.comm.world};
}
// coarse right-hand side g_Pi = sum over ALL patches: per-rank partials summed in rank order
void coarse_allsum(ieti_ctx &c, cudaStream_t s) {
  if (!c.comm.comm || c.T.n_pi == 0) return;
  c.comm.allgather(c.gPi, c.g_all, c.T.n_pi, s);
  ik_sum_ranks(c.T.n_pi, c.comm.world, c.g_all, c.gPi, s);
}

// ---- C2 inner PCG (R19): per patch PCG on K, preconditioner N_1, x0 = 0, rel. tol inner_tol ----
// q is read from the Neumann fine rhs box (BN.b, written by k_iface_t / k_full_t); x lands in IX.
void inner_graph_head(ieti_ctx &c, BatchedPcg &S, bool first, cudaStream_t s) {
  const int Lf = c.L - 1;
  Batch &B = *S.B;
  BLevel &bf = B.lv[Lf];
  const GridDesc *g = B.H->lev[Lf].d_g;
  if (first) ik_inner_init(B.nprob, bf.d_pr, g, bf.b, S.R, S.X, S.qn, S.active, S.its, S.ctr, s);
  else ik_copy(bf.n, S.R, bf.b, s);
  ncycles(c, B, 1, s);                                               // z = N_1(r) in the batch's x
  ik_inner_dir(B.nprob, bf.d_pr, g, S.R, bf.x, S.P, S.rho, S.active, first ? 1 : 0, s);
  ik_inner_begin(S.ctr, s);
  S.applyA(S.P, S.AP, s);
  ik_inner_step(B.nprob, bf.d_pr, g, S.P, S.AP, S.X, S.R, S.rho, S.qn, S.active, S.its, S.ctr, S.tol, S.proj, c.p,
                c.dim, s);
  CK(cudaMemcpyAsync(S.ctr_host, S.ctr, 3 * sizeof(int), cudaMemcpyDeviceToHost, s));
}

void read_timing(ieti_ctx &c, int gid);

template <typename F>
cudaGraphExec_t capture(ieti_ctx &c, int gid, F body, size_t *kn);

void batched_pcg_alloc(ieti_ctx &c, BatchedPcg &S, Batch &B) {
  const long long nb = B.lv[c.L - 1].n;
  S.B = &B;
  S.X = c.alloc<double>(nb); S.R = c.alloc<double>(nb); S.P = c.alloc<double>(nb); S.AP = c.alloc<double>(nb);
  S.rho = c.alloc<double>(B.nprob); S.qn = c.alloc<double>(B.nprob);
  S.active = c.alloc<int>(B.nprob); S.its = c.alloc<int>(B.nprob); S.ctr = c.alloc<int>(3);
  if (!S.ctr_host) {
    CK(cudaMallocHost(&S.ctr_host, 3 * sizeof(int)));
    S.ctr_host[0] = S.ctr_host[1] = S.ctr_host[2] = 0;
  }
}

void batched_pcg_capture(ieti_ctx &c, BatchedPcg &S, int gid_init, int gid_body) {
  size_t ka, kb;
  S.g_init = capture(c, gid_init, [&]() { inner_graph_head(c, S, true, c.st); }, &ka);
  S.g_body = capture(c, gid_body, [&]() { inner_graph_head(c, S, false, c.st); }, &kb);
  S.kn[0] = (int)ka;
  S.kn[1] = (int)kb;
}

// runs the whole loop (host-driven; one 8-byte read per iteration); returns the iterations
int batched_pcg_run(ieti_ctx &c, BatchedPcg &S, cudaStream_t s, int tgid_init, int tgid_body) {
  CK(cudaGraphLaunch(S.g_init, s));
  c.inner_launches += S.kn[0];
  CK(cudaStreamSynchronize(s));
  if (tgid_init >= 0) read_timing(c, tgid_init);
  int steps = 1;
  while (S.ctr_host[1] > 0 && steps < S.maxit) {
    CK(cudaGraphLaunch(S.g_body, s));
    c.inner_launches += S.kn[1];
    CK(cudaStreamSynchronize(s));
    if (tgid_body >= 0) read_timing(c, tgid_body);
    ++steps;
  }
  return steps;
}

// C2: the inner local solves (R19); logs the per-patch counts
void inner_run(ieti_ctx &c, cudaStream_t s) {
  batched_pcg_run(c, c.ipcg, s, 4, 5);
  std::vector<int> its(c.npatch);
  CK(cudaMemcpy(its.data(), c.ipcg.its, c.npatch * sizeof(int), cudaMemcpyDeviceToHost));
  c.inner_log.insert(c.inner_log.end(), its.begin(), its.end());
}

// q = F^ pin  (all on device): pre (B^T, coarse), local Neumann solve, post (interface result, B)
void op_F_pre(ieti_ctx &c, double *pin, cudaStream_t s) {
  const int Lf = c.L - 1;
  halo_fwd(c, pin, s);
  // the Neumann rhs pool is zero except at Gamma (written by k_iface_t): one memset of the pool
  CK(cudaMemsetAsync(c.BN.lv[Lf].b, 0, sizeof(double) * c.BN.lv[Lf].n, s));
  ik_iface_t(c.npatch, c.d_pif, c.d_gbox, c.d_bt_ptr, c.d_bt_m, c.d_bt_w, c.phiG, c.d_crow, c.d_cw, pin, c.t_all,
             c.BN.lv[Lf].b, c.rG, s);
  ik_gather_pi(c.T.n_pi, c.d_gpi_ptr, c.d_gpi_src, c.t_all, c.gPi, s);
  coarse_allsum(c, s);
  ik_gemv(c.T.n_pi, c.Sinv, c.gPi, c.uPi, s);
}

void op_F_post(ieti_ctx &c, const double *xN, double *qout, cudaStream_t s) {
  ik_iface_w(c.npatch, c.d_pif, c.d_gbox, c.phiG, c.d_cptr, c.d_cidx, c.d_cw, c.d_R, c.uPi, xN, c.cvec, c.wG, s);
  ik_jump(c.T.n_lambda, c.d_gp, c.d_gm, c.wG, qout, s);
  halo_rev(c, qout, s);
}

// a host-driven inner loop: run now, or (while a program is captured) end the current segment,
// append the loop as its own step and continue capturing into a new segment
void run_loop(ieti_ctx &c, int which, cudaStream_t s) {
  NvtxRange nv(which == 1 ? "inner PCG (Neumann)" : "inner PCG (Dirichlet)");
  if (which == 1) inner_run(c, s);
  else batched_pcg_run(c, c.dpcg, s, 8, 9);
  // an inner solve that stopped at its iteration cap, or broke down, makes the outer solve report it
  BatchedPcg &S = (which == 1) ? c.ipcg : c.dpcg;
  if (S.ctr_host[1] > 0) c.inner_unconverged = true;
  if (S.ctr_host[2] > 0) c.inner_breakdown = true;
}

void end_segment(ieti_ctx &c);

void host_loop(ieti_ctx &c, int which, cudaStream_t s) {
  if (!c.rec_segs) {
    run_loop(c, which, s);
    return;
  }
  end_segment(c);
  ieti_ctx::Seg sg;
  sg.loop = which;
  c.rec_segs->push_back(sg);
  CK(cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal));
}

// local Neumann solve N (R2) or the inner PCG (R19); returns the solution's box pool
// x = A^-1 b per problem by the factored bands: gather b (box) -> v, substitutions, scatter -> x box
const double *direct_solve(ieti_ctx &c, ieti_ctx::Direct &D, const double *b, double *x, long long nbox,
                           cudaStream_t s) {
  ik_gather_pos(D.nv, D.d_pos, b, D.v, s);
  ik_band_solve(D.nprob, D.max_bw, D.d_desc, D.band, D.up, D.d_voff, D.v, s);
  CK(cudaMemsetAsync(x, 0, (size_t)nbox * sizeof(double), s));
  ik_scatter_pos(D.nv, D.d_pos, D.v, x, s);
  return x;
}

const double *local_neumann(ieti_ctx &c, cudaStream_t s) {
  if (c.direct_N) {
    BLevel &bf = c.BN.lv[c.L - 1];
    return direct_solve(c, c.dirN, bf.b, bf.x, bf.n, s);
  }
  if (c.pcg_mode) {
    host_loop(c, 1, s);
    return c.IX;
  }
  ncycles(c, c.BN, c.a.cycles, s);
  return c.BN.lv[c.L - 1].x;
}

// local Dirichlet solve D in M_sD: c_D V-cycles, or the inner PCG on K_II (R27)
const double *local_dirichlet(ieti_ctx &c, cudaStream_t s) {
  if (c.direct_D) {
    BLevel &bf = c.BD.lv[c.L - 1];
    return direct_solve(c, c.dirD, bf.b, bf.x, bf.n, s);
  }
  if (c.dpcg_mode) {
    host_loop(c, 2, s);
    return c.dpcg.X;
  }
  ncycles(c, c.BD, c.a.dirichlet_cycles, s);
  return c.BD.lv[c.L - 1].x;
}

void op_F(ieti_ctx &c, double *pin, double *qout, cudaStream_t s) {
  op_F_pre(c, pin, s);
  const double *x = local_neumann(c, s);
  op_F_post(c, x, qout, s);
}

// z = M_sD r
void op_MsD(ieti_ctx &c, double *rin, double *zout, cudaStream_t s) {
  const int Lf = c.L - 1;
  const GridDesc *gN = c.HN.lev[Lf].d_g;
  const ProbDesc *pN = c.BN.lv[Lf].d_pr;
  halo_fwd(c, rin, s);
  ik_bdt(c.ngamma, c.d_gabs, c.d_bdt_ptr, c.d_bdt_m, c.d_bdt_w, rin, c.vbox, s);         // v = B_D^T r
  // the inner Dirichlet PCG uses the rhs box as its preconditioner input (ik_copy R -> b): the
  // rows outside the band would keep the previous call's residual, so clear the box first
  if (c.dpcg_mode) CK(cudaMemsetAsync(c.BD.lv[Lf].b, 0, sizeof(double) * c.BD.lv[Lf].n, s));
  launch_rowlist(c.dim, c.p, gN, pN, c.RB.blk, c.RB.nblk, c.RB.coef, c.RB.ld, c.RB.pos, c.RB.out, c.vbox, nullptr,
                 c.BD.lv[Lf].b, 0, s);                                                  // b_D = -K_IG v (band)
  const double *zI = local_dirichlet(c, s);                                              // z_I = D(b_D)
  launch_rowlist(c.dim, c.p, gN, pN, c.RG.blk, c.RG.nblk, c.RG.coef, c.RG.ld, c.RG.pos, c.RG.out, zI,
                 c.vbox, c.yG, 1, s);                                                   // y_G = K_G. (v + z_I)
  ik_bd_gather(c.T.n_lambda, c.d_bd_ptr, c.d_bd_g, c.d_bd_w, nullptr, c.yG, zout, s);   // z = B_D y
  halo_rev(c, zout, s);
}

// x = Ktilde^{-1}(fbox - B^T lam) over full patches; result box in ubox (if want_u) and B w into dout
void op_full_pre(ieti_ctx &c, double *lam, cudaStream_t s, const double *fin = nullptr) {
  const int Lf = c.L - 1;
  if (lam) halo_fwd(c, lam, s);
  ik_full_t(c.npatch, c.d_pif, c.d_gbox, c.d_bt_ptr, c.d_bt_m, c.d_bt_w, c.phiF, c.d_crow, c.d_cw, lam,
            fin ? fin : c.fbox, c.t_all, c.BN.lv[Lf].b, s, c.ngamma, c.full_t_npi, c.rGt);
  ik_gather_pi(c.T.n_pi, c.d_gpi_ptr, c.d_gpi_src, c.t_all, c.gPi, s);
  coarse_allsum(c, s);
  ik_gemv(c.T.n_pi, c.Sinv, c.gPi, c.uPi, s);
}

void op_full_post(ieti_ctx &c, const double *xN, double *dout, bool want_u, cudaStream_t s, double *uout = nullptr) {
  const int Lf = c.L - 1;
  ik_iface_w(c.npatch, c.d_pif, c.d_gbox, c.phiG, c.d_cptr, c.d_cidx, c.d_cw, c.d_R, c.uPi, xN, c.cvec, c.wG, s);
  if (dout) {
    ik_jump(c.T.n_lambda, c.d_gp, c.d_gm, c.wG, dout, s);
    halo_rev(c, dout, s);
  }
  if (want_u) ik_full_u(c.npatch, c.BN.lv[Lf].maxbox, c.d_pif, c.phiF, c.cvec, xN, uout ? uout : c.ubox, s);
}

void op_full(ieti_ctx &c, double *lam, double *dout, bool want_u, cudaStream_t s) {
  op_full_pre(c, lam, s);
  const double *x = local_neumann(c, s);
  op_full_post(c, x, dout, want_u, s);
}

void lattice_in(ieti_ctx &c, const double *lat, double *box, bool interior_only, bool mask_active, cudaStream_t s) {
  const int Lf = c.L - 1;
  ik_lattice_to_box(c.dim, c.p, c.npatch, c.maxlat, c.HN.lev[Lf].d_g, c.BN.lv[Lf].d_pr, c.d_lat_off, lat, box,
                    interior_only ? 1 : 0, s);
  if (mask_active) ik_mask_box(c.dim, c.p, c.npatch, c.BN.lv[Lf].maxbox, c.HN.lev[Lf].d_g, c.BN.lv[Lf].d_pr, box, s);
}

void lattice_out(ieti_ctx &c, const double *box, double *lat, cudaStream_t s) {
  const int Lf = c.L - 1;
  ik_box_to_lattice(c.dim, c.p, c.npatch, c.maxlat, c.HN.lev[Lf].d_g, c.BN.lv[Lf].d_pr, c.d_lat_off, box, lat, s);
}

// ------------------------------------------------------------------------------------------
// MG-MG-S operators (R28-R31; oracle/saddle.py).  V~_h vectors and functionals are torn patch
// vectors in the fine Neumann boxes; multiplier vectors as in the dual PCG.
// ------------------------------------------------------------------------------------------
long long bp_n(ieti_ctx &c) { return c.BN.lv[c.L - 1].n; }

// sc[slot] = a . b over the local box (all ranks summed in rank order)
void bp_dot_box(ieti_ctx &c, const double *a, const double *b, int slot, cudaStream_t s) {
  ik_dot_partial(bp_n(c), a, b, c.bpartial, c.nb_box, s);
  auto r = allsum(c, c.bpartial, c.nb_box, s);
  ik_store_scalar(r.first, r.second, c.bsc, slot, 0, s);
}
// sc[slot] = a . b over the owned multipliers
void bp_dot_lam(ieti_ctx &c, const double *a, const double *b, int slot, cudaStream_t s) {
  ik_dot_partial(c.n_own, a, b, c.partial, c.nb_dot, s);
  auto r = allsum(c, c.partial, c.nb_dot, s);
  ik_store_scalar(r.first, r.second, c.bsc, slot, 0, s);
}

// K~ u = (K^(k) u^(k))_k, the true stiffness (mass term of floating patches removed, R4)
void bp_kt(ieti_ctx &c, const double *in, double *out, cudaStream_t s) {
  apply_level(c, c.BN, c.L - 1, in, out, 1.0, true, s);
}

// out = r^ = P^T r + C^T W R g (R31; in == out allowed: k_full_t copies r into the rhs box first)
void bp_can(ieti_ctx &c, const double *in, double *out, cudaStream_t s) {
  const int Lf = c.L - 1;
  ik_full_t(c.npatch, c.d_pif, c.d_gbox, c.d_bt_ptr, c.d_bt_m, c.d_bt_w, c.phiF, c.d_crow, c.d_cw, nullptr, in,
            c.t_all, c.BN.lv[Lf].b, s, c.ngamma, c.full_t_npi, c.rGt);
  ik_gather_pi(c.T.n_pi, c.d_gpi_ptr, c.d_gpi_src, c.t_all, c.gPi, s);
  coarse_allsum(c, s);
  ik_can_add(c.npatch, c.d_pif, c.d_gbox, c.d_crow, c.d_cw, c.d_R, c.gPi, c.invmult, c.BN.lv[Lf].b, out, s);
}

// out = scale * (Phibar S_PiPi^-1 Phibar^T in + P N_c P^T in)  (R29: K^~^-1 with scale = 1/s)
void bp_khat(ieti_ctx &c, const double *in, double *out, double scale, cudaStream_t s) {
  op_full_pre(c, nullptr, s, in);
  const double *x = local_neumann(c, s);
  op_full_post(c, x, nullptr, true, s, out);
  if (scale != 1.0) ik_scale_copy(bp_n(c), scale, out, out, s);
}

// lout = B~ u (owned rows complete after the reverse halo)
void bp_B(ieti_ctx &c, const double *box, double *lout, cudaStream_t s) {
  ik_jump_box(c.T.n_lambda, c.d_gp, c.d_gm, c.d_gabs, box, lout, s);
  halo_rev(c, lout, s);
}

// box += B~^T lam
void bp_Bt_add(ieti_ctx &c, double *lam, double *box, cudaStream_t s) {
  halo_fwd(c, lam, s);
  ik_bt_add(c.ngamma, c.d_gabs, c.d_bt_ptr, c.d_bt_m, c.d_bt_w, lam, box, s);
}

// ------------------------------------------------------------------------------------------
// PCG
// ------------------------------------------------------------------------------------------
size_t kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  CK(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) CK(cudaGraphGetNodes(g, nodes.data(), &n));
  size_t k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    CK(cudaGraphNodeGetType(nd, &t));
    if (t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

template <typename F>
cudaGraphExec_t capture(ieti_ctx &c, int gid, F body, size_t *kn) {
  cudaGraph_t g;
  c.rec_graph = gid;
  CK(cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal));
  body();
  CK(cudaStreamEndCapture(c.st, &g));
  c.rec_graph = -1;
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, g, 0));
  *kn = kernel_nodes(g);
  cudaGraphDestroy(g);
  return ex;
}

void end_segment(ieti_ctx &c) {
  cudaGraph_t g;
  CK(cudaStreamEndCapture(c.st, &g));
  size_t nn = 0;
  CK(cudaGraphGetNodes(g, nullptr, &nn));
  if (nn > 0) {
    ieti_ctx::Seg sg;
    CK(cudaGraphInstantiate(&sg.g, g, 0));
    sg.kn = (int)kernel_nodes(g);
    c.rec_segs->push_back(sg);
  }
  cudaGraphDestroy(g);
}

// captures body() as program gid (segments split at the host-driven loops); returns its kernels
template <typename F>
size_t capture_prog(ieti_ctx &c, int gid, F body) {
  c.rec_graph = gid;
  c.rec_segs = &c.prog[gid];
  CK(cudaStreamBeginCapture(c.st, cudaStreamCaptureModeThreadLocal));
  body();
  end_segment(c);
  c.rec_segs = nullptr;
  c.rec_graph = -1;
  size_t k = 0;
  for (auto &sg : c.prog[gid]) k += sg.kn;
  return k;
}

// program gid: stored as a host function (run eagerly in loopback test groups, whose collectives
// are host-mediated and cannot sit inside a graph) and, otherwise, captured as graph segments
size_t define_prog(ieti_ctx &c, int gid, std::function<void()> fn) {
  c.prog_fn[gid] = std::move(fn);
  if (c.comm.loop) return 0;
  return capture_prog(c, gid, c.prog_fn[gid]);
}

void capture_graphs(ieti_ctx &c) {
  const long long n = c.n_own;            // PCG vector work and dots over the OWNED multipliers
  cudaStream_t s = c.st;
  size_t k0 = 0, k1 = 0, k2 = 0, k3 = 0;
  // g0: lambda = 0, r = d^ = B Ktilde^{-1} f, ||r0||, z = M r, rho = r.z, p = z
  auto g0_head = [&c, s]() {
    CK(cudaMemsetAsync(c.lam, 0, std::max(1, c.T.n_lambda) * sizeof(double), s));
    op_full_pre(c, nullptr, s);
  };
  auto g0_tail = [&c, s, n](const double *xN) {
    op_full_post(c, xN, c.r, false, s);
    CK(cudaMemsetAsync(c.sc, 0, 16 * sizeof(double), s));
    ik_dot_partial(n, c.r, c.r, c.partial, c.nb_dot, s);
    auto a1 = allsum(c, c.partial, c.nb_dot, s);
    ik_store_scalar(a1.first, a1.second, c.sc, 7, 1, s);
    op_MsD(c, c.r, c.z, s);
    ik_dot_partial(n, c.r, c.z, c.partial, c.nb_dot, s);
    auto a2 = allsum(c, c.partial, c.nb_dot, s);
    ik_store_scalar(a2.first, a2.second, c.sc, 0, 0, s);
    ik_copy(n, c.z, c.pv, s);
    CK(cudaMemcpyAsync(c.sc_host, c.sc, 16 * sizeof(double), cudaMemcpyDeviceToHost, s));
  };
  // g1: q = F^ p, alpha, lambda/r update, ||r||
  auto g1_tail = [&c, s, n](const double *xN) {
    op_F_post(c, xN, c.q, s);
    ik_dot_partial(n, c.pv, c.q, c.partial, c.nb_dot, s);
    auto a1 = allsum(c, c.partial, c.nb_dot, s);
    ik_pcg_alpha(a1.first, a1.second, c.sc, s);
    ik_pcg_update(n, c.sc, c.pv, c.q, c.lam, c.r, c.partial, c.nb_dot, s);
    auto a2 = allsum(c, c.partial, c.nb_dot, s);
    ik_store_scalar(a2.first, a2.second, c.sc, 4, 1, s);
    CK(cudaMemcpyAsync(c.sc_host, c.sc, 16 * sizeof(double), cudaMemcpyDeviceToHost, s));
  };
  if (c.pcg_mode) batched_pcg_capture(c, c.ipcg, 4, 5);
  if (c.dpcg_mode) batched_pcg_capture(c, c.dpcg, 8, 9);
  k0 = define_prog(c, 0, [&c, s, g0_head, g0_tail]() {
    g0_head();
    g0_tail(local_neumann(c, s));
  });
  k1 = define_prog(c, 1, [&c, s, g1_tail]() {
    op_F_pre(c, c.pv, s);
    g1_tail(local_neumann(c, s));
  });
  // g2: z = M_sD r, beta, p update
  k2 = define_prog(c, 2, [&c, s, n]() {
    op_MsD(c, c.r, c.z, s);
    ik_dot_partial(n, c.r, c.z, c.partial, c.nb_dot, s);
    auto a1 = allsum(c, c.partial, c.nb_dot, s);
    ik_pcg_beta(a1.first, a1.second, c.sc, s);
    ik_pcg_p(n, c.sc, c.z, c.pv, c.nb_dot, s);
  });
  // g3: recovery u = Ktilde^{-1}(f - B^T lambda)
  k3 = define_prog(c, 3, [&c, s]() { op_full(c, c.lam, nullptr, true, s); });
  c.kn[0] = (int)k0; c.kn[1] = (int)k1; c.kn[2] = (int)k2; c.kn[3] = (int)k3;
  c.launches_per_iter = (int)(k1 + k2);
}

void read_timing(ieti_ctx &c, int gid) {
  if (!c.timing_on) return;
  for (const auto &tp : c.tpairs[gid]) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c.tev[tp.e0], c.tev[tp.e1]) == cudaSuccess) {
      c.t_acc[tp.cls] += ms;
      c.n_acc[tp.cls] += tp.launches;
      c.b_acc[tp.cls] += tp.bytes;
      c.b3_acc[tp.cls] += tp.bytes3;
    }
  }
}

// run program gid (0: d^ and start, 1: F^ half-iteration, 2: M_sD half-iteration, 3: recovery):
// its captured segments and, between them, the host-driven inner loops; returns the launches
long long launch_graph(ieti_ctx &c, int gid, cudaStream_t s) {
  long long n = 0;
  if (c.comm.loop) {                      // loopback test group: the body runs eagerly on c.st
    c.prog_fn[gid]();
    return 0;
  }
  for (auto &sg : c.prog[gid]) {
    if (sg.g) {
      CK(cudaGraphLaunch(sg.g, s));
      n += sg.kn;
    } else {
      const long long before = c.inner_launches;
      run_loop(c, sg.loop, s);
      n += c.inner_launches - before;
    }
  }
  return n;
}

// full solve; c.fbox holds the masked rhs box
// solve-phase timing: ph_mark(c, i, s) records event i (0: start, 1: after d^ and the PCG start,
// 2: after the loop, 3: after the recovery); the previous solve's phases are accumulated first
void ph_flush(ieti_ctx &c) {
  if (!c.ph_pending) return;
  CK(cudaEventSynchronize(c.ph_ev[3]));
  float ms;
  for (int i = 0; i < 3; ++i)
    if (cudaEventElapsedTime(&ms, c.ph_ev[i], c.ph_ev[i + 1]) == cudaSuccess) c.ph_acc[i] += ms;
  c.ph_acc[3] += 1;
  c.ph_pending = false;
}
void ph_mark(ieti_ctx &c, int i, cudaStream_t s) {
  if (!c.timing_on) return;
  if (i == 0) ph_flush(c);
  if (!c.ph_ev[i]) CK(cudaEventCreate(&c.ph_ev[i]));
  CK(cudaEventRecord(c.ph_ev[i], s));
  if (i == 3) c.ph_pending = true;
}

int pcg_solve(ieti_ctx &c, int fixed_iters, int *iters, double *rel_res, cudaStream_t s) {
  int status = IETI_OK;
  long long launches = 0;
  c.inner_log.clear();
  c.inner_unconverged = c.inner_breakdown = false;
  NvtxRange nv_solve("ieti solve");
  ph_mark(c, 0, s);
  {
    NvtxRange nv("d^ and PCG start");
    launches += launch_graph(c, 0, s);
  }
  ph_mark(c, 1, s);
  CK(cudaStreamSynchronize(s));
  const double r0 = c.sc_host[7];
  int k = 0;
  double rel = 0.0;
  const double tol = (fixed_iters >= 0) ? -1.0 : c.a.pcg_tol;
  const int maxit = (fixed_iters >= 0) ? fixed_iters : c.a.pcg_maxit;
  bool g2_pending = false;
  if (!std::isfinite(r0)) status = IETI_E_BREAKDOWN;    // non-finite data: reported, not a crash
  // gate on the GLOBAL multiplier count: a rank without local multipliers still takes part in the
  // collectives of every iteration
  if (status == IETI_OK && r0 > 0.0 && c.n_lambda_global > 0) {
    rel = 1.0;
    for (k = 1; k <= maxit; ++k) {
      NvtxRange nv("PCG iteration");
      launches += launch_graph(c, 1, s);
      CK(cudaStreamSynchronize(s));
      read_timing(c, 1);
      if (g2_pending) { read_timing(c, 2); g2_pending = false; }
      if (c.sc_host[6] != 0.0) { status = IETI_E_BREAKDOWN; --k; break; }
      double rn = c.sc_host[4];
      rel = rn / r0;
      if (!std::isfinite(rn)) { status = IETI_E_BREAKDOWN; break; }
      if (rn <= tol * r0 || k == maxit) break;
      launches += launch_graph(c, 2, s);
      g2_pending = true;
    }
    if (k > maxit) k = maxit;
    if (status == IETI_OK && fixed_iters < 0 && rel > tol) status = IETI_NOT_CONVERGED;
  }
  *iters = k;
  *rel_res = rel;
  ph_mark(c, 2, s);
  {
    NvtxRange nv("recovery");
    launches += launch_graph(c, 3, s);
  }
  ph_mark(c, 3, s);
  if (g2_pending) { CK(cudaStreamSynchronize(s)); read_timing(c, 2); }
  c.last_launches = launches + 3;   // + lattice in/mask/out kernels
  if (c.pcg_mode || c.dpcg_mode) {
    CK(cudaStreamSynchronize(s));     // the recovery's inner loops ran host-driven: flags are final
    if (status == IETI_OK && c.inner_breakdown) {
      status = IETI_E_BREAKDOWN;
      c.err = "an inner local PCG broke down (p.Ap <= 0 or non-finite)";
    } else if (status == IETI_OK && c.inner_unconverged) {
      status = IETI_NOT_CONVERGED;
      c.err = "an inner local PCG stopped at its iteration cap (inner_maxit / dirichlet_maxit)";
    }
  }
  return status;
}

// ---- MG-MG-S: calibration (R30), programs and solve (R31) ----------------------------------

// smallest eigenvalue of the symmetric tridiagonal (d, e) by Sturm-sequence bisection
double tridiag_min_eig(const std::vector<double> &d, const std::vector<double> &e, double *maxeig) {
  const int m = (int)d.size();
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {       // Gershgorin bounds
    const double r = (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i < m - 1 ? std::fabs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  auto count_below = [&](double x) {  // eigenvalues < x
    int cnt = 0;
    double q = d[0] - x;
    if (q < 0) ++cnt;
    for (int i = 1; i < m; ++i) {
      const double qq = (q == 0.0) ? 1e-300 : q;
      q = d[i] - x - e[i - 1] * e[i - 1] / qq;
      if (q < 0) ++cnt;
    }
    return cnt;
  };
  auto bisect = [&](int k) {          // k-th smallest (0-based)
    double a = lo, b = hi;
    for (int it = 0; it < 200 && b - a > 1e-16 * std::max(std::fabs(a), std::fabs(b)); ++it) {
      const double mid = 0.5 * (a + b);
      if (count_below(mid) > k) b = mid; else a = mid;
    }
    return 0.5 * (a + b);
  };
  if (maxeig) *maxeig = bisect(m - 1);
  return bisect(0);
}

void set_slot(ieti_ctx &c, int slot, double v) {
  CK(cudaMemcpyAsync(c.bsc + slot, &v, sizeof(double), cudaMemcpyHostToDevice, c.st));
  CK(cudaStreamSynchronize(c.st));
}
double get_slot(ieti_ctx &c, int slot) {
  double v = 0.0;
  CK(cudaMemcpyAsync(&v, c.bsc + slot, sizeof(double), cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  return v;
}

// R30: theta_min of K^~_1^-1 K~ from the Lanczos matrix of `lanczos_steps` PCG steps on K~ x = b0,
// b0_i = ((i+1) * 2654435761 mod 2^32) / 2^32 - 1/2 over the globally concatenated active dofs
// (oracle/saddle.py start_vector); s = (1 - margin) theta_min.  Eager, at setup.
void bp_calibrate(ieti_ctx &c) {
  cudaStream_t s = c.st;
  const long long n = bp_n(c);
  // b0 on the local patches' full lattices, active dofs numbered globally
  std::vector<double> lat(c.ndofs, 0.0);
  for (int k = 0; k < c.npatch; ++k) {
    const GridDesc &g = c.HN.lev[c.L - 1].g[k];
    long long cnt = c.act_off_g[c.glob_patch[k]];
    const long long nf = c.lat_off[k + 1] - c.lat_off[k];
    for (long long f = 0; f < nf; ++f) {
      const int i0 = (int)(f % g.M[0]), i1 = (int)((f / g.M[0]) % g.M[1]);
      const int i2 = (c.dim == 3) ? (int)(f / ((long long)g.M[0] * g.M[1])) : 0;
      const bool act = i0 >= g.lo[0] && i0 < g.hi[0] && i1 >= g.lo[1] && i1 < g.hi[1] &&
                       (c.dim == 2 || (i2 >= g.lo[2] && i2 < g.hi[2]));
      if (!act) continue;
      const unsigned long long v = ((unsigned long long)(cnt + 1) * 2654435761ull) % 4294967296ull;
      lat[c.lat_off[k] + f] = (double)v / 4294967296.0 - 0.5;
      ++cnt;
    }
  }
  CK(cudaMemcpyAsync(c.lat_tmp, lat.data(), c.ndofs * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  lattice_in(c, c.lat_tmp, c.b_rho, false, true, s);          // r = b0 (x0 = 0)
  bp_khat(c, c.b_rho, c.b_r, 1.0, s);                           // z = K^_1^-1 r
  ik_copy(n, c.b_r, c.b_p, s);
  bp_dot_box(c, c.b_rho, c.b_r, 8, s);
  double rho = get_slot(c, 8);
  const double rho0 = rho;
  std::vector<double> alphas, betas;
  const int steps = c.a.lanczos_steps > 0 ? c.a.lanczos_steps : 40;
  for (int it = 0; it < steps; ++it) {
    bp_kt(c, c.b_p, c.b_Kp, s);                                  // q = K p
    bp_dot_box(c, c.b_p, c.b_Kp, 9, s);
    const double a = rho / get_slot(c, 9);
    set_slot(c, 2, a);
    ik_axpy_s(n, c.bsc, 2, -1.0, c.b_Kp, c.b_rho, s);           // r -= a q
    bp_khat(c, c.b_rho, c.b_r, 1.0, s);                         // z
    bp_dot_box(c, c.b_rho, c.b_r, 8, s);
    const double rho_new = get_slot(c, 8);
    alphas.push_back(a);
    if (!(rho_new > 1e-24 * rho0)) break;                       // Krylov space exhausted
    const double bta = rho_new / rho;
    betas.push_back(bta);
    rho = rho_new;
    set_slot(c, 3, bta);
    ik_xpby_s(n, c.bsc, 3, c.b_r, c.b_p, s);                    // p = z + b p
  }
  const int m = (int)alphas.size();
  std::vector<double> d(m), e(std::max(0, m - 1));
  d[0] = 1.0 / alphas[0];
  for (int j = 1; j < m; ++j) d[j] = 1.0 / alphas[j] + betas[j - 1] / alphas[j - 1];
  for (int j = 0; j < m - 1; ++j) e[j] = std::sqrt(betas[j]) / alphas[j];
  c.bp_theta_min = tridiag_min_eig(d, e, &c.bp_theta_max);
  c.bp_steps = m;
  const double margin = c.a.khat_margin > 0 ? c.a.khat_margin : 0.05;
  // rounded DOWN to 3 significant digits, m / 10^k with m integer and 10^k exact (oracle/saddle.py
  // floor_sig3): the rounding-level spread of the Lanczos estimate does not reach s
  {
    const double xs = (1.0 - margin) * c.bp_theta_min;
    const int k = 2 - (int)std::floor(std::log10(xs));
    auto p10 = [](int e) { double v = 1.0; for (int i = 0; i < e; ++i) v *= 10.0; return v; };
    c.bp_s = (k >= 0) ? std::floor(xs * p10(k)) / p10(k) : std::floor(xs / p10(-k)) * p10(-k);
  }
  if (!(c.bp_s > 0.0) || !std::isfinite(c.bp_s)) throw IetiError(IETI_E_NOT_SPD, "BPCG calibration failed");
}

// programs 10 (start), 11 (first half-iteration), 12 (second half); scalars in c.bsc (device)
void capture_bpcg(ieti_ctx &c) {
  cudaStream_t s = c.st;
  const long long n = bp_n(c), nl = c.n_own;
  const double is = 1.0 / c.bp_s;
  const size_t lbytes = std::max(1, c.T.n_lambda) * sizeof(double);
  // 4: u = 0, lambda = 0, rho = (can(f), 0); r_u = K^-1 rho_u; Kr; s_l; r_l = M_sD s_l; gamma; p = r
  c.kn[10] = (int)define_prog(c, 10, [&c, s, n, nl, is, lbytes]() {
    CK(cudaMemsetAsync(c.bsc, 0, 32 * sizeof(double), s));
    CK(cudaMemsetAsync(c.b_u, 0, n * sizeof(double), s));
    CK(cudaMemsetAsync(c.lam, 0, lbytes, s));
    CK(cudaMemsetAsync(c.l_rho, 0, lbytes, s));
    bp_can(c, c.fbox, c.b_rho, s);
    bp_dot_box(c, c.b_rho, c.b_rho, 11, s);
    ik_bp_scalar(3, c.bsc, s);
    bp_khat(c, c.b_rho, c.b_r, is, s);
    bp_kt(c, c.b_r, c.b_Kr, s);
    bp_B(c, c.b_r, c.l_s, s);
    ik_sub(nl, c.l_s, c.l_rho, c.l_s, s);
    op_MsD(c, c.l_s, c.l_r, s);
    bp_dot_box(c, c.b_r, c.b_Kr, 8, s);
    bp_dot_box(c, c.b_r, c.b_rho, 9, s);
    bp_dot_lam(c, c.l_r, c.l_s, 10, s);
    ik_bp_scalar(2, c.bsc, s);
    ik_copy(n, c.b_r, c.b_p, s);
    ik_copy(n, c.b_Kr, c.b_Kp, s);
    ik_copy(nl, c.l_r, c.l_p, s);
    CK(cudaMemcpyAsync(c.bsc_host, c.bsc, 16 * sizeof(double), cudaMemcpyDeviceToHost, s));
  });
  // 5: a = (can(Kp + B^T p_l), B p_u); w = K^-1 a_u; delta, alpha; x += alpha p; rho -= alpha a; ||rho||
  c.kn[11] = (int)define_prog(c, 11, [&c, s, n, nl, is]() {
    ik_copy(n, c.b_Kp, c.b_a, s);
    bp_Bt_add(c, c.l_p, c.b_a, s);
    bp_can(c, c.b_a, c.b_a, s);
    bp_B(c, c.b_p, c.l_a, s);
    bp_khat(c, c.b_a, c.b_w, is, s);
    bp_dot_box(c, c.b_a, c.b_w, 8, s);
    bp_dot_box(c, c.b_p, c.b_a, 9, s);
    bp_dot_lam(c, c.l_p, c.l_a, 10, s);
    ik_bp_scalar(0, c.bsc, s);
    ik_axpy_s(n, c.bsc, 2, 1.0, c.b_p, c.b_u, s);
    ik_axpy_s(nl, c.bsc, 2, 1.0, c.l_p, c.lam, s);
    ik_axpy_s(n, c.bsc, 2, -1.0, c.b_a, c.b_rho, s);
    ik_axpy_s(nl, c.bsc, 2, -1.0, c.l_a, c.l_rho, s);
    bp_dot_box(c, c.b_rho, c.b_rho, 11, s);
    bp_dot_lam(c, c.l_rho, c.l_rho, 12, s);
    ik_bp_scalar(3, c.bsc, s);
    CK(cudaMemcpyAsync(c.bsc_host, c.bsc, 16 * sizeof(double), cudaMemcpyDeviceToHost, s));
  });
  // 6: r_u -= alpha w; Kr; s_l = B r_u - rho_l; r_l = M_sD s_l; gamma', beta; p = r + beta p; Kp
  c.kn[12] = (int)define_prog(c, 12, [&c, s, n, nl]() {
    ik_axpy_s(n, c.bsc, 2, -1.0, c.b_w, c.b_r, s);
    bp_kt(c, c.b_r, c.b_Kr, s);
    bp_B(c, c.b_r, c.l_s, s);
    ik_sub(nl, c.l_s, c.l_rho, c.l_s, s);
    op_MsD(c, c.l_s, c.l_r, s);
    bp_dot_box(c, c.b_r, c.b_Kr, 8, s);
    bp_dot_box(c, c.b_r, c.b_rho, 9, s);
    bp_dot_lam(c, c.l_r, c.l_s, 10, s);
    ik_bp_scalar(1, c.bsc, s);
    ik_xpby_s(n, c.bsc, 3, c.b_r, c.b_p, s);
    ik_xpby_s(nl, c.bsc, 3, c.l_r, c.l_p, s);
    ik_xpby_s(n, c.bsc, 3, c.b_Kr, c.b_Kp, s);
  });
  c.launches_per_iter = c.kn[11] + c.kn[12];
}

// BPCG solve (R31); the solution box is c.b_u, lambda in c.lam; c.fbox holds the masked rhs box
int bp_solve(ieti_ctx &c, int fixed_iters, int *iters, double *rel_res, cudaStream_t s) {
  int status = IETI_OK;
  long long launches = 0;
  c.inner_log.clear();
  NvtxRange nv_solve("ieti BPCG solve");
  ph_mark(c, 0, s);
  launches += launch_graph(c, 10, s);
  ph_mark(c, 1, s);
  CK(cudaStreamSynchronize(s));
  read_timing(c, 10);
  bool g12_pending = false;
  const double r0 = std::sqrt(c.bsc_host[4]);
  int k = 0;
  double rel = 0.0;
  const double tol = (fixed_iters >= 0) ? -1.0 : c.a.pcg_tol;
  const int maxit = (fixed_iters >= 0) ? fixed_iters : c.a.pcg_maxit;
  if (!std::isfinite(r0)) status = IETI_E_BREAKDOWN;
  if (status == IETI_OK && r0 > 0.0) {
    rel = 1.0;
    for (k = 1; k <= maxit; ++k) {
      NvtxRange nv("BPCG iteration");
      launches += launch_graph(c, 11, s);
      CK(cudaStreamSynchronize(s));
      read_timing(c, 11);
      if (g12_pending) { read_timing(c, 12); g12_pending = false; }
      if (c.bsc_host[6] != 0.0) { status = IETI_E_BREAKDOWN; --k; break; }
      const double rn = std::sqrt(c.bsc_host[4]);
      rel = rn / r0;
      if (!std::isfinite(rn)) { status = IETI_E_BREAKDOWN; break; }
      if (rn <= tol * r0 || k == maxit) break;
      launches += launch_graph(c, 12, s);
      g12_pending = true;
    }
    if (k > maxit) k = maxit;
    if (status == IETI_OK && fixed_iters < 0 && rel > tol) status = IETI_NOT_CONVERGED;
  }
  *iters = k;
  *rel_res = rel;
  ph_mark(c, 2, s);
  ph_mark(c, 3, s);
  if (g12_pending) { CK(cudaStreamSynchronize(s)); read_timing(c, 12); }
  c.last_launches = launches + 3;
  return status;
}

// the configured outer iteration; returns the status and the solution box
int outer_solve(ieti_ctx &c, int fixed_iters, int *iters, double *rel_res, cudaStream_t s, const double **ubox) {
  if (c.bp_mode) {
    *ubox = c.b_u;
    return bp_solve(c, fixed_iters, iters, rel_res, s);
  }
  *ubox = c.ubox;
  return pcg_solve(c, fixed_iters, iters, rel_res, s);
}

void stage_check(ieti_ctx &c, const char *stage) {
  cudaError_t e = cudaStreamSynchronize(c.st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) throw IetiError(IETI_E_CUDA, std::string("setup stage '") + stage + "': " + cudaGetErrorString(e));
  // per-stage setup wall time (stderr with IETI_VERBOSE=1)
  static thread_local std::chrono::steady_clock::time_point last;
  auto now = std::chrono::steady_clock::now();
  if (std::string(stage) == "begin") { last = now; return; }
  double ms = std::chrono::duration<double, std::milli>(now - last).count();
  last = now;
  c.stage_ms.push_back({stage, ms});
  nvtxMarkA(stage);
  const char *v = getenv("IETI_VERBOSE");
  if (v && v[0] == '1') fprintf(stderr, "[ieti setup] %-14s %9.1f ms\n", stage, ms);
}

// direct local solvers: assemble per patch the lower band of K (Neumann: active dofs, the mass term
// of floating patches removed, the last dof pinned on floating patches) or K_II (Dirichlet: interior
// dofs, Gamma columns dropped) in lexicographic order from the fine stencils, factor on the device
void setup_direct(ieti_ctx &c, bool neumann) {
  const int Lf = c.L - 1, d = c.dim, p = c.p, W1 = 2 * p + 1;
  Level &Lv = (neumann ? c.HN : c.HD).lev[Lf];
  BLevel &bl = (neumann ? c.BN : c.BD).lv[Lf];
  ieti_ctx::Direct &D = neumann ? c.dirN : c.dirD;
  D.nprob = c.npatch;
  std::vector<long long> pos, voff;
  long long len = 0;
  for (int k = 0; k < c.npatch; ++k) {
    const GridDesc &g = Lv.g[k];
    int nd[3] = {1, 1, 1};
    for (int dd = 0; dd < d; ++dd) nd[dd] = g.hi[dd] - g.lo[dd];
    const bool pin = neumann && c.T.floating[k];
    const int n = g.nrows - (pin ? 1 : 0);
    const int bw = p * (1 + nd[0] + (d == 3 ? nd[0] * nd[1] : 0));
    D.desc.push_back(BandDesc{n, bw, len});
    D.max_bw = std::max(D.max_bw, bw);
    voff.push_back((long long)pos.size());
    for (int a = 0; a < n; ++a) {
      int i[3] = {g.lo[0] + a % nd[0], g.lo[1] + (a / nd[0]) % nd[1], g.lo[2] + a / (nd[0] * nd[1])};
      pos.push_back(bl.pr[k].vec_off + sl_pos(g, p, d, i));
    }
    len += (long long)n * (bw + 1);
  }
  D.len = len;
  D.nv = (long long)pos.size();
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const double need = 2.0 * len * sizeof(double);
  if (need > 0.8 * (double)free_b)
    throw IetiError(IETI_E_NOMEM, "direct local solver: the banded factors need " + std::to_string(need / 1e9) +
                                      " GB, more than the device has free (the paper's OoM rows, P:323, P:337)");
  D.band = c.alloc<double>(len);
  D.up = c.alloc<double>(len);
  D.v = c.alloc<double>(D.nv);
  D.d_pos = c.upload(pos);
  D.d_voff = c.upload(voff);
  D.d_desc = c.upload(D.desc);
  // host assembly of each band from the stencil, one patch at a time
  for (int k = 0; k < c.npatch; ++k) {
    const GridDesc &g = Lv.g[k];
    const BandDesc &B = D.desc[k];
    int nd[3] = {1, 1, 1};
    for (int dd = 0; dd < d; ++dd) nd[dd] = g.hi[dd] - g.lo[dd];
    const int Spad = c.S;                            // every layout stores ld x S doubles
    std::vector<double> blk((size_t)g.ld * Spad);
    CK(cudaMemcpy(blk.data(), Lv.coef + g.coef_off, blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
    const bool massfix = neumann && c.T.floating[k];
    std::vector<std::vector<double>> M1(d);
    if (massfix)
      for (int dd = 0; dd < d; ++dd) M1[dd] = mass_1d(c.T.patch[k].knots[dd], p);
    std::vector<double> band((size_t)B.n * (B.bw + 1), 0.0);
    for (int a = 0; a < B.n; ++a) {
      int i[3] = {g.lo[0] + a % nd[0], g.lo[1] + (a / nd[0]) % nd[1], g.lo[2] + a / (nd[0] * nd[1])};
      int col = 0, pw = 1;
      for (int dd = 0; dd < d; ++dd) { col += (i[dd] % (p + 1)) * pw; pw *= (p + 1); }
      const ColourInfo &ci = Lv.ci[g.col_off + col];
      int j[3];
      for (int dd = 0; dd < 3; ++dd) j[dd] = (dd < d) ? (i[dd] - ci.first[dd]) / (p + 1) : 0;
      const int r = ci.start + j[0] + ci.n[0] * (j[1] + ci.n[1] * j[2]);
      for (int o = 0; o < c.S; ++o) {
        const int od[3] = {o % W1 - p, (o / W1) % W1 - p, (d == 3) ? o / (W1 * W1) - p : 0};
        int q[3], inside = 1;
        for (int dd = 0; dd < 3; ++dd) {
          q[dd] = i[dd] + od[dd];
          if (dd < d && (q[dd] < g.lo[dd] || q[dd] >= g.hi[dd])) inside = 0;
        }
        if (!inside) continue;
        const int b = (q[0] - g.lo[0]) + nd[0] * ((q[1] - g.lo[1]) + nd[1] * (d == 3 ? q[2] - g.lo[2] : 0));
        if (b > a || b >= B.n) continue;                     // lower triangle; the pinned dof is the last
        double v = blk[cidx(g, o, r) - g.coef_off];
        if (massfix) {
          double m = 1.0;
          for (int dd = 0; dd < d; ++dd) {
            const int Md = g.M[dd];
            m *= M1[dd][(size_t)i[dd] * Md + q[dd]];
          }
          v -= c.a.alpha_reg * m;                            // the stored stencil is K + alpha Mhat (R4)
        }
        band[(size_t)a * (B.bw + 1) + (b - a + B.bw)] = v;
      }
    }
    CK(cudaMemcpyAsync(D.band + B.off, band.data(), band.size() * sizeof(double), cudaMemcpyHostToDevice, c.st));
    CK(cudaStreamSynchronize(c.st));
  }
  long long max_len = 0;
  for (const auto &B : D.desc) max_len = std::max(max_len, (long long)B.n * (B.bw + 1));
  int *d_info = c.alloc<int>(c.npatch);
  ik_band_factor(c.npatch, D.d_desc, D.band, D.up, max_len, d_info, c.st);
  std::vector<int> info(c.npatch);
  CK(cudaMemcpyAsync(info.data(), d_info, c.npatch * sizeof(int), cudaMemcpyDeviceToHost, c.st));
  CK(cudaStreamSynchronize(c.st));
  for (int k = 0; k < c.npatch; ++k)
    if (info[k]) throw IetiError(IETI_E_NOT_SPD, "direct local solver: non-positive pivot in patch " + std::to_string(k));
}

// geometry_scope OWNED: rank r passed the patches k with owner[k] == r (ascending id).  Every rank
// packs them as doubles [p_d.., n_knots_d.., knots.., ctrl..] per patch, the blocks are all-gathered
// (padded to the longest) and decoded in rank / patch-id order into the global arrays.
void gather_geometry(ieti_ctx &c, const std::vector<int> &owner, std::vector<int> &deg, std::vector<int> &nk,
                     std::vector<double> &kn, std::vector<double> &ct) {
  const ieti_setup_args &a = c.a;
  const int d = a.dim, world = c.comm.world, N = a.n_patches;
  std::vector<double> mine;
  long long koff = 0, coff = 0;
  for (int k = 0, j = 0; k < N; ++k) {
    if (owner[k] != a.rank) continue;
    long long nknot = 0, nctrl = 1;
    for (int e = 0; e < d; ++e) mine.push_back(a.degree[j * d + e]);
    for (int e = 0; e < d; ++e) {
      mine.push_back(a.n_knots[j * d + e]);
      nknot += a.n_knots[j * d + e];
      nctrl *= a.n_knots[j * d + e] - a.degree[j * d + e] - 1;
    }
    mine.insert(mine.end(), a.knots + koff, a.knots + koff + nknot);
    mine.insert(mine.end(), a.ctrl + coff, a.ctrl + coff + nctrl * d);
    koff += nknot;
    coff += nctrl * d;
    ++j;
  }
  auto gather = [&](const std::vector<double> &h, size_t count) {
    double *ds = nullptr, *dr = nullptr;
    CK(cudaMalloc(&ds, std::max<size_t>(1, count) * sizeof(double)));
    CK(cudaMalloc(&dr, std::max<size_t>(1, count * world) * sizeof(double)));
    CK(cudaMemcpyAsync(ds, h.data(), count * sizeof(double), cudaMemcpyHostToDevice, c.st));
    c.comm.allgather(ds, dr, count, c.st);
    std::vector<double> out(count * world);
    CK(cudaMemcpyAsync(out.data(), dr, out.size() * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    cudaFree(ds);
    cudaFree(dr);
    return out;
  };
  const std::vector<double> lens = gather(std::vector<double>{(double)mine.size()}, 1);
  size_t L = 0;
  for (double v : lens) L = std::max(L, (size_t)v);
  mine.resize(L, 0.0);
  const std::vector<double> all = gather(mine, L);
  std::vector<std::vector<double>> per(N);
  std::vector<size_t> pos(world, 0);
  for (int k = 0; k < N; ++k) {                 // each rank's block holds its patches in ascending id
    const int r = owner[k];
    const double *b = all.data() + (size_t)r * L + pos[r];
    long long nknot = 0, nctrl = 1;
    for (int e = 0; e < d; ++e) {
      nknot += (long long)b[d + e];
      nctrl *= (long long)b[d + e] - (long long)b[e] - 1;
    }
    const size_t len = 2 * d + nknot + nctrl * d;
    if (pos[r] + len > (size_t)lens[r]) throw IetiError(IETI_E_ARG, "owned geometry blocks inconsistent with patch_owner");
    per[k].assign(b, b + len);
    pos[r] += len;
  }
  deg.clear(); nk.clear(); kn.clear(); ct.clear();
  for (int k = 0; k < N; ++k) {
    const std::vector<double> &b = per[k];
    long long nknot = 0;
    for (int e = 0; e < d; ++e) deg.push_back((int)b[e]);
    for (int e = 0; e < d; ++e) { nk.push_back((int)b[d + e]); nknot += (long long)b[d + e]; }
    kn.insert(kn.end(), b.begin() + 2 * d, b.begin() + 2 * d + nknot);
    ct.insert(ct.end(), b.begin() + 2 * d + nknot, b.end());
  }
}

void setup_all(ieti_ctx &c) {
  NvtxRange nv("ieti_setup");
  auto t0 = std::chrono::steady_clock::now();
  const ieti_setup_args &a = c.a;
  CK(cudaSetDevice(a.device));
  CK(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
  for (int k = 0; k < 3; ++k) {
    CK(cudaStreamCreateWithFlags(&c.st_aux[k], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c.ev_join[k], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
  {
    const char *xc = getenv("IETI_XGCONC");
    c.xgconc = (xc && xc[0] == '0') ? 0 : 1;
    const char *xb = getenv("IETI_XG_BIG");
    c.xg_big = xb ? std::max(1, std::min(4, atoi(xb))) : 1;
    const char *xs = getenv("IETI_XG_SMALL");
    c.xg_small = xs ? std::max(1, std::min(4, atoi(xs))) : 2;
  }
  stage_check(c, "begin");
  const int world = std::max(1, a.world);
  if (a.n_patches <= 0 || a.dim < 2 || a.dim > 3) throw IetiError(IETI_E_ARG, "bad dim or patch count");
  std::vector<int> owner = a.patch_owner ? std::vector<int>(a.patch_owner, a.patch_owner + a.n_patches)
                                         : default_owner(a.n_patches, world);
  {
    // conditions every rank evaluates identically, before the first collective: a
    // rank that would own nothing must not leave the others waiting in ncclCommInitRank
    std::vector<int> cnt(world, 0);
    for (int o : owner) {
      if (o < 0 || o >= world) throw IetiError(IETI_E_ARG, "patch_owner entry outside [0, world)");
      ++cnt[o];
    }
    for (int r = 0; r < world; ++r)
      if (cnt[r] == 0) throw IetiError(IETI_E_ARG, "every rank must own at least one patch");
  }
  {
    // IETI_NCCL_SELFTEST=1 on one rank: route the reductions through a 1-rank NCCL communicator
    // (loads NCCL, captures its collectives into the graphs) to exercise the multi-GPU path
    const char *st = getenv("IETI_NCCL_SELFTEST");
    if (world == 1 && st && st[0] == '1') {
      unsigned char uid[128];
      std::string e;
      if (comm_unique_id(uid, e) != 0) throw IetiError(IETI_E_NCCL, e);
      c.comm.init(uid, 0, 1, true);
    } else {
      c.comm.init(a.nccl_unique_id, a.rank, world);
    }
  }
  // geometry: every rank's own patches (geometry_scope OWNED) are all-gathered into the global
  // description the topology needs (interface matching)
  const int *g_degree = a.degree, *g_nknots = a.n_knots;
  const double *g_knots = a.knots, *g_ctrl = a.ctrl;
  std::vector<int> v_deg, v_nk;
  std::vector<double> v_kn, v_ct;
  if (a.geometry_scope == IETI_GEOMETRY_OWNED && world > 1) {
    gather_geometry(c, owner, v_deg, v_nk, v_kn, v_ct);
    g_degree = v_deg.data(); g_nknots = v_nk.data(); g_knots = v_kn.data(); g_ctrl = v_ct.data();
  }
  int rc = build_topology(a.dim, a.n_patches, g_degree, g_nknots, g_knots, g_ctrl, a.primal, c.T);
  if (rc != 0) throw IetiError(rc == -9 ? IETI_E_UNSUPPORTED : (rc == -3 ? IETI_E_TOPOLOGY : IETI_E_ARG), c.T.err);
  c.n_lambda_global = c.T.n_lambda;
  c.n_patches_global = c.T.n_patches;
  {
    // global facts the BPCG needs (R29-R31): patches per primal entity, and the position of each
    // patch's active dofs in the globally concatenated active numbering (calibration start vector)
    c.pi_mult.assign(std::max(1, c.T.n_pi), 0.0);
    for (int k = 0; k < c.T.n_patches; ++k)
      for (int g : c.T.R[k]) c.pi_mult[g] += 1.0;
    c.act_off_g.assign(c.T.n_patches + 1, 0);
    for (int k = 0; k < c.T.n_patches; ++k) {
      long long cnt = 1;
      for (int d = 0; d < a.dim; ++d) {
        const int M = g_nknots[k * a.dim + d] - g_degree[k * a.dim + d] - 1;
        cnt *= M - c.T.dir_side[k][2 * d] - c.T.dir_side[k][2 * d + 1];
      }
      c.act_off_g[k + 1] = c.act_off_g[k] + cnt;
    }
  }
  {
    // partition (every rank holds the global topology; keeps the local view, partition.cpp)
    Topo L;
    if (build_partition(c.T, owner, a.rank, world, L, c.plan) != 0) throw IetiError(IETI_E_ARG, L.err);
    c.T = std::move(L);
    c.n_own = c.plan.n_own;
    c.glob_patch = c.plan.local_patches;
  }
  c.dim = a.dim;
  c.p = c.T.p;
  c.P1 = c.p + 1;
  c.npatch = c.T.n_patches;             // local (owned) patches
  c.S = (int)ipow(2 * c.p + 1, c.dim);
  c.ncol = (int)ipow(c.p + 1, c.dim);
  {
    // fused small-level V-cycle (k_vcycle_fused): IETI_FUSE=1 forces it, =0 disables it; by
    // default only batches of >= 128 problems fuse (measured: C5 level 1 gains, batches of 4-64
    // patches lose to per-phase launches)
    const char *nf = getenv("IETI_FUSE");
    c.fuse_mode = (nf && nf[0] == '1') ? 1 : ((nf && nf[0] == '0') ? 0 : -1);
    const char *ps = getenv("IETI_PSWEEP");
    c.psweep = (ps && ps[0] == '1') ? 1 : 0;
    const char *cl = getenv("IETI_CLSWEEP");
    c.clsweep = (cl && cl[0] == '0') ? 0 : 1;
    const char *ccs = getenv("IETI_CLCS");
    c.clcs = ccs ? atoi(ccs) : 0;
    const char *cmx = getenv("IETI_CLMAX_MB");
    if (cmx) c.cl_max_mb = atof(cmx);
    const char *tl = getenv("IETI_TILE");
    const char *ost = getenv("IETI_STENCIL"), *osp = getenv("IETI_SPLIT");
    // the opt-in split / TMA big-level kernels address offset-major rows only
    c.tiled = ((tl && tl[0] == '0') || (ost && std::string(ost) == "tma") || (osp && atoi(osp) > 0)) ? 0 : 1;
    const char *crp = getenv("IETI_CLREP");
    c.clrep = (crp && crp[0] == '1') ? 1 : 0;
    const char *cgl = getenv("IETI_CLGLOBAL");
    c.clglobal = (cgl && cgl[0] == '1') ? 1 : 0;
    c.d_bar = c.alloc<unsigned>(1);
    const char *fm = getenv("IETI_FUSE_MB");
    if (fm && atof(fm) > 0) c.fuse_max_mb = atof(fm);
    const char *pf = getenv("IETI_PF");
    c.prefetch_on = !(pf && pf[0] == '0');
    const char *pm = getenv("IETI_PFMAX");
    if (pm && atof(pm) > 0) c.prefetch_max_mb = atof(pm);
    const char *xg = getenv("IETI_XGROUP_MB");
    if (xg) c.xgroup_mb = atof(xg);
    const char *lp = getenv("IETI_L2P");
    if (lp && lp[0] == '1') {
      int maxp = 0, maxw = 0;
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, a.device);
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, a.device);
      if (maxp > 0 && maxw > 0) {
        c.l2_persist_bytes = (size_t)maxp;
        c.l2_window_max = (size_t)maxw;
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c.l2_persist_bytes));
        c.l2_persist = true;
      }
    }
  }
  {
    // colour of a+o for a of colour col: per direction (col_d + o_d) mod (p+1) (R6)
    std::vector<short> olist((size_t)c.ncol * c.S);
    c.h_nlow.assign(c.ncol, 0);
    const int P1 = c.p + 1, W1 = 2 * c.p + 1;
    for (int col = 0; col < c.ncol; ++col) {
      std::vector<short> lo, hi;
      for (int o = 0; o < c.S; ++o) {
        int cc = col, oo = o, tc = 0, pw = 1;
        for (int d = 0; d < c.dim; ++d) {
          const int cd = cc % P1, od = oo % W1 - c.p;
          cc /= P1;
          oo /= W1;
          tc += (((cd + od) % P1 + P1) % P1) * pw;
          pw *= P1;
        }
        if (tc < col) lo.push_back((short)o);
        else if (tc > col) hi.push_back((short)o);
      }
      if ((int)(lo.size() + hi.size()) != c.S - 1) throw IetiError(IETI_E_ARG, "colour offset lists");
      c.h_nlow[col] = (short)lo.size();
      std::copy(lo.begin(), lo.end(), olist.begin() + (size_t)col * c.S);
      std::copy(hi.begin(), hi.end(), olist.begin() + (size_t)col * c.S + lo.size());
    }
    c.d_olist = c.upload(olist);
    c.h_olist = olist;
    c.d_nlow = c.upload(c.h_nlow);
  }
  for (int k = 0; k < c.npatch; ++k) c.n_floating += c.T.floating[k];
  stage_check(c, "topology");
  setup_knots_levels(c);
  // lattice / box offsets
  c.lat_off.assign(c.npatch + 1, 0);
  std::vector<int> Mall;
  for (int k = 0; k < c.npatch; ++k) {
    long long n = 1;
    for (int i = 0; i < 3; ++i) {
      int M = (i < c.dim) ? c.T.patch[k].M[i] : 1;
      Mall.push_back(M);
      n *= M;
    }
    c.lat_off[k + 1] = c.lat_off[k] + n;
    c.maxlat = std::max(c.maxlat, n);
  }
  c.ndofs = c.lat_off[c.npatch];
  c.HN.dirichlet = false;
  c.HD.dirichlet = true;
  c.HN.lev.assign(c.L, Level());
  c.HD.lev.assign(c.L, Level());
  for (int l = 0; l < c.L; ++l) {
    build_level_desc(c, c.HN, l);
    build_level_desc(c, c.HD, l);
    for (Hier *H : {&c.HN, &c.HD}) {
      Level &Lv = H->lev[l];
      Lv.d_g = c.upload(Lv.g);
      Lv.d_ci = c.upload(Lv.ci);
      upload_level(c, Lv);
    }
  }
  std::vector<int> ident(c.npatch);
  for (int k = 0; k < c.npatch; ++k) ident[k] = k;
  build_batch(c, c.BN, c.HN, ident);
  build_batch(c, c.BD, c.HD, ident);
  {
    // modes 6/7 on the finest level when a solve runs >= 2 V-cycles (IETI_USWEEP=0: off, A/B)
    const char *e = getenv("IETI_USWEEP");
    const bool on = !(e && e[0] == '0');
    BLevel &fn = c.BN.lv[c.L - 1], &fd = c.BD.lv[c.L - 1];
    if (on && c.a.cycles >= 2) fn.U = c.alloc<double>(fn.n);
    if (on && c.a.dirichlet_cycles >= 2) fd.U = c.alloc<double>(fd.n);
  }
  c.box_off.assign(c.npatch, 0);
  for (int k = 0; k < c.npatch; ++k) c.box_off[k] = c.BN.lv[c.L - 1].pr[k].vec_off;
  for (int k = 0; k < c.npatch; ++k)
    if (c.BD.lv[c.L - 1].pr[k].vec_off != c.box_off[k]) throw IetiError(IETI_E_ARG, "box layout mismatch");
  c.maxbox = c.BN.lv[c.L - 1].maxbox;
  c.d_M = c.upload(Mall);
  c.d_lat_off = c.upload(c.lat_off);
  c.d_box_off = c.upload(c.box_off);
  setup_transfers(c);
  stage_check(c, "transfers");
  setup_assembly_tables(c);
  setup_fine_stencils(c);
  stage_check(c, "fine stencils");
  setup_galerkin(c, c.HN);
  setup_galerkin(c, c.HD);
  stage_check(c, "galerkin");
  setup_coarsest(c, c.HN);
  setup_coarsest(c, c.HD);
  stage_check(c, "coarsest");
  setup_interface(c);
  stage_check(c, "interface");
  setup_rowlists(c);
  stage_check(c, "row lists");
  const long long nbox = c.BN.lv[c.L - 1].n;
  c.vbox = c.alloc<double>(nbox);
  c.ybox = c.alloc<double>(nbox);
  c.fbox = c.alloc<double>(nbox);
  c.ubox = c.alloc<double>(nbox);
  const long long nl = std::max(1, c.T.n_lambda);
  c.lam = c.alloc<double>(nl);
  c.r = c.alloc<double>(nl);
  c.z = c.alloc<double>(nl);
  c.pv = c.alloc<double>(nl);
  c.q = c.alloc<double>(nl);
  c.nb_dot = (int)std::max<long long>(1, std::min<long long>(296, (c.n_own + 255) / 256));
  if (c.comm.comm) {
    const Plan &P = c.plan;
    const int nx = std::max(1, std::max(P.send_ptr.back(), P.recv_ptr.back()));
    c.xs = c.alloc<double>(nx);
    c.xr = c.alloc<double>(nx);
    c.d_send_idx = c.upload(P.send_idx);
    c.d_recv_idx = c.upload(P.recv_idx);
    c.d_rsum_ptr = c.upload(P.rsum_ptr);
    c.d_rsum_src = c.upload(P.rsum_src);
    c.g_all = c.alloc<double>((long long)std::max(1, c.T.n_pi) * c.comm.world);
    c.red_send = c.alloc<double>(1);
    c.red_all = c.alloc<double>(c.comm.world);
  }
  c.partial = c.alloc<double>(c.nb_dot);
  c.sc = c.alloc<double>(16);
  CK(cudaMallocHost(&c.sc_host, 16 * sizeof(double)));
  memset(c.sc_host, 0, 16 * sizeof(double));
  c.lat_tmp = c.alloc<double>(c.ndofs);
  c.lat_tmp2 = c.alloc<double>(c.ndofs);
  if (c.pcg_mode) {
    batched_pcg_alloc(c, c.ipcg, c.BN);
    c.IX = c.ipcg.X;
    c.ipcg.tol = c.a.inner_tol;
    c.ipcg.maxit = c.a.inner_maxit;
    c.ipcg.applyA = [&c](const double *x, double *y, cudaStream_t s) {
      apply_level(c, c.BN, c.L - 1, x, y, 1.0, true, s);   // the true K (R4 mass removed)
    };
  }
  if (c.dpcg_mode) {
    batched_pcg_alloc(c, c.dpcg, c.BD);
    c.dpcg.tol = c.a.dirichlet_tol;
    c.dpcg.maxit = c.a.dirichlet_maxit;
    c.dpcg.applyA = [&c](const double *x, double *y, cudaStream_t s) {
      apply_level(c, c.BD, c.L - 1, x, y, 1.0, false, s);  // K_II (the Dirichlet stencils carry no mass term)
    };
  }
  setup_primal_basis(c);
  stage_check(c, "primal basis");
  CK(cudaStreamSynchronize(c.st));
  if (c.direct_N) setup_direct(c, true);
  if (c.direct_D) setup_direct(c, false);
  if (c.direct_N || c.direct_D) stage_check(c, "direct local solvers");
  {
    // MG-MG-S vectors (also used by the diagnostics OP_KT / OP_CAN / OP_KHAT in either mode)
    const long long nb = c.BN.lv[c.L - 1].n, nl = std::max(1, c.T.n_lambda);
    for (double **v : {&c.b_u, &c.b_rho, &c.b_r, &c.b_Kr, &c.b_p, &c.b_Kp, &c.b_a, &c.b_w}) *v = c.alloc<double>(nb);
    for (double **v : {&c.l_rho, &c.l_s, &c.l_r, &c.l_p, &c.l_a}) *v = c.alloc<double>(nl);
    c.nb_box = (int)std::max<long long>(1, std::min<long long>(592, (nb + 255) / 256));
    c.bpartial = c.alloc<double>(c.nb_box);
    c.bsc = c.alloc<double>(32);
    CK(cudaMallocHost(&c.bsc_host, 32 * sizeof(double)));
    memset(c.bsc_host, 0, 32 * sizeof(double));
    std::vector<double> inv(c.pi_mult.size());
    for (size_t i = 0; i < inv.size(); ++i) inv[i] = c.pi_mult[i] > 0 ? 1.0 / c.pi_mult[i] : 0.0;
    c.invmult = c.upload(inv);
  }
  if (c.bp_mode) {
    bp_calibrate(c);
    stage_check(c, "BPCG calibration");
  }
  // graphs (loopback test groups: the same programs, run eagerly -- define_prog)
  if (c.bp_mode) capture_bpcg(c);
  else capture_graphs(c);
  stage_check(c, "graphs");
  c.setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// ==========================================================================================
// C ABI
// ==========================================================================================

namespace {
// every entry point runs on the context's device and restores the caller's current device
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int run_guarded(ieti_ctx *c, const std::function<int()> &f) {
  DeviceGuard dg(c ? c->a.device : -1);
  try {
    return f();
  } catch (const IetiError &e) {
    if (c) c->err = e.what();
    else g_setup_err = e.what();
    return e.code;
  } catch (const CommError &e) {
    if (c) c->err = e.what();
    else g_setup_err = e.what();
    return IETI_E_NCCL;
  } catch (const std::exception &e) {
    if (c) c->err = e.what();
    else g_setup_err = e.what();
    return IETI_E_ARG;
  }
}
}  // namespace

extern "C" {

int ieti_setup(const ieti_setup_args *a, ieti_ctx **out) {
  if (!a || !out) { g_setup_err = "null argument"; return IETI_E_ARG; }
  *out = nullptr;
  if (a->world > 1 && (a->rank < 0 || a->rank >= a->world || !a->nccl_unique_id)) {
    g_setup_err = "world > 1 needs 0 <= rank < world and an NCCL unique id (ieti_nccl_unique_id)";
    return IETI_E_ARG;
  }
  ieti_ctx *c = new ieti_ctx();
  c->a = *a;
  if (c->a.cycles <= 0) c->a.cycles = 2;
  if (c->a.dirichlet_cycles <= 0) c->a.dirichlet_cycles = 2;
  if (c->a.pcg_maxit <= 0) c->a.pcg_maxit = 500;
  if (c->a.pcg_tol <= 0) c->a.pcg_tol = 1e-8;
  if (c->a.inner_maxit <= 0) c->a.inner_maxit = 200;
  if (c->a.alpha_reg < 0) c->a.alpha_reg = 1e-2;
  if (c->a.local_mode != IETI_LOCAL_VCYCLES && c->a.local_mode != IETI_LOCAL_PCG &&
      c->a.local_mode != IETI_LOCAL_DIRECT) {
    g_setup_err = "unknown local_mode";
    delete c;
    return IETI_E_ARG;
  }
  if (c->a.inner_tol <= 0) c->a.inner_tol = 1e-6;
  if (c->a.nu_pre <= 0) c->a.nu_pre = 1;
  if (c->a.nu_post <= 0) c->a.nu_post = 1;
  c->pcg_mode = (c->a.local_mode == IETI_LOCAL_PCG);
  c->direct_N = (c->a.local_mode == IETI_LOCAL_DIRECT);
  if (c->a.dirichlet_mode != IETI_DIRICHLET_VCYCLES && c->a.dirichlet_mode != IETI_DIRICHLET_PCG &&
      c->a.dirichlet_mode != IETI_DIRICHLET_DIRECT) {
    g_setup_err = "unknown dirichlet_mode";
    delete c;
    return IETI_E_ARG;
  }
  c->dpcg_mode = (c->a.dirichlet_mode == IETI_DIRICHLET_PCG);
  c->direct_D = (c->a.dirichlet_mode == IETI_DIRICHLET_DIRECT);
  if (c->a.outer_mode != IETI_OUTER_DUAL_PCG && c->a.outer_mode != IETI_OUTER_BPCG) {
    g_setup_err = "unknown outer_mode";
    delete c;
    return IETI_E_ARG;
  }
  c->bp_mode = (c->a.outer_mode == IETI_OUTER_BPCG);
  if (c->bp_mode && (c->pcg_mode || c->direct_N)) {
    g_setup_err = "outer_mode BPCG (MG-MG-S) uses fixed V-cycles in K^~ (local_mode IETI_LOCAL_VCYCLES)";
    delete c;
    return IETI_E_ARG;
  }
  if (c->a.dirichlet_tol <= 0) c->a.dirichlet_tol = 1e-12;
  if (c->a.dirichlet_maxit <= 0) c->a.dirichlet_maxit = 500;
  int rc;
  {
    DeviceGuard dg(c->a.device);
    rc = run_guarded(nullptr, [&]() { setup_all(*c); return IETI_OK; });
  }
  if (rc != IETI_OK) {
    if (g_setup_err.empty()) g_setup_err = c->err;
    delete c;
    return rc;
  }
  *out = c;
  return IETI_OK;
}

int ieti_assemble_load_builtin(ieti_ctx *c, int f_id, double *rhs) {
  if (!c || !rhs) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    const int d = c->dim, p = c->p;
    long long maxq = 0;
    for (int k = 0; k < c->npatch; ++k) { int nq[3]; long long nqt; nq_of(*c, k, nq, nqt); maxq = std::max(maxq, nqt); }
    size_t mark = c->allocs.size();
    double *G = c->alloc<double>(maxq * (d == 3 ? 6 : 3));
    double *X = c->alloc<double>(maxq * d);
    double *dw = c->alloc<double>(maxq);
    double *fw = c->alloc<double>(maxq);
    int *bad = c->alloc<int>(1);
    for (int k = 0; k < c->npatch; ++k) {
      int nq[3]; long long nqt;
      nq_of(*c, k, nq, nqt);
      int M[3] = {c->T.patch[k].M[0], c->T.patch[k].M[1], c->T.patch[k].M[2]};
      launch_geometry2(d, p, nq, M, c->d_val, c->d_der, c->d_toff + 3 * k, c->d_wq, c->d_woff + 3 * k,
                       c->d_ctrl + c->ctrl_off[k], G, X, dw, bad, c->st);
      launch_eval_f2(d, f_id, X, dw, nqt, fw, c->st);
      const GridDesc &g = c->HN.lev[c->L - 1].g[k];
      launch_load2(d, p, M, c->T.patch[k].melem, g.lo, g.hi, c->d_val, c->d_toff + 3 * k, fw,
                   c->lat_tmp + c->lat_off[k], c->st);
    }
    CK(cudaMemcpyAsync(rhs, c->lat_tmp, c->ndofs * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaGetLastError());
    for (size_t i = mark; i < c->allocs.size(); ++i) cudaFree(c->allocs[i]);
    c->allocs.resize(mark);
    return IETI_OK;
  });
}

// quadrature points of the owned patches (p+1 Gauss points per element and direction, q_1 fastest)
int ieti_quadrature_points(ieti_ctx *c, double *xq, long long *n_points) {
  if (!c) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    long long tot = 0, maxq = 0;
    for (int k = 0; k < c->npatch; ++k) {
      int nq[3];
      long long nqt;
      nq_of(*c, k, nq, nqt);
      tot += nqt;
      maxq = std::max(maxq, nqt);
    }
    if (n_points) *n_points = tot;
    if (!xq) return IETI_OK;
    const int d = c->dim, p = c->p;
    size_t mark = c->allocs.size();
    double *G = c->alloc<double>(maxq * (d == 3 ? 6 : 3));
    double *X = c->alloc<double>(maxq * d);
    double *dw = c->alloc<double>(maxq);
    int *bad = c->alloc<int>(1);
    long long off = 0;
    for (int k = 0; k < c->npatch; ++k) {
      int nq[3];
      long long nqt;
      nq_of(*c, k, nq, nqt);
      int M[3] = {c->T.patch[k].M[0], c->T.patch[k].M[1], c->T.patch[k].M[2]};
      launch_geometry2(d, p, nq, M, c->d_val, c->d_der, c->d_toff + 3 * k, c->d_wq, c->d_woff + 3 * k,
                       c->d_ctrl + c->ctrl_off[k], G, X, dw, bad, c->st);
      CK(cudaMemcpyAsync(xq + off * d, X, nqt * d * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      off += nqt;
    }
    for (size_t i = mark; i < c->allocs.size(); ++i) cudaFree(c->allocs[i]);
    c->allocs.resize(mark);
    return IETI_OK;
  });
}

// patch loads f_a = sum_q f(x_q) w_q |det J| N_a(x_q) from f at the points of ieti_quadrature_points
int ieti_assemble_load(ieti_ctx *c, const double *f_at_qp, double *rhs) {
  if (!c || !f_at_qp || !rhs) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    const int d = c->dim, p = c->p;
    long long maxq = 0;
    for (int k = 0; k < c->npatch; ++k) { int nq[3]; long long nqt; nq_of(*c, k, nq, nqt); maxq = std::max(maxq, nqt); }
    size_t mark = c->allocs.size();
    double *G = c->alloc<double>(maxq * (d == 3 ? 6 : 3));
    double *X = c->alloc<double>(maxq * d);
    double *dw = c->alloc<double>(maxq);
    double *fq = c->alloc<double>(maxq);
    double *fw = c->alloc<double>(maxq);
    int *bad = c->alloc<int>(1);
    long long off = 0;
    for (int k = 0; k < c->npatch; ++k) {
      int nq[3];
      long long nqt;
      nq_of(*c, k, nq, nqt);
      int M[3] = {c->T.patch[k].M[0], c->T.patch[k].M[1], c->T.patch[k].M[2]};
      launch_geometry2(d, p, nq, M, c->d_val, c->d_der, c->d_toff + 3 * k, c->d_wq, c->d_woff + 3 * k,
                       c->d_ctrl + c->ctrl_off[k], G, X, dw, bad, c->st);
      CK(cudaMemcpyAsync(fq, f_at_qp + off, nqt * sizeof(double), cudaMemcpyHostToDevice, c->st));
      launch_mul(nqt, fq, dw, fw, c->st);
      const GridDesc &g = c->HN.lev[c->L - 1].g[k];
      launch_load2(d, p, M, c->T.patch[k].melem, g.lo, g.hi, c->d_val, c->d_toff + 3 * k, fw,
                   c->lat_tmp + c->lat_off[k], c->st);
      off += nqt;
    }
    CK(cudaMemcpyAsync(rhs, c->lat_tmp, c->ndofs * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaGetLastError());
    for (size_t i = mark; i < c->allocs.size(); ++i) cudaFree(c->allocs[i]);
    c->allocs.resize(mark);
    return IETI_OK;
  });
}

int ieti_solve_device(ieti_ctx *c, const double *d_rhs, double *d_u, double *d_lambda, int *iters, double *rel_res,
                      void *cuda_stream) {
  if (!c || !d_rhs || !d_u) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    cudaStream_t ext = (cudaStream_t)cuda_stream;
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, ext));
    CK(cudaStreamWaitEvent(c->st, ev, 0));
    lattice_in(*c, d_rhs, c->fbox, false, true, c->st);
    int it = 0;
    double rr = 0;
    const double *ub = nullptr;
    int status = outer_solve(*c, -1, &it, &rr, c->st, &ub);
    lattice_out(*c, ub, d_u, c->st);
    if (d_lambda && c->n_own)
      CK(cudaMemcpyAsync(d_lambda, c->lam, c->n_own * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    CK(cudaEventRecord(ev, c->st));
    CK(cudaStreamWaitEvent(ext, ev, 0));
    CK(cudaEventDestroy(ev));
    CK(cudaGetLastError());
    if (iters) *iters = it;
    if (rel_res) *rel_res = rr;
    return status;
  });
}

static int solve_host(ieti_ctx *c, const double *rhs, int fixed, double *u, double *lambda, int *iters,
                      double *rel_res) {
  return run_guarded(c, [&]() {
    CK(cudaMemcpyAsync(c->lat_tmp, rhs, c->ndofs * sizeof(double), cudaMemcpyHostToDevice, c->st));
    lattice_in(*c, c->lat_tmp, c->fbox, false, true, c->st);
    int it = 0;
    double rr = 0;
    const double *ub = nullptr;
    int status = outer_solve(*c, fixed, &it, &rr, c->st, &ub);
    lattice_out(*c, ub, c->lat_tmp, c->st);
    CK(cudaMemcpyAsync(u, c->lat_tmp, c->ndofs * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    if (lambda && c->n_own)
      CK(cudaMemcpyAsync(lambda, c->lam, c->n_own * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaGetLastError());
    if (iters) *iters = it;
    if (rel_res) *rel_res = rr;
    return status;
  });
}

int ieti_solve(ieti_ctx *c, const double *rhs, double *u, double *lambda, int *iters, double *rel_res) {
  if (!c || !rhs || !u) return IETI_E_ARG;
  return solve_host(c, rhs, -1, u, lambda, iters, rel_res);
}

int ieti_solve_fixed(ieti_ctx *c, const double *rhs, int iters, double *u, double *lambda, double *rel_res) {
  if (!c || !rhs || !u || iters < 0) return IETI_E_ARG;
  int it = 0;
  return solve_host(c, rhs, iters, u, lambda, &it, rel_res);
}

int ieti_info(const ieti_ctx *c, long long info[16]) {
  if (!c || !info) return IETI_E_ARG;
  for (int i = 0; i < 16; ++i) info[i] = 0;
  info[0] = c->dim; info[1] = c->p; info[2] = c->npatch; info[3] = c->ndofs; info[4] = c->T.n_lambda;
  info[14] = c->n_own; info[15] = c->comm.world;
  info[5] = c->T.n_pi; info[6] = c->L; info[7] = c->n_floating; info[8] = c->stencil_bytes; info[9] = c->ncol;
  info[10] = (long long)c->setup_ms; info[11] = c->basis_its; info[12] = c->launches_per_iter;
  info[13] = (long long)c->bytes_alloc;
  return IETI_OK;
}

int ieti_multiplier_map(const ieti_ctx *c, int *kp, int *ap, int *km, int *am) {
  if (!c) return IETI_E_ARG;
  for (int i = 0; i < c->T.n_lambda; ++i) {
    if (kp) kp[i] = c->plan.gkp[i];
    if (ap) ap[i] = c->T.map_[i];
    if (km) km[i] = c->plan.gkm[i];
    if (am) am[i] = c->T.mam[i];
  }
  return IETI_OK;
}

int ieti_apply(ieti_ctx *c, int op, const double *in, double *out) {
  if (!c || !in || !out) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    cudaStream_t s = c->st;
    const long long nl = c->T.n_lambda;
    const int Lf = c->L - 1;
    switch (op) {
      case IETI_OP_F:
      case IETI_OP_MSD: {
        CK(cudaMemcpyAsync(c->pv, in, nl * sizeof(double), cudaMemcpyHostToDevice, s));
        if (op == IETI_OP_F) op_F(*c, c->pv, c->q, s); else op_MsD(*c, c->pv, c->q, s);
        CK(cudaMemcpyAsync(out, c->q, nl * sizeof(double), cudaMemcpyDeviceToHost, s));
        break;
      }
      case IETI_OP_D: {
        CK(cudaMemcpyAsync(c->lat_tmp, in, c->ndofs * sizeof(double), cudaMemcpyHostToDevice, s));
        lattice_in(*c, c->lat_tmp, c->fbox, false, true, s);
        op_full(*c, nullptr, c->q, false, s);
        CK(cudaMemcpyAsync(out, c->q, nl * sizeof(double), cudaMemcpyDeviceToHost, s));
        break;
      }
      case IETI_OP_KTINV: {
        CK(cudaMemcpyAsync(c->lat_tmp, in, c->ndofs * sizeof(double), cudaMemcpyHostToDevice, s));
        lattice_in(*c, c->lat_tmp, c->fbox, false, true, s);
        op_full(*c, nullptr, nullptr, true, s);
        lattice_out(*c, c->ubox, c->lat_tmp, s);
        CK(cudaMemcpyAsync(out, c->lat_tmp, c->ndofs * sizeof(double), cudaMemcpyDeviceToHost, s));
        break;
      }
      case IETI_OP_NEUMANN:
      case IETI_OP_VCYCLE_N: {
        CK(cudaMemcpyAsync(c->lat_tmp, in, c->ndofs * sizeof(double), cudaMemcpyHostToDevice, s));
        lattice_in(*c, c->lat_tmp, c->BN.lv[Lf].b, false, true, s);
        const double *xo = c->BN.lv[Lf].x;
        if (op == IETI_OP_NEUMANN) xo = local_neumann(*c, s);   // c V-cycles, or the inner PCG (C2)
        else ncycles(*c, c->BN, 1, s);
        lattice_out(*c, xo, c->lat_tmp, s);
        CK(cudaMemcpyAsync(out, c->lat_tmp, c->ndofs * sizeof(double), cudaMemcpyDeviceToHost, s));
        break;
      }
      case IETI_OP_DIRICHLET: {
        CK(cudaMemcpyAsync(c->lat_tmp, in, c->ndofs * sizeof(double), cudaMemcpyHostToDevice, s));
        lattice_in(*c, c->lat_tmp, c->BD.lv[Lf].b, true, false, s);
        lattice_out(*c, local_dirichlet(*c, s), c->lat_tmp, s);   // c_D V-cycles, or the inner PCG (R27)
        CK(cudaMemsetAsync(c->BD.lv[Lf].b, 0, c->BD.lv[Lf].n * sizeof(double), s));
        CK(cudaMemcpyAsync(out, c->lat_tmp, c->ndofs * sizeof(double), cudaMemcpyDeviceToHost, s));
        break;
      }
      case IETI_OP_KT:
      case IETI_OP_CAN:
      case IETI_OP_KHAT: {
        if (op == IETI_OP_KHAT && !c->bp_mode) throw IetiError(IETI_E_ARG, "OP_KHAT needs outer_mode BPCG");
        CK(cudaMemcpyAsync(c->lat_tmp, in, c->ndofs * sizeof(double), cudaMemcpyHostToDevice, s));
        lattice_in(*c, c->lat_tmp, c->b_a, false, true, s);
        if (op == IETI_OP_KT) bp_kt(*c, c->b_a, c->b_w, s);
        else if (op == IETI_OP_CAN) bp_can(*c, c->b_a, c->b_w, s);
        else bp_khat(*c, c->b_a, c->b_w, 1.0 / c->bp_s, s);
        lattice_out(*c, c->b_w, c->lat_tmp, s);
        CK(cudaMemcpyAsync(out, c->lat_tmp, c->ndofs * sizeof(double), cudaMemcpyDeviceToHost, s));
        break;
      }
      default:
        throw IetiError(IETI_E_ARG, "unknown op");
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    return IETI_OK;
  });
}

int ieti_get_stencil(ieti_ctx *c, int hier, int level, int patch, double *out, int *n_rows) {
  if (!c || hier < 0 || hier > 1 || level < 0 || level >= c->L || patch < 0 || patch >= c->npatch) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    Level &Lv = (hier == 0 ? c->HN : c->HD).lev[level];
    const GridDesc &g = Lv.g[patch];
    if (n_rows) *n_rows = g.nrows;
    if (!out) return IETI_OK;
    const int Spad = c->S;                           // every layout stores ld x S doubles
    std::vector<double> blk((size_t)g.ld * Spad);
    CK(cudaMemcpy(blk.data(), Lv.coef + g.coef_off, blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
    const int p = c->p;
    int n0 = g.hi[0] - g.lo[0], n1 = g.hi[1] - g.lo[1];
    for (int a = 0; a < g.nrows; ++a) {
      int i[3] = {g.lo[0] + a % n0, g.lo[1] + (a / n0) % n1, g.lo[2] + a / (n0 * n1)};
      int col = 0, pw = 1;
      for (int dd = 0; dd < c->dim; ++dd) { col += (i[dd] % (p + 1)) * pw; pw *= (p + 1); }
      const ColourInfo &ci = Lv.ci[g.col_off + col];
      int j[3];
      for (int dd = 0; dd < 3; ++dd) j[dd] = (dd < c->dim) ? (i[dd] - ci.first[dd]) / (p + 1) : 0;
      int r = ci.start + j[0] + ci.n[0] * (j[1] + ci.n[1] * j[2]);
      for (int o = 0; o < c->S; ++o) out[(size_t)a * c->S + o] = blk[cidx(g, o, r) - g.coef_off];
    }
    return IETI_OK;
  });
}

int ieti_get_primal_basis(ieti_ctx *c, int patch, double *out, int *n_pi_k) {
  if (!c || patch < 0 || patch >= c->npatch) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    const PatchIface &P = c->pif[patch];
    if (n_pi_k) *n_pi_k = P.npi;
    if (!out) return IETI_OK;
    std::vector<double> blk((size_t)P.npi * P.box);
    if (!blk.empty())
      CK(cudaMemcpy(blk.data(), c->phiF + P.phif_off, blk.size() * sizeof(double), cudaMemcpyDeviceToHost));
    const GridDesc &g = c->HN.lev[c->L - 1].g[patch];
    const int p = c->p;
    long long n = c->lat_off[patch + 1] - c->lat_off[patch];
    for (int j = 0; j < P.npi; ++j)
      for (long long t = 0; t < n; ++t) {
        int i[3] = {(int)(t % g.M[0]), (int)((t / g.M[0]) % g.M[1]), (int)(t / ((long long)g.M[0] * g.M[1]))};
        out[(size_t)j * n + t] = blk[(size_t)j * P.box + box_pos_host(g, p, c->dim, i)];
      }
    return IETI_OK;
  });
}

int ieti_timing(ieti_ctx *c, int enable, int reset, double t_ms[8], long long n[8], double bytes[8]) {
  if (!c) return IETI_E_ARG;
  if (reset) {
    for (int i = 0; i < 8; ++i) { c->t_acc[i] = 0; c->n_acc[i] = 0; c->b_acc[i] = 0; c->b3_acc[i] = 0; }
  }
  for (int i = 0; i < 8; ++i) {
    if (t_ms) t_ms[i] = c->t_acc[i];
    if (n) n[i] = c->n_acc[i];
    if (bytes) bytes[i] = c->b_acc[i];
  }
  if (n) n[7] = c->last_launches;
  if (t_ms) t_ms[7] = (double)c->launches_per_iter;
  if (t_ms) t_ms[6] = c->fused_fine ? 1.0 : 0.0;
  c->timing_on = enable != 0;
  return IETI_OK;
}

int ieti_local_multipliers(const ieti_ctx *c, int *global_ids, int *local_patches) {
  if (!c) return IETI_E_ARG;
  if (global_ids)
    for (size_t j = 0; j < c->plan.local_mult.size(); ++j) global_ids[j] = c->plan.local_mult[j];
  if (local_patches)
    for (size_t j = 0; j < c->plan.local_patches.size(); ++j) local_patches[j] = c->plan.local_patches[j];
  return IETI_OK;
}

static int host_plan(const ieti_setup_args *a, int rank, int world, Plan &P) {
  if (!a || world < 1 || rank < 0 || rank >= world) { g_setup_err = "bad rank/world"; return IETI_E_ARG; }
  Topo G, L;
  int rc = build_topology(a->dim, a->n_patches, a->degree, a->n_knots, a->knots, a->ctrl, a->primal, G);
  if (rc != 0) { g_setup_err = G.err; return rc == -3 ? IETI_E_TOPOLOGY : IETI_E_ARG; }
  std::vector<int> owner = a->patch_owner ? std::vector<int>(a->patch_owner, a->patch_owner + a->n_patches)
                                          : default_owner(a->n_patches, world);
  if (build_partition(G, owner, rank, world, L, P) != 0) { g_setup_err = L.err; return IETI_E_ARG; }
  return IETI_OK;
}

int ieti_plan_info(const ieti_setup_args *a, int rank, int world, long long out[6]) {
  Plan P;
  int rc = host_plan(a, rank, world, P);
  if (rc != IETI_OK) return rc;
  out[0] = (long long)P.local_patches.size(); out[1] = (long long)P.local_mult.size(); out[2] = P.n_own;
  out[3] = (long long)P.peers.size(); out[4] = P.send_ptr.back(); out[5] = P.recv_ptr.back();
  return IETI_OK;
}

int ieti_plan_get(const ieti_setup_args *a, int rank, int world, int *local_patches, int *local_mult, int *peers,
                  int *send_ptr, int *send_idx, int *recv_ptr, int *recv_idx) {
  Plan P;
  int rc = host_plan(a, rank, world, P);
  if (rc != IETI_OK) return rc;
  auto put = [](int *dst, const std::vector<int> &v) { if (dst) std::copy(v.begin(), v.end(), dst); };
  put(local_patches, P.local_patches); put(local_mult, P.local_mult); put(peers, P.peers);
  put(send_ptr, P.send_ptr); put(send_idx, P.send_idx); put(recv_ptr, P.recv_ptr); put(recv_idx, P.recv_idx);
  return IETI_OK;
}

int ieti_nccl_unique_id(void *out128) {
  if (!out128) return IETI_E_ARG;
  return comm_unique_id(out128, g_setup_err) == 0 ? IETI_OK : IETI_E_NCCL;
}

int ieti_inner_log(const ieti_ctx *c, int *counts, int max_calls, int *n_calls) {
  if (!c) return IETI_E_ARG;
  const int nc = c->npatch ? (int)(c->inner_log.size() / c->npatch) : 0;
  if (n_calls) *n_calls = nc;
  if (counts)
    for (int i = 0; i < std::min(nc, max_calls) * c->npatch; ++i) counts[i] = c->inner_log[i];
  return IETI_OK;
}

const char *ieti_last_error(const ieti_ctx *c) { return c ? c->err.c_str() : g_setup_err.c_str(); }

int ieti_phase_times(ieti_ctx *c, int reset, double out[16]) {
  if (!c || !out) return IETI_E_ARG;
  return run_guarded(c, [&]() {
    ph_flush(*c);
    for (int i = 0; i < 16; ++i) out[i] = 0.0;
    for (int i = 0; i < 4; ++i) out[i] = c->ph_acc[i];
    out[4] = c->t_acc[2]; out[5] = c->b_acc[2]; out[6] = c->b3_acc[2]; out[7] = (double)c->n_acc[2];
    out[8] = c->t_acc[3]; out[9] = c->b_acc[3]; out[10] = c->b3_acc[3]; out[11] = (double)c->n_acc[3];
    if (reset) {
      for (double &v : c->ph_acc) v = 0.0;
      for (int i = 2; i <= 3; ++i) { c->t_acc[i] = 0; c->b_acc[i] = 0; c->b3_acc[i] = 0; c->n_acc[i] = 0; }
    }
    return IETI_OK;
  });
}

int ieti_bpcg_info(const ieti_ctx *c, double out[4]) {
  if (!c || !out || !c->bp_mode) return IETI_E_ARG;
  out[0] = c->bp_s;
  out[1] = c->bp_theta_min;
  out[2] = c->bp_theta_max;
  out[3] = c->bp_steps;
  return IETI_OK;
}

void ieti_destroy(ieti_ctx *c) {
  if (!c) return;
  DeviceGuard dg(c->a.device);
  delete c;
}

}  // extern "C"
