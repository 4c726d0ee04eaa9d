// kernels_ieti.cu -- interface, coarse-space and Krylov-vector kernels of the dual PCG (fp64).
//
// F^ p   (App. A.1 of SURVEY; Eq. (4), Eq. (7)):
//   k_iface_t   r_G = B^T p (gather by Gamma dof), t = Phibar_G^T r_G, b_N = r - C^T t   (one block per patch)
//   k_gather_pi g_Pi = sum_k R_k^T t_k   (fixed order)
//   k_gemv      u_Pi = S_PiPi^{-1} g_Pi   (explicit inverse, replicated)
//   k_iface_w   w_G = x_G + Phibar_G (R u_Pi - C x)                             (one block per patch)
//   k_jump      (F^p)_i = w(k+,a+) - w(k-,a-)
// M_sD r: k_bdt (v = B_D^T r into the Gamma entries of a box), spmv, k_bd_gather.
// PCG: deterministic two-pass dot products (fixed block count, fixed tree).
#include "layout.cuh"

#include <algorithm>
#include <cmath>

namespace {

constexpr int NT = 256;

__device__ __forceinline__ double block_sum(double v, double *sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) sh[32] = s;
  }
  __syncthreads();
  return sh[32];
}

// mode 0: r_G = B^T lam (Gamma only);  mode 1: r = f - B^T lam on the whole box (d^, recovery)
// The patch's fine rhs box is zeroed by the caller (one memset of the pool: only Gamma entries are
// nonzero in F^); t = Phibar_G^T r_G with one warp per primal column (no block-wide reductions).
__global__ void k_iface_t(const PatchIface *__restrict__ pif, const int *__restrict__ gbox,
                          const int *__restrict__ bt_ptr, const int *__restrict__ bt_m, const double *__restrict__ bt_w,
                          const double *__restrict__ phiG, const int *__restrict__ crow, const double *__restrict__ cw,
                          const double *__restrict__ lam, double *t_all, double *bN, double *rG) {
  __shared__ double tl[64];
  const PatchIface P = pif[blockIdx.x];
  double *bb = bN + P.box_off;
  for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
    const int gi = P.g_off + g;
    double s = 0.0;
    for (int e = bt_ptr[gi]; e < bt_ptr[gi + 1]; ++e) s = fma(bt_w[e], lam[bt_m[e]], s);
    rG[gi] = s;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = threadIdx.x >> 5; j < P.npi; j += nw) {
    const double *ph = phiG + P.phi_off + (long long)j * P.ng;
    const double *r = rG + P.g_off;
    double s = 0.0;
    for (int g = lane; g < P.ng; g += 32) s = fma(ph[g], r[g], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      tl[j] = s;
      t_all[P.pi_off + j] = s;
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
    const int gi = P.g_off + g;
    const int j = crow[gi];
    double v = rG[gi];
    if (j >= 0) v -= cw[gi] * tl[j];
    bb[gbox[gi]] = v;
  }
}

// full version: r = f_box - B^T lam at Gamma; t = Phibar^T r (full); bN = r - C^T t
__global__ void k_full_t(const PatchIface *__restrict__ pif, const int *__restrict__ gbox,
                         const int *__restrict__ bt_ptr, const int *__restrict__ bt_m, const double *__restrict__ bt_w,
                         const double *__restrict__ phiF, const int *__restrict__ crow, const double *__restrict__ cw,
                         const double *__restrict__ lam, const double *__restrict__ fbox, double *t_all, double *bN) {
  __shared__ double sh[40];
  const PatchIface P = pif[blockIdx.x];
  double *bb = bN + P.box_off;
  const double *ff = fbox + P.box_off;
  for (int t = threadIdx.x; t < P.box; t += blockDim.x) bb[t] = ff[t];
  __syncthreads();
  if (lam != nullptr) {
    for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
      const int gi = P.g_off + g;
      double s = 0.0;
      for (int e = bt_ptr[gi]; e < bt_ptr[gi + 1]; ++e) s = fma(bt_w[e], lam[bt_m[e]], s);
      bb[gbox[gi]] -= s;
    }
  }
  __syncthreads();
  for (int j = 0; j < P.npi; ++j) {
    const double *ph = phiF + P.phif_off + (long long)j * P.box;
    double s = 0.0;
    for (int t = threadIdx.x; t < P.box; t += blockDim.x) s = fma(ph[t], bb[t], s);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) t_all[P.pi_off + j] = s;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
    const int gi = P.g_off + g;
    const int j = crow[gi];
    if (j >= 0) bb[gbox[gi]] -= cw[gi] * t_all[P.pi_off + j];
  }
}

__global__ void k_full_bt(int ngamma, const int *__restrict__ bt_ptr, const int *__restrict__ bt_m,
                          const double *__restrict__ bt_w, const double *__restrict__ lam, double *rG) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngamma) return;
  double s = 0.0;
  for (int e = bt_ptr[g]; e < bt_ptr[g + 1]; ++e) s = fma(bt_w[e], lam[bt_m[e]], s);
  rG[g] = s;
}

// t_(k,j) = sum_box Phibar_j f - sum_Gamma Phibar_j (B^T lam)   (block (k, j))
__global__ void k_full_dot(const PatchIface *__restrict__ pif, const int *__restrict__ gbox,
                           const double *__restrict__ phiF, const double *__restrict__ rG,
                           const double *__restrict__ fbox, double *t_all) {
  __shared__ double sh[40];
  const PatchIface P = pif[blockIdx.x];
  const int j = blockIdx.y;
  if (j >= P.npi) return;
  const double *ph = phiF + P.phif_off + (long long)j * P.box;
  const double *ff = fbox + P.box_off;
  double s = 0.0;
  for (int t = threadIdx.x; t < P.box; t += blockDim.x) s = fma(ph[t], ff[t], s);
  if (rG)
    for (int g = threadIdx.x; g < P.ng; g += blockDim.x) s = fma(-ph[gbox[P.g_off + g]], rG[P.g_off + g], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) t_all[P.pi_off + j] = s;
}

// bN = f - B^T lam - C^T t on the patch's box
__global__ void k_full_bn(const PatchIface *__restrict__ pif, const int *__restrict__ gbox,
                          const int *__restrict__ crow, const double *__restrict__ cw, const double *__restrict__ rG,
                          const double *__restrict__ fbox, const double *__restrict__ t_all, double *bN) {
  const PatchIface P = pif[blockIdx.x];
  double *bb = bN + P.box_off;
  const double *ff = fbox + P.box_off;
  for (int t = threadIdx.x; t < P.box; t += blockDim.x) bb[t] = ff[t];
  __syncthreads();
  for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
    const int gi = P.g_off + g;
    double v = bb[gbox[gi]];
    if (rG) v -= rG[gi];
    const int j = crow[gi];
    if (j >= 0) v -= cw[gi] * t_all[P.pi_off + j];
    bb[gbox[gi]] = v;
  }
}

__global__ void k_gather_pi(int n_pi, const int *__restrict__ ptr, const int *__restrict__ src,
                            const double *__restrict__ t_all, double *g) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pi) return;
  double s = 0.0;
  for (int e = ptr[i]; e < ptr[i + 1]; ++e) s += t_all[src[e]];
  g[i] = s;
}

// y = A x, A dense n x n row-major (warp per row)
__global__ void k_gemv(int n, const double *__restrict__ A, const double *__restrict__ x, double *y) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s = fma(A[(long long)row * n + c], x[c], s);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

// w_G = x_G + Phibar_G (R u_Pi - C x);  c_loc = R u_Pi - C x kept in cvec.  (C x)_j sums over the
// Gamma entries of constraint row j (CSR c_ptr / c_idx, one warp per row, no block-wide reductions)
__global__ void k_iface_w(const PatchIface *__restrict__ pif, const int *__restrict__ gbox,
                          const double *__restrict__ phiG, const int *__restrict__ c_ptr, const int *__restrict__ c_idx,
                          const double *__restrict__ cw, const int *__restrict__ Rg, const double *__restrict__ uPi,
                          const double *__restrict__ xN, double *cvec, double *wG) {
  __shared__ double cl[64];
  const PatchIface P = pif[blockIdx.x];
  const double *xx = xN + P.box_off;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = threadIdx.x >> 5; j < P.npi; j += nw) {
    double s = 0.0;
    for (int e = c_ptr[P.pi_off + j] + lane; e < c_ptr[P.pi_off + j + 1]; e += 32) {
      const int gi = P.g_off + c_idx[e];
      s = fma(cw[gi], xx[gbox[gi]], s);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const double c = uPi[Rg[P.pi_off + j]] - s;
      cl[j] = c;
      cvec[P.pi_off + j] = c;
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
    const int gi = P.g_off + g;
    double v = xx[gbox[gi]];
    for (int j = 0; j < P.npi; ++j) v = fma(phiG[P.phi_off + (long long)j * P.ng + g], cl[j], v);
    wG[gi] = v;
  }
}

// recovery: u_box = x + Phibar (R u_Pi - C x) over the whole box (cvec from k_iface_w)
__global__ void k_full_u(const PatchIface *__restrict__ pif, const double *__restrict__ phiF,
                         const double *__restrict__ cvec, const double *__restrict__ xN, double *ubox) {
  const PatchIface P = pif[blockIdx.y];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.box) return;
  double v = xN[P.box_off + t];
  for (int j = 0; j < P.npi; ++j) v = fma(phiF[P.phif_off + (long long)j * P.box + t], cvec[P.pi_off + j], v);
  ubox[P.box_off + t] = v;
}

__global__ void k_jump(int n, const int *__restrict__ gp, const int *__restrict__ gm, const double *__restrict__ wG,
                       double *q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // a side on a remote patch (multi-GPU) contributes 0 here and is added by the owner (k_rsum)
  const double wp = (gp[i] >= 0) ? wG[gp[i]] : 0.0;
  const double wm = (gm[i] >= 0) ? wG[gm[i]] : 0.0;
  q[i] = wp - wm;
}

// v(Gamma entries of a box) = B_D^T r
__global__ void k_bdt(int ngamma, const long long *__restrict__ gabs, const int *__restrict__ ptr,
                      const int *__restrict__ m, const double *__restrict__ w, const double *__restrict__ r,
                      double *vbox) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngamma) return;
  double s = 0.0;
  for (int e = ptr[g]; e < ptr[g + 1]; ++e) s = fma(w[e], r[m[e]], s);
  vbox[gabs[g]] = s;
}

// z_i = sum_e w_e y[gabs[idx_e]]  (B_D gather) ; with w = +-1 pairs this is also B
__global__ void k_bd_gather(int n, const int *__restrict__ ptr, const int *__restrict__ gi,
                            const double *__restrict__ w, const long long *__restrict__ gabs,
                            const double *__restrict__ y, double *z) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int e = ptr[i]; e < ptr[i + 1]; ++e) s = fma(w[e], y[gabs ? gabs[gi[e]] : (long long)gi[e]], s);
  z[i] = s;
}

// ------------------------------------------------------------------------------------------
// PCG scalars and vectors
// ------------------------------------------------------------------------------------------
__global__ void k_dot_partial(long long n, const double *__restrict__ a, const double *__restrict__ b,
                              double *partial) {
  __shared__ double sh[40];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__device__ double reduce_partials(const double *partial, int nb, double *sh) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
  return block_sum(s, sh);
}

// sc layout: 0 rho, 1 pq, 2 alpha, 3 beta, 4 rr, 5 rz, 6 breakdown, 7 r0, 8 iter flag
__global__ void k_pcg_alpha(const double *partial, int nb, double *sc) {
  __shared__ double sh[40];
  double pq = reduce_partials(partial, nb, sh);
  if (threadIdx.x == 0) {
    sc[1] = pq;
    if (!(pq > 0.0) || !isfinite(pq)) { sc[6] = 1.0; sc[2] = 0.0; }
    else sc[2] = sc[0] / pq;
  }
}

// lam += alpha p ; r -= alpha q ; partial (r.r)
__global__ void k_pcg_update(long long n, const double *sc, const double *__restrict__ p, const double *__restrict__ q,
                             double *lam, double *r, double *partial) {
  __shared__ double sh[40];
  const double alpha = sc[2];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    lam[i] = fma(alpha, p[i], lam[i]);
    double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_store_scalar(const double *partial, int nb, double *sc, int slot, int take_sqrt) {
  __shared__ double sh[40];
  double v = reduce_partials(partial, nb, sh);
  if (threadIdx.x == 0) sc[slot] = take_sqrt ? sqrt(v) : v;
}

__global__ void k_pcg_beta(const double *partial, int nb, double *sc) {
  __shared__ double sh[40];
  double rz = reduce_partials(partial, nb, sh);
  if (threadIdx.x == 0) {
    sc[5] = rz;
    sc[3] = rz / sc[0];
    sc[0] = rz;
  }
}

// p = z + beta p
__global__ void k_pcg_p(long long n, const double *sc, const double *__restrict__ z, double *p) {
  const double beta = sc[3];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

__global__ void k_copy(long long n, const double *a, double *b) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

__global__ void k_scale_copy(long long n, double s, const double *a, double *b) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = s * a[i];
}

// box <-> full-lattice copies of the finest level (blockIdx.y = patch; sub-lattice layout)
__global__ void k_lattice_to_box(int dim, int p, const GridDesc *__restrict__ g_, const ProbDesc *__restrict__ pr_,
                                 const long long *__restrict__ loff, const double *__restrict__ lat, double *box,
                                 int only_interior) {
  const int k = blockIdx.y;
  const ProbDesc pr = pr_[k];
  const GridDesc &g = g_[pr.grid];
  const long long n = (long long)g.M[0] * g.M[1] * g.M[2];
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int i[3] = {(int)(t % g.M[0]), (int)((t / g.M[0]) % g.M[1]), (int)(t / ((long long)g.M[0] * g.M[1]))};
  double v = lat[loff[k] + t];
  if (only_interior) {
    bool in = (i[0] > 0 && i[0] < g.M[0] - 1 && i[1] > 0 && i[1] < g.M[1] - 1);
    if (dim == 3) in = in && (i[2] > 0 && i[2] < g.M[2] - 1);
    if (!in) v = 0.0;
  }
  box[pr.vec_off + sl_pos(g, p, dim, i)] = v;
}

__global__ void k_box_to_lattice(int dim, int p, const GridDesc *__restrict__ g_, const ProbDesc *__restrict__ pr_,
                                 const long long *__restrict__ loff, const double *__restrict__ box, double *lat) {
  const int k = blockIdx.y;
  const ProbDesc pr = pr_[k];
  const GridDesc &g = g_[pr.grid];
  const long long n = (long long)g.M[0] * g.M[1] * g.M[2];
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int i[3] = {(int)(t % g.M[0]), (int)((t / g.M[0]) % g.M[1]), (int)(t / ((long long)g.M[0] * g.M[1]))};
  lat[loff[k] + t] = box[pr.vec_off + sl_pos(g, p, dim, i)];
}

// zero every box entry that is not an active lattice point of its grid (blockIdx.y = problem)
__global__ void k_mask_box(int dim, int p, const GridDesc *__restrict__ g_, const ProbDesc *__restrict__ pr_,
                           double *v) {
  const ProbDesc pr = pr_[blockIdx.y];
  const GridDesc &g = g_[pr.grid];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.box) return;
  const int P1 = p + 1;
  int c = t / g.sb, rem = t % g.sb;
  int q[3] = {rem % g.ns[0], (rem / g.ns[0]) % g.ns[1], (dim == 3) ? rem / (g.ns[0] * g.ns[1]) : 0};
  bool in = true;
  for (int d = 0; d < dim; ++d) {
    int cd = c % P1;
    c /= P1;
    int i = cd + P1 * q[d];
    in = in && (i >= g.lo[d]) && (i < g.hi[d]);
  }
  if (!in) v[pr.vec_off + t] = 0.0;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// launchers (thin; all shapes decided by the host code in solver.cu)
// ------------------------------------------------------------------------------------------

void ik_iface_t(int npatch, const void *pif, const int *gbox, const int *bt_ptr, const int *bt_m, const double *bt_w,
                const double *phiG, const int *crow, const double *cw, const double *lam, double *t_all, double *bN,
                double *rG, cudaStream_t s) {
  k_iface_t<<<npatch, NT, 0, s>>>((const PatchIface *)pif, gbox, bt_ptr, bt_m, bt_w, phiG, crow, cw, lam, t_all, bN, rG);
}
void ik_full_t(int npatch, const void *pif, const int *gbox, const int *bt_ptr, const int *bt_m, const double *bt_w,
               const double *phiF, const int *crow, const double *cw, const double *lam, const double *fbox,
               double *t_all, double *bN, cudaStream_t s, int ngamma, int max_npi, double *rG) {
  if (max_npi <= 0 || !rG) {
    k_full_t<<<npatch, NT, 0, s>>>((const PatchIface *)pif, gbox, bt_ptr, bt_m, bt_w, phiF, crow, cw, lam, fbox, t_all, bN);
    return;
  }
  // wide form: r_G = B^T lam; t_(k,j) = Phibar_j^T (f - B^T lam), one block per (patch, column)
  // (the full basis is the stream: C5 2.5 GB); then bN = f - B^T lam - C^T t per patch
  if (lam && ngamma > 0) k_full_bt<<<(ngamma + 255) / 256, 256, 0, s>>>(ngamma, bt_ptr, bt_m, bt_w, lam, rG);
  k_full_dot<<<dim3((unsigned)npatch, (unsigned)max_npi), NT, 0, s>>>((const PatchIface *)pif, gbox, phiF,
                                                                      lam ? rG : nullptr, fbox, t_all);
  k_full_bn<<<npatch, NT, 0, s>>>((const PatchIface *)pif, gbox, crow, cw, lam ? rG : nullptr, fbox, t_all, bN);
}
void ik_gather_pi(int n_pi, const int *ptr, const int *src, const double *t_all, double *g, cudaStream_t s) {
  if (n_pi > 0) k_gather_pi<<<(n_pi + 127) / 128, 128, 0, s>>>(n_pi, ptr, src, t_all, g);
}
void ik_gemv(int n, const double *A, const double *x, double *y, cudaStream_t s) {
  if (n > 0) k_gemv<<<(n * 32 + 255) / 256, 256, 0, s>>>(n, A, x, y);
}
void ik_iface_w(int npatch, const void *pif, const int *gbox, const double *phiG, const int *c_ptr, const int *c_idx,
                const double *cw, const int *Rg, const double *uPi, const double *xN, double *cvec, double *wG,
                cudaStream_t s) {
  k_iface_w<<<npatch, NT, 0, s>>>((const PatchIface *)pif, gbox, phiG, c_ptr, c_idx, cw, Rg, uPi, xN, cvec, wG);
}
void ik_full_u(int npatch, int maxbox, const void *pif, const double *phiF, const double *cvec, const double *xN,
               double *ubox, cudaStream_t s) {
  dim3 grid((maxbox + 255) / 256, npatch);
  k_full_u<<<grid, 256, 0, s>>>((const PatchIface *)pif, phiF, cvec, xN, ubox);
}
void ik_jump(int n, const int *gp, const int *gm, const double *wG, double *q, cudaStream_t s) {
  if (n > 0) k_jump<<<(n + 255) / 256, 256, 0, s>>>(n, gp, gm, wG, q);
}
void ik_bdt(int ngamma, const long long *gabs, const int *ptr, const int *m, const double *w, const double *r,
            double *vbox, cudaStream_t s) {
  if (ngamma > 0) k_bdt<<<(ngamma + 255) / 256, 256, 0, s>>>(ngamma, gabs, ptr, m, w, r, vbox);
}
void ik_bd_gather(int n, const int *ptr, const int *gi, const double *w, const long long *gabs, const double *y,
                  double *z, cudaStream_t s) {
  if (n > 0) k_bd_gather<<<(n + 255) / 256, 256, 0, s>>>(n, ptr, gi, w, gabs, y, z);
}
void ik_dot_partial(long long n, const double *a, const double *b, double *partial, int nb, cudaStream_t s) {
  k_dot_partial<<<nb, NT, 0, s>>>(n, a, b, partial);
}
void ik_pcg_alpha(const double *partial, int nb, double *sc, cudaStream_t s) { k_pcg_alpha<<<1, NT, 0, s>>>(partial, nb, sc); }
void ik_pcg_update(long long n, const double *sc, const double *p, const double *q, double *lam, double *r,
                   double *partial, int nb, cudaStream_t s) {
  k_pcg_update<<<nb, NT, 0, s>>>(n, sc, p, q, lam, r, partial);
}
void ik_store_scalar(const double *partial, int nb, double *sc, int slot, int take_sqrt, cudaStream_t s) {
  k_store_scalar<<<1, NT, 0, s>>>(partial, nb, sc, slot, take_sqrt);
}
void ik_pcg_beta(const double *partial, int nb, double *sc, cudaStream_t s) { k_pcg_beta<<<1, NT, 0, s>>>(partial, nb, sc); }
void ik_pcg_p(long long n, const double *sc, const double *z, double *p, int nb, cudaStream_t s) {
  k_pcg_p<<<nb, NT, 0, s>>>(n, sc, z, p);
}
void ik_copy(long long n, const double *a, double *b, cudaStream_t s) {
  if (n > 0) k_copy<<<(unsigned)std::min<long long>((n + 255) / 256, 4096), 256, 0, s>>>(n, a, b);
}
void ik_scale_copy(long long n, double sc, const double *a, double *b, cudaStream_t s) {
  if (n > 0) k_scale_copy<<<(unsigned)std::min<long long>((n + 255) / 256, 4096), 256, 0, s>>>(n, sc, a, b);
}
void ik_lattice_to_box(int dim, int p, int npatch, long long maxn, const GridDesc *g, const ProbDesc *pr,
                       const long long *loff, const double *lat, double *box, int only_interior, cudaStream_t s) {
  dim3 grid((unsigned)((maxn + 255) / 256), npatch);
  k_lattice_to_box<<<grid, 256, 0, s>>>(dim, p, g, pr, loff, lat, box, only_interior);
}
void ik_box_to_lattice(int dim, int p, int npatch, long long maxn, const GridDesc *g, const ProbDesc *pr,
                       const long long *loff, const double *box, double *lat, cudaStream_t s) {
  dim3 grid((unsigned)((maxn + 255) / 256), npatch);
  k_box_to_lattice<<<grid, 256, 0, s>>>(dim, p, g, pr, loff, box, lat);
}
void ik_mask_box(int dim, int p, int nprob, int maxbox, const GridDesc *g, const ProbDesc *pr, double *v, cudaStream_t s) {
  dim3 grid((maxbox + 255) / 256, nprob);
  k_mask_box<<<grid, 256, 0, s>>>(dim, p, g, pr, v);
}

// ------------------------------------------------------------------------------------------
// C2: per-patch inner PCG on K with a one-V-cycle preconditioner (reading R19).
// One thread block per patch (problem); scalars per patch in device arrays; ctr[0] = inner
// iteration number, ctr[1] = number of patches still active after the current step.
// ------------------------------------------------------------------------------------------
namespace {

// r = q, x = 0, qn = ||q||, active = (qn > 0), its = 0
__global__ void k_inner_init(const ProbDesc *__restrict__ pr, const GridDesc *__restrict__ g,
                             const double *__restrict__ q, double *r, double *x, double *qn, int *active, int *its,
                             int *ctr) {
  __shared__ double sh[40];
  const ProbDesc P = pr[blockIdx.x];
  const int n = g[P.grid].box;
  double s = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const double v = q[P.vec_off + t];
    r[P.vec_off + t] = v;
    x[P.vec_off + t] = 0.0;
    s = fma(v, v, s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) {
    qn[blockIdx.x] = sqrt(s);
    active[blockIdx.x] = (s > 0.0) ? 1 : 0;
    its[blockIdx.x] = 0;
    if (blockIdx.x == 0) { ctr[0] = 0; ctr[1] = 0; ctr[2] = 0; }
  }
}

// rho_new = r.z; first: p = z, rho = rho_new (every patch, as the textbook start);
// otherwise on active patches: beta = rho_new / rho, p = z + beta p, rho = rho_new
__global__ void k_inner_dir(const ProbDesc *__restrict__ pr, const GridDesc *__restrict__ g,
                            const double *__restrict__ r, const double *__restrict__ z, double *p, double *rho,
                            const int *__restrict__ active, int first) {
  __shared__ double sh[40];
  const ProbDesc P = pr[blockIdx.x];
  const int n = g[P.grid].box;
  double s = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) s = fma(r[P.vec_off + t], z[P.vec_off + t], s);
  s = block_sum(s, sh);
  if (first) {
    for (int t = threadIdx.x; t < n; t += blockDim.x) p[P.vec_off + t] = z[P.vec_off + t];
    if (threadIdx.x == 0) rho[blockIdx.x] = s;
    return;
  }
  if (!active[blockIdx.x]) return;
  const double beta = s / rho[blockIdx.x];
  for (int t = threadIdx.x; t < n; t += blockDim.x) p[P.vec_off + t] = fma(beta, p[P.vec_off + t], z[P.vec_off + t]);
  __syncthreads();
  if (threadIdx.x == 0) rho[blockIdx.x] = s;
}

__global__ void k_inner_begin(int *ctr) {
  ctr[0] += 1;
  ctr[1] = 0;
}

// alpha = rho / p.Ap; x += alpha p; r -= alpha Ap; stop the patch when ||r|| <= tol ||q||
// proj (optional, per problem): keep r in range(K) = {1^T r = 0} on floating patches (subtract the
// mean over the active lattice points) -- rounding otherwise feeds the kernel of the singular K,
// which the regularised V-cycle amplifies by ~1/alpha (primal-basis setup only)
__global__ void k_inner_step(const ProbDesc *__restrict__ pr, const GridDesc *__restrict__ g,
                             const double *__restrict__ p, const double *__restrict__ Ap, double *x, double *r,
                             const double *__restrict__ rho, const double *__restrict__ qn, int *active, int *its,
                             int *ctr, double tol, const int *__restrict__ proj, int pdeg, int dim) {
  __shared__ double sh[40];
  if (!active[blockIdx.x]) return;
  const ProbDesc P = pr[blockIdx.x];
  const GridDesc &G = g[P.grid];
  const int n = G.box;
  double s = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) s = fma(p[P.vec_off + t], Ap[P.vec_off + t], s);
  s = block_sum(s, sh);
  if (!(s > 0.0) || !isfinite(s)) {
    // p.Ap <= 0: p = 0 (the residual vanished to rounding: stop) or a breakdown (negative or
    // non-finite curvature: stop the patch and count it, reported by the solve -- ADVICE r1)
    if (threadIdx.x == 0) {
      active[blockIdx.x] = 0;
      its[blockIdx.x] = ctr[0];
      if (!isfinite(s) || s < 0.0) atomicAdd(&ctr[2], 1);
    }
    return;
  }
  const double alpha = rho[blockIdx.x] / s;
  double rr = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const long long i = P.vec_off + t;
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    rr = fma(ri, ri, rr);
  }
  if (proj && proj[blockIdx.x]) {
    const int P1 = pdeg + 1;
    auto is_act = [&](int t) {
      int c = t / G.sb, rem = t % G.sb;
      const int q[3] = {rem % G.ns[0], (rem / G.ns[0]) % G.ns[1], (dim == 3) ? rem / (G.ns[0] * G.ns[1]) : 0};
      bool in = true;
      for (int d = 0; d < dim; ++d) {
        const int i = c % P1 + P1 * q[d];
        c /= P1;
        in = in && i >= G.lo[d] && i < G.hi[d];
      }
      return in;
    };
    double sr = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) sr += r[P.vec_off + t];   // non-active entries are 0
    sr = block_sum(sr, sh);
    const double mean = sr / (double)G.nrows;
    rr = 0.0;
    for (int t = threadIdx.x; t < n; t += blockDim.x)
      if (is_act(t)) {
        const double ri = r[P.vec_off + t] - mean;
        r[P.vec_off + t] = ri;
        rr = fma(ri, ri, rr);
      }
  }
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) {
    its[blockIdx.x] = ctr[0];
    if (sqrt(rr) <= tol * qn[blockIdx.x]) active[blockIdx.x] = 0;
    else atomicAdd(&ctr[1], 1);
  }
}

}  // namespace

void ik_inner_init(int nprob, const ProbDesc *pr, const GridDesc *g, const double *q, double *r, double *x, double *qn,
                   int *active, int *its, int *ctr, cudaStream_t s) {
  k_inner_init<<<nprob, NT, 0, s>>>(pr, g, q, r, x, qn, active, its, ctr);
}
void ik_inner_dir(int nprob, const ProbDesc *pr, const GridDesc *g, const double *r, const double *z, double *p,
                  double *rho, const int *active, int first, cudaStream_t s) {
  k_inner_dir<<<nprob, NT, 0, s>>>(pr, g, r, z, p, rho, active, first);
}
void ik_inner_begin(int *ctr, cudaStream_t s) { k_inner_begin<<<1, 1, 0, s>>>(ctr); }
void ik_inner_step(int nprob, const ProbDesc *pr, const GridDesc *g, const double *p, const double *Ap, double *x,
                   double *r, const double *rho, const double *qn, int *active, int *its, int *ctr, double tol,
                   const int *proj, int pdeg, int dim, cudaStream_t s) {
  k_inner_step<<<nprob, NT, 0, s>>>(pr, g, p, Ap, x, r, rho, qn, active, its, ctr, tol, proj, pdeg, dim);
}

// ------------------------------------------------------------------------------------------
// multi-GPU exchange helpers (partition.cpp plan; comm.cpp collectives)
// ------------------------------------------------------------------------------------------
namespace {
__global__ void k_pack(int n, const int *__restrict__ idx, const double *__restrict__ src, double *dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[idx[e]];
}
__global__ void k_unpack(int n, const int *__restrict__ idx, const double *__restrict__ src, double *dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[idx[e]] = src[e];
}
// owner rows: v[j] += received partials in ascending peer order (deterministic)
__global__ void k_rsum(int n_own, const int *__restrict__ ptr, const int *__restrict__ srcpos,
                       const double *__restrict__ recv, double *v) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_own || ptr[j] == ptr[j + 1]) return;
  double s = v[j];
  for (int e = ptr[j]; e < ptr[j + 1]; ++e) s += recv[srcpos[e]];
  v[j] = s;
}
// out[i] = sum_r all[r*n + i] in rank order
__global__ void k_sum_ranks(int n, int world, const double *__restrict__ all, double *out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += all[(long long)r * n + i];
  out[i] = s;
}
__global__ void k_reduce_to(const double *partial, int nb, double *out) {
  __shared__ double sh[40];
  double v = reduce_partials(partial, nb, sh);
  if (threadIdx.x == 0) out[0] = v;
}
}  // namespace

void ik_pack(int n, const int *idx, const double *src, double *dst, cudaStream_t s) {
  if (n > 0) k_pack<<<(n + 255) / 256, 256, 0, s>>>(n, idx, src, dst);
}
void ik_unpack(int n, const int *idx, const double *src, double *dst, cudaStream_t s) {
  if (n > 0) k_unpack<<<(n + 255) / 256, 256, 0, s>>>(n, idx, src, dst);
}
void ik_rsum(int n_own, const int *ptr, const int *srcpos, const double *recv, double *v, cudaStream_t s) {
  if (n_own > 0) k_rsum<<<(n_own + 255) / 256, 256, 0, s>>>(n_own, ptr, srcpos, recv, v);
}
void ik_sum_ranks(int n, int world, const double *all, double *out, cudaStream_t s) {
  if (n > 0) k_sum_ranks<<<(n + 255) / 256, 256, 0, s>>>(n, world, all, out);
}
void ik_reduce_to(const double *partial, int nb, double *out, cudaStream_t s) {
  k_reduce_to<<<1, NT, 0, s>>>(partial, nb, out);
}

// ------------------------------------------------------------------------------------------
// MG-MG-S: Bramble-Pasciak CG on the saddle point Eq. (2) (DESIGN.md
// R28-R31).  Vectors of V~_h and its functionals live in fine-level Neumann boxes (torn patch
// vectors, R28); multiplier vectors as in the dual PCG.
// ------------------------------------------------------------------------------------------
namespace {

// out = bN + C^T W R g : the null-part-free representative of a functional (R31); bN holds
// P^T r = r - C^T Phibar^T r (k_full_t), g = sum_k R_k^T Phibar_k^T r_k, W = 1 / multiplicity
__global__ void k_can_add(const PatchIface *__restrict__ pif, const int *__restrict__ gbox,
                          const int *__restrict__ crow, const double *__restrict__ cw, const int *__restrict__ R,
                          const double *__restrict__ g, const double *__restrict__ invmult,
                          const double *__restrict__ bN, double *out) {
  const PatchIface P = pif[blockIdx.x];
  const double *bb = bN + P.box_off;
  double *oo = out + P.box_off;
  for (int t = threadIdx.x; t < P.box; t += blockDim.x) oo[t] = bb[t];
  __syncthreads();
  for (int gg = threadIdx.x; gg < P.ng; gg += blockDim.x) {
    const int gi = P.g_off + gg;
    const int j = crow[gi];
    if (j >= 0) {
      const int gid = R[P.pi_off + j];
      oo[gbox[gi]] = fma(cw[gi], g[gid] * invmult[gid], oo[gbox[gi]]);
    }
  }
}

// box (Gamma entries) += B^T lam
__global__ void k_bt_add(int ngamma, const long long *__restrict__ gabs, const int *__restrict__ ptr,
                         const int *__restrict__ m, const double *__restrict__ w, const double *__restrict__ lam,
                         double *box) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngamma) return;
  double s = 0.0;
  for (int e = ptr[g]; e < ptr[g + 1]; ++e) s = fma(w[e], lam[m[e]], s);
  box[gabs[g]] += s;
}

// q_i = u(k+, a+) - u(k-, a-) read from a box vector (B u); remote sides contribute 0 (k_rsum)
__global__ void k_jump_box(int n, const int *__restrict__ gp, const int *__restrict__ gm,
                           const long long *__restrict__ gabs, const double *__restrict__ box, double *q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double wp = (gp[i] >= 0) ? box[gabs[gp[i]]] : 0.0;
  const double wm = (gm[i] >= 0) ? box[gabs[gm[i]]] : 0.0;
  q[i] = wp - wm;
}

// y += sign * sc[slot] * x
__global__ void k_axpy_s(long long n, const double *__restrict__ sc, int slot, double sign,
                         const double *__restrict__ x, double *y) {
  const double a = sign * sc[slot];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

// y = x + sc[slot] * y
__global__ void k_xpby_s(long long n, const double *__restrict__ sc, int slot, const double *__restrict__ x,
                         double *y) {
  const double b = sc[slot];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(b, y[i], x[i]);
}

// out = a - b
__global__ void k_sub(long long n, const double *__restrict__ a, const double *__restrict__ b, double *out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

// scalar steps (slots: 0 gamma, 1 delta, 2 alpha, 3 beta, 4 ||rho||^2, 6 breakdown, 8.. dot values)
//   op 0 (delta): delta = d8 - d9 - d10; alpha = gamma / delta; breakdown unless delta, gamma > 0
//   op 1 (gamma): gamma' = d8 - d9 + d10; beta = gamma' / gamma; gamma = gamma'
//   op 2 (gamma, first): gamma = d8 - d9 + d10
//   op 3 (residual): ||rho||^2 = d11 + d12
__global__ void k_bp_scalar(int op, double *sc) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (op == 0) {
    const double delta = sc[8] - sc[9] - sc[10];
    sc[1] = delta;
    const bool ok = isfinite(delta) && delta > 0.0 && isfinite(sc[0]) && sc[0] > 0.0;
    if (!ok) sc[6] = 1.0;
    sc[2] = ok ? sc[0] / delta : 0.0;
  } else if (op == 1 || op == 2) {
    const double g = sc[8] - sc[9] + sc[10];
    if (op == 1) sc[3] = g / sc[0];
    sc[0] = g;
  } else {
    sc[4] = sc[11] + sc[12];
  }
}

}  // namespace

static unsigned vgrid(long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 4096); }

void ik_can_add(int npatch, const void *pif, const int *gbox, const int *crow, const double *cw, const int *R,
                const double *g, const double *invmult, const double *bN, double *out, cudaStream_t s) {
  if (npatch > 0) k_can_add<<<npatch, NT, 0, s>>>((const PatchIface *)pif, gbox, crow, cw, R, g, invmult, bN, out);
}
void ik_bt_add(int ngamma, const long long *gabs, const int *ptr, const int *m, const double *w, const double *lam,
               double *box, cudaStream_t s) {
  if (ngamma > 0) k_bt_add<<<(ngamma + 255) / 256, 256, 0, s>>>(ngamma, gabs, ptr, m, w, lam, box);
}
void ik_jump_box(int n, const int *gp, const int *gm, const long long *gabs, const double *box, double *q,
                 cudaStream_t s) {
  if (n > 0) k_jump_box<<<(n + 255) / 256, 256, 0, s>>>(n, gp, gm, gabs, box, q);
}
void ik_axpy_s(long long n, const double *sc, int slot, double sign, const double *x, double *y, cudaStream_t s) {
  if (n > 0) k_axpy_s<<<vgrid(n), 256, 0, s>>>(n, sc, slot, sign, x, y);
}
void ik_xpby_s(long long n, const double *sc, int slot, const double *x, double *y, cudaStream_t s) {
  if (n > 0) k_xpby_s<<<vgrid(n), 256, 0, s>>>(n, sc, slot, x, y);
}
void ik_sub(long long n, const double *a, const double *b, double *out, cudaStream_t s) {
  if (n > 0) k_sub<<<vgrid(n), 256, 0, s>>>(n, a, b, out);
}
void ik_bp_scalar(int op, double *sc, cudaStream_t s) { k_bp_scalar<<<1, 32, 0, s>>>(op, sc); }
