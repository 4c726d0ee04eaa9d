// kernels_basis.cu -- per-problem ("segmented") kernels for the primal-basis setup (Eq. (6)).
//
// The energy-minimising basis Phibar^(k) (Eq. (6)) is assembled from Y = K^+ C^T (I - 11^T/n)
// (floating) or Y = K^{-1} C^T, computed by batched PCG over all (patch, column) problems
// (solver.cu, BatchedPcg).  These kernels provide the non-stencil pieces: right-hand sides,
// per-problem dot products and vector updates, C y, the combination Phibar = Y M + 1 c^T and
// column extraction.  One thread block per problem.
#include "internal.h"

namespace {
constexpr int NT = 256;

__device__ __forceinline__ double bsum(double v, double *sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) sh[32] = s;
  }
  __syncthreads();
  return sh[32];
}

__global__ void k_rhs_ct(const int *__restrict__ prob_patch, const int *__restrict__ prob_col,
                         const ProbDesc *__restrict__ pr, const PatchIface *__restrict__ pif,
                         const int *__restrict__ gbox, const int *__restrict__ crow, const double *__restrict__ cw,
                         double *b) {
  const PatchIface P = pif[prob_patch[blockIdx.x]];
  const int col = prob_col[blockIdx.x];
  const long long off = pr[blockIdx.x].vec_off;
  // C^T e_j; on floating patches C^T (e_j - 1/n_Pi), which is consistent (1^T C^T = 1^T) because
  // every constraint row sums to one on constants
  const double sub = P.floating ? 1.0 / P.npi : 0.0;
  for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
    const int gi = P.g_off + g;
    if (crow[gi] >= 0) b[off + gbox[gi]] = cw[gi] * (((crow[gi] == col) ? 1.0 : 0.0) - sub);
  }
}

__global__ void k_seg_dot(const ProbDesc *__restrict__ pr, const GridDesc *__restrict__ g,
                          const double *__restrict__ a, const double *__restrict__ b, double *out) {
  __shared__ double sh[40];
  const ProbDesc P = pr[blockIdx.x];
  const int n = g[P.grid].box;
  double s = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) s = fma(a[P.vec_off + t], b[P.vec_off + t], s);
  s = bsum(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void k_seg_axpy(const ProbDesc *__restrict__ pr, const GridDesc *__restrict__ g, const double *coef,
                           double sign, const double *__restrict__ x, double *y, const int *active) {
  if (active && !active[blockIdx.x]) return;
  const ProbDesc P = pr[blockIdx.x];
  const int n = g[P.grid].box;
  const double a = sign * coef[blockIdx.x];
  for (int t = threadIdx.x; t < n; t += blockDim.x) y[P.vec_off + t] = fma(a, x[P.vec_off + t], y[P.vec_off + t]);
}

__global__ void k_seg_xpby(const ProbDesc *__restrict__ pr, const GridDesc *__restrict__ g, const double *__restrict__ z,
                           const double *beta, double *p, const int *active) {
  if (active && !active[blockIdx.x]) return;
  const ProbDesc P = pr[blockIdx.x];
  const int n = g[P.grid].box;
  const double b = beta[blockIdx.x];
  for (int t = threadIdx.x; t < n; t += blockDim.x) p[P.vec_off + t] = fma(b, p[P.vec_off + t], z[P.vec_off + t]);
}

__global__ void k_cx(const int *__restrict__ prob_patch, const ProbDesc *__restrict__ pr,
                     const PatchIface *__restrict__ pif, const int *__restrict__ gbox, const int *__restrict__ crow,
                     const double *__restrict__ cw, const double *__restrict__ x, double *out, int stride) {
  __shared__ double sh[40];
  const PatchIface P = pif[prob_patch[blockIdx.x]];
  const long long off = pr[blockIdx.x].vec_off;
  for (int j = 0; j < P.npi; ++j) {
    double s = 0.0;
    for (int g = threadIdx.x; g < P.ng; g += blockDim.x) {
      const int gi = P.g_off + g;
      if (crow[gi] == j) s = fma(cw[gi], x[off + gbox[gi]], s);
    }
    s = bsum(s, sh);
    if (threadIdx.x == 0) out[(long long)blockIdx.x * stride + j] = s;
  }
}
}  // namespace

void bk_rhs_ct(int nprob, const int *prob_patch, const int *prob_col, const ProbDesc *pr, const void *pif,
               const int *gbox, const int *crow, const double *cw, double *b, cudaStream_t s) {
  if (nprob > 0) k_rhs_ct<<<nprob, NT, 0, s>>>(prob_patch, prob_col, pr, (const PatchIface *)pif, gbox, crow, cw, b);
}
void bk_seg_dot(int nprob, const ProbDesc *pr, const GridDesc *g, const double *a, const double *b, double *out,
                cudaStream_t s) {
  if (nprob > 0) k_seg_dot<<<nprob, NT, 0, s>>>(pr, g, a, b, out);
}
void bk_seg_axpy(int nprob, const ProbDesc *pr, const GridDesc *g, const double *coef, double sign, const double *x,
                 double *y, const int *active, cudaStream_t s) {
  if (nprob > 0) k_seg_axpy<<<nprob, NT, 0, s>>>(pr, g, coef, sign, x, y, active);
}
void bk_seg_xpby(int nprob, const ProbDesc *pr, const GridDesc *g, const double *z, const double *beta, double *p,
                 const int *active, cudaStream_t s) {
  if (nprob > 0) k_seg_xpby<<<nprob, NT, 0, s>>>(pr, g, z, beta, p, active);
}
void bk_cx(int nprob, const int *prob_patch, const ProbDesc *pr, const void *pif, const int *gbox, const int *crow,
           const double *cw, const double *x, double *out, int out_stride, cudaStream_t s) {
  if (nprob > 0) k_cx<<<nprob, NT, 0, s>>>(prob_patch, pr, (const PatchIface *)pif, gbox, crow, cw, x, out, out_stride);
}

// ---- combination / extraction kernels -------------------------------------------------------
namespace {
// dst[patch k][col j][t] = sum_i src[k][i][t] * M_k[i][j] + c_k[j] * [t is an active lattice point]
// (Phibar = Y M + 1 c^T; c = 0 on non-floating patches)
__global__ void k_combine(const PatchIface *__restrict__ pif, const long long *__restrict__ hoff,
                          const double *__restrict__ Hm, const double *__restrict__ cconst,
                          const GridDesc *__restrict__ g_, int p, int dim, const double *__restrict__ src,
                          double *dst) {
  const PatchIface P = pif[blockIdx.y];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.box) return;
  const double *H = Hm + hoff[blockIdx.y];
  bool act = false;
  if (P.floating) {
    const GridDesc &g = g_[blockIdx.y];
    const int P1 = p + 1;
    int c = t / g.sb, rem = t % g.sb;
    int q[3] = {rem % g.ns[0], (rem / g.ns[0]) % g.ns[1], (dim == 3) ? rem / (g.ns[0] * g.ns[1]) : 0};
    act = true;
    for (int d = 0; d < dim; ++d) {
      const int i = c % P1 + P1 * q[d];
      c /= P1;
      act = act && i >= g.lo[d] && i < g.hi[d];
    }
  }
  const double *cc = cconst + P.pi_off;
  for (int j = 0; j < P.npi; ++j) {
    double s = act ? cc[j] : 0.0;
    for (int i = 0; i < P.npi; ++i) s = fma(src[P.phif_off + (long long)i * P.box + t], H[i * P.npi + j], s);
    dst[P.phif_off + (long long)j * P.box + t] = s;
  }
}

// out[p*stride + i] = Phibar_k[:, i] . y_p   for every problem p = (k, j)
__global__ void k_phi_dots(const int *__restrict__ prob_patch, const ProbDesc *__restrict__ pr,
                           const PatchIface *__restrict__ pif, const double *__restrict__ phif,
                           const double *__restrict__ y, double *out, int stride) {
  __shared__ double sh[40];
  const PatchIface P = pif[prob_patch[blockIdx.x]];
  const long long off = pr[blockIdx.x].vec_off;
  for (int i = 0; i < P.npi; ++i) {
    double s = 0.0;
    for (int t = threadIdx.x; t < P.box; t += blockDim.x) s = fma(phif[P.phif_off + (long long)i * P.box + t], y[off + t], s);
    s = bsum(s, sh);
    if (threadIdx.x == 0) out[(long long)blockIdx.x * stride + i] = s;
  }
}

// phiG[k][j][g] = phif[k][j][gbox[g]]
__global__ void k_extract_gamma(const PatchIface *__restrict__ pif, const int *__restrict__ gbox,
                                const double *__restrict__ phif, double *phiG) {
  const PatchIface P = pif[blockIdx.y];
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.ng) return;
  for (int j = 0; j < P.npi; ++j)
    phiG[P.phi_off + (long long)j * P.ng + g] = phif[P.phif_off + (long long)j * P.box + gbox[P.g_off + g]];
}

// copy problem vectors <-> per-patch column pools (phif layout)
__global__ void k_prob_to_cols(const int *__restrict__ prob_patch, const int *__restrict__ prob_col,
                               const ProbDesc *__restrict__ pr, const PatchIface *__restrict__ pif,
                               const double *__restrict__ x, double *cols, int to_cols) {
  const PatchIface P = pif[prob_patch[blockIdx.y]];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.box) return;
  const long long a = pr[blockIdx.y].vec_off + t;
  const long long b = P.phif_off + (long long)prob_col[blockIdx.y] * P.box + t;
  if (to_cols) cols[b] = x[a];
  else ((double *)x)[a] = cols[b];
}
}  // namespace

void bk_combine(int npatch, int maxbox, const void *pif, const long long *hoff, const double *Hm,
                const double *cconst, const GridDesc *g, int p, int dim, const double *src, double *dst,
                cudaStream_t s) {
  dim3 grid((maxbox + 255) / 256, npatch);
  k_combine<<<grid, 256, 0, s>>>((const PatchIface *)pif, hoff, Hm, cconst, g, p, dim, src, dst);
}
void bk_phi_dots(int nprob, const int *prob_patch, const ProbDesc *pr, const void *pif, const double *phif,
                 const double *y, double *out, int stride, cudaStream_t s) {
  if (nprob > 0) k_phi_dots<<<nprob, NT, 0, s>>>(prob_patch, pr, (const PatchIface *)pif, phif, y, out, stride);
}
void bk_extract_gamma(int npatch, int maxng, const void *pif, const int *gbox, const double *phif, double *phiG,
                      cudaStream_t s) {
  if (maxng <= 0) return;
  dim3 grid((maxng + 255) / 256, npatch);
  k_extract_gamma<<<grid, 256, 0, s>>>((const PatchIface *)pif, gbox, phif, phiG);
}
void bk_prob_cols(int nprob, int maxbox, const int *prob_patch, const int *prob_col, const ProbDesc *pr,
                  const void *pif, const double *x, double *cols, int to_cols, cudaStream_t s) {
  if (nprob <= 0) return;
  dim3 grid((maxbox + 255) / 256, nprob);
  k_prob_to_cols<<<grid, 256, 0, s>>>(prob_patch, prob_col, pr, (const PatchIface *)pif, x, cols, to_cols);
}
