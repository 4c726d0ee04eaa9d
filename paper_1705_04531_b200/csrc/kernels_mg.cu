// kernels_mg.cu -- batched per-patch geometric multigrid kernels for sm_100a (fp64).
//
//  * k_sgs       one colour phase of the (p+1)^d-colour Gauss-Seidel smoother (R5, R6):
//                x_a += (b_a - sum_o A[a,o] x[a+o]) / A[a,a] for every row a of colour c of every
//                problem in the batch.  Rows of one colour are decoupled (|i_d - j_d| >= p+1 in
//                some d => A_ij = 0), so the phase is one launch.
//  * k_residual  y = s (b - A x)  or  y = s A (x + x2)  [+ on-the-fly beta * Mhat term]
//  * k_restrict  b_c = P^T r_f,  x_c = 0        (P = P_1 (x) ... (x) P_d, knot insertion, R8)
//  * k_prolong   x_f += P x_c
//  * k_coarse    x = A_0^{-1} b (explicit inverse of the coarsest Galerkin matrix, R9)
//  * Galerkin    A_{l-1} = P^T A_l P in stencil form, two stages (setup only)
//
// One thread per stencil row, rows of a colour contiguous in the offset-major coefficient
// array: each of the (2p+1)^d coefficient loads of a warp is one 256-byte coalesced
// transaction; x (<= ~0.5 MB per patch) is served from L1/L2.
#include "internal.h"

#include <algorithm>
#include <cstdio>

namespace {

template <int D, int P>
struct St {
  static constexpr int W1 = 2 * P + 1;
  static constexpr int S = (D == 3) ? W1 * W1 * W1 : W1 * W1;
  static constexpr int CENTER = (D == 3) ? P + W1 * (P + W1 * P) : P + W1 * P;
};

__device__ __forceinline__ void decode_colour_row(const ColourInfo &ci, int j, int P1, int *i) {
  int j0 = j % ci.n[0];
  int t = j / ci.n[0];
  int j1 = t % ci.n[1];
  int j2 = t / ci.n[1];
  i[0] = ci.first[0] + P1 * j0;
  i[1] = ci.first[1] + P1 * j1;
  i[2] = ci.first[2] + P1 * j2;
}

template <int D, int P>
__device__ __forceinline__ long long box_pos(const GridDesc &g, const int *i) {
  long long z = (D == 3) ? (i[2] + P) : 0;
  return (long long)(i[0] + P) + (long long)g.pad[0] * ((i[1] + P) + (long long)g.pad[1] * z);
}

// sum_o A[r,o] * x[pos + off(o)]  (coefficients offset-major with leading dimension ld)
template <int D, int P>
__device__ __forceinline__ double stencil_dot(const double *__restrict__ c, long long ld, const double *xb,
                                              int s1, long long s2) {
  constexpr int W1 = 2 * P + 1;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  int o = 0;
#pragma unroll
  for (int o2 = (D == 3 ? -P : 0); o2 <= (D == 3 ? P : 0); ++o2) {
#pragma unroll
    for (int o1 = -P; o1 <= P; ++o1) {
      const double *xr = xb + o1 * s1 + o2 * s2;
#pragma unroll
      for (int o0 = -P; o0 <= P; ++o0, ++o) {
        double a = __ldg(c + o * ld);
        double v = xr[o0];
        switch (o & 3) {
          case 0: acc0 = fma(a, v, acc0); break;
          case 1: acc1 = fma(a, v, acc1); break;
          case 2: acc2 = fma(a, v, acc2); break;
          default: acc3 = fma(a, v, acc3); break;
        }
      }
    }
  }
  (void)W1;
  return (acc0 + acc1) + (acc2 + acc3);
}

template <int D, int P>
__global__ void __launch_bounds__(128) k_sgs(LevelView lv, const BlockEntry *__restrict__ blocks,
                                             double *x, const double *__restrict__ b) {
  const BlockEntry be = blocks[blockIdx.x];
  if ((int)threadIdx.x >= be.nrow) return;
  const ProbDesc pr = lv.probs[be.prob];
  const GridDesc &g = lv.grids[pr.grid];
  const ColourInfo ci = lv.cinfo[g.col_off + be.colour];
  const int j = be.row0 + threadIdx.x;
  int i[3];
  decode_colour_row(ci, j, P + 1, i);
  const long long pos = pr.vec_off + box_pos<D, P>(g, i);
  const long long ld = g.ld;
  const double *c = lv.coef + g.coef_off + ci.start + j;
  const int s1 = g.pad[0];
  const long long s2 = (long long)g.pad[0] * g.pad[1];
  double sum = stencil_dot<D, P>(c, ld, x + pos, s1, s2);
  double diag = __ldg(c + St<D, P>::CENTER * ld);
  x[pos] += (b[pos] - sum) / diag;
}

template <int D, int P>
__global__ void __launch_bounds__(128) k_residual(LevelView lv, const BlockEntry *__restrict__ blocks,
                                                  const double *x, const double *x2, const double *b,
                                                  double *y, double scale, int use_mass) {
  const BlockEntry be = blocks[blockIdx.x];
  if ((int)threadIdx.x >= be.nrow) return;
  const ProbDesc pr = lv.probs[be.prob];
  const GridDesc &g = lv.grids[pr.grid];
  const ColourInfo ci = lv.cinfo[g.col_off + be.colour];
  const int j = be.row0 + threadIdx.x;
  int i[3];
  decode_colour_row(ci, j, P + 1, i);
  const long long pos = pr.vec_off + box_pos<D, P>(g, i);
  const long long ld = g.ld;
  const double *c = lv.coef + g.coef_off + ci.start + j;
  const int s1 = g.pad[0];
  const long long s2 = (long long)g.pad[0] * g.pad[1];
  double sum;
  if (x2 == nullptr) {
    sum = stencil_dot<D, P>(c, ld, x + pos, s1, s2);
  } else {
    constexpr int W1 = 2 * P + 1;
    double acc = 0.0;
    int o = 0;
    for (int o2 = (D == 3 ? -P : 0); o2 <= (D == 3 ? P : 0); ++o2)
      for (int o1 = -P; o1 <= P; ++o1)
#pragma unroll
        for (int o0 = -P; o0 <= P; ++o0, ++o) {
          long long q = pos + o0 + o1 * s1 + o2 * s2;
          acc = fma(__ldg(c + o * ld), x[q] + x2[q], acc);
        }
    (void)W1;
    sum = acc;
  }
  if (use_mass && g.mass_beta != 0.0) {
    // + beta * (M_1 (x) ... (x) M_d) applied on the fly from the 1D mass tables (R4)
    constexpr int W1 = 2 * P + 1;
    const double *m0 = lv.mass + g.mass_off + (long long)i[0] * W1;
    const double *m1 = lv.mass + g.mass_off + (long long)g.M[0] * W1 + (long long)i[1] * W1;
    const double *m2 = lv.mass + g.mass_off + (long long)(g.M[0] + g.M[1]) * W1 + (long long)i[2] * W1;
    double acc = 0.0;
    for (int o2 = (D == 3 ? -P : 0); o2 <= (D == 3 ? P : 0); ++o2) {
      double w2 = (D == 3) ? m2[o2 + P] : 1.0;
      for (int o1 = -P; o1 <= P; ++o1) {
        double w12 = w2 * m1[o1 + P];
        for (int o0 = -P; o0 <= P; ++o0) {
          long long q = pos + o0 + o1 * s1 + o2 * s2;
          double v = x[q] + (x2 ? x2[q] : 0.0);
          acc = fma(w12 * m0[o0 + P], v, acc);
        }
      }
    }
    sum = fma(g.mass_beta, acc, sum);
  }
  y[pos] = (b != nullptr) ? scale * (b[pos] - sum) : scale * sum;
}

// -------- transfers ---------------------------------------------------------------------
__device__ __forceinline__ void decode_point(const GridDesc &g, int t, int *i) {
  int n0 = g.hi[0] - g.lo[0], n1 = g.hi[1] - g.lo[1];
  i[0] = g.lo[0] + t % n0;
  t /= n0;
  i[1] = g.lo[1] + t % n1;
  i[2] = g.lo[2] + t / n1;
}

template <int D, int P>
__global__ void k_restrict(const GridDesc *gc_, const GridDesc *gf_, const TransDesc *td_, const ProbDesc *pc_,
                           const ProbDesc *pf_, const int *__restrict__ ipool, const double *__restrict__ wpool,
                           const BlockEntry *__restrict__ blocks, const double *rf, double *bc, double *xc) {
  const BlockEntry be = blocks[blockIdx.x];
  if ((int)threadIdx.x >= be.nrow) return;
  const ProbDesc pc = pc_[be.prob], pf = pf_[be.prob];
  const GridDesc &gc = gc_[pc.grid];
  const GridDesc &gf = gf_[pf.grid];
  const TransDesc &td = td_[pc.grid];
  int a[3];
  decode_point(gc, be.row0 + threadIdx.x, a);
  constexpr int NW = P + 2;
  int f[3];
  const double *w[3];
  for (int d = 0; d < 3; ++d) {
    if (d < D) {
      f[d] = ipool[td.rc_off[d] + a[d]];
      w[d] = wpool + td.rw_off[d] + (long long)a[d] * NW;
    } else {
      f[d] = 0;
      w[d] = nullptr;
    }
  }
  const long long s1 = gf.pad[0], s2 = (long long)gf.pad[0] * gf.pad[1];
  double acc = 0.0;
  for (int t2 = 0; t2 < (D == 3 ? NW : 1); ++t2) {
    double w2 = (D == 3) ? w[2][t2] : 1.0;
    if (w2 == 0.0) continue;
    for (int t1 = 0; t1 < NW; ++t1) {
      double w12 = w2 * w[1][t1];
      if (w12 == 0.0) continue;
      int ii[3] = {f[0], f[1] + t1, f[2] + t2};
      const double *r = rf + pf.vec_off + box_pos<D, P>(gf, ii);
#pragma unroll
      for (int t0 = 0; t0 < NW; ++t0) acc = fma(w12 * w[0][t0], r[t0], acc);
    }
  }
  (void)s1; (void)s2;
  const long long q = pc.vec_off + box_pos<D, P>(gc, a);
  bc[q] = acc;
  if (xc) xc[q] = 0.0;
}

template <int D, int P>
__global__ void k_prolong(const GridDesc *gc_, const GridDesc *gf_, const TransDesc *td_, const ProbDesc *pc_,
                          const ProbDesc *pf_, const int *__restrict__ ipool, const double *__restrict__ wpool,
                          const BlockEntry *__restrict__ blocks, const double *xc, double *xf) {
  const BlockEntry be = blocks[blockIdx.x];
  if ((int)threadIdx.x >= be.nrow) return;
  const ProbDesc pc = pc_[be.prob], pf = pf_[be.prob];
  const GridDesc &gc = gc_[pc.grid];
  const GridDesc &gf = gf_[pf.grid];
  const TransDesc &td = td_[pc.grid];
  int i[3];
  decode_point(gf, be.row0 + threadIdx.x, i);
  const int W = td.W;
  int c[3];
  const double *w[3];
  for (int d = 0; d < 3; ++d) {
    if (d < D) {
      c[d] = ipool[td.pf_off[d] + i[d]];
      w[d] = wpool + td.pw_off[d] + (long long)i[d] * W;
    } else {
      c[d] = 0;
      w[d] = nullptr;
    }
  }
  double acc = 0.0;
  for (int t2 = 0; t2 < (D == 3 ? W : 1); ++t2) {
    double w2 = (D == 3) ? w[2][t2] : 1.0;
    if (w2 == 0.0) continue;
    for (int t1 = 0; t1 < W; ++t1) {
      double w12 = w2 * w[1][t1];
      if (w12 == 0.0) continue;
      int aa[3] = {c[0], c[1] + t1, c[2] + t2};
      const double *e = xc + pc.vec_off + box_pos<D, P>(gc, aa);
      for (int t0 = 0; t0 < W; ++t0) acc = fma(w12 * w[0][t0], e[t0], acc);
    }
  }
  xf[pf.vec_off + box_pos<D, P>(gf, i)] += acc;
}

// -------- coarsest solve: x = A0^{-1} b (one block per problem) ------------------------------
template <int D, int P>
__global__ void k_coarse(const GridDesc *g_, const ProbDesc *pr_, const long long *inv_off, const double *inv,
                         const double *b, double *x) {
  extern __shared__ double sb[];
  const ProbDesc pr = pr_[blockIdx.x];
  const GridDesc &g = g_[pr.grid];
  const int n = g.nrows;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    int i[3];
    decode_point(g, t, i);
    sb[t] = b[pr.vec_off + box_pos<D, P>(g, i)];
  }
  __syncthreads();
  const double *A = inv + inv_off[pr.grid];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < n; r += nw) {
    double acc = 0.0;
    for (int c = lane; c < n; c += 32) acc = fma(A[(long long)r * n + c], sb[c], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      int i[3];
      decode_point(g, r, i);
      x[pr.vec_off + box_pos<D, P>(g, i)] = acc;
    }
  }
}

// -------- Galerkin A_c = P^T A_f P (setup) ------------------------------------------------
// stage 1: B[i][t] = sum_o A_f[i, i+o] P[i+o, cw(i)+t]   (fine row i, coarse window t in CW^D)
template <int D, int P>
__global__ void k_galerkin_ap(GridDesc gf, const ColourInfo *cif, GridDesc gc, TransDesc td, int CW,
                              const int *__restrict__ cwin, const int *__restrict__ ipool,
                              const double *__restrict__ wpool, const double *__restrict__ coef_f, double *B,
                              int ncol) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= gf.nrows) return;
  // find colour of colour-major row r (linear scan over colours; setup only)
  int c = 0;
  while (c + 1 < ncol && cif[gf.col_off + c + 1].start <= r) ++c;
  const ColourInfo ci = cif[gf.col_off + c];
  int i[3];
  decode_colour_row(ci, r - ci.start, P + 1, i);
  int cw[3] = {0, 0, 0};
  for (int d = 0; d < D; ++d) cw[d] = cwin[d * 4096 + i[d]];
  const int CWD = (D == 3) ? CW * CW * CW : CW * CW;
  double *Bi = B + (long long)r * CWD;
  for (int t = 0; t < CWD; ++t) Bi[t] = 0.0;
  const int W = td.W;
  int o = 0;
  for (int o2 = (D == 3 ? -P : 0); o2 <= (D == 3 ? P : 0); ++o2)
    for (int o1 = -P; o1 <= P; ++o1)
      for (int o0 = -P; o0 <= P; ++o0, ++o) {
        int j[3] = {i[0] + o0, i[1] + o1, i[2] + o2};
        bool in = true;
        for (int d = 0; d < D; ++d) in &= (j[d] >= gf.lo[d] && j[d] < gf.hi[d]);
        if (!in) continue;
        double a = coef_f[gf.coef_off + (long long)o * gf.ld + r];
        if (a == 0.0) continue;
        // coarse contributors of fine j: c(j_d) + s_d, weights pw
        int cj[3];
        const double *pw[3];
        for (int d = 0; d < D; ++d) {
          cj[d] = ipool[td.pf_off[d] + j[d]];
          pw[d] = wpool + td.pw_off[d] + (long long)j[d] * W;
        }
        for (int s2 = 0; s2 < (D == 3 ? W : 1); ++s2) {
          double w2 = (D == 3) ? pw[2][s2] : 1.0;
          if (w2 == 0.0) continue;
          int b2 = (D == 3) ? cj[2] + s2 : 0;
          if (D == 3 && (b2 < gc.lo[2] || b2 >= gc.hi[2])) continue;
          int t2 = (D == 3) ? b2 - cw[2] : 0;
          for (int s1 = 0; s1 < W; ++s1) {
            double w12 = w2 * pw[1][s1];
            if (w12 == 0.0) continue;
            int b1 = cj[1] + s1;
            if (b1 < gc.lo[1] || b1 >= gc.hi[1]) continue;
            int t1 = b1 - cw[1];
            for (int s0 = 0; s0 < W; ++s0) {
              double w = w12 * pw[0][s0];
              if (w == 0.0) continue;
              int b0 = cj[0] + s0;
              if (b0 < gc.lo[0] || b0 >= gc.hi[0]) continue;
              int t0 = b0 - cw[0];
              Bi[t0 + CW * (t1 + CW * t2)] += a * w;
            }
          }
        }
      }
}

// stage 2: A_c[a, a+oc] = sum_{i in supp(a)} P[i,a] B[i][a+oc-cw(i)]
template <int D, int P>
__global__ void k_galerkin_ptb(GridDesc gf, const ColourInfo *cif, GridDesc gc, const ColourInfo *cic, TransDesc td,
                               int CW, const int *__restrict__ cwin, const int *__restrict__ ipool,
                               const double *__restrict__ wpool, const double *__restrict__ B, double *coef_c,
                               int ncol) {
  constexpr int S = St<D, P>::S;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)gc.nrows * S) return;
  const int r = (int)(tid / S);
  const int o = (int)(tid % S);
  int c = 0;
  while (c + 1 < ncol && cic[gc.col_off + c + 1].start <= r) ++c;
  const ColourInfo ci = cic[gc.col_off + c];
  int a[3];
  decode_colour_row(ci, r - ci.start, P + 1, a);
  constexpr int W1 = 2 * P + 1;
  int oc[3] = {o % W1 - P, (o / W1) % W1 - P, (D == 3) ? o / (W1 * W1) - P : 0};
  int bb[3] = {a[0] + oc[0], a[1] + oc[1], a[2] + oc[2]};
  double val = 0.0;
  bool inb = true;
  for (int d = 0; d < D; ++d) inb &= (bb[d] >= gc.lo[d] && bb[d] < gc.hi[d]);
  if (inb) {
    constexpr int NW = P + 2;
    int f[3];
    const double *w[3];
    for (int d = 0; d < D; ++d) {
      f[d] = ipool[td.rc_off[d] + a[d]];
      w[d] = wpool + td.rw_off[d] + (long long)a[d] * NW;
    }
    for (int t2 = 0; t2 < (D == 3 ? NW : 1); ++t2) {
      double w2 = (D == 3) ? w[2][t2] : 1.0;
      if (w2 == 0.0) continue;
      int i2 = (D == 3) ? f[2] + t2 : 0;
      if (D == 3 && (i2 < gf.lo[2] || i2 >= gf.hi[2])) continue;
      for (int t1 = 0; t1 < NW; ++t1) {
        double w12 = w2 * w[1][t1];
        if (w12 == 0.0) continue;
        int i1 = f[1] + t1;
        if (i1 < gf.lo[1] || i1 >= gf.hi[1]) continue;
        for (int t0 = 0; t0 < NW; ++t0) {
          double ww = w12 * w[0][t0];
          if (ww == 0.0) continue;
          int i0 = f[0] + t0;
          if (i0 < gf.lo[0] || i0 >= gf.hi[0]) continue;
          // fine row index (colour-major) of i
          int ii[3] = {i0, i1, i2};
          int col = 0, pw = 1;
          int jj[3];
          for (int d = 0; d < D; ++d) { col += (ii[d] % (P + 1)) * pw; pw *= (P + 1); }
          const ColourInfo cf = cif[gf.col_off + col];
          for (int d = 0; d < 3; ++d) jj[d] = (d < D) ? (ii[d] - cf.first[d]) / (P + 1) : 0;
          int rf = cf.start + jj[0] + cf.n[0] * (jj[1] + cf.n[1] * jj[2]);
          int t[3] = {0, 0, 0};
          bool ok = true;
          for (int d = 0; d < D; ++d) {
            t[d] = bb[d] - cwin[d * 4096 + ii[d]];
            ok &= (t[d] >= 0 && t[d] < CW);
          }
          if (!ok) continue;
          const int CWD = (D == 3) ? CW * CW * CW : CW * CW;
          val = fma(ww, B[(long long)rf * CWD + t[0] + CW * (t[1] + CW * t[2])], val);
        }
      }
    }
  }
  coef_c[gc.coef_off + (long long)o * gc.ld + r] = val;
}

// dense active-box matrix (lexicographic active order) of a grid from its stencil
template <int D, int P>
__global__ void k_dense_from_stencil(const GridDesc *g_, const ColourInfo *ci_, const double *coef, double *dense,
                                     const long long *dense_off, int ncol) {
  const GridDesc &g = g_[blockIdx.y];
  constexpr int S = St<D, P>::S;
  constexpr int W1 = 2 * P + 1;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)g.nrows * S) return;
  const int a = (int)(tid / S);        // lexicographic active index
  const int o = (int)(tid % S);
  int i[3];
  decode_point(g, a, i);
  int col = 0, pw = 1;
  for (int d = 0; d < D; ++d) { col += (i[d] % (P + 1)) * pw; pw *= (P + 1); }
  const ColourInfo cf = ci_[g.col_off + col];
  int jj[3];
  for (int d = 0; d < 3; ++d) jj[d] = (d < D) ? (i[d] - cf.first[d]) / (P + 1) : 0;
  const int r = cf.start + jj[0] + cf.n[0] * (jj[1] + cf.n[1] * jj[2]);
  int oc[3] = {o % W1 - P, (o / W1) % W1 - P, (D == 3) ? o / (W1 * W1) - P : 0};
  int b[3] = {i[0] + oc[0], i[1] + oc[1], i[2] + oc[2]};
  for (int d = 0; d < D; ++d)
    if (b[d] < g.lo[d] || b[d] >= g.hi[d]) return;
  int n0 = g.hi[0] - g.lo[0], n1 = g.hi[1] - g.lo[1];
  int bcol = (b[0] - g.lo[0]) + n0 * ((b[1] - g.lo[1]) + n1 * (D == 3 ? b[2] - g.lo[2] : 0));
  dense[dense_off[blockIdx.y] + (long long)a * g.nrows + bcol] = coef[g.coef_off + (long long)o * g.ld + r];
}


// SPD inverse of one dense matrix per block: Cholesky into scratch, then A^{-1} = L^{-T} L^{-1}
__global__ void k_spd_inverse2(double *dense, const long long *dense_off, const int *n_, double *scratch,
                               const long long *scratch_off, int *fail) {
  double *A = dense + dense_off[blockIdx.x];
  double *Lm = scratch + scratch_off[blockIdx.x];      // n*n: L (lower), then Linv
  const int n = n_[blockIdx.x];
  for (long long t = threadIdx.x; t < (long long)n * n; t += blockDim.x) Lm[t] = A[t];
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double s = Lm[(long long)j * n + j];
      for (int k = 0; k < j; ++k) s -= Lm[(long long)j * n + k] * Lm[(long long)j * n + k];
      if (!(s > 0.0)) { atomicExch(fail, 1); s = 1.0; }
      Lm[(long long)j * n + j] = sqrt(s);
    }
    __syncthreads();
    const double djj = Lm[(long long)j * n + j];
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double s = Lm[(long long)i * n + j];
      for (int k = 0; k < j; ++k) s -= Lm[(long long)i * n + k] * Lm[(long long)j * n + k];
      Lm[(long long)i * n + j] = s / djj;
    }
    __syncthreads();
  }
  // A^{-1} = L^{-T} L^{-1}: column c of A^{-1} = L^{-T} (L^{-1} e_c): forward then backward solve
  // one thread per column c, result written to A (column c), using A's column as work vector
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    // forward: y = L^{-1} e_c  (y_i = 0 for i < c)
    for (int i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      if (i > c)
        for (int k = c; k < i; ++k) s -= Lm[(long long)i * n + k] * A[(long long)k * n + c];
      A[(long long)i * n + c] = (i < c) ? 0.0 : s / Lm[(long long)i * n + i];
    }
    // backward: z = L^{-T} y
    for (int i = n - 1; i >= 0; --i) {
      double s = A[(long long)i * n + c];
      for (int k = i + 1; k < n; ++k) s -= Lm[(long long)k * n + i] * A[(long long)k * n + c];
      A[(long long)i * n + c] = s / Lm[(long long)i * n + i];
    }
  }
}
}  // namespace

// ------------------------------------------------------------------------------------------
#define DISPATCH_DP(dim, p, KERNEL_CALL)                                         \
  do {                                                                           \
    if (dim == 2) {                                                              \
      switch (p) {                                                               \
        case 1: { constexpr int D = 2, P = 1; KERNEL_CALL; } break;              \
        case 2: { constexpr int D = 2, P = 2; KERNEL_CALL; } break;              \
        case 3: { constexpr int D = 2, P = 3; KERNEL_CALL; } break;              \
        case 4: { constexpr int D = 2, P = 4; KERNEL_CALL; } break;              \
      }                                                                          \
    } else {                                                                     \
      switch (p) {                                                               \
        case 1: { constexpr int D = 3, P = 1; KERNEL_CALL; } break;              \
        case 2: { constexpr int D = 3, P = 2; KERNEL_CALL; } break;              \
        case 3: { constexpr int D = 3, P = 3; KERNEL_CALL; } break;              \
        case 4: { constexpr int D = 3, P = 4; KERNEL_CALL; } break;              \
      }                                                                          \
    }                                                                            \
  } while (0)

void launch_sgs_phase(int dim, int p, const LevelView &lv, const BlockEntry *blocks, int nblocks, int nthr,
                      double *x, const double *b, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (k_sgs<D, P><<<nblocks, nthr, 0, s>>>(lv, blocks, x, b)));
}

void launch_residual(int dim, int p, const LevelView &lv, const BlockEntry *blocks, int nblocks, int nthr,
                     const double *x, const double *x2, const double *b, double *y, double scale,
                     bool use_mass, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (k_residual<D, P><<<nblocks, nthr, 0, s>>>(lv, blocks, x, x2, b, y, scale, use_mass ? 1 : 0)));
}

void launch_restrict(int dim, int p, const GridDesc *gc, const GridDesc *gf, const TransDesc *td,
                     const ProbDesc *pc, const ProbDesc *pf, const int *ipool, const double *wpool,
                     const BlockEntry *blocks, int nblocks, int nthr, const double *rf, double *bc, double *xc,
                     cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (k_restrict<D, P><<<nblocks, nthr, 0, s>>>(gc, gf, td, pc, pf, ipool, wpool, blocks, rf, bc, xc)));
}

void launch_prolong(int dim, int p, const GridDesc *gc, const GridDesc *gf, const TransDesc *td,
                    const ProbDesc *pc, const ProbDesc *pf, const int *ipool, const double *wpool,
                    const BlockEntry *blocks, int nblocks, int nthr, const double *xc, double *xf,
                    cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (k_prolong<D, P><<<nblocks, nthr, 0, s>>>(gc, gf, td, pc, pf, ipool, wpool, blocks, xc, xf)));
}

void launch_coarse_solve(const GridDesc *g, const ProbDesc *pr, const long long *inv_off, const double *inv,
                         int nprob, int dim, int p, const double *b, double *x, int max_rows, cudaStream_t s) {
  if (nprob <= 0) return;
  size_t smem = (size_t)std::max(1, max_rows) * sizeof(double);
  DISPATCH_DP(dim, p, ({
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_coarse<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_coarse<D, P><<<nprob, 256, smem, s>>>(g, pr, inv_off, inv, b, x);
  }));
}

void launch_galerkin_stages(int dim, int p, const GridDesc &gf, const ColourInfo *cif, const GridDesc &gc,
                            const ColourInfo *cic, const TransDesc &td, int CW, const int *cwin, const int *ipool,
                            const double *wpool, const double *coef_f, double *coef_c, double *B, int ncol,
                            cudaStream_t s) {
  int nthr = 128;
  int nb1 = (gf.nrows + nthr - 1) / nthr;
  int S = 1;
  for (int d = 0; d < dim; ++d) S *= (2 * p + 1);
  long long n2 = (long long)gc.nrows * S;
  int nb2 = (int)((n2 + nthr - 1) / nthr);
  DISPATCH_DP(dim, p, (k_galerkin_ap<D, P><<<nb1, nthr, 0, s>>>(gf, cif, gc, td, CW, cwin, ipool, wpool, coef_f, B, ncol)));
  DISPATCH_DP(dim, p, (k_galerkin_ptb<D, P><<<nb2, nthr, 0, s>>>(gf, cif, gc, cic, td, CW, cwin, ipool, wpool, B, coef_c, ncol)));
}

void launch_dense_from_stencil(int dim, int p, const GridDesc *g, const ColourInfo *ci, const double *coef,
                               int ngrid, double *dense, const long long *dense_off, cudaStream_t s, int max_rows) {
  int S = 1;
  for (int d = 0; d < dim; ++d) S *= (2 * p + 1);
  long long n = (long long)max_rows * S;
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)ngrid);
  int ncol = 1;
  for (int d = 0; d < dim; ++d) ncol *= (p + 1);
  DISPATCH_DP(dim, p, (k_dense_from_stencil<D, P><<<grid, 128, 0, s>>>(g, ci, coef, dense, dense_off, ncol)));
}

void launch_spd_inverse2(double *dense, const long long *dense_off, const int *n, int ngrid, double *scratch,
                         const long long *scratch_off, int *fail, cudaStream_t s) {
  if (ngrid <= 0) return;
  k_spd_inverse2<<<ngrid, 256, 0, s>>>(dense, dense_off, n, scratch, scratch_off, fail);
}
