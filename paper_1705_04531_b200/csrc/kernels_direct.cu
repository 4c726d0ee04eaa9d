// kernels_direct.cu -- batched banded Cholesky: the direct local solvers of the paper's D-D and MG-D
// variants ("direct solvers everywhere"; the paper uses PARDISO, A34 out of scope).
//
// Per patch the local matrix (K_II for the Dirichlet problems of M_sD; K -- with one
// dof pinned on floating patches, K^+ -- for the Neumann problems, whose right-hand sides are the
// consistent P^T r, App. A.1) is stored as a lower band in lexicographic dof order (half bandwidth
// bw = p (M_1 + ... ) + p: every coupling |i_d - j_d| <= p lies within it):
//     B[i][k] = A[i][i - bw + k],  k = 0..bw  (k = bw the diagonal; entries left of column 0 are 0)
// k_band_chol factors A = L L^T in place (right-looking, column by column, one block per patch);
// k_band_tr writes U[i][k] = L[i + k][i] so that the backward substitution reads rows.  The
// triangular solves run one warp per patch (each row: a bw-term dot product with the last bw
// solution values, kept in shared memory).  3D bands grow like p M^2: C5 patches would need
// 1.3 GB each (the paper's OoM rows) and are refused at setup.
#include "internal.h"

#include <algorithm>
#include <cmath>

namespace {

// in-place lower-band Cholesky of problem blockIdx.x; info[prob] = 0 ok, j+1 if pivot j <= 0
__global__ void k_band_chol(const BandDesc *__restrict__ bd, double *band, int *info) {
  const BandDesc D = bd[blockIdx.x];
  const int n = D.n, bw = D.bw, ld = bw + 1;
  double *B = band + D.off;
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double a = B[(long long)j * ld + bw];
      if (!(a > 0.0) && !bad) bad = j + 1;
      piv = sqrt(fabs(a) > 0 ? fabs(a) : 1.0);
      B[(long long)j * ld + bw] = piv;
    }
    __syncthreads();
    const int m = min(bw, n - 1 - j);             // rows j+1 .. j+m below the pivot
    for (int t = threadIdx.x; t < m; t += blockDim.x) {
      const int i = j + 1 + t;
      B[(long long)i * ld + (j - i + bw)] /= piv;   // L[i][j]
    }
    __syncthreads();
    // trailing update A[i][k] -= L[i][j] L[k][j], j < k <= i <= j + m
    const int tot = m * (m + 1) / 2;
    for (int t = threadIdx.x; t < tot; t += blockDim.x) {
      // t -> (a, b) with 0 <= b <= a < m : a = floor((sqrt(8t+1)-1)/2)
      int a = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((a + 1) * (a + 2) / 2 <= t) ++a;
      while (a * (a + 1) / 2 > t) --a;
      const int b = t - a * (a + 1) / 2;
      const int i = j + 1 + a, k = j + 1 + b;
      const double lij = B[(long long)i * ld + (j - i + bw)];
      const double lkj = B[(long long)k * ld + (j - k + bw)];
      B[(long long)i * ld + (k - i + bw)] -= lij * lkj;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) info[blockIdx.x] = bad;
}

// U[i][k] = L[i + k][i]
__global__ void k_band_tr(const BandDesc *__restrict__ bd, const double *__restrict__ band, double *up) {
  const BandDesc D = bd[blockIdx.y];
  const int ld = D.bw + 1;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < (long long)D.n * ld;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / ld), k = (int)(e % ld);
    const int r = i + k;
    up[D.off + e] = (r < D.n) ? band[D.off + (long long)r * ld + (D.bw - k)] : 0.0;
  }
}

// forward + backward substitution, one warp per problem; v (length n) in / out
__global__ void k_band_solve(const BandDesc *__restrict__ bd, const double *__restrict__ band,
                             const double *__restrict__ up, const long long *__restrict__ voff, double *v) {
  extern __shared__ double win[];                    // ring of the last bw + 1 solution values
  const BandDesc D = bd[blockIdx.x];
  const int n = D.n, bw = D.bw, ld = bw + 1, lane = threadIdx.x;
  const double *L = band + D.off;
  const double *U = up + D.off;
  double *x = v + voff[blockIdx.x];
  const int R = ld;                                  // ring length
  for (int t = lane; t < R; t += 32) win[t] = 0.0;
  __syncwarp();
  // forward: y_i = (b_i - sum_{k<bw} L[i][k] y_{i-bw+k}) / L[i][bw]
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    const double *row = L + (long long)i * ld;
    for (int k = lane; k < bw; k += 32) {
      const int jj = i - bw + k;
      if (jj >= 0) s = fma(row[k], win[jj % R], s);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const double y = (x[i] - s) / row[bw];
      win[i % R] = y;
      x[i] = y;
    }
    __syncwarp();
  }
  for (int t = lane; t < R; t += 32) win[t] = 0.0;
  __syncwarp();
  // backward: x_i = (y_i - sum_{k=1..bw} U[i][k] x_{i+k}) / U[i][0]
  for (int i = n - 1; i >= 0; --i) {
    double s = 0.0;
    const double *row = U + (long long)i * ld;
    for (int k = 1 + lane; k <= bw; k += 32) {
      const int jj = i + k;
      if (jj < n) s = fma(row[k], win[jj % R], s);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const double xi = (x[i] - s) / row[0];
      win[i % R] = xi;
      x[i] = xi;
    }
    __syncwarp();
  }
}

__global__ void k_gather_pos(long long n, const long long *__restrict__ pos, const double *__restrict__ box, double *v) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    v[t] = box[pos[t]];
}
__global__ void k_scatter_pos(long long n, const long long *__restrict__ pos, const double *__restrict__ v, double *box) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    box[pos[t]] = v[t];
}

}  // namespace

void ik_band_factor(int nprob, const BandDesc *bd, double *band, double *up, long long max_len, int *info,
                    cudaStream_t s) {
  if (nprob <= 0) return;
  k_band_chol<<<nprob, 1024, 0, s>>>(bd, band, info);
  const unsigned gx = (unsigned)std::min<long long>(4096, (max_len + 255) / 256);
  k_band_tr<<<dim3(std::max(1u, gx), (unsigned)nprob), 256, 0, s>>>(bd, band, up);
}

void ik_band_solve(int nprob, int max_bw, const BandDesc *bd, const double *band, const double *up,
                   const long long *voff, double *v, cudaStream_t s) {
  if (nprob <= 0) return;
  const size_t smem = (size_t)(max_bw + 1) * sizeof(double);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(k_band_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = smem;
  }
  k_band_solve<<<nprob, 32, smem, s>>>(bd, band, up, voff, v);
}

void ik_gather_pos(long long n, const long long *pos, const double *box, double *v, cudaStream_t s) {
  if (n > 0) k_gather_pos<<<(unsigned)std::min<long long>(4096, (n + 255) / 256), 256, 0, s>>>(n, pos, box, v);
}
void ik_scatter_pos(long long n, const long long *pos, const double *v, double *box, cudaStream_t s) {
  if (n > 0) k_scatter_pos<<<(unsigned)std::min<long long>(4096, (n + 255) / 256), 256, 0, s>>>(n, pos, v, box);
}
