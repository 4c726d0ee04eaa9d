// layout.cuh -- HBM layout of level vectors and stencil coefficients (host + device).
//
// Vectors: compact "sub-lattice boxes".  The full lattice of a grid is split into its (p+1)^d
// colour sub-lattices i_d = c_d + (p+1) j_d (R6 colours); every sub-lattice is stored as a
// box of ns_d = ceil(M_d/(p+1)) points per direction (no halo), sub-lattices one after the
// other.  Consecutive rows of one colour are then consecutive in memory, and so are their
// neighbours a+o for every fixed offset o: a colour phase reads x with unit stride for each
// of its (2p+1)^d offsets.  A neighbour a+o outside the lattice has a ZERO (padded)
// coefficient (R24); its computed address wraps into an adjacent sub-lattice row, another
// colour's box, the next patch or the pool's zero guard band, all finite values, so the
// product is an exact zero and no bounds check is needed.  Entries of the box that are not
// active lattice points are kept zero (Dirichlet elimination, dummy slots).  Without halos the
// box is ~1.1x the lattice (C5 fine: 46,656 vs 42,875 doubles), so every level vector of all
// patches stays L2-resident across the colour phases (C5: 96 MB of 126 MB).
//
// Coefficients: padded full stencil rows ((2p+1)^d, R24) of the ACTIVE rows in colour-major
// order, addressed coef[coef_off + (o / tg) * (ld * tg) + r * tg + (o % tg)]:
//   tg = -S (bandwidth-bound levels, one thread per row, default): row tiles of 32,
//          coef[coef_off + (r / 32) * 32 S + o * 32 + r % 32]: a warp reads 32 consecutive rows of
//          one offset (256 B), and its successive offsets are ADJACENT 256-B runs, so a warp walks
//          one contiguous S * 256-B block (DRAM page locality; +4 % on the finest phase measured);
//   tg = 1 (IETI_TILE=0, and the opt-in split / TMA big-level kernels): offset-major, a warp
//          reads 32 consecutive rows of one offset, successive offsets ld * 8 B apart;
//   tg = S (small, latency-bound levels, 4 threads per row): row-major, the 4 threads of a row
//          take interleaved offsets and read consecutive coefficients of the row.
#pragma once
#include "internal.h"

#ifdef __CUDACC__
#define IETI_HD __host__ __device__ __forceinline__
#else
#define IETI_HD inline
#endif

// position of full-lattice index i (all i_d >= 0) in the grid's sub-lattice box
IETI_HD long long sl_pos(const GridDesc &g, int p, int dim, const int *i) {
  const int P1 = p + 1;
  int c = 0, pw = 1;
  int j[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) {
    c += (i[d] % P1) * pw;
    pw *= P1;
    j[d] = i[d] / P1;
  }
  long long z = (dim == 3) ? j[2] : 0;
  return (long long)c * g.sb + j[0] + (long long)g.ns[0] * (j[1] + (long long)g.ns[1] * z);
}

// sl_pos is separable: sl_pos(i) = sum_d sl_term(d, i_d)
IETI_HD long long sl_term(const GridDesc &g, int p, int d, int id) {
  const int P1 = p + 1;
  long long cw = g.sb, st = 1;
  for (int e = 0; e < d; ++e) { cw *= P1; st *= g.ns[e]; }
  return (long long)(id % P1) * cw + (long long)(id / P1) * st;
}

// box offset of the neighbour a+o of any point a of colour `colour` (o = flattened offset)
// (exact for neighbours inside the lattice; otherwise a finite wrap-around read, see above)
IETI_HD int sl_delta(const GridDesc &g, int p, int dim, int colour, int o) {
  const int P1 = p + 1, W1 = 2 * p + 1;
  int cc = colour, oo = o, dc = 0, pw = 1, sh[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) {
    int cd = cc % P1;
    cc /= P1;
    int od = oo % W1 - p;
    oo /= W1;
    int s = cd + od;                          // in [-p, 2p]
    int shd = (s < 0) ? -1 : (s >= P1 ? 1 : 0);
    int cn = s - shd * P1;
    dc += (cn - cd) * pw;
    pw *= P1;
    sh[d] = shd;
  }
  return dc * g.sb + sh[0] + g.ns[0] * (sh[1] + g.ns[1] * sh[2]);
}

IETI_HD long long cidx(const GridDesc &g, int o, long long r) {
  const int tg = g.tg;
  if (tg < 0)   // row tiles (bandwidth-bound levels): [r / 32][o][r % 32], S = -tg offsets per row
    return g.coef_off + (r >> 5) * (32LL * -tg) + (long long)o * 32 + (r & 31);
  return g.coef_off + (long long)(o / tg) * ((long long)g.ld * tg) + r * tg + (o % tg);
}

// colour-major row index of an active lattice point (host + device)
IETI_HD int cm_row(const GridDesc &g, const ColourInfo *ci_grid, int p, int dim, const int *i) {
  const int P1 = p + 1;
  int col = 0, pw = 1;
  for (int d = 0; d < dim; ++d) { col += (i[d] % P1) * pw; pw *= P1; }
  const ColourInfo &ci = ci_grid[col];
  int j[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) j[d] = (i[d] - ci.first[d]) / P1;
  return ci.start + j[0] + ci.n[0] * (j[1] + ci.n[1] * j[2]);
}

#ifdef __CUDACC__
// stencil shape of degree P in D dimensions: W1 = 2P+1 per direction, S = W1^D offsets, CENTER =
// the flattened zero offset (shared by the stencil kernels of kernels_mg.cu and kernels_sweep.cu)
template <int D, int P>
struct St {
  static constexpr int W1 = 2 * P + 1;
  static constexpr int S = (D == 3) ? W1 * W1 * W1 : W1 * W1;
  static constexpr int CENTER = (D == 3) ? P + W1 * (P + W1 * P) : P + W1 * P;
};

template <int D, int P>
__device__ __forceinline__ long long row_pos(const GridDesc &g, const ColourInfo &ci, int colour, int j) {
  // sub-lattice box position of row j of colour `colour` (rows of a colour are the sub-lattice
  // points first_d + (p+1) jj_d, i.e. sub-lattice index first_d/(p+1) + jj_d)
  constexpr int P1 = P + 1;
  int j0 = j % ci.n[0];
  int t = j / ci.n[0];
  int j1 = t % ci.n[1];
  int j2 = t / ci.n[1];
  int q0 = ci.first[0] / P1 + j0;
  int q1 = ci.first[1] / P1 + j1;
  int q2 = (D == 3) ? ci.first[2] / P1 + j2 : 0;
  return (long long)colour * g.sb + q0 + (long long)g.ns[0] * (q1 + (long long)g.ns[1] * q2);
}

#endif
