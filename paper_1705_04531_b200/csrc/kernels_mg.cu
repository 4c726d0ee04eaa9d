// kernels_mg.cu -- batched per-patch geometric multigrid kernels for sm_100a (fp64).
//
//  * k_stencil<MODE=0>  one colour phase of the (p+1)^d-colour Gauss-Seidel smoother (R5, R6):
//                x_a += (b_a - sum_o A[a,o] x[a+o]) / A[a,a] for every row a of colour c of every
//                problem in the batch.  Rows of one colour are decoupled (|i_d - j_d| >= p+1 in
//                some d => A_ij = 0), so the phase is one launch.
//  * k_stencil<MODE=1>  r = b - A x  ;  <MODE=2>  y = s A x
//  * k_rowlist   y = A x over an explicit row list (Gamma rows / interior band rows of M_sD)
//  * k_restrict  b_c = P^T r_f, x_c = 0   (P = P_1 (x) ... (x) P_d from knot insertion, R8)
//  * k_prolong   x_f += P x_c
//  * k_coarse    x = A_0^{-1} b (explicit inverse of the coarsest Galerkin matrix, R9)
//  * Galerkin    A_{l-1} = P^T A_l P in stencil form, two stages (setup only)
//
// Stencil kernels: tg threads per row (tg = 1 on fine levels, 4 on small coarse levels),
// coefficient loads batched 8 at a time for memory-level parallelism, the per-colour neighbour
// offsets of the sub-lattice layout in shared memory.  Each coefficient stream and each x
// gather of a warp is a run of consecutive addresses (layout.cuh).
#include "layout.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef IETI_KB1
#define IETI_KB1 8    // min resident blocks of the one-thread-per-row stencil kernels (finest levels); 10 (48 regs)
                      // measured slower: C5 0.714 vs 0.788 of peak, C3 332 vs 375 it/s (tools/gpu/ab_kb.sh)
#endif

// Stencil modes (one launch = one colour phase, or all rows for MODE 1/2):
//  0  SGS phase        x_a += delta, delta = (b_a - sum_o A[a,o] x[a+o]) / A_aa; dx_a = delta if dx
//  1  residual         y_a = b_a - sum_o A[a,o] x[a+o]
//  2  apply            y_a = scale * sum_o A[a,o] x[a+o]
//  4  SGS phase from x = 0 (first forward sweep of a level visit): only neighbours of LOWER
//     colours are nonzero, so only their coefficients are streamed:
//                      x_a = (b_a - sum_{col(a+o) < col(a)} A[a,o] x[a+o]) / A_aa
//  5  residual right after a forward sweep: row a's residual was zeroed by its own update and
//     changed afterwards only by the updates dx of HIGHER colours, so
//                      y_a = - sum_{col(a+o) > col(a)} A[a,o] dx[a+o]
//     (mathematically b - A x; streams half the coefficients).  dx = x after a sweep from 0.
//  7  backward SGS phase that also records U_a = sum_{col(a+o) > col(a)} A[a,o] x[a+o] (into y):
//     the higher colours are final when colour col(a) runs backwards, and x is not touched again
//     before the next cycle's forward sweep reaches row a
//  6  forward SGS phase of the next cycle: higher-colour neighbours still hold the values U_a
//     was computed from, so only LOWER-colour coefficients are streamed:
//                      x_a += delta, delta = (b_a - sum_{lower} A x - A_aa x_a - U_a) / A_aa
//     (same arithmetic as mode 0 up to summation order; dx_a = delta if dx)
// Offsets are processed from a per-block list (offset, box delta) in shared memory; TPR threads
// share a row, each taking a contiguous chunk of the list, so for a fixed list entry the lanes
// of a warp read consecutive rows of the offset-major coefficient table (coalesced).
// list of (offset, box delta) pairs for a colour phase / residual of grid g (GridDesc::ent_off)
template <int D, int P>
__device__ __forceinline__ const int2 *entry_list(const LevelView &lv, const GridDesc &g, int colour, int mode,
                                                  const short *__restrict__ nlow, int &n) {
  constexpr int S = St<D, P>::S;
  const int2 *E = lv.ent + g.ent_off + (long long)colour * (2 * S);
  if (mode == 4) {
    n = nlow[colour];
    return E + S;
  }
  if (mode == 5) {
    const int nl = nlow[colour];
    n = S - 1 - nl;
    return E + S + nl;
  }
  n = S;
  return E;
}

// one colour-block entry of a stencil launch (the body of k_stencil, shared with the persistent
// sweep k_sweep).  PDL: programmatic-dependent-launch wait between the static prologue and the
// first read of x (per-phase launches only).  XCG: read x through L2 only (ld.global.cg) -- in the
// persistent sweep the other SMs' updates of earlier phases are not visible to a stale L1 line.
template <int D, int P, int TPR, int MODE, int NB, bool PDL, bool XCG>
__device__ __forceinline__ void stencil_entry(const LevelView &lv, const BlockEntry be, const ProbDesc &pr,
                                              const GridDesc &g, double *x, const double *__restrict__ b,
                                              double *y, double scale, const double *__restrict__ dsrc, double *dx,
                                              const short *__restrict__ olist, const short *__restrict__ nlow,
                                              int2 *E) {
  constexpr int S = St<D, P>::S;
  constexpr int CEN = St<D, P>::CENTER;
  // (offset, box delta) list of this colour, computed in shared memory (cheaper on the critical
  // path than copying the precomputed table: measured on B200)
  int n, nsplit = 0;
  if (MODE >= 4) {
    const int nl = nlow[be.colour];
    n = (MODE == 4 || MODE == 6) ? nl : (MODE == 5 ? S - 1 - nl : S - 1);
    nsplit = nl;                                   // MODE 7: entries [0, nl) lower, [nl, S-1) upper
    const short *ol = olist + (long long)be.colour * S + ((MODE == 5) ? nl : 0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int o = ol[i];
      E[i] = make_int2(o, sl_delta(g, P, D, be.colour, o));
    }
  } else {
    n = S;
    for (int o = threadIdx.x; o < S; o += blockDim.x) E[o] = make_int2(o, sl_delta(g, P, D, be.colour, o));
  }
  __syncthreads();
  const int rl = threadIdx.x / TPR;
  const int gi = threadIdx.x % TPR;
  const bool valid = rl < be.nrow;
  double acc = 0.0, accu = 0.0, diag = 1.0, bval = 0.0;
  long long pos = 0;
  int r = 0;
  if (valid) {
    const ColourInfo ci = lv.cinfo[g.col_off + be.colour];
    const int j = be.row0 + rl;
    pos = pr.vec_off + row_pos<D, P>(g, ci, be.colour, j);
    r = ci.start + j;
    // the diagonal (static) is fetched before the dependency wait, b right after it: neither
    // load sits on the critical path behind the accumulation
    if ((MODE == 0 || MODE == 4 || MODE >= 6) && gi == 0) diag = __ldg(lv.coef + cidx(g, CEN, r));
  }
  // programmatic dependent launch: the prologue above reads only static data; let the next
  // phase's grid launch now and wait for the previous grid's results only here
  if (PDL) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (valid) {
    if ((MODE == 0 || MODE == 4 || MODE == 1 || MODE >= 6) && gi == 0) bval = __ldcs(b + pos);
    // offset-major rows (GridDesc::tg == 1: coef[o][r], a warp reads consecutive rows per
    // offset) or row-major rows (tg == S: coef[r][o]); the list is interleaved over the TPR
    // threads of a row, so every warp-load is a few fully used contiguous runs either way
    const bool omaj = (g.tg == 1), tiled = (g.tg < 0);
    const long long ostr = omaj ? g.ld : (tiled ? 32 : 1);
    const double *c = lv.coef + g.coef_off +
                      (omaj ? (long long)r
                            : tiled ? ((long long)r >> 5) * (32LL * St<D, P>::S) + (r & 31) : (long long)r * St<D, P>::S);
    const double *xb = ((MODE == 5) ? dsrc : x) + pos;
#ifdef IETI_DEBUG_BOUNDS
    // debug builds: every neighbour gather of this row must stay inside the level's vector pool
    // (the sub-lattice layout relies on wrapped reads landing in finite, zero-coefficient data)
    for (int i = gi; i < n; i += TPR) {
      const long long at = pos + E[i].y;
      if (at < 0 || at >= lv.nvec) {
        printf("IETI_DEBUG_BOUNDS: k_stencil mode %d prob %d colour %d row %d reads %lld outside [0, %lld)\n", MODE,
               be.prob, be.colour, be.row0 + rl, at, lv.nvec);
        asm volatile("trap;");
      }
    }
#endif
    // partial sum of list entries [i0, i1) (this thread's interleave), NB loads in flight
    auto range_sum = [&](int i0, int i1) {
      double s0 = 0.0, s1 = 0.0;
      int i = i0 + gi;
      for (; i + (NB - 1) * TPR < i1; i += NB * TPR) {
        double a[NB], v[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int2 e = E[i + u * TPR];
          // natural-order lists (MODE 0/1/2): the coefficient address does not wait for the list
          const int oc = (MODE >= 4) ? e.x : (i + u * TPR);
          // coefficients stream through once per sweep: evict-first keeps the level vectors in L2
          a[u] = __ldcs(c + (long long)oc * ostr);
          v[u] = XCG ? __ldcg(xb + e.y) : xb[e.y];
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          if (u & 1) s1 = fma(a[u], v[u], s1);
          else s0 = fma(a[u], v[u], s0);
        }
      }
      for (; i < i1; i += TPR) {
        const int2 e = E[i];
        const int oc = (MODE >= 4) ? e.x : i;
        s0 = fma(__ldcs(c + (long long)oc * ostr), XCG ? __ldcg(xb + e.y) : xb[e.y], s0);
      }
      return s0 + s1;
    };
    if (MODE == 7) {
      acc = range_sum(0, nsplit);
      accu = range_sum(nsplit, n);
    } else {
      acc = range_sum(0, n);
    }
  }
  if (TPR > 1) {
#pragma unroll
    for (int m = 1; m < TPR; m <<= 1) {
      acc += __shfl_xor_sync(FULL, acc, m);
      if (MODE == 7) accu += __shfl_xor_sync(FULL, accu, m);
    }
  }
  if (valid && gi == 0) {
    if (MODE == 6 || MODE == 7) {
      const double xa = XCG ? __ldcg(x + pos) : x[pos];
      const double u = (MODE == 6) ? __ldcs(y + pos) : accu;
      const double delta = (bval - (acc + diag * xa + u)) / diag;
      x[pos] = xa + delta;
      if (MODE == 7) __stcs(y + pos, accu);
      else if (dx) __stcs(dx + pos, delta);
      return;
    }
    // b is read and dx / y written once per sweep: streaming (evict-first) accesses keep x in L2
    if (MODE == 0 || MODE == 4) {
      const double delta = (bval - acc) / diag;
      if (MODE == 4) {
        x[pos] = delta;
      } else {
        x[pos] = (XCG ? __ldcg(x + pos) : x[pos]) + delta;
        if (dx) __stcs(dx + pos, delta);
      }
    } else if (MODE == 1) {
      __stcs(y + pos, bval - acc);
    } else if (MODE == 5) {
      __stcs(y + pos, -acc);
    } else {
      y[pos] = scale * acc;
    }
  }
}

template <int D, int P, int TPR, int MODE, int NB = 8>
__global__ void __launch_bounds__(128, (NB > 8 ? 5 : (TPR == 1 ? IETI_KB1 : 8))) k_stencil(LevelView lv, const BlockEntry *__restrict__ blocks, double *x,
                                                    const double *__restrict__ b, double *y, double scale,
                                                    const double *__restrict__ dsrc, double *dx,
                                                    const short *__restrict__ olist, const short *__restrict__ nlow,
                                                    int pcol) {
  constexpr int S = St<D, P>::S;
  constexpr int CEN = St<D, P>::CENTER;
  __shared__ int2 E[S];
  const BlockEntry be = blocks[blockIdx.x];
  const ProbDesc pr = lv.probs[be.prob];
  const GridDesc &g = lv.grids[pr.grid];
  if (TPR > 1 && pcol >= 0 && threadIdx.x == 0 && g.tg > 1) {
    // latency-bound small levels (row-major rows): prefetch this block's share of the NEXT colour
    // phase's coefficient block of the same patch into L2 (cp.async.bulk.prefetch), so that
    // phase's load batches hit L2 instead of HBM
    const ColourInfo cc = lv.cinfo[g.col_off + be.colour], cn = lv.cinfo[g.col_off + pcol];
    const long long n = (long long)cc.n[0] * cc.n[1] * cc.n[2], nn = (long long)cn.n[0] * cn.n[1] * cn.n[2];
    if (n > 0 && nn > 0) {
      const long long a0 = be.row0 * nn / n, a1 = (be.row0 + be.nrow) * nn / n;
      long long lo = g.coef_off + (cn.start + a0) * S, hi = g.coef_off + (cn.start + a1) * S;
      lo &= ~1LL;
      hi = (hi + 1) & ~1LL;
      if (hi > lo)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lv.coef + lo), "r"((unsigned)((hi - lo) * 8))
                     : "memory");
    }
  }
  stencil_entry<D, P, TPR, MODE, NB, true, false>(lv, be, pr, g, x, b, y, scale, dsrc, dx, olist, nlow, E);
}

// ---- persistent sweep: all colour phases of one sweep in ONE launch --------------------------
// A sweep is (p+1)^d dependent colour phases (R6).  Launched one kernel per phase, each phase pays
// a launch gap, a ramp-up and a drain (~3-4 us against a 36 us finest phase of C5, most of a small
// level's ~5 us phase).  Here the grid stays resident (cooperative launch: co-residency is checked by
// the driver, never a hang) and the phases are separated by a grid barrier; each block takes the
// colour blocks b, b + gridDim, ... of the current phase (ptab: per phase the first entry and the
// count, in sweep order).  x is read through L2 (ld.global.cg) because earlier phases' updates
// come from other SMs.  Same arithmetic per row as k_stencil (R23).
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned &target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    volatile unsigned *vb = bar;
    while (*vb < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

template <int D, int P, int TPR, int MODE>
__global__ void __launch_bounds__(128, 8) k_sweep(LevelView lv, const BlockEntry *__restrict__ blocks,
                                                  const int2 *__restrict__ ptab, int nphase, unsigned *bar,
                                                  double *x, const double *__restrict__ b, double *y, double *dx,
                                                  const short *__restrict__ olist, const short *__restrict__ nlow) {
  constexpr int S = St<D, P>::S;
  __shared__ int2 E[S];
  unsigned target = 0;
  for (int ph = 0; ph < nphase; ++ph) {
    const int2 pt = ptab[ph];
    for (int e = blockIdx.x; e < pt.y; e += gridDim.x) {
      const BlockEntry be = blocks[pt.x + e];
      const ProbDesc pr = lv.probs[be.prob];
      const GridDesc &g = lv.grids[pr.grid];
      stencil_entry<D, P, TPR, MODE, 8, false, true>(lv, be, pr, g, x, b, y, 1.0, nullptr, dx, olist, nlow, E);
      __syncthreads();                               // E is rebuilt by the next entry
    }
    if (ph + 1 < nphase) grid_sync(bar, target);
  }
}

// ---- split-row variant for the bandwidth-bound big levels (one row per TWO threads) -----------
// A colour phase of the finest level has too few rows (C5: ~80 k per x-group) to keep enough loads
// in flight with one thread per row (21-23 % warps active, DRAM at 50-55 % of peak: the phase is a
// chain of ~43 dependent load batches per thread).  Here every row is shared by two warps: warp pair
// (2q, 2q+1) of a 256-thread block covers the same 32 consecutive rows, warp 2q the first half of
// the row's (offset, delta) list and warp 2q+1 the second half, so every warp-load is still one
// 256-byte run of the offset-major coefficient table, twice as many warps are resident and each
// thread's chain is half as long.  The partial sums meet in shared memory (R23: summation order
// only).  Same modes as k_stencil<.., TPR = 1, ..>.
template <int D, int P, int MODE, int NB = 8>
__global__ void __launch_bounds__(256, (NB > 4 ? 4 : 6)) k_stencil_split(LevelView lv, const BlockEntry *__restrict__ blocks, double *x,
                                                         const double *__restrict__ b, double *y, double scale,
                                                         const double *__restrict__ dsrc, double *dx,
                                                         const short *__restrict__ olist,
                                                         const short *__restrict__ nlow) {
  constexpr int S = St<D, P>::S;
  constexpr int CEN = St<D, P>::CENTER;
  __shared__ int2 E[S];
  __shared__ double part[2][128];
  const BlockEntry be = blocks[blockIdx.x];
  const ProbDesc pr = lv.probs[be.prob];
  const GridDesc &g = lv.grids[pr.grid];
  int n, nsplit = 0;
  if (MODE >= 4) {
    const int nl = nlow[be.colour];
    n = (MODE == 4 || MODE == 6) ? nl : (MODE == 5 ? S - 1 - nl : S - 1);
    nsplit = nl;
    const short *ol = olist + (long long)be.colour * S + ((MODE == 5) ? nl : 0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int o = ol[i];
      E[i] = make_int2(o, sl_delta(g, P, D, be.colour, o));
    }
  } else {
    n = S;
    for (int o = threadIdx.x; o < S; o += blockDim.x) E[o] = make_int2(o, sl_delta(g, P, D, be.colour, o));
  }
  __syncthreads();
  const int half = (threadIdx.x >> 5) & 1;
  const int rl = ((threadIdx.x >> 6) << 5) | (threadIdx.x & 31);
  const bool valid = rl < be.nrow;
  double acc = 0.0, accu = 0.0, diag = 1.0, bval = 0.0;
  long long pos = 0;
  int r = 0;
  if (valid) {
    const ColourInfo ci = lv.cinfo[g.col_off + be.colour];
    const int j = be.row0 + rl;
    pos = pr.vec_off + row_pos<D, P>(g, ci, be.colour, j);
    r = ci.start + j;
    if ((MODE == 0 || MODE == 4 || MODE >= 6) && half == 0) diag = __ldg(lv.coef + cidx(g, CEN, r));
  }
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (valid) {
    if ((MODE == 0 || MODE == 4 || MODE == 1 || MODE >= 6) && half == 0) bval = __ldcs(b + pos);
    const long long ostr = g.ld;                         // offset-major (tg == 1)
    const double *c = lv.coef + g.coef_off + (long long)r;
    const double *xb = ((MODE == 5) ? dsrc : x) + pos;
    auto range_sum = [&](int i0, int i1) {
      double s0 = 0.0, s1 = 0.0;
      int i = i0;
      for (; i + NB - 1 < i1; i += NB) {
        double a[NB], v[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int2 e = E[i + u];
          const int oc = (MODE >= 4) ? e.x : (i + u);
          a[u] = __ldcs(c + (long long)oc * ostr);
          v[u] = xb[e.y];
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          if (u & 1) s1 = fma(a[u], v[u], s1);
          else s0 = fma(a[u], v[u], s0);
        }
      }
      for (; i < i1; ++i) {
        const int2 e = E[i];
        const int oc = (MODE >= 4) ? e.x : i;
        s0 = fma(__ldcs(c + (long long)oc * ostr), xb[e.y], s0);
      }
      return s0 + s1;
    };
    const int mid = n / 2;
    const int lo = half ? mid : 0, hi = half ? n : mid;
    if (MODE == 7) {
      acc = range_sum(lo, min(hi, nsplit) > lo ? min(hi, nsplit) : lo);
      accu = range_sum(max(lo, nsplit), hi > max(lo, nsplit) ? hi : max(lo, nsplit));
    } else {
      acc = range_sum(lo, hi);
    }
  }
  if (half == 1) {
    part[0][rl] = acc;
    part[1][rl] = accu;
  }
  __syncthreads();
  if (!valid || half == 1) return;
  acc += part[0][rl];
  accu += part[1][rl];
  if (MODE == 6 || MODE == 7) {
    const double xa = x[pos];
    const double u = (MODE == 6) ? __ldcs(y + pos) : accu;
    const double delta = (bval - (acc + diag * xa + u)) / diag;
    x[pos] = xa + delta;
    if (MODE == 7) __stcs(y + pos, accu);
    else if (dx) __stcs(dx + pos, delta);
    return;
  }
  if (MODE == 0 || MODE == 4) {
    const double delta = (bval - acc) / diag;
    if (MODE == 4) {
      x[pos] = delta;
    } else {
      x[pos] += delta;
      if (dx) __stcs(dx + pos, delta);
    }
  } else if (MODE == 1) {
    __stcs(y + pos, bval - acc);
  } else if (MODE == 5) {
    __stcs(y + pos, -acc);
  } else {
    y[pos] = scale * acc;
  }
}

// ---- TMA-fed variant for large grids (one thread per row) ------------------------------------
// Same modes and accumulation order as k_stencil<.., TPR = 1, ..> (entries alternate between two
// accumulators).  The coefficient stream of the block's rows -- for every list entry one
// contiguous slab coef[o][r0 .. r0+nrow) -- is fetched by the Tensor Memory Accelerator
// (cp.async.bulk, L2 evict-first) into a ring of TST stages x TPU entries in shared memory,
// completion tracked by one mbarrier per stage; thread 0 refills a stage after the block has
// consumed it.  Coefficient bytes in flight therefore cost no registers; the registers hold the
// x gathers (L2 hits), prefetched one stage ahead.
constexpr int TPU = 8;                 // list entries per stage
constexpr int TST = 4;                 // stages in the ring
constexpr int TSL = 130;               // slab length (doubles): 128 rows + alignment shift, even

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int D, int P, int MODE>
__global__ void __launch_bounds__(128, 6) k_stencil_tma(LevelView lv, const BlockEntry *__restrict__ blocks,
                                                        double *x, const double *__restrict__ b, double *y,
                                                        double scale, const double *__restrict__ dsrc, double *dx,
                                                        const short *__restrict__ olist,
                                                        const short *__restrict__ nlow) {
  constexpr int S = St<D, P>::S;
  constexpr int CEN = St<D, P>::CENTER;
  extern __shared__ __align__(16) double csm[];   // [TST][TPU][TSL]
  __shared__ __align__(8) unsigned long long bar[TST];
  __shared__ int2 ent[S];
  __shared__ int n_sh;
  const BlockEntry be = blocks[blockIdx.x];
  const ProbDesc pr = lv.probs[be.prob];
  const GridDesc &g = lv.grids[pr.grid];
  {
    int ne;
    const int2 *E = entry_list<D, P>(lv, g, be.colour, MODE, nlow, ne);
    for (int i = threadIdx.x; i < ne; i += blockDim.x) ent[i] = __ldg(E + i);
    if (threadIdx.x == 0) n_sh = ne;
  }
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int st = 0; st < TST; ++st) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[st])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int n = n_sh;
  const bool valid = tid < be.nrow;
  const ColourInfo ci = lv.cinfo[g.col_off + be.colour];
  const int r0 = ci.start + be.row0;
  const long long ld = g.ld;
  const long long cbase = g.coef_off + r0;
  const int shift = (int)(cbase & 1);               // 16-byte aligned slabs (ld is even)
  const int slab = (be.nrow + shift + 1) & ~1;       // doubles per slab (multiple of 2 = 16 bytes)
  const int j = be.row0 + (valid ? tid : 0);
  const long long pos = pr.vec_off + row_pos<D, P>(g, ci, be.colour, j);
  const double *xb = ((MODE == 5) ? dsrc : x) + pos;
  const int nst = (n + TPU - 1) / TPU;
  unsigned long long pol = 0;
  if (tid == 0) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int st) {                         // thread 0 only
    if (st >= nst) return;
    const int slot = st % TST;
    const int i0 = st * TPU, cnt = min(TPU, n - i0);
    const unsigned bytes = (unsigned)(cnt * slab * 8);
    const unsigned mb = smem_u32(&bar[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    for (int u = 0; u < cnt; ++u) {
      const double *src = lv.coef + cbase - shift + (long long)ent[i0 + u].x * ld;
      const unsigned dst = smem_u32(csm + (slot * TPU + u) * TSL);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
          ::"r"(dst), "l"(src), "r"(slab * 8), "r"(mb), "l"(pol) : "memory");
    }
  };
  if (tid == 0)
    for (int st = 0; st < TST; ++st) issue(st);
  auto loadx = [&](int st, double *v) {
    const int i0 = st * TPU;
#pragma unroll
    for (int u = 0; u < TPU; ++u) v[u] = (valid && st < nst && i0 + u < n) ? xb[ent[i0 + u].y] : 0.0;
  };
  double vc[TPU], vn[TPU];
  loadx(0, vc);
  double acc = 0.0, acc1 = 0.0;
  for (int st = 0; st < nst; ++st) {
    loadx(st + 1, vn);
    const int slot = st % TST;
    const unsigned mb = smem_u32(&bar[slot]);
    const unsigned parity = (unsigned)((st / TST) & 1);
    unsigned done = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(mb), "r"(parity) : "memory");
    } while (!done);
    const double *cs = csm + slot * TPU * TSL + shift + tid;
    const int i0 = st * TPU;
#pragma unroll
    for (int u = 0; u < TPU; ++u) {
      if (i0 + u < n) {
        const double a = valid ? cs[u * TSL] : 0.0;
        if (u & 1) acc1 = fma(a, vc[u], acc1);
        else acc = fma(a, vc[u], acc);
      }
    }
#pragma unroll
    for (int u = 0; u < TPU; ++u) vc[u] = vn[u];
    __syncthreads();                                 // slot consumed by every thread
    if (tid == 0) issue(st + TST);
  }
  acc += acc1;
  if (!valid) return;
  const int r = r0 + tid;
  if (MODE == 0 || MODE == 4) {
    const double diag = __ldg(lv.coef + g.coef_off + (long long)CEN * g.ld + r);
    const double delta = (b[pos] - acc) / diag;
    if (MODE == 4) {
      x[pos] = delta;
    } else {
      x[pos] += delta;
      if (dx) dx[pos] = delta;
    }
  } else if (MODE == 1) {
    y[pos] = b[pos] - acc;
  } else if (MODE == 5) {
    y[pos] = -acc;
  } else {
    y[pos] = scale * acc;
  }
}

// y = A x over a row list (rows grouped by (patch, colour)); out_mode 0: y[vec_off + out] = -acc
// (band rows, interior box positions), 1: y[out] = acc (compact Gamma index).  Coefficients of the
// list are offset-major [o][row] with leading dimension ld.
template <int D, int P>
__global__ void __launch_bounds__(128, 8) k_rowlist(const GridDesc *__restrict__ grids, const ProbDesc *__restrict__ probs,
                                                    const BlockEntry *__restrict__ blocks, const double *__restrict__ coef,
                                                    long long ld, const int *__restrict__ rpos,
                                                    const int *__restrict__ rout, const double *__restrict__ x,
                                                    const double *__restrict__ x2, double *y, int out_mode) {
  constexpr int S = St<D, P>::S;
  __shared__ int dl[S];
  const BlockEntry be = blocks[blockIdx.x];
  const ProbDesc pr = probs[be.prob];
  const GridDesc &g = grids[pr.grid];
  for (int o = threadIdx.x; o < S; o += blockDim.x) dl[o] = sl_delta(g, P, D, be.colour, o);
  __syncthreads();
  if ((int)threadIdx.x >= be.nrow) return;
  const int row = be.row0 + threadIdx.x;
  const long long pos = pr.vec_off + rpos[row];
  const double *c = coef + row;
  double acc = 0.0, acc1 = 0.0;
#pragma unroll
  for (int t0 = 0; t0 < S; t0 += 8) {
    double a[8], v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (t0 + u < S) {
        a[u] = __ldcs(c + (long long)(t0 + u) * ld);
        const long long q = pos + dl[t0 + u];
        v[u] = x[q] + (x2 ? x2[q] : 0.0);
      }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (t0 + u < S) {
        if (u & 1) acc1 = fma(a[u], v[u], acc1);
        else acc = fma(a[u], v[u], acc);
      }
  }
  acc += acc1;
  if (out_mode == 0) y[pr.vec_off + rout[row]] = -acc;
  else y[rout[row]] = acc;
}

// -------- transfers ---------------------------------------------------------------------
__device__ __forceinline__ void decode_point(const GridDesc &g, int t, int *i) {
  int n0 = g.hi[0] - g.lo[0], n1 = g.hi[1] - g.lo[1];
  i[0] = g.lo[0] + t % n0;
  t /= n0;
  i[1] = g.lo[1] + t % n1;
  i[2] = g.lo[2] + t / n1;
}

// b_c[a] = (P^T r_f)[a] for coarse point a (active-box index t); x_c[a] = 0
template <int D, int P, bool PDL = false>
__device__ __forceinline__ void restrict_point(const GridDesc &gc, const GridDesc &gf, const TransDesc &td,
                                               long long coff, long long foff, const int *__restrict__ ipool,
                                               const double *__restrict__ wpool, int t, const double *rf, double *bc,
                                               double *xc) {
  int a[3];
  decode_point(gc, t, a);
  constexpr int NW = P + 2;
  int f[3] = {0, 0, 0};
  const double *w[3] = {nullptr, nullptr, nullptr};
  for (int d = 0; d < D; ++d) {
    f[d] = ipool[td.rc_off[d] + a[d]];
    w[d] = wpool + td.rw_off[d] + (long long)a[d] * NW;
  }
  // box positions are separable (layout.cuh sl_term): one table per direction; constant trip
  // counts, fully unrolled (the tables stay in registers), zero weights multiply finite values
  long long pt[3][NW];
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int t = 0; t < NW; ++t) pt[d][t] = (d < D) ? sl_term(gf, P, d, f[d] + t) : 0;
  double w0[NW], w1[NW], w2v[NW];
#pragma unroll
  for (int t = 0; t < NW; ++t) {
    w0[t] = w[0][t];
    w1[t] = w[1][t];
    w2v[t] = (D == 3) ? w[2][t] : 1.0;
  }
  // programmatic dependent launch (IETI_PDL_TR): everything above is static (descriptors, windows,
  // weights); the fine residual written by the previous grid is read only after the wait
  if (PDL) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const double *r = rf + foff;
  double acc = 0.0;
#pragma unroll
  for (int t2 = 0; t2 < (D == 3 ? NW : 1); ++t2) {
    const double w2 = w2v[t2];
#pragma unroll
    for (int t1 = 0; t1 < NW; ++t1) {
      const double w12 = w2 * w1[t1];
      const double *rr = r + pt[1][t1] + pt[2][t2];
      double s1 = 0.0;
#pragma unroll
      for (int t0 = 0; t0 < NW; ++t0) s1 = fma(w0[t0], rr[pt[0][t0]], s1);
      acc = fma(w12, s1, acc);
    }
  }
  const long long q = coff + sl_pos(gc, P, D, a);
  bc[q] = acc;
  if (xc) xc[q] = 0.0;
}

// x_f[i] += (P x_c)[i] for fine point i (active-box index t)
template <int D, int P, bool PDL = false>
__device__ __forceinline__ void prolong_point(const GridDesc &gc, const GridDesc &gf, const TransDesc &td,
                                              long long coff, long long foff, const int *__restrict__ ipool,
                                              const double *__restrict__ wpool, int t, const double *xc, double *xf) {
  int i[3];
  decode_point(gf, t, i);
  constexpr int W = P / 2 + 2;                   // window of coarse contributors (TransDesc::W, host)
  int c[3] = {0, 0, 0};
  const double *w[3] = {nullptr, nullptr, nullptr};
  for (int d = 0; d < D; ++d) {
    c[d] = ipool[td.pf_off[d] + i[d]];
    w[d] = wpool + td.pw_off[d] + (long long)i[d] * W;
  }
  // constant trip counts, fully unrolled: position tables and weights stay in registers
  long long pt[3][W];
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int t = 0; t < W; ++t) pt[d][t] = (d < D) ? sl_term(gc, P, d, c[d] + t) : 0;
  double w0[W], w1[W], w2v[W];
#pragma unroll
  for (int t = 0; t < W; ++t) {
    w0[t] = w[0][t];
    w1[t] = w[1][t];
    w2v[t] = (D == 3) ? w[2][t] : 1.0;
  }
  // programmatic dependent launch (IETI_PDL_TR): the coarse correction of the previous grid is read
  // only after the wait; descriptors, windows and weights above are static
  if (PDL) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const double *e = xc + coff;
  double acc = 0.0;
#pragma unroll
  for (int t2 = 0; t2 < (D == 3 ? W : 1); ++t2) {
    const double w2 = w2v[t2];
#pragma unroll
    for (int t1 = 0; t1 < W; ++t1) {
      const double w12 = w2 * w1[t1];
      const double *ee = e + pt[1][t1] + pt[2][t2];
      double s1 = 0.0;
#pragma unroll
      for (int t0 = 0; t0 < W; ++t0) s1 = fma(w0[t0], ee[pt[0][t0]], s1);
      acc = fma(w12, s1, acc);
    }
  }
  xf[foff + sl_pos(gf, P, D, i)] += acc;
}

template <int D, int P>
__global__ void k_restrict(const GridDesc *gc_, const GridDesc *gf_, const TransDesc *td_, const ProbDesc *pc_,
                           const ProbDesc *pf_, const int *__restrict__ ipool, const double *__restrict__ wpool,
                           const BlockEntry *__restrict__ blocks, const double *rf, double *bc, double *xc) {
  const BlockEntry be = blocks[blockIdx.x];
  if ((int)threadIdx.x >= be.nrow) return;
  const ProbDesc pc = pc_[be.prob], pf = pf_[be.prob];
  restrict_point<D, P, true>(gc_[pc.grid], gf_[pf.grid], td_[pc.grid], pc.vec_off, pf.vec_off, ipool, wpool,
                       be.row0 + threadIdx.x, rf, bc, xc);
}

template <int D, int P>
__global__ void k_prolong(const GridDesc *gc_, const GridDesc *gf_, const TransDesc *td_, const ProbDesc *pc_,
                          const ProbDesc *pf_, const int *__restrict__ ipool, const double *__restrict__ wpool,
                          const BlockEntry *__restrict__ blocks, const double *xc, double *xf) {
  const BlockEntry be = blocks[blockIdx.x];
  if ((int)threadIdx.x >= be.nrow) return;
  const ProbDesc pc = pc_[be.prob], pf = pf_[be.prob];
  prolong_point<D, P, true>(gc_[pc.grid], gf_[pf.grid], td_[pc.grid], pc.vec_off, pf.vec_off, ipool, wpool,
                      be.row0 + threadIdx.x, xc, xf);
}

// ---- fused V-cycle on the small levels (one thread-block cluster per problem) ----------------
// V_ltop(x, b) of O7 for every problem of a batch in ONE launch.  A cluster of `cs` CTAs owns one
// problem; every colour phase of levels ltop..1 (forward, residual, backward) gives each CTA a
// contiguous slice of the colour's rows, whose row-major coefficients (GridDesc::tg == S) are one
// contiguous block: the Tensor Memory Accelerator prefetches the NEXT phase's block into L2
// (cp.async.bulk.prefetch.L2) while the current phase computes, so a phase costs L2 latencies
// plus a cluster barrier instead of a kernel launch and an HBM round trip per batch (no shared
// memory is spent on coefficients, so every cluster of the batch is resident at once).
// Restriction, the coarsest solve (explicit inverse, R9) and prolongation run in between.
template <int D, int P>
__global__ void __launch_bounds__(256, 4) k_vcycle_fused(const FusedArgs a) {
  namespace cg = cooperative_groups;
  constexpr int S = St<D, P>::S;
  constexpr int CEN = St<D, P>::CENTER;
  __shared__ int2 ent[S];
  extern __shared__ __align__(16) double dsm[];   // coarsest rhs
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks();
  const int cr = (int)cl.block_rank();
  const int pb = blockIdx.x / cs;
  const int tid = threadIdx.x;
  const int ncol = a.ncol;
  const int tprf = a.tprf;                       // threads per row (power of two <= 32)
  const int rpp = blockDim.x / tprf;             // rows per pass
  const int sub = tid % tprf;
  double *bsm = dsm;
  auto csync = [&]() {
    if (cs == 1) __syncthreads();
    else cl.sync();
  };
  // staged phases: down part per level l = ltop..1: C forward then C residual colours; up part
  // per level l = 1..ltop: C backward colours (descending)
  const int nstage = 3 * ncol * a.ltop;
  auto stage_desc = [&](int k, int &l, int &col, int &mode) {
    const int nd = 2 * ncol * a.ltop;
    if (k < nd) {
      l = a.ltop - k / (2 * ncol);
      const int w = k % (2 * ncol);
      const bool zero = (l < a.ltop) || a.zero_top;
      if (w < ncol) { col = w; mode = zero ? 4 : 0; }
      else { col = w - ncol; mode = 5; }
    } else {
      const int k2 = k - nd;
      l = 1 + k2 / ncol;
      col = ncol - 1 - k2 % ncol;
      mode = 0;
    }
  };
  // this CTA's row slice of colour col at level l: [rb, re) of the colour's rows
  auto slice = [&](int l, int col, int &rb, int &re, long long &cbase) {
    const FusedLevel &L = a.lev[l];
    const ProbDesc pr = L.probs[pb];
    const GridDesc &g = L.grids[pr.grid];
    const ColourInfo ci = L.cinfo[g.col_off + col];
    const int nr = ci.n[0] * ci.n[1] * ci.n[2];
    rb = (int)((long long)nr * cr / cs);
    re = (int)((long long)nr * (cr + 1) / cs);
    cbase = g.coef_off + (long long)(ci.start + rb) * S;
  };
  auto prefetch = [&](int k) {                   // thread 0: staged phase k's coefficients -> L2
    if (k >= nstage) return;
    int l, col, mode, rb, re;
    long long cbase;
    stage_desc(k, l, col, mode);
    slice(l, col, rb, re, cbase);
    const int shift = (int)(cbase & 1);
    const unsigned bytes = (unsigned)((((long long)(re - rb) * S + shift + 1) & ~1LL) * 8);
    if (bytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.lev[l].coef + cbase - shift), "r"(bytes)
                   : "memory");
  };
  if (tid == 0) prefetch(0);
  int k = 0;                                     // next staged phase
  // one staged phase: rows of this CTA's slice, coefficients from shared memory
  auto run_stage = [&]() {
    int l, col, mode, rb, re;
    long long cbase;
    stage_desc(k, l, col, mode);
    slice(l, col, rb, re, cbase);
    const FusedLevel &L = a.lev[l];
    const ProbDesc pr = L.probs[pb];
    const GridDesc &g = L.grids[pr.grid];
    const ColourInfo ci = L.cinfo[g.col_off + col];
    int n;
    if (mode == 4 || mode == 5) {
      const int nl = a.nlow[col];
      n = (mode == 4) ? nl : (S - 1 - nl);
      const short *ol = a.olist + (long long)col * S + ((mode == 4) ? 0 : nl);
      for (int i = tid; i < n; i += blockDim.x) {
        const int o = ol[i];
        ent[i] = make_int2(o, sl_delta(g, P, D, col, o));
      }
    } else {
      n = S;
      for (int o = tid; o < S; o += blockDim.x) ent[o] = make_int2(o, sl_delta(g, P, D, col, o));
    }
    __syncthreads();                             // ent ready
    if (tid == 0) prefetch(k + 1);               // overlaps the next phase's HBM fetch with this one
    const double *cb = L.coef + cbase;
    const double *dsrc = (mode == 5) ? (((l < a.ltop) || a.zero_top) ? L.x : L.d) : L.x;
    const int nrow = re - rb;
    for (int r0 = 0; r0 < nrow; r0 += rpp) {
      const int rl = r0 + tid / tprf;
      const bool valid = rl < nrow;
      double acc = 0.0, acc1 = 0.0;
      long long pos = 0;
      if (valid) {
        pos = pr.vec_off + row_pos<D, P>(g, ci, col, rb + rl);
        const double *cr_ = cb + (long long)rl * S;
        const double *xb = dsrc + pos;
        int i = sub;
        for (; i + 3 * tprf < n; i += 4 * tprf) {
          double av[4], v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int2 e = ent[i + u * tprf];
            av[u] = __ldcs(cr_ + e.x);
            v[u] = xb[e.y];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (u & 1) acc1 = fma(av[u], v[u], acc1);
            else acc = fma(av[u], v[u], acc);
          }
        }
        for (; i < n; i += tprf) {
          const int2 e = ent[i];
          acc = fma(__ldcs(cr_ + e.x), xb[e.y], acc);
        }
        acc += acc1;
      }
      for (int m = 1; m < tprf; m <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
      if (valid && sub == 0) {
        if (mode == 0 || mode == 4) {
          const double diag = cb[(long long)rl * S + CEN];
          const double delta = (L.b[pos] - acc) / diag;
          if (mode == 4) {
            L.x[pos] = delta;
          } else {
            L.x[pos] += delta;
            if (L.d && l == a.ltop && !a.zero_top && k < 2 * ncol * a.ltop) L.d[pos] = delta;
          }
        } else {
          L.r[pos] = -acc;
        }
      }
    }
    ++k;
    __syncthreads();                             // ent reusable
  };
  // ---- down: pre-smoothing, residual (from the increments, MODE 5), restriction ---------------
  for (int l = a.ltop; l >= 1; --l) {
    for (int col = 0; col < ncol; ++col) {
      run_stage();
      csync();
    }
    for (int col = 0; col < ncol; ++col) run_stage();
    csync();
    const FusedLevel &L = a.lev[l], &C = a.lev[l - 1];
    const ProbDesc pc = C.probs[pb], pf = L.probs[pb];
    const GridDesc &gc = C.grids[pc.grid], &gf = L.grids[pf.grid];
    const TransDesc &td = L.td[pc.grid];
    for (int t = cr * blockDim.x + tid; t < gc.nrows; t += cs * blockDim.x)
      restrict_point<D, P>(gc, gf, td, pc.vec_off, pf.vec_off, L.ip, L.wp, t, L.r, C.b, C.x);
    csync();
  }
  // ---- coarsest: x0 = A0^{-1} b0 ------------------------------------------------------------------
  {
    const FusedLevel &L = a.lev[0];
    const ProbDesc pr = L.probs[pb];
    const GridDesc &g = L.grids[pr.grid];
    const int n0 = g.nrows;
    for (int t = tid; t < n0; t += blockDim.x) {
      int i[3];
      decode_point(g, t, i);
      bsm[t] = L.b[pr.vec_off + sl_pos(g, P, D, i)];
    }
    __syncthreads();
    const double *A = a.inv + a.inv_off[pr.grid];
    const int lane = tid & 31, nw = (cs * blockDim.x) >> 5, w = (cr * blockDim.x + tid) >> 5;
    for (int rr = w; rr < n0; rr += nw) {
      double acc = 0.0;
      for (int cc = lane; cc < n0; cc += 32) acc = fma(A[(long long)rr * n0 + cc], bsm[cc], acc);
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        int i[3];
        decode_point(g, rr, i);
        L.x[pr.vec_off + sl_pos(g, P, D, i)] = acc;
      }
    }
    csync();
  }
  // ---- up: prolongation and post-smoothing ---------------------------------------------------------
  for (int l = 1; l <= a.ltop; ++l) {
    const FusedLevel &L = a.lev[l], &C = a.lev[l - 1];
    const ProbDesc pc = C.probs[pb], pf = L.probs[pb];
    const GridDesc &gc = C.grids[pc.grid], &gf = L.grids[pf.grid];
    const TransDesc &td = L.td[pc.grid];
    for (int t = cr * blockDim.x + tid; t < gf.nrows; t += cs * blockDim.x)
      prolong_point<D, P>(gc, gf, td, pc.vec_off, pf.vec_off, L.ip, L.wp, t, C.x, L.x);
    csync();
    for (int col = 0; col < ncol; ++col) {
      run_stage();
      csync();
    }
  }
}

// -------- coarsest solve: x = A0^{-1} b (one block per problem) ------------------------------
template <int D, int P>
__global__ void k_coarse(const GridDesc *g_, const ProbDesc *pr_, const long long *inv_off, const double *inv,
                         const double *b, double *x) {
  // grid (problems, row splits): every block stages the problem's rhs in shared memory and takes the
  // rows blockIdx.y, blockIdx.y + gridDim.y, ... (one warp per row, lanes over the columns)
  extern __shared__ double sb[];
  const ProbDesc pr = pr_[blockIdx.x];
  const GridDesc &g = g_[pr.grid];
  const int n = g.nrows;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    int i[3];
    decode_point(g, t, i);
    sb[t] = b[pr.vec_off + sl_pos(g, P, D, i)];
  }
  __syncthreads();
  const double *A = inv + inv_off[pr.grid];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = blockIdx.y * nw + warp; r < n; r += nw * gridDim.y) {
    const double *Ar = A + (long long)r * n;
    double acc = 0.0;
    int c = lane;
    // 8 row loads in flight per lane, then the FMAs in column order (same order as one at a time)
    for (; c + 7 * 32 < n; c += 8 * 32) {
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldcs(Ar + c + u * 32);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fma(a[u], sb[c + u * 32], acc);
    }
    for (; c < n; c += 32) acc = fma(__ldcs(Ar + c), sb[c], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
    if (lane == 0) {
      int i[3];
      decode_point(g, r, i);
      x[pr.vec_off + sl_pos(g, P, D, i)] = acc;
    }
  }
}

// -------- Galerkin A_c = P^T A_f P (setup) ------------------------------------------------
__device__ __forceinline__ void colour_row_lattice(const ColourInfo &ci, int j, int P1, int *i) {
  int j0 = j % ci.n[0], t = j / ci.n[0];
  i[0] = ci.first[0] + P1 * j0;
  i[1] = ci.first[1] + P1 * (t % ci.n[1]);
  i[2] = ci.first[2] + P1 * (t / ci.n[1]);
}

// stage 1: B[i][t] = sum_o A_f[i, i+o] P[i+o, cw(i)+t]   (fine row i, coarse window t in CW^D)
template <int D, int P>
__global__ void k_galerkin_ap(GridDesc gf, const ColourInfo *cif, GridDesc gc, TransDesc td, int CW,
                              const int *__restrict__ cwin, const int *__restrict__ ipool,
                              const double *__restrict__ wpool, const double *__restrict__ coef_f, double *B,
                              int ncol) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= gf.nrows) return;
  int c = 0;
  while (c + 1 < ncol && cif[gf.col_off + c + 1].start <= r) ++c;
  const ColourInfo ci = cif[gf.col_off + c];
  int i[3];
  colour_row_lattice(ci, r - ci.start, P + 1, i);
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
        double a = coef_f[cidx(gf, o, r)];
        if (a == 0.0) continue;
        int cj[3] = {0, 0, 0};
        const double *pw[3] = {nullptr, nullptr, nullptr};
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
  const int r = (int)(tid % gc.nrows);
  const int o = (int)(tid / gc.nrows);
  int c = 0;
  while (c + 1 < ncol && cic[gc.col_off + c + 1].start <= r) ++c;
  const ColourInfo ci = cic[gc.col_off + c];
  int a[3];
  colour_row_lattice(ci, r - ci.start, P + 1, a);
  constexpr int W1 = 2 * P + 1;
  int oc[3] = {o % W1 - P, (o / W1) % W1 - P, (D == 3) ? o / (W1 * W1) - P : 0};
  int bb[3] = {a[0] + oc[0], a[1] + oc[1], a[2] + oc[2]};
  double val = 0.0;
  bool inb = true;
  for (int d = 0; d < D; ++d) inb &= (bb[d] >= gc.lo[d] && bb[d] < gc.hi[d]);
  if (inb) {
    constexpr int NW = P + 2;
    int f[3] = {0, 0, 0};
    const double *w[3] = {nullptr, nullptr, nullptr};
    for (int d = 0; d < D; ++d) {
      f[d] = ipool[td.rc_off[d] + a[d]];
      w[d] = wpool + td.rw_off[d] + (long long)a[d] * NW;
    }
    const int CWD = (D == 3) ? CW * CW * CW : CW * CW;
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
          int ii[3] = {i0, i1, i2};
          int rf = cm_row(gf, cif + gf.col_off, P, D, ii);
          int t[3] = {0, 0, 0};
          bool ok = true;
          for (int d = 0; d < D; ++d) {
            t[d] = bb[d] - cwin[d * 4096 + ii[d]];
            ok &= (t[d] >= 0 && t[d] < CW);
          }
          if (!ok) continue;
          val = fma(ww, B[(long long)rf * CWD + t[0] + CW * (t[1] + CW * t[2])], val);
        }
      }
    }
  }
  coef_c[cidx(gc, o, r)] = val;
}

// dense active-box matrix (lexicographic active order) of a grid from its stencil
template <int D, int P>
__global__ void k_dense_from_stencil(const GridDesc *g_, const ColourInfo *ci_, const double *coef, double *dense,
                                     const long long *dense_off) {
  const GridDesc &g = g_[blockIdx.y];
  constexpr int S = St<D, P>::S;
  constexpr int W1 = 2 * P + 1;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)g.nrows * S) return;
  const int a = (int)(tid / S);        // lexicographic active index
  const int o = (int)(tid % S);
  int i[3];
  decode_point(g, a, i);
  const int r = cm_row(g, ci_ + g.col_off, P, D, i);
  int oc[3] = {o % W1 - P, (o / W1) % W1 - P, (D == 3) ? o / (W1 * W1) - P : 0};
  int b[3] = {i[0] + oc[0], i[1] + oc[1], i[2] + oc[2]};
  for (int d = 0; d < D; ++d)
    if (b[d] < g.lo[d] || b[d] >= g.hi[d]) return;
  int n0 = g.hi[0] - g.lo[0], n1 = g.hi[1] - g.lo[1];
  int bcol = (b[0] - g.lo[0]) + n0 * ((b[1] - g.lo[1]) + n1 * (D == 3 ? b[2] - g.lo[2] : 0));
  dense[dense_off[blockIdx.y] + (long long)a * g.nrows + bcol] = coef[cidx(g, o, r)];
}

// SPD inverse of one dense matrix per block: Cholesky into scratch, then A^{-1} = L^{-T} L^{-1}
__global__ void k_spd_inverse2(double *dense, const long long *dense_off, const int *n_, double *scratch,
                               const long long *scratch_off, int *fail) {
  double *A = dense + dense_off[blockIdx.x];
  double *Lm = scratch + scratch_off[blockIdx.x];
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
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    for (int i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      if (i > c)
        for (int k = c; k < i; ++k) s -= Lm[(long long)i * n + k] * A[(long long)k * n + c];
      A[(long long)i * n + c] = (i < c) ? 0.0 : s / Lm[(long long)i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = A[(long long)i * n + c];
      for (int k = i + 1; k < n; ++k) s -= Lm[(long long)k * n + i] * A[(long long)k * n + c];
      A[(long long)i * n + c] = s / Lm[(long long)i * n + i];
    }
  }
}

// y += beta * (M_1 (x) ... (x) M_d) x on floating grids (setup only: true K = (K + alpha M) - alpha M)
template <int D, int P>
__global__ void k_mass_add(LevelView lv, const BlockEntry *__restrict__ blocks, const double *x, double *y) {
  const BlockEntry be = blocks[blockIdx.x];
  if ((int)threadIdx.x >= be.nrow) return;
  const ProbDesc pr = lv.probs[be.prob];
  const GridDesc &g = lv.grids[pr.grid];
  if (g.mass_beta == 0.0) return;
  constexpr int W1 = 2 * P + 1;
  const ColourInfo ci = lv.cinfo[g.col_off + be.colour];
  int i[3];
  colour_row_lattice(ci, be.row0 + threadIdx.x, P + 1, i);
  const long long pos = pr.vec_off + sl_pos(g, P, D, i);
  const int2 *__restrict__ E = lv.ent + g.ent_off + (long long)be.colour * (2 * St<D, P>::S);   // natural order
  const double *m0 = lv.mass + g.mass_off + (long long)i[0] * W1;
  const double *m1 = lv.mass + g.mass_off + (long long)g.M[0] * W1 + (long long)i[1] * W1;
  const double *m2 = lv.mass + g.mass_off + (long long)(g.M[0] + g.M[1]) * W1 + (long long)i[2] * W1;
  double acc = 0.0;
  int o = 0;
  for (int o2 = (D == 3 ? -P : 0); o2 <= (D == 3 ? P : 0); ++o2) {
    const double w2 = (D == 3) ? m2[o2 + P] : 1.0;
    for (int o1 = -P; o1 <= P; ++o1) {
      const double w12 = w2 * m1[o1 + P];
      for (int o0 = -P; o0 <= P; ++o0, ++o) acc = fma(w12 * m0[o0 + P], x[pos + E[o].y], acc);
    }
  }
  y[pos] += g.mass_beta * acc;
}

// dst[o*ld + row] = A_src[row's source row, o] + beta * prod_d Mhat_d  (beta = source grid's mass_beta)
template <int D, int P>
__global__ void k_extract_rows(const GridDesc *__restrict__ g_, const double *__restrict__ coef,
                               const double *__restrict__ mass, const int *__restrict__ rgrid,
                               const int *__restrict__ rrow, const int *__restrict__ rflat, long long nrows,
                               double *dst, long long ostride, long long rstride) {
  constexpr int S = St<D, P>::S;
  constexpr int W1 = 2 * P + 1;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= nrows * S) return;
  const long long row = tid % nrows;
  const int o = (int)(tid / nrows);
  const GridDesc &g = g_[rgrid[row]];
  double v = coef[cidx(g, o, rrow[row])];
  if (g.mass_beta != 0.0 && mass != nullptr) {
    int f = rflat[row];
    const int oc[3] = {o % W1, (o / W1) % W1, o / (W1 * W1)};
    double m = 1.0;
    long long off = 0;
    for (int d = 0; d < D; ++d) {
      const int i = f % g.M[d];
      f /= g.M[d];
      m *= mass[g.mass_off + off + (long long)i * W1 + oc[d]];
      off += (long long)g.M[d] * W1;
    }
    v += g.mass_beta * m;
  }
  // ostride < 0: row tiles of 32 (layout.cuh, tg = -S)
  if (ostride < 0) dst[(row >> 5) * (32LL * S) + (long long)o * 32 + (row & 31)] = v;
  else dst[o * ostride + row * rstride] = v;
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
        case 5: { constexpr int D = 2, P = 5; KERNEL_CALL; } break;              \
        case 6: { constexpr int D = 2, P = 6; KERNEL_CALL; } break;              \
        case 7: { constexpr int D = 2, P = 7; KERNEL_CALL; } break;              \
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

template <int D, int P, int MODE>
static void stencil_tpr(int tpr, int nblocks, const LevelView &lv, const BlockEntry *blocks, double *x,
                        const double *b, double *y, double scale, const double *dsrc, double *dx,
                        const short *olist, const short *nlow, cudaStream_t s, int pcol = -1) {
  // read per launch (graphs capture once): the TMA-fed variant is opt-in, measured slower
  const char *e_st = getenv("IETI_STENCIL");
  const int use_tma = (e_st && std::string(e_st) == "tma") ? 1 : 0;
  if (tpr == 1 && use_tma && MODE < 6) {
    // large grids: TMA-fed coefficient stream (k_stencil_tma)
    if constexpr (MODE < 6) {
      constexpr size_t smem = (size_t)TST * TPU * TSL * sizeof(double);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_stencil_tma<D, P, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
      }
      k_stencil_tma<D, P, MODE><<<nblocks, 128, smem, s>>>(lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow);
    }
  } else {
    const char *e_pdl = getenv("IETI_PDL");
    const int pdl = (e_pdl && e_pdl[0] == '0') ? 0 : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)nblocks);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    // PDL pays on the latency-bound small levels (C2 +18 %, C3 +9 %) and costs ~4 % on the
    // bandwidth-bound one-thread-per-row levels (early dependents hold SM slots): small levels only
    cfg.numAttrs = (pdl && tpr >= 4) ? 1 : 0;
    const char *e_nb = getenv("IETI_BATCH");           // A/B: 16-deep load batches on the big levels
    const char *e_sp = getenv("IETI_SPLIT");           // A/B: two threads (warps) per row on the big levels
    const int split = e_sp ? atoi(e_sp) : 0;          // 1: 8-deep batches (4 blocks/SM), 2: 4-deep (6 blocks/SM)
    if (tpr == 1 && split) {
      cfg.blockDim = dim3(256);
      if (split == 2)
        cudaLaunchKernelEx(&cfg, k_stencil_split<D, P, MODE, 4>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow);
      else
        cudaLaunchKernelEx(&cfg, k_stencil_split<D, P, MODE, 8>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow);
    } else if (tpr == 1 && e_nb && atoi(e_nb) == 16)
      cudaLaunchKernelEx(&cfg, k_stencil<D, P, 1, MODE, 16>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow, pcol);
    else if (tpr == 1)
      cudaLaunchKernelEx(&cfg, k_stencil<D, P, 1, MODE>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow, pcol);
    else if (tpr == 2)
      cudaLaunchKernelEx(&cfg, k_stencil<D, P, 2, MODE>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow, pcol);
    else if (tpr == 8)
      cudaLaunchKernelEx(&cfg, k_stencil<D, P, 8, MODE>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow, pcol);
    else if (tpr == 16)
      cudaLaunchKernelEx(&cfg, k_stencil<D, P, 16, MODE>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow, pcol);
    else
      cudaLaunchKernelEx(&cfg, k_stencil<D, P, 4, MODE>, lv, blocks, x, b, y, scale, dsrc, dx, olist, nlow, pcol);
  }
}

// persistent sweep (k_sweep): mode 0 (dx optional), 4 (from x = 0), 6 (reads U from u), 7 (writes U);
// returns false (nothing launched) if the cooperative grid cannot be resident
template <int D, int P, int TPR, int MODE>
static bool sweep_launch(const LevelView &lv, const BlockEntry *blocks, const int2 *ptab, int nphase, int maxent,
                         unsigned *bar, double *x, const double *b, double *u, double *dx, const short *olist,
                         const short *nlow, cudaStream_t s) {
  static int per_sm = -1, nsm = 0;
  if (per_sm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep<D, P, TPR, MODE>, 128, 0) != cudaSuccess)
      per_sm = 0;
  }
  const int grid = std::min(maxent, per_sm * nsm);
  if (grid <= 0) return false;
  cudaMemsetAsync(bar, 0, sizeof(unsigned), s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_sweep<D, P, TPR, MODE>, lv, blocks, ptab, nphase, bar, x, b, u, dx, olist,
                            nlow) == cudaSuccess;
}

template <int D, int P, int MODE>
static bool sweep_tpr(int tpr, const LevelView &lv, const BlockEntry *blocks, const int2 *ptab, int nphase, int maxent,
                      unsigned *bar, double *x, const double *b, double *u, double *dx, const short *olist,
                      const short *nlow, cudaStream_t s) {
  switch (tpr) {
    case 1: return sweep_launch<D, P, 1, MODE>(lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s);
    case 2: return sweep_launch<D, P, 2, MODE>(lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s);
    case 8: return sweep_launch<D, P, 8, MODE>(lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s);
    case 16: return sweep_launch<D, P, 16, MODE>(lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s);
    default: return sweep_launch<D, P, 4, MODE>(lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s);
  }
}

bool launch_sweep(int dim, int p, int tpr, int mode, const LevelView &lv, const BlockEntry *blocks, const int2 *ptab,
                  int nphase, int maxent, unsigned *bar, double *x, const double *b, double *u, double *dx,
                  const short *olist, const short *nlow, cudaStream_t s) {
  bool ok = false;
  DISPATCH_DP(dim, p, (ok = (mode == 4)   ? sweep_tpr<D, P, 4>(tpr, lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s)
                            : (mode == 6) ? sweep_tpr<D, P, 6>(tpr, lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s)
                            : (mode == 7) ? sweep_tpr<D, P, 7>(tpr, lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s)
                                          : sweep_tpr<D, P, 0>(tpr, lv, blocks, ptab, nphase, maxent, bar, x, b, u, dx, olist, nlow, s)));
  return ok;
}

void launch_sgs_phase(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks, double *x,
                      const double *b, double *dx, int pcol, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (stencil_tpr<D, P, 0>(tpr, nblocks, lv, blocks, x, b, nullptr, 1.0, nullptr, dx, nullptr,
                                            nullptr, s, pcol)));
}

// mode 6 (forward, reads U from u) / 7 (backward, writes U to u): the two sweeps around a cycle
// boundary of the finest level share the higher-colour partial sums (see the mode list above)
void launch_sgs_phase_u(int dim, int p, int tpr, int mode, const LevelView &lv, const BlockEntry *blocks,
                        int nblocks, double *x, const double *b, double *u, double *dx, const short *olist,
                        const short *nlow, int pcol, cudaStream_t s) {
  if (nblocks <= 0) return;
  if (mode == 6)
    DISPATCH_DP(dim, p, (stencil_tpr<D, P, 6>(tpr, nblocks, lv, blocks, x, b, u, 1.0, nullptr, dx, olist, nlow, s,
                                              pcol)));
  else
    DISPATCH_DP(dim, p, (stencil_tpr<D, P, 7>(tpr, nblocks, lv, blocks, x, b, u, 1.0, nullptr, nullptr, olist, nlow,
                                              s, pcol)));
}
void launch_sgs_phase_zero(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                           double *x, const double *b, const short *olist, const short *nlow, int pcol, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (stencil_tpr<D, P, 4>(tpr, nblocks, lv, blocks, x, b, nullptr, 1.0, nullptr, nullptr, olist,
                                            nlow, s, pcol)));
}

void launch_residual(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                     const double *x, const double *b, double *y, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (stencil_tpr<D, P, 1>(tpr, nblocks, lv, blocks, (double *)x, b, y, 1.0, nullptr, nullptr,
                                            nullptr, nullptr, s)));
}

void launch_residual_upper(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                           const double *dsrc, double *y, const short *olist, const short *nlow, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (stencil_tpr<D, P, 5>(tpr, nblocks, lv, blocks, nullptr, nullptr, y, 1.0, dsrc, nullptr, olist,
                                            nlow, s)));
}

void launch_apply(int dim, int p, int tpr, const LevelView &lv, const BlockEntry *blocks, int nblocks,
                  const double *x, double *y, double scale, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (stencil_tpr<D, P, 2>(tpr, nblocks, lv, blocks, (double *)x, nullptr, y, scale, nullptr,
                                            nullptr, nullptr, nullptr, s)));
}

void launch_mass_add(int dim, int p, const LevelView &lv, const BlockEntry *blocks, int nblocks, int nthr,
                     const double *x, double *y, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (k_mass_add<D, P><<<nblocks, nthr, 0, s>>>(lv, blocks, x, y)));
}

void launch_rowlist(int dim, int p, const GridDesc *grids, const ProbDesc *probs, const BlockEntry *blocks, int nblocks,
                    const double *coef, long long ld, const int *rpos, const int *rout, const double *x,
                    const double *x2, double *y, int out_mode, cudaStream_t s) {
  if (nblocks <= 0) return;
  DISPATCH_DP(dim, p, (k_rowlist<D, P><<<nblocks, 128, 0, s>>>(grids, probs, blocks, coef, ld, rpos, rout, x, x2, y,
                                                               out_mode)));
}

// transfer kernels: launched with programmatic stream serialization on latency-bound batches (the static
// prologue of k_restrict / k_prolong overlaps the previous grid's tail); IETI_PDL_TR=0 switches it off
static void transfer_cfg(cudaLaunchConfig_t &cfg, cudaLaunchAttribute *at, int nblocks, int nthr, cudaStream_t s) {
  static const int pdl = [] {
    const char *e = getenv("IETI_PDL_TR");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  cfg.gridDim = dim3((unsigned)nblocks);
  cfg.blockDim = dim3((unsigned)nthr);
  cfg.stream = s;
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // bandwidth-bound batches (more than ~2 waves of blocks) gain nothing from an early launch
  cfg.numAttrs = (pdl && nblocks <= 4096) ? 1 : 0;
}

void launch_restrict(int dim, int p, const GridDesc *gc, const GridDesc *gf, const TransDesc *td,
                     const ProbDesc *pc, const ProbDesc *pf, const int *ipool, const double *wpool,
                     const BlockEntry *blocks, int nblocks, int nthr, const double *rf, double *bc, double *xc,
                     cudaStream_t s) {
  if (nblocks <= 0) return;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  transfer_cfg(cfg, at, nblocks, nthr, s);
  DISPATCH_DP(dim, p, (cudaLaunchKernelEx(&cfg, k_restrict<D, P>, gc, gf, td, pc, pf, ipool, wpool, blocks, rf, bc, xc)));
}

void launch_prolong(int dim, int p, const GridDesc *gc, const GridDesc *gf, const TransDesc *td,
                    const ProbDesc *pc, const ProbDesc *pf, const int *ipool, const double *wpool,
                    const BlockEntry *blocks, int nblocks, int nthr, const double *xc, double *xf,
                    cudaStream_t s) {
  if (nblocks <= 0) return;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  transfer_cfg(cfg, at, nblocks, nthr, s);
  DISPATCH_DP(dim, p, (cudaLaunchKernelEx(&cfg, k_prolong<D, P>, gc, gf, td, pc, pf, ipool, wpool, blocks, xc, xf)));
}

void launch_coarse_solve(const GridDesc *g, const ProbDesc *pr, const long long *inv_off, const double *inv,
                         int nprob, int dim, int p, const double *b, double *x, int max_rows, cudaStream_t s) {
  if (nprob <= 0) return;
  size_t smem = (size_t)std::max(1, max_rows) * sizeof(double);
  DISPATCH_DP(dim, p, ({
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_coarse<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // row splits: >= 2 blocks per SM over the batch (C4: 64 problems x 8), at most one warp per row
    int ny = 1;
    while (ny < 16 && nprob * ny < 296 && ny * 8 < max_rows) ny *= 2;
    k_coarse<D, P><<<dim3((unsigned)nprob, (unsigned)ny), 256, smem, s>>>(g, pr, inv_off, inv, b, x);
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
  DISPATCH_DP(dim, p, (k_dense_from_stencil<D, P><<<grid, 128, 0, s>>>(g, ci, coef, dense, dense_off)));
}

void launch_spd_inverse2(double *dense, const long long *dense_off, const int *n, int ngrid, double *scratch,
                         const long long *scratch_off, int *fail, cudaStream_t s) {
  if (ngrid <= 0) return;
  k_spd_inverse2<<<ngrid, 256, 0, s>>>(dense, dense_off, n, scratch, scratch_off, fail);
}

void launch_extract_rows(int dim, int p, const GridDesc *g, const double *coef, const double *mass, const int *rgrid,
                         const int *rrow, const int *rflat, long long nrows, double *dst, long long ostride,
                         long long rstride, cudaStream_t s) {
  if (nrows <= 0) return;
  int S = 1;
  for (int d = 0; d < dim; ++d) S *= (2 * p + 1);
  long long n = nrows * S;
  DISPATCH_DP(dim, p, (k_extract_rows<D, P><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, coef, mass, rgrid, rrow,
                                                                                       rflat, nrows, dst, ostride,
                                                                                       rstride)));
}

void launch_vcycle_fused(int dim, int p, const FusedArgs &a, int nprob, int cs, cudaStream_t s) {
  if (nprob <= 0) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nprob * cs));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = (size_t)std::max(1, a.max_coarse_rows) * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DISPATCH_DP(dim, p, ({
    auto kern = k_vcycle_fused<D, P>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
    cudaLaunchKernelEx(&cfg, kern, a);
  }));
}
