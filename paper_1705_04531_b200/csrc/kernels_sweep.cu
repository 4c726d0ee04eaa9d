// kernels_sweep.cu -- one colour-Gauss-Seidel SWEEP per launch on the latency-bound levels
// (R5, R6): one thread-block cluster per problem, the (p+1)^d colour phases separated by a
// cluster barrier instead of a kernel launch each.
//
// Why: on the small, row-major levels (GridDesc::tg == S) a colour phase moves a few MB; launched
// one kernel per phase it costs a launch gap plus two dependent HBM round trips (coefficients,
// then the reduction) -- ~6 us on C4 against ~2 us of bytes.  The coefficients of a phase do not
// depend on x, only the neighbour gathers do.  So here every CTA owns a contiguous row slice of
// each colour of its problem (row-major rows: one contiguous slab of nrow * S doubles), and the
// Tensor Memory Accelerator copies the NEXT phase's slab into shared memory (cp.async.bulk +
// mbarrier, double buffer) while the current phase computes and while the cluster waits at the
// barrier.  The critical path of a phase is then: barrier -> x gathers (L2) -> reduction -> x
// store.  x stays in global memory; the barrier's release / acquire (MEMBAR.GPU before the
// arrive, CCTL.IVALL after the wait) makes the other CTAs' updates visible.
//
// Arithmetic per row is exactly that of k_stencil<.., TPR, MODE 0 / 4, NB = 8> (same list order,
// same 8-deep batches with two partial sums, same shuffle reduction), so both paths give bitwise
// identical iterates (R23: no reordering at all).
#include "layout.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int MAXCOL = 64;                         // (p+1)^d colours of every supported (d, p)

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  // release: this CTA's x stores are visible cluster-wide before the arrive; acquire: the other
  // CTAs' stores are visible after the wait (ptxas: MEMBAR before, L1 invalidate after)
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct SweepArgs {
  LevelView lv;
  double *x;
  const double *b;
  double *dx;               // forward increments (mode 0 only; may be null)
  const short *nlow;        // per colour: number of lower-colour offsets
  int ncol;
  int fwd;                  // 1: colours ascending, 0: descending
  int zero;                 // 1: x = 0 on entry (mode 4 lists: lower colours only)
  int slab;                 // doubles per coefficient buffer (even)
  int rmax;                 // most rows of one CTA's slice of a colour
};

// one cluster of cs CTAs per problem; CTA cr owns rows [nr cr / cs, nr (cr+1) / cs) of every colour.
// Shared memory (dynamic): [2][slab] coefficient slabs | [2][S + 2] (offset, box delta) lists |
// [ncol][rmax] b of the CTA's rows | [ncol][rmax] box positions of the rows (int, relative to the
// problem's vector offset)
template <int D, int P, int TPR>
__global__ void __launch_bounds__(256, 4) k_sweep_cl(const SweepArgs a) {
  constexpr int S = St<D, P>::S;
  constexpr int CEN = St<D, P>::CENTER;
  constexpr int NB = 8;
  constexpr int EL = (S + 2 + 1) & ~1;               // entries per list buffer (even: 16-byte buffers)
  extern __shared__ __align__(16) double csm[];
  int2 *Eb = reinterpret_cast<int2 *>(csm + 2 * a.slab);
  double *sb = reinterpret_cast<double *>(Eb + 2 * EL);
  int *spos = reinterpret_cast<int *>(sb + a.ncol * a.rmax);
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ int srb[MAXCOL], snr[MAXCOL];
  const int cs = (int)cluster_size(), cr = (int)cluster_rank();
  const int pb = blockIdx.x / cs;
  const LevelView &lv = a.lv;
  const ProbDesc pr = lv.probs[pb];
  const GridDesc &g = lv.grids[pr.grid];
  const int tid = threadIdx.x;
  const int rpp = blockDim.x / TPR;                  // rows per pass
  const int gi = tid % TPR;
  const long long coef_off = g.coef_off;
  const int ent_off = g.ent_off;
  // per colour: this CTA's row slice, and the box position of every row of it (computed once here,
  // off the phases' critical path; the cluster barriers invalidate L1, so nothing is re-read later)
  for (int col = tid; col < a.ncol; col += blockDim.x) {
    const ColourInfo ci = lv.cinfo[g.col_off + col];
    const int nr = ci.n[0] * ci.n[1] * ci.n[2];
    srb[col] = ci.start + nr * cr / cs;            // first (colour-major) row of the slice
    snr[col] = nr * (cr + 1) / cs - nr * cr / cs;
  }
  for (int t = tid; t < a.ncol * a.rmax; t += blockDim.x) {
    const int col = t / a.rmax, rl = t % a.rmax;
    const ColourInfo ci = lv.cinfo[g.col_off + col];
    const int nr = ci.n[0] * ci.n[1] * ci.n[2];
    const int j = nr * cr / cs + rl;
    spos[t] = (j < nr) ? (int)row_pos<D, P>(g, ci, col, j) : 0;
    sb[t] = (j < nr) ? __ldcs(a.b + pr.vec_off + spos[t]) : 0.0;   // b is constant over the sweep
  }
  unsigned long long pol = 0;
  if (tid == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  auto colour_of = [&](int ph) { return a.fwd ? ph : a.ncol - 1 - ph; };
  // 16-byte aligned source of a slab starting at double offset `at` (shift = 0 / 1 doubles)
  auto slab_shift = [&](int col) { return (int)((coef_off + (long long)srb[col] * S) & 1); };
  // (offset, box delta) list of a colour in the precomputed table (GridDesc::ent_off): natural
  // order (S entries) or, from x = 0, the lower-colour offsets (solver.cu olist order)
  auto list_at = [&](int col, int &n) {
    const long long e0 = ent_off + (long long)col * 2 * S + (a.zero ? S : 0);
    n = a.zero ? a.nlow[col] : S;
    return e0;
  };
  // thread 0: the slab and the list of phase ph -> buffers ph & 1, one mbarrier transaction
  auto issue = [&](int ph) {
    const int col = colour_of(ph), nrow = snr[col];
    const unsigned mb = smem_u32(&bar[ph & 1]);
    const long long gstart = coef_off + (long long)srb[col] * S;
    const int shift = (int)(gstart & 1);
    const unsigned cbytes = nrow ? (unsigned)((((long long)nrow * S + shift + 1) & ~1LL) * 8) : 0u;
    int n;
    const long long e0 = list_at(col, n);
    const int eshift = (int)(e0 & 1);
    const unsigned ebytes = n ? (unsigned)(((n + eshift + 1) & ~1) * 8) : 0u;
    if (cbytes + ebytes == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
      return;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(cbytes + ebytes) : "memory");
    if (cbytes)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
          ::"r"(smem_u32(csm + (ph & 1) * a.slab)), "l"(lv.coef + gstart - shift), "r"(cbytes), "r"(mb), "l"(pol)
          : "memory");
    if (ebytes)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(Eb + (ph & 1) * EL)), "l"(lv.ent + e0 - eshift), "r"(ebytes), "r"(mb)
                   : "memory");
  };
  if (tid == 0) issue(0);
  constexpr int KM = (S + TPR - 1) / TPR;            // most list entries per thread
  for (int ph = 0; ph < a.ncol; ++ph) {
    const int buf = ph & 1;
    // the other buffers were consumed in phase ph - 1 by every thread (the cluster barrier below)
    if (tid == 0 && ph + 1 < a.ncol) issue(ph + 1);
    const int col = colour_of(ph);
    const int nrow = snr[col];
    int n;
    const long long e0 = list_at(col, n);
    const int2 *e = Eb + buf * EL + (e0 & 1);
    const double *cb = csm + buf * a.slab + slab_shift(col);
    const int *rpos = spos + col * a.rmax;
    {
      const unsigned mb = smem_u32(&bar[buf]);
      const unsigned parity = (unsigned)((ph >> 1) & 1);
      unsigned done = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(mb), "r"(parity) : "memory");
      } while (!done);
    }
    for (int r0 = 0; r0 < nrow; r0 += rpp) {
      const int rl = r0 + tid / TPR;
      const bool valid = rl < nrow;
      double acc = 0.0, bval = 0.0, diag = 1.0, xa = 0.0;
      const long long pos = pr.vec_off + (valid ? rpos[rl] : 0);
      if (valid) {
        if (gi == 0) {
          bval = sb[col * a.rmax + rl];
          diag = cb[(long long)rl * S + CEN];
        }
        const double *c = cb + (long long)rl * S;
        const double *xb = a.x + pos;
        // k_stencil's range_sum (interleaved entries, 8-deep batches with two partial sums, the
        // tail into the first): entry k of this thread is list entry gi + k TPR
        double s0 = 0.0, s1 = 0.0;
        if constexpr (KM <= 24) {
          // every gather of the row issued at once (one L2 round trip), then the same FMA order
          const int K = (n > gi) ? (n - gi + TPR - 1) / TPR : 0;
          const int KB = (K / NB) * NB;
          double v[KM];
#pragma unroll
          for (int k = 0; k < KM; ++k) v[k] = (k < K) ? xb[e[gi + k * TPR].y] : 0.0;
          if (!a.zero && gi == CEN % TPR) xa = v[CEN / TPR];   // x_a itself (the centre entry)
#pragma unroll
          for (int k = 0; k < KM; ++k) {
            const int i = gi + k * TPR;
            if (k < KB) {
              const double cv = c[a.zero ? e[i].x : i];
              if (k & 1) s1 = fma(cv, v[k], s1);
              else s0 = fma(cv, v[k], s0);
            } else if (k < K) {
              s0 = fma(c[a.zero ? e[i].x : i], v[k], s0);
            }
          }
        } else {
          int i = gi;
          for (; i + (NB - 1) * TPR < n; i += NB * TPR) {
            double av[NB], v[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
              const int2 en = e[i + u * TPR];
              av[u] = c[a.zero ? en.x : (i + u * TPR)];
              v[u] = xb[en.y];
              if (!a.zero && i + u * TPR == CEN) xa = v[u];
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) {
              if (u & 1) s1 = fma(av[u], v[u], s1);
              else s0 = fma(av[u], v[u], s0);
            }
          }
          for (; i < n; i += TPR) {
            const int2 en = e[i];
            const double v = xb[en.y];
            if (!a.zero && i == CEN) xa = v;
            s0 = fma(c[a.zero ? en.x : i], v, s0);
          }
        }
        acc = s0 + s1;
      }
#pragma unroll
      for (int m = 1; m < TPR; m <<= 1) acc += __shfl_xor_sync(FULL, acc, m);
      if (TPR > 1 && !a.zero) xa = __shfl_sync(FULL, xa, (threadIdx.x & 31 & ~(TPR - 1)) + CEN % TPR);
      if (valid && gi == 0) {
        const double delta = (bval - acc) / diag;
        if (a.zero) {
          a.x[pos] = delta;
        } else {
          a.x[pos] = xa + delta;
          if (a.dx) __stcs(a.dx + pos, delta);
        }
      }
    }
    cluster_barrier();
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------
#define SW_DISPATCH_DP(dim, p, KERNEL_CALL)                                      \
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

template <int D, int P, int TPR>
static int sweep_cl_launch(const SweepArgs &a, int nprob, int cs, int nthr, cudaStream_t s, bool query) {
  auto kern = k_sweep_cl<D, P, TPR>;
  constexpr int S = St<D, P>::S, EL = (S + 2 + 1) & ~1;
  const size_t smem = (size_t)2 * a.slab * sizeof(double) + (size_t)2 * EL * sizeof(int2) +
                      (size_t)a.ncol * a.rmax * (sizeof(double) + sizeof(int));
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return -1;
  if (cs > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nprob * cs));
  cfg.blockDim = dim3((unsigned)nthr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (query) {
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    return ncl;
  }
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? 1 : -1;
}

template <int D, int P>
static int sweep_cl_tpr(int tpr, const SweepArgs &a, int nprob, int cs, int nthr, cudaStream_t s, bool query) {
  switch (tpr) {
    case 2: return sweep_cl_launch<D, P, 2>(a, nprob, cs, nthr, s, query);
    case 4: return sweep_cl_launch<D, P, 4>(a, nprob, cs, nthr, s, query);
    case 8: return sweep_cl_launch<D, P, 8>(a, nprob, cs, nthr, s, query);
    case 16: return sweep_cl_launch<D, P, 16>(a, nprob, cs, nthr, s, query);
    default: return -1;
  }
}

// query: the number of clusters that can be co-resident (0 / -1: this configuration cannot run);
// launch: 1 on success, -1 on a launch error
int launch_sweep_cluster(int dim, int p, int tpr, const LevelView &lv, int nprob, int cs, int nthr, int slab, int rmax, int ncol,
                         bool fwd, bool zero, double *x, const double *b, double *dx, const short *nlow,
                         cudaStream_t s, bool query) {
  SweepArgs a{lv, x, b, dx, nlow, ncol, fwd ? 1 : 0, zero ? 1 : 0, slab, rmax};
  int r = -1;
  SW_DISPATCH_DP(dim, p, (r = sweep_cl_tpr<D, P>(tpr, a, nprob, cs, nthr, s, query)));
  return r;
}
