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
#include <type_traits>
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
  double *dx;               // forward increments (modes 0 and 6; may be null)
  double *U;                // higher-colour sums: read by mode 6, written by mode 7
  const short *nlow;        // per colour: number of lower-colour offsets
  int ncol;
  int fwd;                  // 1: colours ascending, 0: descending
  int slab;                 // doubles per coefficient buffer (even); 0: coefficients read from global
                            // memory, the next phase's rows prefetched into L2 (levels whose slabs do
                            // not fit in shared memory next to all the problem's resident clusters)
  int rmax;                 // most rows of one CTA's slice of a colour
  int rep;                  // > 0: every CTA keeps a replica of its problem's x box in shared memory
                            // (rep doubles >= box + 2 guard, even); updates are broadcast to all the
                            // cluster's replicas through distributed shared memory, so the gathers
                            // never leave the SM and no global store sits before a barrier
  int guard;                // replica guard on each side (>= the widest wrapped neighbour offset)
};

// Modes as k_stencil (kernels_mg.cu): 0 full SGS phase (natural list, x_a is the centre gather),
// 4 from x = 0 (lower-colour list), 6 forward with U (lower-colour list, U_a read), 7 backward
// recording U (lower then higher list, two partial sums).
// One cluster of cs CTAs per problem; CTA cr owns rows [nr cr / cs, nr (cr+1) / cs) of every colour.
// Shared memory (dynamic): [2][slab] coefficient slabs | [2][S + 2] (offset, box delta) lists |
// [ncol][rmax] b of the CTA's rows | [ncol][rmax] box positions of the rows (int, relative to the
// problem's vector offset)
template <int D, int P, int TPR, int MODE, bool REP>
__global__ void __launch_bounds__(512, 2) k_sweep_cl(const SweepArgs a) {
  constexpr int S = St<D, P>::S;
  constexpr int CEN = St<D, P>::CENTER;
  constexpr int NB = 8;
  constexpr int EL = (S + 2 + 1) & ~1;               // entries per list buffer (even: 16-byte buffers)
  constexpr bool NAT = (MODE == 0);                  // natural-order list: coefficient index = list index
  extern __shared__ __align__(16) double smem_dyn[];
  double *xs = smem_dyn;                             // REP: [guard | box | guard] replica of x
  double *csm = smem_dyn + (REP ? a.rep : 0);
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
  // per colour: this CTA's row slice, and the box position and b of every row of it (computed once
  // here, off the phases' critical path; the cluster barriers invalidate L1)
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
    spos[t] = (j < nr) ? (int)row_pos<D, P>(g, ci, col, j) : -1;
  }
  unsigned long long pol = 0;
  if (tid == 0) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();                                   // srb / snr and the mbarriers are ready for thread 0's issue(0)
  auto colour_of = [&](int ph) { return a.fwd ? ph : a.ncol - 1 - ph; };
  // (offset, box delta) list of a colour in the precomputed table (GridDesc::ent_off): [c][0] the
  // natural order (S entries), [c][1] the lower-colour offsets then the higher ones (S - 1)
  auto list_at = [&](int col, int &n) {
    const long long e0 = ent_off + (long long)col * 2 * S + (NAT ? 0 : S);
    n = NAT ? S : (MODE == 7 ? S - 1 : a.nlow[col]);
    return e0;
  };
  // thread 0: the list (and the slab, or its L2 prefetch) of phase ph -> buffers ph & 1
  auto issue = [&](int ph) {
    const int col = colour_of(ph), nrow = snr[col];
    const unsigned mb = smem_u32(&bar[ph & 1]);
    const long long gstart = coef_off + (long long)srb[col] * S;
    const int shift = (int)(gstart & 1);
    const unsigned rbytes = nrow ? (unsigned)((((long long)nrow * S + shift + 1) & ~1LL) * 8) : 0u;
    const unsigned cbytes = a.slab ? rbytes : 0u;
    if (!a.slab && rbytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lv.coef + gstart - shift), "r"(rbytes)
                   : "memory");
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
  // programmatic dependent launch (opt-in, IETI_PDL_CL=1): everything above -- descriptors, row positions, phase 0's
  // list and coefficient slab (or its L2 prefetch) -- is static and overlaps the previous grid's tail; b
  // and x, which that grid may have written, are read only after the wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int t = tid; t < a.ncol * a.rmax; t += blockDim.x)
    sb[t] = (spos[t] >= 0) ? __ldcs(a.b + pr.vec_off + spos[t]) : 0.0;   // b is constant over the sweep
  if constexpr (REP) {
    // the replica holds exactly the global values of [vec_off - guard, vec_off + box + guard) (the
    // pool's guard bands and the neighbouring boxes), so wrapped zero-coefficient gathers read the
    // same finite values as the global path: bitwise equal results
    const double *src = a.x + pr.vec_off - a.guard;
    for (int t = tid; t < g.box + 2 * a.guard; t += blockDim.x) xs[t] = src[t];
  }
  __syncthreads();
  // every replica is loaded before any CTA of the cluster broadcasts an update into it
  if constexpr (REP) cluster_barrier();
  constexpr int KM = (S + TPR - 1) / TPR;            // most list entries per thread
  for (int ph = 0; ph < a.ncol; ++ph) {
    const int buf = ph & 1;
    // the other buffers were consumed in phase ph - 1 by every thread (the cluster barrier below)
    if (tid == 0 && ph + 1 < a.ncol) issue(ph + 1);
    // the next grid may start its static prologue during this sweep's last phase
    if (ph + 1 == a.ncol) asm volatile("griddepcontrol.launch_dependents;");
    const int col = colour_of(ph);
    const int nrow = snr[col];
    int n;
    const long long e0 = list_at(col, n);
    const int nl = a.nlow[col];
    const int2 *e = Eb + buf * EL + (e0 & 1);
    const double *cb = a.slab ? csm + buf * a.slab + (int)((coef_off + (long long)srb[col] * S) & 1)
                              : lv.coef + coef_off + (long long)srb[col] * S;
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
      double acc = 0.0, accu = 0.0, bval = 0.0, diag = 1.0, xa = 0.0, uval = 0.0;
      const int lpos = valid ? rpos[rl] : 0;         // box position
      const long long pos = pr.vec_off + lpos;
      if (valid) {
        const double *c = cb + (long long)rl * S;
        const double *xb = REP ? xs + a.guard + lpos : a.x + pos;
        if (gi == 0 || REP) {                        // REP: every lane of the row forms the update
          bval = sb[col * a.rmax + rl];
          diag = c[CEN];
          if (MODE == 6 || MODE == 7) xa = xb[0];        // issued with the gathers (independent)
          if (MODE == 6 && gi == 0) uval = __ldcs(a.U + pos);
        }
        // k_stencil's range_sum over list entries [i0, i1): entry k of this thread is
        // i0 + gi + k TPR; 8-deep batches alternate two partial sums, the tail goes to the first
        // k_stencil's range_sum over list entries [i0, i1): entry k of this thread is
        // i0 + gi + k TPR; full 8-entry batches alternate two partial sums (odd k into the second),
        // the tail goes to the first.  Loads are issued PF entries at a time (coefficient and x
        // gather together), then the FMAs run in that order: with coefficient slabs in shared
        // memory PF covers the whole range (one L2 round trip for the gathers); from global memory
        // PF = 8 bounds the registers
        auto range_sum = [&](int i0, int i1, auto pf_tag, auto glob_tag) {
          constexpr int PF = decltype(pf_tag)::value;
          constexpr bool GLOB = decltype(glob_tag)::value;   // coefficients from global memory
          const int K = (i1 - i0 > gi) ? (i1 - i0 - gi + TPR - 1) / TPR : 0;
          const int KB = (K / NB) * NB;
          double s0 = 0.0, s1 = 0.0;
          for (int k0 = 0; k0 < K; k0 += PF) {
            double v[PF], cv[GLOB ? PF : 1];
#pragma unroll
            for (int u = 0; u < PF; ++u) {
              const int k = k0 + u, i = i0 + gi + k * TPR;
              if (k < K) {
                const int2 en = e[i];
                if (GLOB) cv[GLOB ? u : 0] = c[NAT ? i : en.x];
                v[u] = xb[en.y];
                if (NAT && i == CEN) xa = v[u];            // x_a itself (the centre entry)
              } else {
                v[u] = 0.0;
                if (GLOB) cv[GLOB ? u : 0] = 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < PF; ++u) {
              const int k = k0 + u, i = i0 + gi + k * TPR;
              if (k < K) {
                const double w = GLOB ? cv[GLOB ? u : 0] : c[NAT ? i : e[i].x];   // slab: shared memory
                if (k < KB && (k & 1)) s1 = fma(w, v[u], s1);
                else s0 = fma(w, v[u], s0);
              }
            }
          }
          return s0 + s1;
        };
        auto rsum = [&](int i0, int i1) {
          if constexpr (KM <= (MODE == 7 ? 12 : 24)) {   // mode 7: two ranges, registers for both
            if (a.slab) return range_sum(i0, i1, std::integral_constant<int, KM>(), std::false_type());
          }
          if (a.slab) return range_sum(i0, i1, std::integral_constant<int, NB>(), std::false_type());
          return range_sum(i0, i1, std::integral_constant<int, NB>(), std::true_type());
        };
        if (MODE == 7) {
          acc = rsum(0, nl);
          accu = rsum(nl, n);
        } else {
          acc = rsum(0, n);
        }
      }
#pragma unroll
      for (int m = 1; m < TPR; m <<= 1) {
        acc += __shfl_xor_sync(FULL, acc, m);
        if (MODE == 7) accu += __shfl_xor_sync(FULL, accu, m);
      }
      if (NAT && TPR > 1) xa = __shfl_sync(FULL, xa, (threadIdx.x & 31 & ~(TPR - 1)) + CEN % TPR);
      if (MODE == 6 && REP && TPR > 1) uval = __shfl_sync(FULL, uval, threadIdx.x & 31 & ~(TPR - 1));
      // the update (same expression in every lane that forms it: identical values)
      double xnew = 0.0, delta = 0.0;
      if (MODE == 6 || MODE == 7) {
        const double u = (MODE == 6) ? uval : accu;
        delta = (bval - (acc + diag * xa + u)) / diag;
        xnew = xa + delta;
      } else {
        delta = (bval - acc) / diag;
        xnew = (MODE == 4) ? delta : xa + delta;
      }
      if (valid && gi == 0) {
        if (!REP) a.x[pos] = xnew;
        if (MODE == 7) __stcs(a.U + pos, accu);
        else if ((MODE == 0 || MODE == 6) && a.dx) __stcs(a.dx + pos, delta);
      }
      if constexpr (REP) {
        // lane gi of the row writes the replicas of ranks gi, gi + TPR, ... (local: plain store)
        if (valid) {
          const unsigned la = smem_u32(xs + a.guard + lpos);
          for (int r = gi; r < cs; r += TPR) {
            if (r == cr) {
              xs[a.guard + lpos] = xnew;
            } else {
              unsigned ra;
              asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r));
              asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(xnew) : "memory");
            }
          }
        }
      }
    }
    cluster_barrier();
  }
  if constexpr (REP) {
    // every replica is final (the last barrier): CTA cr writes its share of the box back
    const int box = g.box;
    double *dst = a.x + pr.vec_off;
    for (int t = box * cr / cs + tid; t < box * (cr + 1) / cs; t += blockDim.x) dst[t] = xs[a.guard + t];
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

template <int D, int P, int TPR, int MODE>
static int sweep_cl_launch(const SweepArgs &a, int nprob, int cs, int nthr, cudaStream_t s, bool query) {
  auto kern = a.rep ? k_sweep_cl<D, P, TPR, MODE, true> : k_sweep_cl<D, P, TPR, MODE, false>;
  constexpr int S = St<D, P>::S, EL = (S + 2 + 1) & ~1;
  const size_t smem = (size_t)(a.rep + 2 * a.slab) * sizeof(double) + (size_t)2 * EL * sizeof(int2) +
                      (size_t)a.ncol * a.rmax * (sizeof(double) + sizeof(int));
  // one fixed ceiling per kernel (the host caps a configuration at 112 KB): the attribute is a property
  // of the function, not of a launch, and graph nodes / profiler replays of earlier launches with
  // larger buffers must stay valid after a later launch with smaller ones
  static bool attr[2] = {false, false};
  if (!attr[a.rep ? 1 : 0]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      return -1;
    attr[a.rep ? 1 : 0] = true;
  }
  if (smem > 200 * 1024) return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nprob * cs));
  cfg.blockDim = dim3((unsigned)nthr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // programmatic dependent launch of the sweep: opt-in (IETI_PDL_CL=1), measured slower on B200 (C3 -6 %,
  // C4 / C2 -1.5 %: the early CTAs of the next sweep take SM slots and shared memory from the running one)
  static const int pdl = [] {
    const char *e = getenv("IETI_PDL_CL");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && !query) ? 2 : 1;
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

template <int D, int P, int MODE>
static int sweep_cl_tpr(int tpr, const SweepArgs &a, int nprob, int cs, int nthr, cudaStream_t s, bool query) {
  switch (tpr) {
    case 2: return sweep_cl_launch<D, P, 2, MODE>(a, nprob, cs, nthr, s, query);
    case 4: return sweep_cl_launch<D, P, 4, MODE>(a, nprob, cs, nthr, s, query);
    case 8: return sweep_cl_launch<D, P, 8, MODE>(a, nprob, cs, nthr, s, query);
    case 16: return sweep_cl_launch<D, P, 16, MODE>(a, nprob, cs, nthr, s, query);
    default: return -1;
  }
}

// query: the number of clusters that can be co-resident (0 / -1: this configuration cannot run);
// launch: 1 on success, -1 on a launch error.  mode: 0, 4, 6, 7 (k_stencil's SGS phase modes)
int launch_sweep_cluster(int dim, int p, int tpr, int mode, const LevelView &lv, int nprob, int cs, int nthr, int slab,
                         int rmax, int rep, int guard, int ncol, bool fwd, double *x, const double *b, double *dx,
                         double *U, const short *nlow, cudaStream_t s, bool query) {
  SweepArgs a{lv, x, b, dx, U, nlow, ncol, fwd ? 1 : 0, slab, rmax, rep, guard};
  int r = -1;
  switch (mode) {
    case 0: SW_DISPATCH_DP(dim, p, (r = sweep_cl_tpr<D, P, 0>(tpr, a, nprob, cs, nthr, s, query))); break;
    case 4: SW_DISPATCH_DP(dim, p, (r = sweep_cl_tpr<D, P, 4>(tpr, a, nprob, cs, nthr, s, query))); break;
    case 6: SW_DISPATCH_DP(dim, p, (r = sweep_cl_tpr<D, P, 6>(tpr, a, nprob, cs, nthr, s, query))); break;
    case 7: SW_DISPATCH_DP(dim, p, (r = sweep_cl_tpr<D, P, 7>(tpr, a, nprob, cs, nthr, s, query))); break;
    default: break;
  }
  return r;
}
