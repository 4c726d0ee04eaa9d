// sweep.cu -- standalone A/B microbenchmark of the finest-level colour-SGS phase of C5
// (3D, p = 3, 35^3 lattice per patch, 343-coefficient offset-major stencil rows, compact
// sub-lattice boxes; same addressing as paper_1705_04531_b200/csrc/layout.cuh).
// Not part of the product: it isolates the design choices of one sweep (launch shape, load
// depth, rows per thread, cluster-persistent phases) on synthetic data, so that each can be
// timed in seconds instead of a full library rebuild.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sweep sweep.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <algorithm>
#include <string>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

constexpr int P = 3, P1 = 4, W1 = 7, S = 343, CEN = 3 + 7 * (3 + 7 * 3), NCOL = 64;
constexpr int M = 35, NS = 9, SB = NS * NS * NS, BOX = NCOL * SB;

struct Geo {
  int npatch;
  int ld;                // rows per patch padded to 32
  int cstart[NCOL];      // colour-major first row
  int cn[NCOL][3];       // rows per dim of each colour
  long long guard;       // doubles of zero guard before the first patch box
};
__constant__ Geo G;
__device__ short g_ord[NCOL * S];   // per colour: offsets sorted by (target colour, shift) (ORD variants)
// per colour: the offsets of one target colour (they share cache lines: shifts of one sub-lattice
// position) spread over CONSECUTIVE load batches, NB apart, instead of one batch (ORD2 variants):
// a batch's loads are in flight together, so partners in one batch all miss L1; one batch apart the
// later ones find the lines the earlier batch filled
__device__ short g_ord2[NCOL * S];
// CHAIN variants: a chain of dependent descriptor loads before the first data load (the library's
// blocks -> probs -> grids -> cinfo walk); every entry is 0, the result shifts the patch index
__device__ int g_chain[4][8192];
// HALF variants (the library's modes 4 / 6: a forward sweep from x = 0 streams only the offsets
// whose target colour is LOWER than the row's): per colour the count and the list, natural order
__device__ short g_low[NCOL * S];
__device__ int g_nlow[NCOL];

__host__ __device__ inline int sl_delta(int colour, int o) {
  int cc = colour, oo = o, dc = 0, pw = 1, sh[3] = {0, 0, 0};
  for (int d = 0; d < 3; ++d) {
    int cd = cc % P1;
    cc /= P1;
    int od = oo % W1 - P;
    oo /= W1;
    int s = cd + od;
    int shd = (s < 0) ? -1 : (s >= P1 ? 1 : 0);
    int cn = s - shd * P1;
    dc += (cn - cd) * pw;
    pw *= P1;
    sh[d] = shd;
  }
  return dc * SB + sh[0] + NS * (sh[1] + NS * sh[2]);
}

__device__ __forceinline__ long long rowpos(int colour, int j) {
  const int n0 = G.cn[colour][0], n1 = G.cn[colour][1];
  int j0 = j % n0, t = j / n0, j1 = t % n1, j2 = t / n1;
  return (long long)colour * SB + j0 + NS * (j1 + NS * j2);
}

// ---- per-phase kernel: RPT consecutive rows per thread, NB-deep batches --------------------------
// loads are volatile inline PTX so that the compiler keeps the batch order (a whole batch of NB
// coefficient + NB x loads is issued before the first FMA; with DB the NEXT batch is issued before
// the FMAs of the current one, so 2 NB loads stay in flight)
__device__ __forceinline__ double ldcs64(const double *p) {
  double v;
  asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ldcs128(const double *p) {
  double2 v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldx64(const double *p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <int NB, int RPT, bool PDL, bool NOX, bool DB, int TILE = 0, int ORD = 0, int CHAIN = 0, bool HALF = false>
__global__ void __launch_bounds__(128, 4) k_phase(const double *__restrict__ coef, double *x, const double *__restrict__ b,
                                                 int colour, int p0, int nbpp) {
  if (CHAIN > 0) {
    int v = g_chain[0][blockIdx.x & 8191];
    if (CHAIN > 1) v = g_chain[1][(v + blockIdx.x) & 8191];
    if (CHAIN > 2) v = g_chain[2][(v + blockIdx.x) & 8191];
    if (CHAIN > 3) v = g_chain[3][(v + blockIdx.x) & 8191];
    p0 += v;
  }
  __shared__ int dl[S + 2 * NB];
  __shared__ short oc[S + 2 * NB];
  for (int o = threadIdx.x; o < S + 2 * NB; o += blockDim.x) {
    const int nl = HALF ? g_nlow[colour] : S;
    const int oo = (o < nl) ? (HALF ? g_low[colour * S + o] : ORD == 1 ? g_ord[colour * S + o] : ORD == 2 ? g_ord2[colour * S + o] : o) : 0;
    oc[o] = (short)oo;
    dl[o] = (o < S) ? sl_delta(colour, oo) : 0;
  }
  const int patch = p0 + blockIdx.x / nbpp;
  const int nr = G.cn[colour][0] * G.cn[colour][1] * G.cn[colour][2];
  const int j0 = (blockIdx.x % nbpp) * 128 * RPT + threadIdx.x * RPT;
  __syncthreads();
  if (PDL) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (j0 >= nr) return;
  const long long vo = G.guard + (long long)patch * BOX;
  // offset-major [o][row] (TILE 0) or row tiles [row / TILE][o][row % TILE] (a warp's coefficient
  // rows are then one contiguous run of S * 256 B)
  const long long rr = G.cstart[colour] + j0;
  const double *c = coef + (long long)patch * S * G.ld +
                    (TILE ? (rr / TILE) * TILE * S + rr % TILE : rr);
  const long long ldo = TILE ? TILE : G.ld;
  long long pos[RPT];
  bool ok[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    ok[q] = j0 + q < nr;
    pos[q] = vo + rowpos(colour, ok[q] ? j0 + q : j0);
  }
  double s0[RPT], s1[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) s0[q] = s1[q] = 0.0;
  const long long ld = ldo;
  const int NL = HALF ? g_nlow[colour] : S;
  auto issue = [&](int o, double (&a)[NB][RPT], double (&v)[NB][RPT]) {
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      // entries past S read offset 0 with a zero weight (masked below): no tail branch
      const int oo = (ORD || HALF) ? oc[o + u] : ((o + u < S) ? o + u : 0);
      const int d = dl[o + u];
      if (RPT == 2) {
        const double2 aa = ldcs128(c + oo * ld);
        a[u][0] = aa.x;
        a[u][1] = aa.y;
      } else {
#pragma unroll
        for (int q = 0; q < RPT; ++q) a[u][q] = ldcs64(c + oo * ld + q);
      }
#pragma unroll
      for (int q = 0; q < RPT; ++q) v[u][q] = NOX ? 1.0 : ldx64(x + pos[q] + d);
    }
  };
  auto consume = [&](int o, double (&a)[NB][RPT], double (&v)[NB][RPT]) {
#pragma unroll
    for (int u = 0; u < NB; ++u)
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const double w = (o + u < NL) ? a[u][q] : 0.0;
        if (u & 1) s1[q] = fma(w, v[u][q], s1[q]);
        else s0[q] = fma(w, v[u][q], s0[q]);
      }
  };
  if (DB) {
    double a0[NB][RPT], v0[NB][RPT], a1[NB][RPT], v1[NB][RPT];
    issue(0, a0, v0);
    for (int o = 0; o < S; o += 2 * NB) {
      issue(o + NB, a1, v1);
      consume(o, a0, v0);
      if (o + 2 * NB < S) issue(o + 2 * NB, a0, v0);
      consume(o + NB, a1, v1);
    }
  } else {
    for (int o = 0; o < NL; o += NB) {
      double a[NB][RPT], v[NB][RPT];
      issue(o, a, v);
      consume(o, a, v);
    }
  }
#pragma unroll
  for (int q = 0; q < RPT; ++q)
    if (ok[q]) {
      const double diag = c[(long long)CEN * ldo + q];
      x[pos[q]] += (__ldcs(b + pos[q]) - (s0[q] + s1[q])) / diag;
    }
}

// ---- cluster-persistent sweep: one cluster per patch, all 64 phases in one launch -----------------
// phases separated by barrier.cluster (release / acquire: the acquire invalidates this SM's L1, so
// the other CTAs' x updates are seen)
template <int NB, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_sweep_cluster(const double *__restrict__ coef, double *x,
                                                          const double *__restrict__ b, int p0) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int cs = (int)cl.num_blocks(), cr = (int)cl.block_rank();
  const int patch = p0 + blockIdx.x / cs;
  __shared__ int dl[S + NB];
  const long long vo = G.guard + (long long)patch * BOX;
  const long long ld = G.ld;
  for (int colour = 0; colour < NCOL; ++colour) {
    for (int o = threadIdx.x; o < S + NB; o += NT) dl[o] = (o < S) ? sl_delta(colour, o) : 0;
    __syncthreads();
    const int nr = G.cn[colour][0] * G.cn[colour][1] * G.cn[colour][2];
    const int rb = nr * cr / cs, re = nr * (cr + 1) / cs;
    for (int j = rb + threadIdx.x; j < re; j += NT) {
      const double *c = coef + (long long)patch * S * ld + G.cstart[colour] + j;
      const long long pos = vo + rowpos(colour, j);
      double s0 = 0, s1 = 0;
      for (int o = 0; o < S; o += NB) {
        double a[NB], v[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int oo = (o + u < S) ? o + u : 0;
          a[u] = ldcs64(c + oo * ld);
          v[u] = ldx64(x + pos + dl[o + u]);
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const double w = (o + u < S) ? a[u] : 0.0;
          if (u & 1) s1 = fma(w, v[u], s1);
          else s0 = fma(w, v[u], s0);
        }
      }
      x[pos] += (__ldcs(b + pos) - (s0 + s1)) / c[(long long)CEN * ld];
    }
    cl.sync();
  }
}

__global__ void k_init(double *coef, long long n, int ld) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long o = (i / ld) % S;
    unsigned h = (unsigned)(i * 2654435761ull);
    coef[i] = (o == CEN) ? 1.0 : 1e-4 * ((h >> 8) * (1.0 / 16777216.0) - 0.5);
  }
}

static double half_rows_bytes = 0;   // per patch: algorithmic bytes of one HALF sweep

int main(int argc, char **argv) {
  const int npatch = argc > 1 ? atoi(argv[1]) : 256;
  const int reps = argc > 2 ? atoi(argv[2]) : 6;
  Geo g{};
  g.npatch = npatch;
  int start = 0;
  for (int c = 0; c < NCOL; ++c) {
    int cc = c, tot = 1;
    for (int d = 0; d < 3; ++d) {
      const int cd = cc % P1;
      cc /= P1;
      g.cn[c][d] = (M - cd + P) / P1;
      tot *= g.cn[c][d];
    }
    g.cstart[c] = start;
    start += (tot + 127) / 128 * 128;   // colour starts on 128-row tiles (TILE variants, rpt2)
  }
  g.ld = (start + 31) / 32 * 32;
  {
    std::vector<short> ord((size_t)NCOL * S), ord2((size_t)NCOL * S);
    for (int c = 0; c < NCOL; ++c) {
      std::vector<std::pair<int, int>> key;
      for (int o = 0; o < S; ++o) {
        int cc = c, oo = o, tc = 0, sk = 0, pw = 1, pw3 = 1;
        for (int d = 0; d < 3; ++d) {
          const int cd = cc % P1, od = oo % W1 - P;
          cc /= P1;
          oo /= W1;
          const int s = cd + od, sh = (s < 0) ? -1 : (s >= P1 ? 1 : 0);
          tc += (s - sh * P1) * pw;
          sk += (sh + 1) * pw3;
          pw *= P1;
          pw3 *= 3;
        }
        key.push_back({tc * 27 + sk, o});
      }
      std::sort(key.begin(), key.end());
      for (int i = 0; i < S; ++i) ord[(size_t)c * S + i] = (short)key[i].second;
      // ORD2: groups of equal target colour; 8 slots, each emits one member per batch and takes
      // the next group when its group is exhausted (partners land exactly one batch apart)
      std::vector<std::vector<int>> grp;
      for (int i = 0; i < S; ++i) {
        if (i == 0 || key[i].first / 27 != key[i - 1].first / 27) grp.emplace_back();
        grp.back().push_back(key[i].second);
      }
      std::stable_sort(grp.begin(), grp.end(), [](const std::vector<int> &u, const std::vector<int> &v) { return u.size() > v.size(); });
      std::vector<int> seq;
      size_t next = 0;
      std::vector<std::pair<int, int>> slot(8, {-1, 0});
      while ((int)seq.size() < S) {
        for (auto &sl : slot) {
          if (sl.first < 0 || sl.second >= (int)grp[sl.first].size()) {
            sl = {-1, 0};
            if (next < grp.size()) sl = {(int)next++, 0};
          }
          if (sl.first >= 0) seq.push_back(grp[sl.first][sl.second++]);
        }
      }
      for (int i = 0; i < S; ++i) ord2[(size_t)c * S + i] = (short)seq[i];
    }
    CK(cudaMemcpyToSymbol(g_ord, ord.data(), ord.size() * sizeof(short)));
    CK(cudaMemcpyToSymbol(g_ord2, ord2.data(), ord2.size() * sizeof(short)));
    std::vector<short> low((size_t)NCOL * S, 0);
    std::vector<int> nlow(NCOL, 0);
    half_rows_bytes = 0;
    for (int c = 0; c < NCOL; ++c) {
      for (int o = 0; o < S; ++o) {
        int cc = c, oo = o, tc = 0, pw = 1;
        for (int d = 0; d < 3; ++d) {
          const int cd = cc % P1, od = oo % W1 - P;
          cc /= P1;
          oo /= W1;
          const int s2 = cd + od, sh = (s2 < 0) ? -1 : (s2 >= P1 ? 1 : 0);
          tc += (s2 - sh * P1) * pw;
          pw *= P1;
        }
        if (tc < c) low[(size_t)c * S + nlow[c]++] = (short)o;
      }
      int cc = c, tot = 1;
      for (int d = 0; d < 3; ++d) { tot *= (M - cc % P1 + P) / P1; cc /= P1; }
      half_rows_bytes += (double)tot * (nlow[c] + 3) * 8.0;
    }
    CK(cudaMemcpyToSymbol(g_low, low.data(), low.size() * sizeof(short)));
    CK(cudaMemcpyToSymbol(g_nlow, nlow.data(), nlow.size() * sizeof(int)));
  }
  g.guard = BOX;
  CK(cudaMemcpyToSymbol(G, &g, sizeof g));
  const long long ncoef = (long long)npatch * S * g.ld;
  const long long nvec = (long long)npatch * BOX + 2 * g.guard;
  double *coef, *x, *b;
  CK(cudaMalloc(&coef, ncoef * 8));
  CK(cudaMalloc(&x, nvec * 8));
  CK(cudaMalloc(&b, nvec * 8));
  CK(cudaMemset(x, 0, nvec * 8));
  CK(cudaMemset(b, 0, nvec * 8));
  k_init<<<148 * 16, 256>>>(coef, ncoef, g.ld);
  {
    std::vector<double> hb(nvec, 0.0);
    for (long long i = g.guard; i < nvec - g.guard; ++i) hb[i] = 1.0;
    CK(cudaMemcpy(b, hb.data(), nvec * 8, cudaMemcpyHostToDevice));
  }
  CK(cudaDeviceSynchronize());
  int rows_tot = 0;
  for (int c = 0; c < NCOL; ++c) rows_tot += g.cn[c][0] * g.cn[c][1] * g.cn[c][2];
  const double bytes_sweep = (double)npatch * rows_tot * (S + 3) * 8.0;
  printf("# npatch %d rows/patch %d ld %d coef %.1f GB, bytes per sweep %.2f GB\n", npatch, rows_tot, g.ld,
         ncoef * 8e-9, bytes_sweep * 1e-9);
  cudaStream_t st[2];
  CK(cudaStreamCreateWithFlags(&st[0], cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&st[1], cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // one sweep = 64 colour phases over `ngroups` sequential (or concurrent) patch groups
  auto launch_phase = [&](auto kern, int rpt, bool pdl, int colour, int p0, int np, cudaStream_t s) {
    const int nr = g.cn[colour][0] * g.cn[colour][1] * g.cn[colour][2];
    const int nbpp = (nr + 128 * rpt - 1) / (128 * rpt);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(np * nbpp));
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, kern, (const double *)coef, x, (const double *)b, colour, p0, nbpp));
  };
  double bytes_run = 0;   // 0: a full sweep's bytes
  auto run = [&](const char *name, auto sweep) {
    // capture one sweep in a graph (as the library does), then replay
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st[0], cudaStreamCaptureModeGlobal));
    sweep(st[0]);
    CK(cudaStreamEndCapture(st[0], &gr));
    CK(cudaGraphInstantiate(&ge, gr, 0));
    for (int w = 0; w < 2; ++w) CK(cudaGraphLaunch(ge, st[0]));
    CK(cudaStreamSynchronize(st[0]));
    CK(cudaEventRecord(e0, st[0]));
    for (int r = 0; r < reps; ++r) CK(cudaGraphLaunch(ge, st[0]));
    CK(cudaEventRecord(e1, st[0]));
    CK(cudaStreamSynchronize(st[0]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double t = ms * 1e-3 / reps;
    const double by = bytes_run > 0 ? bytes_run : bytes_sweep;
    printf("%-34s sweep %8.3f ms  phase %7.2f us  %7.1f GB/s\n", name, t * 1e3, t * 1e6 / NCOL, by / t * 1e-9);
    fflush(stdout);
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(gr));
  };
  const std::string only = argc > 3 ? argv[3] : "";
  auto want = [&](const char *n) { return only.empty() || only.find(n) != std::string::npos; };

  for (int ng : {1, 2, 4}) {
    const int per = (npatch + ng - 1) / ng;
    char nm[64];
    auto grouped = [&](auto kern, int rpt, bool pdl) {
      return [=, &launch_phase](cudaStream_t s) {
        for (int gi = 0; gi < ng; ++gi)
          for (int c = 0; c < NCOL; ++c)
            launch_phase(kern, rpt, pdl, c, gi * per, std::min(per, npatch - gi * per), s);
      };
    };
    if (want("nb8")) {
      snprintf(nm, sizeof nm, "nb8 rpt1 groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, false>, 1, false));
    }
    if (want("pdl")) {
      snprintf(nm, sizeof nm, "nb8 rpt1 pdl groups%d", ng);
      run(nm, grouped(k_phase<8, 1, true, false, false>, 1, true));
    }
    if (want("nb16")) {
      snprintf(nm, sizeof nm, "nb16 rpt1 groups%d", ng);
      run(nm, grouped(k_phase<16, 1, false, false, false>, 1, false));
    }
    if (want("rpt2")) {
      snprintf(nm, sizeof nm, "nb8 rpt2 groups%d", ng);
      run(nm, grouped(k_phase<8, 2, false, false, false>, 2, false));
    }
    if (want("db")) {
      snprintf(nm, sizeof nm, "nb8 rpt1 DB groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, true>, 1, false));
      snprintf(nm, sizeof nm, "nb4 rpt2 DB groups%d", ng);
      run(nm, grouped(k_phase<4, 2, false, false, true>, 2, false));
      snprintf(nm, sizeof nm, "nb16 rpt1 DB groups%d", ng);
      run(nm, grouped(k_phase<16, 1, false, false, true>, 1, false));
    }
    if (want("tile")) {
      snprintf(nm, sizeof nm, "nb8 rpt1 TILE32 groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, false, 32>, 1, false));
      snprintf(nm, sizeof nm, "nb8 rpt1 TILE128 groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, false, 128>, 1, false));
      snprintf(nm, sizeof nm, "nb8 rpt2 TILE64 groups%d", ng);
      run(nm, grouped(k_phase<8, 2, false, false, false, 64>, 2, false));
      snprintf(nm, sizeof nm, "nb16 rpt1 TILE32 groups%d", ng);
      run(nm, grouped(k_phase<16, 1, false, false, false, 32>, 1, false));
      snprintf(nm, sizeof nm, "nb8 rpt1 NO-X TILE32 groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, true, false, 32>, 1, false));
    }
    if (want("ord")) {
      snprintf(nm, sizeof nm, "nb8 rpt1 ORD groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, false, 0, 1>, 1, false));
      snprintf(nm, sizeof nm, "nb8 rpt1 ORD TILE32 groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, false, 32, 1>, 1, false));
      snprintf(nm, sizeof nm, "nb16 rpt1 ORD TILE32 groups%d", ng);
      run(nm, grouped(k_phase<16, 1, false, false, false, 32, 1>, 1, false));
    }
    if (want("ord2")) {
      snprintf(nm, sizeof nm, "nb8 rpt1 ORD2 groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, false, 0, 2>, 1, false));
      snprintf(nm, sizeof nm, "nb8 rpt1 ORD2 TILE32 groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, false, false, 32, 2>, 1, false));
    }
    if (want("nox")) {
      snprintf(nm, sizeof nm, "nb8 rpt1 NO-X groups%d", ng);
      run(nm, grouped(k_phase<8, 1, false, true, false>, 1, false));
    }
    auto conc_run = [&](const char *nm0, auto kern) {
      snprintf(nm, sizeof nm, "%s concurrent groups%d", nm0, ng);
      run(nm, [&](cudaStream_t s) {
        cudaEvent_t f, j[4];
        CK(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
        CK(cudaEventRecord(f, s));
        std::vector<cudaStream_t> ss(ng);
        for (int gi = 0; gi < ng; ++gi) {
          CK(cudaStreamCreateWithFlags(&ss[gi], cudaStreamNonBlocking));
          CK(cudaStreamWaitEvent(ss[gi], f, 0));
          for (int c = 0; c < NCOL; ++c)
            launch_phase(kern, 1, false, c, gi * per, std::min(per, npatch - gi * per), ss[gi]);
          CK(cudaEventCreateWithFlags(&j[gi], cudaEventDisableTiming));
          CK(cudaEventRecord(j[gi], ss[gi]));
          CK(cudaStreamWaitEvent(s, j[gi], 0));
        }
      });
    };
    if (want("chain") && ng > 1) {
      conc_run("nb8 rpt1 TILE32 chain1", k_phase<8, 1, false, false, false, 32, 0, 1>);
      conc_run("nb8 rpt1 TILE32 chain4", k_phase<8, 1, false, false, false, 32, 0, 4>);
    }
    if (want("half") && ng > 1) {
      bytes_run = half_rows_bytes * npatch;
      conc_run("nb8 rpt1 TILE32 HALF", k_phase<8, 1, false, false, false, 32, 0, 0, true>);
      bytes_run = 0;
    }
    if (want("cord") && ng > 1) {
      conc_run("nb8 rpt1 TILE32", k_phase<8, 1, false, false, false, 32, 0>);
      conc_run("nb8 rpt1 ORD2", k_phase<8, 1, false, false, false, 0, 2>);
      conc_run("nb8 rpt1 ORD2 TILE32", k_phase<8, 1, false, false, false, 32, 2>);
    }
    if (want("conc") && ng > 1) {
      // groups concurrently: group gi on a forked stream (graph branches)
      snprintf(nm, sizeof nm, "nb8 rpt1 concurrent groups%d", ng);
      run(nm, [&](cudaStream_t s) {
        cudaEvent_t f, j[4];
        CK(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
        CK(cudaEventRecord(f, s));
        std::vector<cudaStream_t> ss(ng);
        for (int gi = 0; gi < ng; ++gi) {
          CK(cudaStreamCreateWithFlags(&ss[gi], cudaStreamNonBlocking));
          CK(cudaStreamWaitEvent(ss[gi], f, 0));
          for (int c = 0; c < NCOL; ++c)
            launch_phase(k_phase<8, 1, false, false, false>, 1, false, c, gi * per, std::min(per, npatch - gi * per), ss[gi]);
          CK(cudaEventCreateWithFlags(&j[gi], cudaEventDisableTiming));
          CK(cudaEventRecord(j[gi], ss[gi]));
          CK(cudaStreamWaitEvent(s, j[gi], 0));
        }
      });
    }
  }
  auto cluster_run = [&](const char *nm0, auto kern, int nt, int cs, int ng) {
    const int per = (npatch + ng - 1) / ng;
    char nm[96];
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, nt, 0));
    snprintf(nm, sizeof nm, "%s cs%d nt%d g%d (%d/SM)", nm0, cs, nt, ng, nb);
    run(nm, [&](cudaStream_t s) {
      for (int gi = 0; gi < ng; ++gi) {
        const int np = std::min(per, npatch - gi * per);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(np * cs));
        cfg.blockDim = dim3(nt);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, kern, (const double *)coef, x, (const double *)b, gi * per));
      }
    });
  };
  if (want("clu")) {
    for (int ng : {1, 2}) {
      cluster_run("clu nb8 r80", k_sweep_cluster<8, 128, 6>, 128, 6, ng);
      cluster_run("clu nb8 r64", k_sweep_cluster<8, 128, 8>, 128, 6, ng);
      cluster_run("clu nb8 r64", k_sweep_cluster<8, 128, 8>, 128, 8, ng);
      cluster_run("clu nb16 r128", k_sweep_cluster<16, 128, 4>, 128, 6, ng);
      cluster_run("clu nb16 r80", k_sweep_cluster<16, 128, 6>, 128, 6, ng);
      cluster_run("clu nb8 r64", k_sweep_cluster<8, 192, 5>, 192, 4, ng);
      cluster_run("clu nb8 r64", k_sweep_cluster<8, 256, 4>, 256, 3, ng);
      cluster_run("clu nb8 r64", k_sweep_cluster<8, 96, 10>, 96, 8, ng);
    }
  }
  if (want("check")) {
    // bitwise: one sweep from the same x by the per-phase kernel and by the cluster kernel
    std::vector<double> h1(nvec), h2(nvec);
    CK(cudaMemset(x, 0, nvec * 8));
    for (int c = 0; c < NCOL; ++c) launch_phase(k_phase<8, 1, false, false, false>, 1, false, c, 0, npatch, st[0]);
    CK(cudaStreamSynchronize(st[0]));
    CK(cudaMemcpy(h1.data(), x, nvec * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(x, 0, nvec * 8));
    {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(npatch * 6));
      cfg.blockDim = dim3(128);
      cfg.stream = st[0];
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 6;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k_sweep_cluster<8, 128, 8>, (const double *)coef, x, (const double *)b, 0));
    }
    CK(cudaStreamSynchronize(st[0]));
    CK(cudaMemcpy(h2.data(), x, nvec * 8, cudaMemcpyDeviceToHost));
    long long diff = 0;
    double mx = 0;
    for (long long i = 0; i < nvec; ++i)
      if (h1[i] != h2[i]) {
        ++diff;
        mx = std::max(mx, std::abs(h1[i] - h2[i]));
      }
    printf("check: cluster sweep vs per-phase sweep: %lld of %lld entries differ (max %.3e)\n", diff, nvec, mx);
  }
  // plain stream reference: read the whole coefficient pool once (no gathers)
  return 0;
}
