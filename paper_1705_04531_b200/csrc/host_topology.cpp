// host_topology.cpp -- host-side setup of libieti: knot validation, B-spline utilities,
// multipatch topology, primal constraints and the (scaled) jump operators.
//
//  * Cox-de Boor, Boehm knot insertion for the nested dyadic grids,
//    (p+1)-point Gauss-Legendre rule, 1D parameter mass.
//  * Interfaces: a side is an interface if every control point on it coincides (1e-10*diam)
//    with control points of one other patch; otherwise it is Dirichlet.
//  * Entities by codimension; primal constraints with
//    open-entity averages w_a ~ prod (t_{a+p+1} - t_a)/(p+1)  (reading R13).
//  * Multipliers: non-redundant chains, canonical order; B_D = (B_g B_g^T)^{-1} B_g (R12).
#include "internal.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <map>
#include <numeric>
#include <unordered_map>

// ---------------------------------------------------------------------------------------
// B-spline utilities
// ---------------------------------------------------------------------------------------
static int find_span(const std::vector<double> &t, int p, double x) {
  int M = (int)t.size() - p - 1;
  if (x >= t[M]) return M - 1;
  int lo = p, hi = M;   // t[lo] <= x < t[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) / 2;
    if (x < t[mid]) hi = mid; else lo = mid;
  }
  return lo;
}

// out[(k)*(p+1) + j] = d^k N_{span-p+j}(x), k = 0..nder
void bspline_basis_ders(const std::vector<double> &t, int p, double x, int nder, int &span, double *out) {
  span = find_span(t, p, x);
  std::vector<double> N((p + 1) * (p + 1), 0.0);          // N[q][j]: degree-q values (triangular)
  N[0] = 1.0;
  std::vector<double> val(p + 1, 0.0), prev(p + 1, 0.0);
  // degree-by-degree values on the span; keep all degrees for the derivative formula
  std::vector<std::vector<double>> lev(p + 1, std::vector<double>(p + 1, 0.0));
  lev[0][0] = 1.0;
  for (int q = 1; q <= p; ++q) {
    for (int j = 0; j <= q; ++j) {
      // function index i = span - q + j, degree q
      int i = span - q + j;
      double v = 0.0;
      if (j >= 1) {               // term with N_{i,q-1} = lev[q-1][j-1]
        double den = t[i + q] - t[i];
        if (den > 0) v += (x - t[i]) / den * lev[q - 1][j - 1];
      }
      if (j <= q - 1) {           // term with N_{i+1,q-1} = lev[q-1][j]
        double den = t[i + q + 1] - t[i + 1];
        if (den > 0) v += (t[i + q + 1] - x) / den * lev[q - 1][j];
      }
      lev[q][j] = v;
    }
  }
  for (int j = 0; j <= p; ++j) out[j] = lev[p][j];
  // derivatives: d^k N_{i,p} via the standard coefficient recursion on degree p-k values
  for (int k = 1; k <= nder; ++k) {
    int q = p - k;
    for (int j = 0; j <= p; ++j) {
      int i = span - p + j;
      // a_{k,l} coefficients:  d^k N_{i,p} = p!/(p-k)! sum_{l=0}^k a_{k,l} N_{i+l,p-k}
      std::vector<double> a(k + 1, 0.0), b(k + 1, 0.0);
      a[0] = 1.0;
      for (int kk = 1; kk <= k; ++kk) {
        std::fill(b.begin(), b.end(), 0.0);
        for (int l = 0; l <= kk; ++l) {
          double s = 0.0;
          if (l <= kk - 1) {
            double den = t[i + p - kk + 1 + l] - t[i + l];
            if (den > 0) s += a[l] / den;
          }
          if (l >= 1) {
            double den = t[i + p - kk + l + 1] - t[i + l];
            if (den > 0) s -= a[l - 1] / den;
          }
          b[l] = s;
        }
        a = b;
      }
      double d = 0.0;
      for (int l = 0; l <= k; ++l) {
        int ii = i + l;                     // N_{ii, q}; index within lev[q]: ii - (span - q)
        int jj = ii - (span - q);
        if (jj >= 0 && jj <= q) d += a[l] * lev[q][jj];
      }
      double fac = 1.0;
      for (int r = 0; r < k; ++r) fac *= (p - r);
      out[k * (p + 1) + j] = fac * d;
    }
  }
}

void gauss_legendre01(int n, double *x, double *w) {
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 1; j <= n; ++j) { double p2 = p1; p1 = p0; p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j; }
      double dp = n * (z * p0 - p1) / (z * z - 1.0);
      double dz = p0 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) {
        p0 = 1.0; p1 = 0.0;
        for (int j = 1; j <= n; ++j) { double p2 = p1; p1 = p0; p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j; }
        dp = n * (z * p0 - p1) / (z * z - 1.0);
        x[n - 1 - i] = 0.5 * (z + 1.0);
        w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);   // = 0.5 * 2/((1-z^2) P'^2)
        break;
      }
    }
  }
}

static std::vector<double> distinct(const std::vector<double> &t) {
  std::vector<double> u;
  for (double v : t) if (u.empty() || v != u.back()) u.push_back(v);
  return u;
}

std::vector<double> coarsen_knots(const std::vector<double> &t, int p) {
  std::vector<double> u = distinct(t);
  std::vector<double> tc;
  for (int i = 0; i < p; ++i) tc.push_back(t.front());
  for (size_t i = 0; i < u.size(); i += 2) tc.push_back(u[i]);
  for (int i = 0; i < p; ++i) tc.push_back(t.back());
  return tc;
}

// dense P (Mf x Mc), row-major, by repeated Boehm insertion of the knots of tf not in tc
std::vector<double> knot_insertion_dense(const std::vector<double> &tc, int p, const std::vector<double> &tf,
                                         int &Mf, int &Mc) {
  Mc = (int)tc.size() - p - 1;
  Mf = (int)tf.size() - p - 1;
  std::vector<double> extra;
  {
    size_t i = 0, j = 0;
    while (j < tf.size()) {
      if (i < tc.size() && tc[i] == tf[j]) { ++i; ++j; }
      else { extra.push_back(tf[j]); ++j; }
    }
  }
  std::vector<double> t = tc;
  int M = Mc;
  std::vector<double> P((size_t)M * Mc, 0.0);
  for (int i = 0; i < M; ++i) P[(size_t)i * Mc + i] = 1.0;
  for (double u : extra) {
    int k = find_span(t, p, u);
    std::vector<double> Pn((size_t)(M + 1) * Mc, 0.0);
    for (int i = 0; i <= M; ++i) {
      double a;
      if (i <= k - p) a = 1.0;
      else if (i >= k + 1) a = 0.0;
      else a = (u - t[i]) / (t[i + p] - t[i]);
      for (int c = 0; c < Mc; ++c) {
        double v = 0.0;
        if (i < M) v += a * P[(size_t)i * Mc + c];
        if (i >= 1) v += (1.0 - a) * P[(size_t)(i - 1) * Mc + c];
        Pn[(size_t)i * Mc + c] = v;
      }
    }
    t.insert(std::upper_bound(t.begin(), t.end(), u), u);
    P.swap(Pn);
    ++M;
  }
  return P;
}

std::vector<double> mass_1d(const std::vector<double> &t, int p) {
  int M = (int)t.size() - p - 1;
  std::vector<double> out((size_t)M * M, 0.0);
  std::vector<double> xg(p + 1), wg(p + 1), v((p + 1) * 2);
  gauss_legendre01(p + 1, xg.data(), wg.data());
  std::vector<double> u = distinct(t);
  for (size_t e = 0; e + 1 < u.size(); ++e) {
    double a = u[e], b = u[e + 1];
    for (int q = 0; q <= p; ++q) {
      double x = a + (b - a) * xg[q];
      int span;
      bspline_basis_ders(t, p, x, 0, span, v.data());
      for (int i = 0; i <= p; ++i)
        for (int j = 0; j <= p; ++j)
          out[(size_t)(span - p + i) * M + (span - p + j)] += (b - a) * wg[q] * v[i] * v[j];
    }
  }
  return out;
}

// ---------------------------------------------------------------------------------------
// topology
// ---------------------------------------------------------------------------------------
namespace {
struct DSU {
  std::vector<int> p;
  explicit DSU(int n) : p(n) { std::iota(p.begin(), p.end(), 0); }
  int find(int a) { while (p[a] != a) { p[a] = p[p[a]]; a = p[a]; } return a; }
  void unite(int a, int b) { a = find(a); b = find(b); if (a != b) p[std::max(a, b)] = std::min(a, b); }
};
struct Key3 {
  long long a, b, c;
  bool operator==(const Key3 &o) const { return a == o.a && b == o.b && c == o.c; }
};
struct Key3Hash {
  size_t operator()(const Key3 &k) const {
    uint64_t h = 1469598103934665603ull;
    for (long long v : {k.a, k.b, k.c}) { h ^= (uint64_t)v; h *= 1099511628211ull; }
    return (size_t)h;
  }
};
inline void unravel(long long flat, const int *M, int d, int *idx) {
  for (int k = 0; k < d; ++k) { idx[k] = (int)(flat % M[k]); flat /= M[k]; }
}
}  // namespace

// section timing of the host topology (stderr with IETI_VERBOSE=1)
static void topo_tick(const char *what) {
  static std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  const char *v = getenv("IETI_VERBOSE");
  if (v && v[0] == '1')
    fprintf(stderr, "[ieti topology] before section %s: +%.1f ms\n", what,
            std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

int build_topology(int dim, int n_patches, const int *degree, const int *n_knots, const double *knots,
                   const double *ctrl, unsigned primal, Topo &T) {
  T = Topo();
  T.dim = dim;
  T.n_patches = n_patches;
  if (dim < 2 || dim > 3 || n_patches < 1) { T.err = "dim must be 2 or 3 and n_patches >= 1"; return -1; }
  T.p = degree[0];
  // kernels are instantiated for p = 1..7 in 2D (Table 1's p = 7 rows) and 1..4 in 3D
  if (T.p < 1 || T.p > (dim == 2 ? 7 : 4)) { T.err = "degree must be in 1..7 (2D) / 1..4 (3D)"; return -9; }
  const double *kp = knots;
  const double *cp = ctrl;
  T.patch.resize(n_patches);
  for (int k = 0; k < n_patches; ++k) {
    HostPatch &P = T.patch[k];
    P.p = T.p;
    long long n = 1;
    for (int d = 0; d < 3; ++d) { P.M[d] = 1; P.melem[d] = 1; }
    for (int d = 0; d < dim; ++d) {
      if (degree[k * dim + d] != T.p) { T.err = "all patches/directions must share one degree"; return -9; }
      int nk = n_knots[k * dim + d];
      P.knots[d].assign(kp, kp + nk);
      kp += nk;
      const auto &t = P.knots[d];
      int p = T.p;
      if (nk < 2 * (p + 1)) { T.err = "too few knots"; return -1; }
      for (int i = 1; i < nk; ++i) if (t[i] < t[i - 1]) { T.err = "knot vector decreasing"; return -1; }
      for (int i = 1; i <= p; ++i)
        if (t[i] != t[0] || t[nk - 1 - i] != t[nk - 1]) { T.err = "knot vector not open"; return -1; }
      if (t[0] != 0.0 || t[nk - 1] != 1.0) { T.err = "knot vector must span [0,1]"; return -1; }
      for (int i = p + 1; i < nk - p - 1; ++i)
        if (t[i] == t[i - 1] || t[i] == t[i + 1]) { T.err = "interior knots must be simple"; return -9; }
      P.M[d] = nk - p - 1;
      P.melem[d] = nk - 2 * p - 1;
      if (P.M[d] < p + 1) { T.err = "M < p+1"; return -1; }
      n *= P.M[d];
    }
    P.ctrl.assign(cp, cp + n * dim);
    cp += n * dim;
  }
  topo_tick("0");
  // ---- geometric grouping of boundary dofs (hash grid) ----------------------------------
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (auto &P : T.patch)
    for (size_t i = 0; i < P.ctrl.size(); ++i) {
      int d = (int)(i % dim);
      lo[d] = std::min(lo[d], P.ctrl[i]);
      hi[d] = std::max(hi[d], P.ctrl[i]);
    }
  double diam = 0;
  for (int d = 0; d < dim; ++d) diam = std::max(diam, hi[d] - lo[d]);
  // cells much wider than tol (and far narrower than any mesh width): almost no point lies within tol of
  // a cell face, so almost every point probes its own cell only; which points unite does not depend on it
  const double tol = 1e-10 * diam, cell = 4096.0 * tol;
  std::vector<int> bk;            // patch
  std::vector<long long> bf;      // flat
  std::vector<double> bx;         // coords [3]
  for (int k = 0; k < n_patches; ++k) {
    const HostPatch &P = T.patch[k];
    long long n = 1;
    for (int d = 0; d < dim; ++d) n *= P.M[d];
    int idx[3];
    for (long long f = 0; f < n; ++f) {
      unravel(f, P.M, dim, idx);
      bool bnd = false;
      for (int d = 0; d < dim; ++d) bnd |= (idx[d] == 0 || idx[d] == P.M[d] - 1);
      if (!bnd) continue;
      bk.push_back(k);
      bf.push_back(f);
      for (int d = 0; d < 3; ++d) bx.push_back(d < dim ? P.ctrl[f * dim + d] : 0.0);
    }
  }
  const int nb = (int)bk.size();
  // cells of a uniform grid (edge 4 tol), the boundary points sorted by cell: the points of one cell are
  // one contiguous run (a sort + binary searches instead of a hash map of vectors: 1.8 M points on C5)
  struct CellPt { long long a, b, c; int i; };
  auto keyof = [&](int i, int dx, int dy, int dz) {
    return Key3{(long long)std::floor(bx[3 * i] / cell) + dx, (long long)std::floor(bx[3 * i + 1] / cell) + dy,
                (long long)std::floor(bx[3 * i + 2] / cell) + dz};
  };
  auto cell_less = [](const CellPt &u, const CellPt &v) {
    if (u.a != v.a) return u.a < v.a;
    if (u.b != v.b) return u.b < v.b;
    if (u.c != v.c) return u.c < v.c;
    return u.i < v.i;
  };
  std::vector<CellPt> cells(nb);
  for (int i = 0; i < nb; ++i) {
    const Key3 k = keyof(i, 0, 0, 0);
    cells[i] = CellPt{k.a, k.b, k.c, i};
  }
  std::sort(cells.begin(), cells.end(), cell_less);
  std::vector<int> run_end(nb);                 // by sorted position: end of the position's cell run
  std::vector<int> spos(nb);                    // point -> sorted position
  for (int q = nb - 1; q >= 0; --q) {
    const bool same = q + 1 < nb && cells[q].a == cells[q + 1].a && cells[q].b == cells[q + 1].b && cells[q].c == cells[q + 1].c;
    run_end[q] = same ? run_end[q + 1] : q + 1;
    spos[cells[q].i] = q;
  }
  topo_tick("0a");
  DSU dsu(nb);
  int zr = (dim == 3) ? 1 : 0;
  // a partner within tol can only sit in a neighbouring cell when the point is within tol of
  // that cell face: probe only those neighbours (the own cell only for almost every point)
  auto span = [&](double v, int &lo_, int &hi_) {
    const double f = v / cell - std::floor(v / cell);
    lo_ = (f * cell <= tol) ? -1 : 0;
    hi_ = ((1.0 - f) * cell <= tol) ? 1 : 0;
  };
  auto try_unite = [&](int i, int j) {
    if (j <= i) return;
    double s = 0;
    for (int d = 0; d < 3; ++d) { double q = bx[3 * i + d] - bx[3 * j + d]; s += q * q; }
    if (std::sqrt(s) <= tol) dsu.unite(i, j);
  };
  for (int i = 0; i < nb; ++i) {
    int xl, xh, yl, yh, zl, zh;
    span(bx[3 * i], xl, xh);
    span(bx[3 * i + 1], yl, yh);
    span(bx[3 * i + 2], zl, zh);
    if (!zr) zl = zh = 0;
    for (int dx = xl; dx <= xh; ++dx)
      for (int dy = yl; dy <= yh; ++dy)
        for (int dz = zl; dz <= zh; ++dz) {
          if (dx == 0 && dy == 0 && dz == 0) {
            // own cell: the rest of the run after i (members are sorted by point index)
            for (int q = spos[i] + 1; q < run_end[spos[i]]; ++q) try_unite(i, cells[q].i);
            continue;
          }
          const Key3 k = keyof(i, dx, dy, dz);
          const CellPt probe{k.a, k.b, k.c, -1};
          for (auto it = std::lower_bound(cells.begin(), cells.end(), probe, cell_less);
               it != cells.end() && it->a == k.a && it->b == k.b && it->c == k.c; ++it)
            try_unite(i, it->i);
        }
  }
  topo_tick("0b");
  std::map<int, std::vector<int>> groups_m;        // root -> member indices (ascending)
  for (int i = 0; i < nb; ++i) groups_m[dsu.find(i)].push_back(i);
  topo_tick("0c");
  // lookup (k, flat) -> boundary index
  std::vector<std::unordered_map<long long, int>> bidx(n_patches);
  for (int i = 0; i < nb; ++i) bidx[bk[i]][bf[i]] = i;
  std::vector<int> root(nb);
  for (int i = 0; i < nb; ++i) root[i] = dsu.find(i);
  for (auto &g : groups_m) {
    std::vector<int> ks;
    for (int i : g.second) ks.push_back(bk[i]);
    std::sort(ks.begin(), ks.end());
    if (std::adjacent_find(ks.begin(), ks.end()) != ks.end()) { T.err = "two dofs of one patch coincide"; return -3; }
  }
  topo_tick("1");
  // ---- sides ---------------------------------------------------------------------------
  T.floating.assign(n_patches, 0);
  T.dir_side.assign(n_patches, {0, 0, 0, 0, 0, 0});
  for (int k = 0; k < n_patches; ++k) {
    const HostPatch &P = T.patch[k];
    long long n = 1;
    for (int d = 0; d < dim; ++d) n *= P.M[d];
    int nd = 0;
    for (int d = 0; d < dim; ++d)
      for (int s = 0; s < 2; ++s) {
        std::vector<int> partners;
        bool first = true;
        // the points of side (d, s) only (P.M[e] = 1 for e >= dim), ascending flat index
        const int e1 = (d == 0) ? 1 : 0, e2 = (d == 2) ? 1 : 2;
        const long long st[3] = {1, P.M[0], (long long)P.M[0] * P.M[1]};
        const long long f0 = (s ? P.M[d] - 1 : 0) * st[d];
        for (long long q = 0; q < (long long)P.M[e1] * P.M[e2]; ++q) {
          const long long f = f0 + (q % P.M[e1]) * st[e1] + (q / P.M[e1]) * st[e2];
          std::vector<int> mates;
          for (int j : groups_m[root[bidx[k][f]]]) if (bk[j] != k) mates.push_back(bk[j]);
          std::sort(mates.begin(), mates.end());
          if (first) { partners = mates; first = false; }
          else {
            std::vector<int> tmp;
            std::set_intersection(partners.begin(), partners.end(), mates.begin(), mates.end(), std::back_inserter(tmp));
            partners.swap(tmp);
          }
          if (partners.empty()) break;
        }
        if (partners.empty()) { T.dir_side[k][2 * d + s] = 1; ++nd; }
      }
    T.floating[k] = (nd == 0);
  }
  auto is_active = [&](int k, long long f) {
    int idx[3];
    unravel(f, T.patch[k].M, dim, idx);
    for (int d = 0; d < dim; ++d) {
      if (idx[d] == 0 && T.dir_side[k][2 * d]) return false;
      if (idx[d] == T.patch[k].M[d] - 1 && T.dir_side[k][2 * d + 1]) return false;
    }
    return true;
  };
  topo_tick("2");
  // ---- Gamma lists ---------------------------------------------------------------------
  T.gamma.assign(n_patches, {});
  std::vector<std::unordered_map<long long, int>> gpos(n_patches);
  for (int k = 0; k < n_patches; ++k) {
    std::vector<long long> fl;
    for (auto &kv : bidx[k]) if (is_active(k, kv.first)) fl.push_back(kv.first);
    std::sort(fl.begin(), fl.end());
    for (size_t i = 0; i < fl.size(); ++i) { T.gamma[k].push_back((int)fl[i]); gpos[k][fl[i]] = (int)i; }
  }
  topo_tick("3");
  // ---- active groups and entities ----------------------------------------------------------
  struct Group { std::vector<std::pair<int, long long>> mem; int entity = -1; };
  std::vector<Group> G;
  for (auto &g : groups_m) {
    if (g.second.size() < 2) continue;
    int na = 0;
    for (int i : g.second) na += is_active(bk[i], bf[i]);
    if (na != 0 && na != (int)g.second.size()) { T.err = "non-conforming Dirichlet elimination at an interface"; return -3; }
    if (na == 0) continue;
    Group gr;
    for (int i : g.second) gr.mem.push_back({bk[i], bf[i]});
    std::sort(gr.mem.begin(), gr.mem.end());
    G.push_back(gr);
  }
  auto subcode = [&](int k, long long f, int &codim) {
    int idx[3];
    unravel(f, T.patch[k].M, dim, idx);
    int code = 0, pw = 1;
    codim = 0;
    for (int d = 0; d < dim; ++d) {
      int s = (idx[d] == 0) ? 0 : (idx[d] == T.patch[k].M[d] - 1 ? 1 : 2);
      if (s < 2) ++codim;
      code += s * pw;
      pw *= 3;
    }
    return code;
  };
  struct Entity { int kind; std::map<int, std::vector<long long>> mem; std::vector<int> groups; };
  std::map<std::vector<std::pair<int, int>>, int> ent_id;
  std::vector<Entity> E;
  for (size_t gi = 0; gi < G.size(); ++gi) {
    std::vector<std::pair<int, int>> key;
    int cd0 = -1;
    for (auto &m : G[gi].mem) {
      int cd;
      int c = subcode(m.first, m.second, cd);
      if (cd0 >= 0 && cd != cd0) { T.err = "non-conforming junction"; return -3; }
      cd0 = cd;
      key.push_back({m.first, c});
    }
    auto it = ent_id.find(key);
    int e;
    if (it == ent_id.end()) {
      e = (int)E.size();
      ent_id[key] = e;
      Entity en;
      en.kind = (cd0 == dim) ? 1 : ((dim == 3 && cd0 == 2) || (dim == 2 && cd0 == 1) ? 2 : 4);
      E.push_back(en);
    } else e = it->second;
    G[gi].entity = e;
    E[e].groups.push_back((int)gi);
    for (auto &m : G[gi].mem) E[e].mem[m.first].push_back(m.second);
  }
  topo_tick("4");
  // ---- primal entities, global order (k1, min flat in k1) ---------------------------------
  std::vector<int> prim;
  for (size_t e = 0; e < E.size(); ++e) {
    for (auto &kv : E[e].mem) std::sort(kv.second.begin(), kv.second.end());
    if (E[e].kind & primal) prim.push_back((int)e);
  }
  std::sort(prim.begin(), prim.end(), [&](int a, int b) {
    auto ka = std::make_pair(E[a].mem.begin()->first, E[a].mem.begin()->second.front());
    auto kb = std::make_pair(E[b].mem.begin()->first, E[b].mem.begin()->second.front());
    return ka < kb;
  });
  T.n_pi = (int)prim.size();
  T.R.assign(n_patches, {});
  T.c_row.assign(n_patches, {});
  T.c_w.assign(n_patches, {});
  for (int k = 0; k < n_patches; ++k) {
    T.c_row[k].assign(T.gamma[k].size(), -1);
    T.c_w[k].assign(T.gamma[k].size(), 0.0);
  }
  std::vector<char> primal_vertex_group(G.size(), 0);
  for (int gid = 0; gid < T.n_pi; ++gid) {
    Entity &en = E[prim[gid]];
    if (en.kind == 1) for (int gi : en.groups) primal_vertex_group[gi] = 1;
    for (auto &kv : en.mem) {
      int k = kv.first;
      int row = (int)T.R[k].size();
      T.R[k].push_back(gid);
      // weights (R13)
      std::vector<double> w(kv.second.size(), 1.0);
      double sum = 0;
      for (size_t j = 0; j < kv.second.size(); ++j) {
        int idx[3];
        unravel(kv.second[j], T.patch[k].M, dim, idx);
        int cd;
        int code = subcode(k, kv.second[j], cd);
        for (int d = 0; d < dim; ++d) {
          int s = (code / (d == 0 ? 1 : (d == 1 ? 3 : 9))) % 3;
          if (s == 2) {
            const auto &t = T.patch[k].knots[d];
            w[j] *= (t[idx[d] + T.p + 1] - t[idx[d]]) / (T.p + 1);
          }
        }
        sum += w[j];
      }
      for (size_t j = 0; j < kv.second.size(); ++j) {
        int gp = gpos[k].at(kv.second[j]);
        T.c_row[k][gp] = row;
        T.c_w[k][gp] = w[j] / sum;
      }
    }
  }
  topo_tick("5");
  // ---- multipliers (R12) -------------------------------------------------------------------
  struct Row { int k1; long long a1; int i; int g; };
  std::vector<Row> rows;
  for (size_t gi = 0; gi < G.size(); ++gi) {
    if (primal_vertex_group[gi]) continue;
    auto &m = G[gi].mem;
    for (size_t i = 0; i + 1 < m.size(); ++i) rows.push_back({m[0].first, m[0].second, (int)i, (int)gi});
  }
  std::sort(rows.begin(), rows.end(), [](const Row &a, const Row &b) {
    if (a.k1 != b.k1) return a.k1 < b.k1;
    if (a.a1 != b.a1) return a.a1 < b.a1;
    return a.i < b.i;
  });
  T.n_lambda = (int)rows.size();
  // (group, chain position) -> multiplier row: one flat table (prefix sums of the chain lengths)
  std::vector<long long> row_base(G.size() + 1, 0);
  for (size_t gi = 0; gi < G.size(); ++gi)
    row_base[gi + 1] = row_base[gi] + (primal_vertex_group[gi] ? 0 : (long long)G[gi].mem.size() - 1);
  std::vector<int> row_tab((size_t)row_base[G.size()], -1);
  for (int r = 0; r < T.n_lambda; ++r) row_tab[(size_t)(row_base[rows[r].g] + rows[r].i)] = r;
  auto row_of = [&](int gi, int i) { return row_tab[(size_t)(row_base[gi] + i)]; };
  T.mkp.resize(T.n_lambda); T.map_.resize(T.n_lambda); T.mkm.resize(T.n_lambda); T.mam.resize(T.n_lambda);
  T.bd_ptr.assign(T.n_lambda + 1, 0);
  std::vector<std::vector<std::tuple<int, int, double>>> bd_rows(T.n_lambda);
  std::vector<std::vector<std::vector<std::pair<int, double>>>> bt(n_patches), bdt(n_patches);
  for (int k = 0; k < n_patches; ++k) { bt[k].resize(T.gamma[k].size()); bdt[k].resize(T.gamma[k].size()); }
  for (int r = 0; r < T.n_lambda; ++r) {
    auto &m = G[rows[r].g].mem;
    int i = rows[r].i;
    T.mkp[r] = m[i].first; T.map_[r] = (int)m[i].second;
    T.mkm[r] = m[i + 1].first; T.mam[r] = (int)m[i + 1].second;
  }
  for (size_t gi = 0; gi < G.size(); ++gi) {
    if (primal_vertex_group[gi]) continue;
    auto &m = G[gi].mem;
    int mm = (int)m.size();
    // W = (B_g B_g^T)^{-1}, B_g B_g^T = tridiag(-1, 2, -1) of size mm-1: closed-form inverse
    // W[i][j] = min(i+1, j+1) * (mm - max(i+1, j+1)) / mm
    int n1 = mm - 1;
    for (int i = 0; i < n1; ++i) {
      int r = row_of((int)gi, i);
      for (int c = 0; c < mm; ++c) {
        // (W B_g)[i][c] = W[i][c] - W[i][c-1]  (B_g[j][c] = +1 if j == c, -1 if j == c-1)
        double v = 0.0;
        if (c < n1) v += (double)std::min(i + 1, c + 1) * (mm - std::max(i + 1, c + 1)) / mm;
        if (c >= 1) v -= (double)std::min(i + 1, c) * (mm - std::max(i + 1, c)) / mm;
        bd_rows[r].push_back({m[c].first, (int)m[c].second, v});
        int gp = gpos[m[c].first].at(m[c].second);
        bdt[m[c].first][gp].push_back({r, v});
      }
    }
    for (int c = 0; c < mm; ++c) {
      int k = m[c].first;
      int gp = gpos[k].at(m[c].second);
      if (c < n1) bt[k][gp].push_back({row_of((int)gi, c), +1.0});
      if (c >= 1) bt[k][gp].push_back({row_of((int)gi, c - 1), -1.0});
    }
  }
  for (int r = 0; r < T.n_lambda; ++r) {
    T.bd_ptr[r + 1] = T.bd_ptr[r] + (int)bd_rows[r].size();
    for (auto &e : bd_rows[r]) { T.bd_k.push_back(std::get<0>(e)); T.bd_a.push_back(std::get<1>(e)); T.bd_w.push_back(std::get<2>(e)); }
  }
  T.bt_ptr.assign(n_patches, {}); T.bt_m.assign(n_patches, {}); T.bt_w.assign(n_patches, {});
  T.bdt_ptr.assign(n_patches, {}); T.bdt_m.assign(n_patches, {}); T.bdt_w.assign(n_patches, {});
  for (int k = 0; k < n_patches; ++k) {
    T.bt_ptr[k].push_back(0);
    T.bdt_ptr[k].push_back(0);
    for (size_t g = 0; g < T.gamma[k].size(); ++g) {
      auto l = bt[k][g];
      std::sort(l.begin(), l.end());
      for (auto &e : l) { T.bt_m[k].push_back(e.first); T.bt_w[k].push_back(e.second); }
      T.bt_ptr[k].push_back((int)T.bt_m[k].size());
      auto l2 = bdt[k][g];
      std::sort(l2.begin(), l2.end());
      for (auto &e : l2) { T.bdt_m[k].push_back(e.first); T.bdt_w[k].push_back(e.second); }
      T.bdt_ptr[k].push_back((int)T.bdt_m[k].size());
    }
  }
  topo_tick("end");
  return 0;
}
