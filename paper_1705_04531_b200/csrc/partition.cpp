// partition.cpp -- patch partition over ranks and the dual-vector exchange plan (multi-GPU).
//
// Patches are the unit of data parallelism (every local solve is per patch); the only
// couplings inside a dual-PCG iteration are the interface lambda / trace exchange, the coarse
// right-hand side and the PCG scalars.  Every rank builds the GLOBAL topology from
// the (replicated) geometry and then keeps a LOCAL view:
//   * local patches   = patches with owner[k] == rank, ascending global id;
//   * local multipliers M_r = multipliers of every dof group with a copy on a local patch
//     (these are the rows of B, B_D and the columns of B^T, B_D^T that touch local data),
//     ordered OWNED first (owner of a multiplier = owner of its k+ patch, R12), then GHOSTS,
//     each part in canonical order.
// Exchange plan (per peer q, lists in canonical order, identical on both sides by construction):
//   fwd_send[q] = my owned multipliers that are in M_q,   fwd_recv[q] = my ghosts owned by q
//   (owner -> ghost copies: before B^T p and B_D^T r);
//   the reverse exchange (ghost partial sums -> owner, after B w and B_D y) uses the same lists
//   with the roles swapped; the owner adds the received partials in ascending peer order.
#include "internal.h"

#include <algorithm>
#include <map>
#include <numeric>

std::vector<int> default_owner(int n_patches, int world) {
  std::vector<int> own(n_patches, 0);
  for (int r = 0; r < world; ++r) {
    const long long a = (long long)n_patches * r / world, b = (long long)n_patches * (r + 1) / world;
    for (long long k = a; k < b; ++k) own[k] = r;
  }
  return own;
}

// multipliers touching rank r's patches (global ids, ascending)
static std::vector<int> touching(const Topo &G, const std::vector<int> &owner, int r) {
  std::vector<int> out;
  for (int i = 0; i < G.n_lambda; ++i) {
    bool t = owner[G.mkp[i]] == r || owner[G.mkm[i]] == r;
    for (int e = G.bd_ptr[i]; e < G.bd_ptr[i + 1] && !t; ++e) t = owner[G.bd_k[e]] == r;
    if (t) out.push_back(i);
  }
  return out;
}

int build_partition(const Topo &G, const std::vector<int> &owner, int rank, int world, Topo &L, Plan &P) {
  if ((int)owner.size() != G.n_patches) { L.err = "patch_owner size mismatch"; return -1; }
  for (int o : owner)
    if (o < 0 || o >= world) { L.err = "patch_owner entry out of range"; return -1; }
  P = Plan();
  P.rank = rank;
  P.world = world;
  // local patches
  std::vector<int> lp_of(G.n_patches, -1);
  for (int k = 0; k < G.n_patches; ++k)
    if (owner[k] == rank) { lp_of[k] = (int)P.local_patches.size(); P.local_patches.push_back(k); }
  // local multipliers: owned first, then ghosts
  std::vector<std::vector<int>> Mq(world);
  for (int q = 0; q < world; ++q) Mq[q] = touching(G, owner, q);
  const std::vector<int> &Mr = Mq[rank];
  for (int i : Mr)
    if (owner[G.mkp[i]] == rank) P.local_mult.push_back(i);
  P.n_own = (int)P.local_mult.size();
  for (int i : Mr)
    if (owner[G.mkp[i]] != rank) P.local_mult.push_back(i);
  std::vector<int> lm_of(G.n_lambda, -1);
  for (size_t j = 0; j < P.local_mult.size(); ++j) lm_of[P.local_mult[j]] = (int)j;
  // exchange lists per peer
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    std::vector<int> snd, rcv;
    {
      // my owned in M_q (canonical order)
      std::vector<char> inq(G.n_lambda, 0);
      for (int i : Mq[q]) inq[i] = 1;
      for (int i : Mr)
        if (owner[G.mkp[i]] == rank && inq[i]) snd.push_back(lm_of[i]);
    }
    for (int i : Mr)
      if (owner[G.mkp[i]] == q) rcv.push_back(lm_of[i]);
    if (snd.empty() && rcv.empty()) continue;
    P.peers.push_back(q);
    P.send_ptr.push_back((int)P.send_idx.size());
    P.send_idx.insert(P.send_idx.end(), snd.begin(), snd.end());
    P.recv_ptr.push_back((int)P.recv_idx.size());
    P.recv_idx.insert(P.recv_idx.end(), rcv.begin(), rcv.end());
  }
  P.send_ptr.push_back((int)P.send_idx.size());
  P.recv_ptr.push_back((int)P.recv_idx.size());
  // reverse-exchange sum plan: for owned row j, received partial positions (in the recv
  // buffer of the reverse exchange = send layout of the forward one), ascending peer order
  P.rsum_ptr.assign(P.n_own + 1, 0);
  {
    std::vector<std::vector<int>> src(P.n_own);
    for (size_t pi = 0; pi < P.peers.size(); ++pi)
      for (int e = P.send_ptr[pi]; e < P.send_ptr[pi + 1]; ++e) src[P.send_idx[e]].push_back(e);
    for (int j = 0; j < P.n_own; ++j) {
      P.rsum_ptr[j + 1] = P.rsum_ptr[j] + (int)src[j].size();
      P.rsum_src.insert(P.rsum_src.end(), src[j].begin(), src[j].end());
    }
  }
  // ---- local topology view ----------------------------------------------------------------
  L = Topo();
  L.dim = G.dim;
  L.p = G.p;
  L.n_patches = (int)P.local_patches.size();
  for (int k : P.local_patches) {
    L.patch.push_back(G.patch[k]);
    L.floating.push_back(G.floating[k]);
    L.dir_side.push_back(G.dir_side[k]);
    L.gamma.push_back(G.gamma[k]);
    L.R.push_back(G.R[k]);
    L.c_row.push_back(G.c_row[k]);
    L.c_w.push_back(G.c_w[k]);
    // B^T and B_D^T lists: same entry order as the global tables (bitwise-identical sums)
    L.bt_ptr.push_back(G.bt_ptr[k]);
    L.bdt_ptr.push_back(G.bdt_ptr[k]);
    std::vector<int> m1, m2;
    for (int i : G.bt_m[k]) m1.push_back(lm_of[i]);
    for (int i : G.bdt_m[k]) m2.push_back(lm_of[i]);
    for (int v : m1)
      if (v < 0) { L.err = "internal: B^T entry outside the local multiplier set"; return -1; }
    for (int v : m2)
      if (v < 0) { L.err = "internal: B_D^T entry outside the local multiplier set"; return -1; }
    L.bt_m.push_back(m1);
    L.bt_w.push_back(G.bt_w[k]);
    L.bdt_m.push_back(m2);
    L.bdt_w.push_back(G.bdt_w[k]);
  }
  L.n_pi = G.n_pi;
  L.n_lambda = (int)P.local_mult.size();
  L.mkp.resize(L.n_lambda); L.map_.resize(L.n_lambda); L.mkm.resize(L.n_lambda); L.mam.resize(L.n_lambda);
  L.bd_ptr.assign(L.n_lambda + 1, 0);
  for (int j = 0; j < L.n_lambda; ++j) {
    const int i = P.local_mult[j];
    P.gkp.push_back(G.mkp[i]);
    P.gkm.push_back(G.mkm[i]);
    L.mkp[j] = lp_of[G.mkp[i]];          // -1 when the patch is remote
    L.map_[j] = G.map_[i];
    L.mkm[j] = lp_of[G.mkm[i]];
    L.mam[j] = G.mam[i];
    for (int e = G.bd_ptr[i]; e < G.bd_ptr[i + 1]; ++e) {
      const int lk = lp_of[G.bd_k[e]];
      if (lk < 0) continue;              // remote entries are summed on their own rank
      L.bd_k.push_back(lk);
      L.bd_a.push_back(G.bd_a[e]);
      L.bd_w.push_back(G.bd_w[e]);
    }
    L.bd_ptr[j + 1] = (int)L.bd_k.size();
  }
  return 0;
}
