// Element partition and face-neighbour halo plan for multi-rank runs (host only).
//
// Rank r owns the contiguous element range [E r / N, E (r+1) / N): element rows in 2D and slabs in
// 3D, because the reference numbers elements e = (k ny + j) nx + i (reference dg/mesh.hpp:312).
// The only cross-element data dependence of the hot path is the neighbour trace inside
// jacobian_apply (ops/linearized.hpp:216-236, ops/discretization.hpp:170-181), so a rank needs
// the state blocks of the off-rank face neighbours of its elements: the halo. Halo slots are
// grouped by owner rank and sorted by global id; the owner sends exactly the elements that have
// a face neighbour on the receiving rank, in ascending order (face adjacency is symmetric), so
// send and receive orders agree without any index exchange.
#include <algorithm>
#include <string>
#include <vector>

#include "tpdg_internal.hpp"

namespace tpdg_gpu {

HaloPlan build_halo_plan(const tpdg_gpu_system* sys, int rank, int nranks, int e_begin, int e_end) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Failure{TPDG_CONFIG, "halo plan: bad rank / nranks"};
  const int d = sys->dim, E = sys->n_elements;
  std::vector<int> owner_lo(nranks + 1);
  for (int r = 0; r <= nranks; ++r) owner_lo[r] = int((int64_t(E) * r) / nranks);
  if (nranks > 1 && (e_begin != owner_lo[rank] || e_end != owner_lo[rank + 1]))
    throw Failure{TPDG_CONFIG, "multi-rank element range must be [E r / N, E (r+1) / N)"};
  auto owner_of = [&](int e) {
    const int r = int(std::upper_bound(owner_lo.begin(), owner_lo.end(), e) - owner_lo.begin()) - 1;
    return std::min(std::max(r, 0), nranks - 1);
  };
  HaloPlan P;
  P.e_begin = e_begin;
  P.e_end = e_end;
  const size_t nl = size_t(e_end - e_begin);
  P.conn.assign(nl * 2 * d * 3, 0);
  std::vector<std::vector<int>> need(nranks);
  for (size_t le = 0; le < nl; ++le)
    for (int f = 0; f < 2 * d; ++f) {
      const int64_t* fc = sys->conn + ((size_t(e_begin) + le) * 2 * d + f) * 3;
      int* out = &P.conn[(le * 2 * d + f) * 3];
      out[1] = int(fc[1]);
      out[2] = int(fc[2]);
      const int64_t nb = fc[0];
      if (nb < 0) {
        out[0] = -1;
      } else if (nb >= e_begin && nb < e_end) {
        out[0] = int(nb - e_begin);
      } else {
        if (nranks == 1) throw Failure{TPDG_CONFIG, "neighbour outside the local range needs nranks > 1"};
        out[0] = -2 - int(nb);
        need[owner_of(int(nb))].push_back(int(nb));
      }
    }
  std::vector<std::pair<int, int>> gid_slot;
  int slot = 0;
  for (int r = 0; r < nranks; ++r) {
    auto& nd = need[r];
    std::sort(nd.begin(), nd.end());
    nd.erase(std::unique(nd.begin(), nd.end()), nd.end());
    if (r == rank || nd.empty()) continue;
    HaloPlan::Peer p;
    p.rank = r;
    p.recv_first = slot;
    p.recv_count = int(nd.size());
    for (int gid : nd) {
      gid_slot.push_back({gid, int(nl) + slot++});
      P.halo_gid.push_back(gid);
    }
    P.peers.push_back(p);
  }
  std::sort(gid_slot.begin(), gid_slot.end());
  for (size_t i = 0; i < P.conn.size(); i += 3)
    if (P.conn[i] <= -2) {
      const int gid = -2 - P.conn[i];
      P.conn[i] = std::lower_bound(gid_slot.begin(), gid_slot.end(), std::make_pair(gid, -1))->second;
    }
  P.n_halo = slot;
  if (nranks > 1)
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      std::vector<int> send;
      for (size_t le = 0; le < nl; ++le)
        for (int f = 0; f < 2 * d; ++f) {
          const int64_t nb = sys->conn[((size_t(e_begin) + le) * 2 * d + f) * 3];
          if (nb >= 0 && (nb < e_begin || nb >= e_end) && owner_of(int(nb)) == r) {
            send.push_back(int(le));
            break;
          }
        }
      if (send.empty()) continue;
      auto it = std::find_if(P.peers.begin(), P.peers.end(), [&](const HaloPlan::Peer& p) { return p.rank == r; });
      if (it == P.peers.end()) {
        HaloPlan::Peer p;
        p.rank = r;
        P.peers.push_back(p);
        it = P.peers.end() - 1;
      }
      it->send_local = send;
    }
  return P;
}

} // namespace tpdg_gpu
