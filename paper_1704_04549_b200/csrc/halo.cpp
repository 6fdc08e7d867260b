// Element partition and face-neighbour halo plan for multi-rank runs (host only).
//
// Rank r owns the contiguous element range [E r / N, E (r+1) / N): element rows in 2D and slabs in
// 3D, because the reference numbers elements e = (k ny + j) nx + i (reference dg/mesh.hpp:312).
// The only cross-element data dependence of the hot path is the neighbour trace inside
// jacobian_apply (ops/linearized.hpp:216-236, ops/discretization.hpp:170-181), and with
// Gauss-Lobatto nodes that trace is the neighbour's face node layer (discretization.hpp:89-97):
// a rank needs, per cut face, n_c q^(d-1) values of the off-rank neighbour, not its element block.
// Off-rank neighbours still get a halo slot (an element-block-sized place where the layers they
// contribute are written, so the operator kernels address them like local neighbours); slots are
// grouped by owner rank and sorted by global id. The owner sends the layers (element, face) of its
// faces whose neighbour is on the receiving rank, ordered by (global element, face); the receiver
// lists the layers it needs, (neighbour, neighbour face), in the same order. Face adjacency is
// symmetric (the neighbour of (nb, nf) is the requesting face), so both lists are the same set in
// the same order without any index exchange.
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
  std::vector<std::vector<int>> need(nranks);                      // remote neighbour elements per owner
  std::vector<std::vector<std::pair<int, int>>> need_layer(nranks);  // (neighbour gid, neighbour face)
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
        need_layer[owner_of(int(nb))].push_back({int(nb), int(fc[1])});
      }
    }
  std::vector<std::pair<int, int>> gid_slot;
  int slot = 0;
  for (int r = 0; r < nranks; ++r) {
    auto& nd = need[r];
    std::sort(nd.begin(), nd.end());
    nd.erase(std::unique(nd.begin(), nd.end()), nd.end());
    for (int gid : nd) {
      gid_slot.push_back({gid, int(nl) + slot++});
      P.halo_gid.push_back(gid);
    }
  }
  std::sort(gid_slot.begin(), gid_slot.end());
  auto slot_of = [&](int gid) {
    return std::lower_bound(gid_slot.begin(), gid_slot.end(), std::make_pair(gid, -1))->second;
  };
  for (size_t i = 0; i < P.conn.size(); i += 3)
    if (P.conn[i] <= -2) P.conn[i] = slot_of(-2 - P.conn[i]);
  P.n_halo = slot;
  if (nranks > 1)
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      HaloPlan::Peer p;
      p.rank = r;
      auto& nlay = need_layer[r];
      std::sort(nlay.begin(), nlay.end());
      nlay.erase(std::unique(nlay.begin(), nlay.end()), nlay.end());
      for (const auto& gf : nlay) {
        p.recv_slot.push_back(slot_of(gf.first) - int(nl));
        p.recv_face.push_back(gf.second);
      }
      for (size_t le = 0; le < nl; ++le)  // ascending (gid, face): the peer's need list, by symmetry
        for (int f = 0; f < 2 * d; ++f) {
          const int64_t nb = sys->conn[((size_t(e_begin) + le) * 2 * d + f) * 3];
          if (nb >= 0 && (nb < e_begin || nb >= e_end) && owner_of(int(nb)) == r) {
            p.send_elem.push_back(int(le));
            p.send_face.push_back(f);
          }
        }
      if (!p.recv_slot.empty() || !p.send_elem.empty()) P.peers.push_back(std::move(p));
    }
  return P;
}

} // namespace tpdg_gpu
