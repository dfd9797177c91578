// Covisibility clustering of cameras for the PoST clustered solve
// (reference clustering.cluster_cameras, pkg/src/powerba/clustering.py:49-101):
// edge weight = number of landmarks two cameras both observe; edges merged
// greedily heaviest first (ties on the smaller camera index pair) under a
// cluster-size cap with union-find; cluster ids ordered by smallest member.
// Host C++: one sort of the camera pairs instead of a Python Counter.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/poba.h"

namespace poba {
int fail(int code, const std::string& msg);
}

extern "C" int poba_cluster_cameras(int64_t n_cam, int64_t n_pt, int64_t n_obs, const int64_t* cam_idx,
                                    const int64_t* pt_idx, int64_t max_cluster_size, int64_t* assignment,
                                    int64_t* n_clusters, int64_t* cut_observations) {
  if (max_cluster_size < 1) return poba::fail(POBA_EINVAL, "max_cluster_size must be at least 1");
  if (n_cam <= 0 || n_pt <= 0 || n_obs <= 0 || !cam_idx || !pt_idx || !assignment || !n_clusters ||
      !cut_observations)
    return poba::fail(POBA_EINVAL, "bad arguments");
  // observations grouped by landmark, cameras in file order inside each landmark
  // (np.lexsort((cam, pt)) sorts by point, then camera)
  std::vector<int64_t> order(n_obs);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return pt_idx[a] != pt_idx[b] ? pt_idx[a] < pt_idx[b] : cam_idx[a] < cam_idx[b];
  });
  for (int64_t i = 0; i < n_obs; ++i)
    if (cam_idx[i] < 0 || cam_idx[i] >= n_cam || pt_idx[i] < 0 || pt_idx[i] >= n_pt)
      return poba::fail(POBA_EINVAL, "camera or point index out of range");
  // every camera pair (ci < cj in landmark order, as the reference enumerates i < j) of every landmark
  std::vector<uint64_t> pairs;
  for (int64_t a = 0; a < n_obs;) {
    int64_t b = a;
    while (b < n_obs && pt_idx[order[b]] == pt_idx[order[a]]) ++b;
    for (int64_t i = a; i < b; ++i)
      for (int64_t j = i + 1; j < b; ++j)
        pairs.push_back(((uint64_t)cam_idx[order[i]] << 32) | (uint64_t)cam_idx[order[j]]);
    a = b;
  }
  std::sort(pairs.begin(), pairs.end());
  struct Edge {
    int64_t w;
    uint32_t ci, cj;
  };
  std::vector<Edge> edges;
  for (size_t a = 0; a < pairs.size();) {
    size_t b = a;
    while (b < pairs.size() && pairs[b] == pairs[a]) ++b;
    edges.push_back(Edge{(int64_t)(b - a), (uint32_t)(pairs[a] >> 32), (uint32_t)(pairs[a] & 0xffffffffu)});
    a = b;
  }
  std::vector<uint64_t>().swap(pairs);
  std::stable_sort(edges.begin(), edges.end(), [](const Edge& x, const Edge& y) {
    if (x.w != y.w) return x.w > y.w;
    if (x.ci != y.ci) return x.ci < y.ci;
    return x.cj < y.cj;
  });
  std::vector<int64_t> parent(n_cam), size(n_cam, 1);
  std::iota(parent.begin(), parent.end(), 0);
  auto find = [&](int64_t a) {
    while (parent[a] != a) {
      parent[a] = parent[parent[a]];
      a = parent[a];
    }
    return a;
  };
  for (const Edge& e : edges) {
    const int64_t ra = find(e.ci), rb = find(e.cj);
    if (ra == rb || size[ra] + size[rb] > max_cluster_size) continue;
    const int64_t keep = std::min(ra, rb), drop = std::max(ra, rb);
    parent[drop] = keep;
    size[keep] += size[drop];
  }
  std::vector<int64_t> root(n_cam), ids(n_cam, -1);
  for (int64_t c = 0; c < n_cam; ++c) root[c] = find(c);
  int64_t nc = 0;
  for (int64_t c = 0; c < n_cam; ++c)  // roots are the smallest member, so this orders ids by smallest member
    if (root[c] == c) ids[c] = nc++;
  for (int64_t c = 0; c < n_cam; ++c) assignment[c] = ids[root[c]];
  *n_clusters = nc;
  // observations of landmarks seen from more than one cluster
  int64_t cut = 0;
  for (int64_t a = 0; a < n_obs;) {
    int64_t b = a;
    bool multi = false;
    const int64_t first = assignment[cam_idx[order[a]]];
    while (b < n_obs && pt_idx[order[b]] == pt_idx[order[a]]) {
      multi |= assignment[cam_idx[order[b]]] != first;
      ++b;
    }
    if (multi) cut += b - a;
    a = b;
  }
  *cut_observations = cut;
  return POBA_OK;
}
