// compute_topology (tree.py:205-239): neighbour lists (same-level cells at
// Chebyshev distance <= 1, sorted by id) and interaction lists (children of
// the parent's neighbours that are not neighbours, sorted).
#include <algorithm>
#include <unordered_map>

#include "engine.h"

namespace ifmm {

static inline uint64_t cell_key(long long x, long long y, long long z) {
  // 21 bits per axis (depth <= 12 in the reference, tree.py:110)
  return ((uint64_t)(x & 0x1fffff) << 42) | ((uint64_t)(y & 0x1fffff) << 21) |
         (uint64_t)(z & 0x1fffff);
}

void Tree::build_topology() {
  nbrs.assign(nc, {});
  inters.assign(nc, {});
  for (const auto& ids : levels) {
    std::unordered_map<uint64_t, int> where;
    where.reserve(ids.size() * 2);
    for (int c : ids) where[cell_key(cell[3 * c], cell[3 * c + 1], cell[3 * c + 2])] = c;
    for (int c : ids) {
      const long long x = cell[3 * c], y = cell[3 * c + 1], z = cell[3 * c + 2];
      auto& out = nbrs[c];
      for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dz = -1; dz <= 1; ++dz) {
            if (x + dx < 0 || y + dy < 0 || z + dz < 0) continue;
            auto it = where.find(cell_key(x + dx, y + dy, z + dz));
            if (it != where.end()) out.push_back(it->second);
          }
      std::sort(out.begin(), out.end());
    }
  }
  for (int l = 2; l <= depth; ++l)
    for (int c : levels[l]) {
      auto& out = inters[c];
      for (int pn : nbrs[parent[c]])
        for (int ch : children[pn])
          if (!adjacent(c, ch)) out.push_back(ch);
      std::sort(out.begin(), out.end());
    }
}

}  // namespace ifmm
