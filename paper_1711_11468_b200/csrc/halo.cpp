// z-slab halo exchange plan (see halo.hpp).
#include "halo.hpp"

#include "common.cuh"

namespace lbmgpu {

std::vector<HaloRow> halo_plan(int nz, int parts, bool ring) {
  std::vector<HaloRow> rows;
  if (parts <= 1) return rows;
  auto nzl = [&](int p) {
    return static_cast<int>(int64_t(nz) * (p + 1) / parts -
                            int64_t(nz) * p / parts);
  };
  const int nb = ring ? parts : parts - 1;
  for (int phase = 0; phase < 2; ++phase)
    for (int b = 0; b < nb; ++b) {
      const int p = b, q = (b + 1) % parts;
      const int top_own = nzl(p), top_ghost = nzl(p) + 1;
      if (phase == 0) {
        rows.push_back({0, q, p, 1, top_ghost, kUpSlot0});
        rows.push_back({0, p, q, top_own, 0, kDownSlot0});
      } else {
        rows.push_back({1, p, q, top_ghost, 1, kUpSlot0});
        rows.push_back({1, q, p, 0, top_own, kDownSlot0});
      }
    }
  return rows;
}

std::vector<HaloRow> halo_plan_os(int nz, int parts) {
  std::vector<HaloRow> rows;
  if (parts <= 1) return rows;
  auto nzl = [&](int p) {
    return static_cast<int>(int64_t(nz) * (p + 1) / parts -
                            int64_t(nz) * p / parts);
  };
  for (int phase = 2; phase < 4; ++phase)
    for (int b = 0; b < parts; ++b) {
      const int p = b, q = (b + 1) % parts;
      const int top_own = nzl(p), top_ghost = nzl(p) + 1;
      if (phase == 2) {
        rows.push_back({2, q, p, 1, top_ghost, kDownSlot0});
        rows.push_back({2, p, q, top_own, 0, kUpSlot0});
      } else {
        rows.push_back({3, p, q, top_ghost, kStageBottom, kUpSlot0});
        rows.push_back({3, p, q, top_ghost, kStageBottom, kDownSlot0});
        rows.push_back({3, q, p, 0, kStageTop, kDownSlot0});
        rows.push_back({3, q, p, 0, kStageTop, kUpSlot0});
      }
    }
  return rows;
}

}  // namespace lbmgpu
