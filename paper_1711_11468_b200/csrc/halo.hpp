// z-slab halo exchange plan for the direct AA sweep (new; the reference has
// no distributed path -- SURVEY.md section 8(e)).
//
// Part p owns z in [z0_p, z1_p) stored in planes zs = 1..nzl_p; planes 0 and
// nzl_p+1 are ghosts.  Across the boundary between part p (below) and part
// q (above):
//   phase 0 (after even, before odd):
//     q plane 1        up-slots   -> p ghost nzl_p+1 up-slots
//     p plane nzl_p    down-slots -> q ghost 0       down-slots
//   phase 1 (after odd):
//     p ghost nzl_p+1  up-slots   -> q plane 1       up-slots
//     q ghost 0        down-slots -> p plane nzl_p   down-slots
// "up"/"down" = the five c_z=+1 / c_z=-1 direction slots, contiguous in the
// [z][slot][y][x] layout (common.cuh).  The AA odd step touches exactly these
// ghost slots and no other part touches them during the same sub-step, so the
// exchange is race-free and the result is bitwise the single-part result.
//
// One-step kernels (blk-push / blk-pull, halo_plan_os), every boundary
// including the z wrap (solid nodes stream too, and total_mass counts them):
//   phase 2 (pull, before every sweep, on the source grid):
//     q plane 1        down-slots -> p ghost nzl_p+1 down-slots
//     p plane nzl_p    up-slots   -> q ghost 0       up-slots
//   phase 3 (push, after every sweep, on the destination grid): the ghost
//   plane holds what the part pushed across the face -- the crossing slot d
//   where the target is fluid, the bounce-back slot opp(d) where it is
//   solid -- so both 5-slot groups travel into the receiver's staging plane
//   (dst_plane kStageBottom / kStageTop) and the receiver merges them by
//   its own node flags:
//     p ghost nzl_p+1  up + down -> q bottom staging
//     q ghost 0        down + up -> p top staging
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace lbmgpu {

struct HaloRow {
  int phase;      // 0 pre-odd, 1 post-odd, 2 pull pre-sweep, 3 push post-sweep
  int src_part, dst_part;
  int src_plane, dst_plane;  // storage planes (dst < 0: staging plane)
  int slot0;      // first of the 5 contiguous slots (0 down, 14 up)
};

// nz planes cut into `parts` slabs [nz*p/parts, nz*(p+1)/parts); ring adds
// the boundary between the last and the first slab (z-periodic exchange).
std::vector<HaloRow> halo_plan(int nz, int parts, bool ring);

// staging planes of the push exchange (HaloRow::dst_plane)
constexpr int kStageBottom = -1;
constexpr int kStageTop = -2;
// phases 2 and 3 for the one-step kernels (always with the z ring)
std::vector<HaloRow> halo_plan_os(int nz, int parts);

// ---- NCCL transport (nccl.cpp), shared by the direct and list engines ----
class NcclTransportImpl;
struct NcclP2P {
  int peer;                // part index (== rank; 0 with one rank)
  const double* send;      // nullptr: no send
  double* recv;            // nullptr: no recv
  size_t count;            // doubles
};
NcclTransportImpl* nccl_create(std::vector<HaloRow> plan, int rank, int nranks,
                               const uint8_t* id128);
// bases[p] / stages[p]: the grid and the two staging planes of slab p if it
// lives in this process (else nullptr)
void nccl_exchange(NcclTransportImpl* t, int phase, const std::vector<double*>& bases,
                   const std::vector<double*>& stages, uint64_t P, cudaStream_t s);
void nccl_wait(NcclTransportImpl* t, int phase, cudaStream_t s);
void nccl_begin(NcclTransportImpl* t, int phase, cudaStream_t s);
void nccl_p2p(NcclTransportImpl* t, const std::vector<NcclP2P>& ops);
void nccl_end(NcclTransportImpl* t, int phase);
cudaStream_t nccl_comm_stream(NcclTransportImpl* t);
double nccl_sum(NcclTransportImpl* t, double v);
void nccl_destroy(NcclTransportImpl* t);

}  // namespace lbmgpu
