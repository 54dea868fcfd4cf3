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
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace lbmgpu {

struct HaloRow {
  int phase;      // 0 pre-odd, 1 post-odd
  int src_part, dst_part;
  int src_plane, dst_plane;  // storage planes
  int slot0;      // first of the 5 contiguous slots (0 down, 14 up)
};

// nz planes cut into `parts` slabs [nz*p/parts, nz*(p+1)/parts); ring adds
// the boundary between the last and the first slab (z-periodic exchange).
std::vector<HaloRow> halo_plan(int nz, int parts, bool ring);

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
void nccl_exchange(NcclTransportImpl* t, int phase, const std::vector<double*>& bases,
                   uint64_t P, cudaStream_t s);
void nccl_wait(NcclTransportImpl* t, int phase, cudaStream_t s);
void nccl_begin(NcclTransportImpl* t, int phase, cudaStream_t s);
void nccl_p2p(NcclTransportImpl* t, const std::vector<NcclP2P>& ops);
void nccl_end(NcclTransportImpl* t, int phase);
cudaStream_t nccl_comm_stream(NcclTransportImpl* t);
double nccl_sum(NcclTransportImpl* t, double v);
void nccl_destroy(NcclTransportImpl* t);

}  // namespace lbmgpu
