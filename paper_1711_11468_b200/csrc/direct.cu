// Direct (full-array) addressing: blk-push-*, blk-pull-*, aa-*, aa-vec-soa.
//
// Reference: FullLattice (src/full_lattice.cpp), FullOsKernel
// (src/kernels_full_os.cpp:47-194), FullAaKernel / FullAaVecKernel
// (src/kernels_full_aa.cpp:46-160,172-347).
//
// Device layout (ours, not the reference's): per z-slab part,
//   SoA  e(zs, slot, y, x) = (zs*19 + slot)*P + y*nx + x     P = nx*ny
//   AoS  e(zs, slot, y, x) = ((zs*ny + y)*nx + x)*19 + slot
// x (the periodic channel axis) is the coalesced axis and each z-plane's
// direction slabs are contiguous, so a z-slab halo is one block per face.
// slot = dslot(d) groups the directions by c_z (common.cuh).  Canonical
// (reference) order is restored only by the snapshot/load gathers.
//
// Full-way bounce-back: the reference runs a solid-node swap sweep after every
// sub-step (full_lattice.cpp:42-56).  Here it is folded into the sweeps:
//  * push: a population streamed into a solid node t is stored directly into
//    slot opp(d) of t (the swap the correction would apply);
//  * pull: a solid node stores its gathered q_d into its own slot opp(d);
//  * AA: the correction sweeps are dropped altogether -- solid slots are read
//    and written only in odd sub-steps and the two swaps per pair cancel
//    (initial solid weights are swap-symmetric).  Bitwise parity with
//    aa-soa / aa-aos is asserted by tests/test_gpu_parity.py.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "direct_args.cuh"
#include "halo.hpp"
#include "tma.cuh"
#include "lbm.hpp"

#include "direct_node.cuh"
#include "direct_aos.cuh"
#include "direct_fused.cuh"
#include "direct_peer.cuh"
#include "direct_job.cuh"

namespace lbmgpu {

// ---- init / canonical transfer / perturbation / macro --------------------
template <bool SOA>
__global__ void k_full_init(double* buf, uint32_t nx, uint32_t ny,
                            uint32_t zs_count, uint64_t P) {
  const uint64_t total = uint64_t(zs_count) * P;
  const Idx<SOA> I{P, nx, ny};
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t zs = static_cast<uint32_t>(i / P);
    const uint32_t r = static_cast<uint32_t>(i - uint64_t(zs) * P);
    const uint32_t y = r / nx, x = r - y * nx;
#pragma unroll
    for (int d = 0; d < kQ; ++d) buf[I(zs, dslot(d), y, x)] = weight(d);
  }
}

struct CanonArgs {
  double* buf;
  const uint32_t* node_of;  // k -> own node id
  const uint64_t* canon;    // k -> canonical index (nullptr: identity k + kbase)
  uint64_t kbase;
  uint64_t k0, k1;          // part-local range
  uint64_t c0;              // canonical index of staging row 0
  uint32_t nx, ny, zoff;
  uint64_t P;
};

template <bool SOA, bool TO_STAGING>
__global__ void k_full_canon(const CanonArgs a, double* staging) {
  const Idx<SOA> I{a.P, a.nx, a.ny};
  for (uint64_t k = a.k0 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
       k < a.k1; k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c = a.canon ? a.canon[k] : k + a.kbase;
    const uint32_t node = a.node_of[k];
    const uint32_t z = static_cast<uint32_t>(node / a.P);
    const uint32_t r = static_cast<uint32_t>(node - uint64_t(z) * a.P);
    const uint32_t y = r / a.nx, x = r - y * a.nx;
    double* row = staging + (c - a.c0) * kQ;
#pragma unroll
    for (int d = 0; d < kQ; ++d) {
      const uint64_t e = I(z + a.zoff, dslot(d), y, x);
      if (TO_STAGING)
        row[d] = a.buf[e];
      else
        a.buf[e] = row[d];
    }
  }
}

template <bool SOA>
__global__ void k_full_perturb(const CanonArgs a, uint64_t seed, double amp) {
  const Idx<SOA> I{a.P, a.nx, a.ny};
  for (uint64_t k = a.k0 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
       k < a.k1; k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c = a.canon ? a.canon[k] : k + a.kbase;
    const uint32_t node = a.node_of[k];
    const uint32_t z = static_cast<uint32_t>(node / a.P);
    const uint32_t r = static_cast<uint32_t>(node - uint64_t(z) * a.P);
    const uint32_t y = r / a.nx, x = r - y * a.nx;
#pragma unroll
    for (int d = 0; d < kQ; ++d)
      a.buf[I(z + a.zoff, dslot(d), y, x)] = perturbed_value(c, d, seed, amp);
  }
}

template <bool SOA>
__global__ void k_full_macro(const CanonArgs a, double* rho, double* u) {
  const Idx<SOA> I{a.P, a.nx, a.ny};
  for (uint64_t k = a.k0 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
       k < a.k1; k += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c = a.canon ? a.canon[k] : k + a.kbase;
    const uint32_t node = a.node_of[k];
    const uint32_t z = static_cast<uint32_t>(node / a.P);
    const uint32_t r = static_cast<uint32_t>(node - uint64_t(z) * a.P);
    const uint32_t y = r / a.nx, x = r - y * a.nx;
    double f[kQ];
#pragma unroll
    for (int d = 0; d < kQ; ++d) f[d] = a.buf[I(z + a.zoff, dslot(d), y, x)];
    double rr, ux, uy, uz;
    macroscopic(f, rr, ux, uy, uz);
    rho[c] = rr;
    u[3 * c] = ux;
    u[3 * c + 1] = uy;
    u[3 * c + 2] = uz;
  }
}

// Copies the part's own planes of the canonical FlagField into the device
// (z, y, x) order the sweeps index with.
__global__ void k_part_flags(const uint8_t* __restrict__ gflags, int nx, int ny,
                             int nz, int z0, int z1,
                             uint8_t* __restrict__ pflags) {
  const uint64_t P = uint64_t(nx) * ny;
  const uint64_t own = uint64_t(z1 - z0) * P;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < own;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t z = static_cast<uint32_t>(i / P);
    const uint32_t r = static_cast<uint32_t>(i - z * P);
    const uint32_t y = r / nx, x = r - y * nx;
    pflags[i] = gflags[(uint64_t(x) * ny + y) * nz + (z + z0)];
  }
}

// Push target mask of a part's own planes: bit d set iff the node x + c_d
// (wrapped on every axis of the whole box, as the single-part push sweep
// stores) is solid.  One 4-byte load per node instead of 18 neighbour flag
// loads; for a z slab it also covers the targets in the ghost planes.
__global__ void k_push_tmask(const uint8_t* __restrict__ gflags, uint32_t nx, uint32_t ny,
                             uint32_t nz, uint32_t z0, uint32_t nzl,
                             uint32_t* __restrict__ tmask) {
  const uint64_t P = uint64_t(nx) * ny, V = P * nzl;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < V;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t z = static_cast<uint32_t>(i / P) + z0;
    const uint32_t r = static_cast<uint32_t>(i % P);
    const uint32_t y = r / nx, x = r - y * nx;
    uint32_t m = 0;
    for (int d = 1; d < kQ; ++d) {
      const uint32_t tx = (x + nx + cx(d)) % nx, ty = (y + ny + cy(d)) % ny,
                     tz = (z + nz + cz(d)) % nz;
      if (gflags[(uint64_t(tx) * ny + ty) * nz + tz]) m |= 1u << d;  // x-major
    }
    tmask[i] = m;
  }
}

// Push halo merge (halo.hpp phase 3) into a boundary plane of the
// destination grid: the staged ghost plane of the neighbour holds, per node
// and crossing direction d, slot d (node fluid) or the bounce-back slot
// opp(d) (node solid); exactly that slot is copied.  `up` = the data came
// from below (crossing slots are the c_z = +1 ones).
__global__ void k_push_halo_merge(DirectArgs a, const double* __restrict__ stage,
                                  uint32_t zown, bool up) {
  const uint32_t P = a.P;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    const uint32_t y = i / a.nx, x = i - y * a.nx;
    const bool solid = solid_node(a, x, y, zown, zown * P + i);
    double* plane = a.dst + uint64_t(zown + a.zoff) * kQ * P + i;
    const int s0 = up ? kUpSlot0 : kDownSlot0;
#pragma unroll
    for (int k = 0; k < kHaloSlots; ++k) {
      const int sc = s0 + k;
      const int s = solid ? dslot(opp(ddir(sc))) : sc;
      plane[uint64_t(s) * P] = stage[uint64_t(s) * P + i];
    }
  }
}

// For each fluid box node in canonical order with z in [z0, z1): its
// canonical index is crank[gi]; its position k within the part is
// prank[gi] (scan of the part mask).  Writes node_of[k] and canon[k].
__global__ void k_part_lists(const uint8_t* __restrict__ gflags,
                             const uint32_t* __restrict__ crank,
                             const uint32_t* __restrict__ prank, int nx, int ny,
                             int nz, int z0, int z1,
                             uint32_t* __restrict__ node_of,
                             uint64_t* __restrict__ canon) {
  const uint64_t V = uint64_t(nx) * ny * nz;
  for (uint64_t gi = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; gi < V;
       gi += uint64_t(gridDim.x) * blockDim.x) {
    const int z = static_cast<int>(gi % nz);
    if (z < z0 || z >= z1 || gflags[gi]) continue;
    const uint64_t r = gi / nz;
    const uint32_t y = static_cast<uint32_t>(r % ny);
    const uint32_t x = static_cast<uint32_t>(r / ny);
    const uint32_t k = prank[gi];
    node_of[k] = (uint32_t(z - z0) * ny + y) * nx + x;
    if (canon) canon[k] = crank[gi];
  }
}

__global__ void k_part_mask(const uint8_t* __restrict__ gflags, int nz, int z0,
                            int z1, uint64_t V, uint8_t* __restrict__ mask) {
  for (uint64_t gi = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; gi < V;
       gi += uint64_t(gridDim.x) * blockDim.x) {
    const int z = static_cast<int>(gi % nz);
    // "solid" (1) unless fluid and inside the part's slab
    mask[gi] = (z >= z0 && z < z1 && gflags[gi] == 0) ? 0 : 1;
  }
}

// ------------------------------------------------------------------ engine
namespace {

int grid_for(uint64_t n, int threads) {
  return static_cast<int>(std::min<uint64_t>(ceil_div(n, threads), 148ull * 64));
}

struct Part {
  int index = 0;            // global slab index (== rank for NCCL)
  int z0 = 0, z1 = 0;
  uint32_t nzl = 0, zoff = 0, nzs = 0;
  DevBuf<double> buf[2];
  DevBuf<uint8_t> flags;
  DevBuf<uint32_t> tmask;   // push: solid-target bits per node (k_push_tmask)
  DevBuf<double> stage;     // push, several parts: bottom / top staging planes (2 x 19 x P)
  DevBuf<uint32_t> node_of;
  DevBuf<uint64_t> canon;   // empty when the part holds the whole box
  DevBuf<unsigned long long> pflag;  // peer transport: epoch flags (direct_peer.cuh)
  uint64_t n_fluid = 0;
  std::vector<uint64_t> canon_host;  // canonical index of each k (sorted)
};

// Address of a plan row's plane: storage plane >= 0 of grid `buf`, or one of
// the part's two staging planes (halo.hpp kStageBottom / kStageTop).
inline double* plane_ptr(const Part& pt, int buf, int plane, int slot0, uint64_t P) {
  if (plane >= 0) return pt.buf[buf].get() + (uint64_t(plane) * kQ + slot0) * P;
  return pt.stage.get() + (uint64_t(-plane - 1) * kQ + slot0) * P;
}

// Halo transport between slabs.  exchange() enqueues one phase of the plan
// on grid `buf` after the work already on `s`; wait() makes `s` wait for its
// completion.
class Transport {
 public:
  virtual ~Transport() = default;
  virtual void exchange(int phase, std::vector<Part>& parts, uint64_t P,
                        cudaStream_t s, int buf = 0) = 0;
  virtual void wait(int phase, cudaStream_t s) { (void)phase; (void)s; }
  virtual double sum(double v) { return v; }
};

// All slabs on this device: the plan's rows become device-to-device copies on
// the compute stream (used for single-GPU emulation of the decomposition).
class LocalTransport final : public Transport {
 public:
  explicit LocalTransport(std::vector<HaloRow> plan) : plan_(std::move(plan)) {}
  void exchange(int phase, std::vector<Part>& parts, uint64_t P,
                cudaStream_t s, int buf) override {
    for (const HaloRow& r : plan_) {
      if (r.phase != phase) continue;
      const double* src = plane_ptr(parts[r.src_part], buf, r.src_plane, r.slot0, P);
      double* dst = plane_ptr(parts[r.dst_part], buf, r.dst_plane, r.slot0, P);
      LBM_CUDA(cudaMemcpyAsync(dst, src, uint64_t(kHaloSlots) * P * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    }
  }

 private:
  std::vector<HaloRow> plan_;
};

}  // namespace

// NCCL transport (nccl.cpp, declared in halo.hpp): one process per GPU,
// slab = rank.

namespace {

class NcclTransport final : public Transport {
 public:
  NcclTransport(std::vector<HaloRow> plan, int rank, int nranks, int nparts,
                const uint8_t* id128)
      : t_(nccl_create(std::move(plan), rank, nranks, id128)),
        bases_(nparts, nullptr),
        stages_(nparts, nullptr) {}
  ~NcclTransport() override { nccl_destroy(t_); }
  void exchange(int phase, std::vector<Part>& parts, uint64_t P,
                cudaStream_t s, int buf) override {
    for (Part& pt : parts) {
      bases_[pt.index] = pt.buf[buf].get();
      stages_[pt.index] = pt.stage.get();
    }
    nccl_exchange(t_, phase, bases_, stages_, P, s);
  }
  void wait(int phase, cudaStream_t s) override { nccl_wait(t_, phase, s); }
  double sum(double v) override { return nccl_sum(t_, v); }

 private:
  NcclTransportImpl* t_;
  std::vector<double*> bases_, stages_;
};

class DirectEngine final : public Engine {
 public:
  DirectEngine(const Descriptor& d, const GeomSpec& g, const DistSpec& dist) {
    desc_ = d;
    LBM_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    nvtxNameCudaStreamA(stream_, "lbmgpu interior");
    rank_ = dist.rank;
    nranks_ = dist.nranks;
    nparts_ = nranks_ > 1 ? nranks_ : std::max(1, dist.virtual_parts);
    if (nparts_ > 1 && !d.soa)
      throw ConfigError("z-slab decomposition needs the SoA layout");
    if (nparts_ > g.nz) throw ConfigError("more z-slab parts than z planes");
    if (dist.transport != 0 && dist.transport != 1)
      throw ConfigError("dist: transport must be 0 (halo copies) or 1 (peer memory)");
    if (dist.transport == 1 && nparts_ < 2)
      throw ConfigError("peer transport: needs a z-slab decomposition (>= 2 slabs)");
    if (nranks_ > 1 && !dist.have_id && dist.transport != 1)
      throw ConfigError("dist: nranks > 1 needs the NCCL unique id");
    {
      int dev = 0;
      LBM_CUDA(cudaGetDevice(&dev));
      LBM_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, dev));
      // tuning knobs (defaults are the measured best)
      if (const char* e = std::getenv("LBMGPU_AA_MINB")) minb_ = std::atoi(e);
      if (const char* e = std::getenv("LBMGPU_TILE_BY")) tile_by_ = static_cast<uint32_t>(std::atoi(e));
      if (const char* e = std::getenv("LBMGPU_PUSH_AS_PULL")) fused_push_as_pull_ = std::atoi(e) != 0;
      if (const char* e = std::getenv("LBMGPU_FUSED_MB"))
        fused_bytes_ = uint64_t(std::atoll(e)) << 20;
    }

    DeviceGeometry geo = build_geometry_device(g, stream_);
    geom_ = g;
    geom_.custom.clear();  // the device flags are kept per part
    nx_ = geo.nx;
    ny_ = geo.ny;
    nz_ = geo.nz;
    n_fluid_ = static_cast<uint64_t>(geo.n_fluid);
    P_ = uint64_t(nx_) * ny_;
    for (int p = 0; p < nparts_; ++p)
      if (P_ * (uint64_t(nz_) * (p + 1) / nparts_ - uint64_t(nz_) * p / nparts_) >=
          (1ull << 31))
        throw ConfigError("direct lattice: more than 2^31 nodes in one slab");

    const uint64_t V = geo.volume();
    DevBuf<uint32_t> crank(V);
    scan_fluid(geo.flags.get(), crank.get(), V, stream_);

    // which slabs live in this process
    std::vector<int> mine;
    if (nranks_ > 1)
      mine.push_back(rank_);
    else
      for (int p = 0; p < nparts_; ++p) mine.push_back(p);
    parts_.resize(mine.size());
    for (size_t i = 0; i < mine.size(); ++i) {
      Part& pt = parts_[i];
      const int p = mine[i];
      pt.index = p;
      pt.z0 = static_cast<int>(int64_t(nz_) * p / nparts_);
      pt.z1 = static_cast<int>(int64_t(nz_) * (p + 1) / nparts_);
      pt.nzl = pt.z1 - pt.z0;
      pt.zoff = nparts_ > 1 ? 1 : 0;
      pt.nzs = pt.nzl + 2 * pt.zoff;
      const uint64_t slots = uint64_t(pt.nzs) * P_ * kQ;
      const int nbuf = d.prop == Prop::Aa ? 1 : 2;
      for (int b = 0; b < nbuf; ++b) {
        pt.buf[b].alloc(slots);
        const int gr = grid_for(uint64_t(pt.nzs) * P_, 256);
        if (d.soa)
          k_full_init<true><<<gr, 256, 0, stream_>>>(pt.buf[b].get(), nx_, ny_, pt.nzs, P_);
        else
          k_full_init<false><<<gr, 256, 0, stream_>>>(pt.buf[b].get(), nx_, ny_, pt.nzs, P_);
        LBM_CHECK_LAUNCH();
      }
      pt.flags.alloc(uint64_t(pt.nzl) * P_);
      k_part_flags<<<grid_for(uint64_t(pt.nzl) * P_, 256), 256, 0, stream_>>>(
          geo.flags.get(), nx_, ny_, nz_, pt.z0, pt.z1, pt.flags.get());
      LBM_CHECK_LAUNCH();
      // push: solid-target masks (required with several parts: the
      // targets in the ghost planes have no flags of their own here)
      if (d.prop == Prop::OsPush) {
        pt.tmask.alloc(uint64_t(pt.nzl) * P_);
        k_push_tmask<<<grid_for(uint64_t(pt.nzl) * P_, 256), 256, 0, stream_>>>(
            geo.flags.get(), nx_, ny_, nz_, pt.z0, pt.nzl, pt.tmask.get());
        LBM_CHECK_LAUNCH();
      }
      if (d.prop == Prop::OsPush && nparts_ > 1) pt.stage.alloc(2 * kQ * P_);
      // the slab's fluid nodes in canonical order
      DevBuf<uint8_t> mask(V);
      DevBuf<uint32_t> prank(V);
      k_part_mask<<<grid_for(V, 256), 256, 0, stream_>>>(geo.flags.get(), nz_,
                                                         pt.z0, pt.z1, V,
                                                         mask.get());
      LBM_CHECK_LAUNCH();
      pt.n_fluid = scan_fluid(mask.get(), prank.get(), V, stream_);
      pt.node_of.alloc(std::max<uint64_t>(pt.n_fluid, 1));
      const bool whole = nparts_ == 1;
      if (!whole) pt.canon.alloc(std::max<uint64_t>(pt.n_fluid, 1));
      k_part_lists<<<grid_for(V, 256), 256, 0, stream_>>>(
          geo.flags.get(), crank.get(), prank.get(), nx_, ny_, nz_, pt.z0,
          pt.z1, pt.node_of.get(), whole ? nullptr : pt.canon.get());
      LBM_CHECK_LAUNCH();
      if (!whole) {
        pt.canon_host.resize(pt.n_fluid);
        if (pt.n_fluid)
          LBM_CUDA(cudaMemcpyAsync(pt.canon_host.data(), pt.canon.get(),
                                   pt.n_fluid * 8, cudaMemcpyDeviceToHost, stream_));
        LBM_CUDA(cudaStreamSynchronize(stream_));
      }
    }
    if (nparts_ > 1) {
      // z-wrap exchange only if a fluid node sits on the z=0 or z=nz-1 plane
      std::vector<uint8_t> hf(V);
      LBM_CUDA(cudaMemcpyAsync(hf.data(), geo.flags.get(), V,
                               cudaMemcpyDeviceToHost, stream_));
      LBM_CUDA(cudaStreamSynchronize(stream_));
      bool end_fluid = false;
      for (uint64_t i = 0; i < V && !end_fluid; i += nz_)
        end_fluid = hf[i] == 0 || hf[i + nz_ - 1] == 0;
      // one-step kernels stream solid nodes too: always the full ring
      std::vector<HaloRow> plan = d.prop == Prop::Aa ? halo_plan(nz_, nparts_, end_fluid)
                                                     : halo_plan_os(nz_, nparts_);
      // NCCL between processes; with one process the copies are local, and
      // an NCCL id selects NCCL self send/recv instead (tests the NCCL path on
      // one GPU).
      // (the peer transport between processes needs NCCL only for the
      // total-mass reduction; without an id there is no Transport at all)
      if (dist.have_id)
        tr_ = std::make_unique<NcclTransport>(std::move(plan), rank_, nranks_,
                                              nparts_, dist.nccl_id.data());
      else if (nranks_ == 1)
        tr_ = std::make_unique<LocalTransport>(std::move(plan));
      ring_ = end_fluid || d.prop != Prop::Aa;  // one-step plans always carry the ring
      if (dist.transport == 1) setup_peer();
    }
    LBM_CUDA(cudaStreamSynchronize(stream_));
  }

  ~DirectEngine() override {
    if (stream_) cudaStreamSynchronize(stream_);
    if (bstream_) {
      cudaStreamSynchronize(bstream_);
      cudaStreamDestroy(bstream_);
    }
    for (cudaEvent_t e : pev_)
      if (e) cudaEventDestroy(e);
    for (void* p : ipc_open_) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t e : job_ev_) cudaEventDestroy(e);
    for (cudaStream_t st : {job_s_in_, job_s_out_, job_k_in_, job_k_out_})
      if (st) cudaStreamDestroy(st);
    if (peer_err_) cudaFreeHost(peer_err_);
    tr_.reset();
    if (stream_) cudaStreamDestroy(stream_);
  }

  int parts() const override { return static_cast<int>(parts_.size()); }
  void part_info(int p, int* z0, int* z1, uint64_t* nf) const override {
    *z0 = parts_.at(p).z0;
    *z1 = parts_.at(p).z1;
    *nf = parts_.at(p).n_fluid;
  }
  bool holds_all() const override { return nranks_ == 1; }

  DirectArgs args(const Part& pt, uint32_t node0, uint32_t count,
                  const TrtArgs& t, int src_buf, int dst_buf) const {
    DirectArgs a;
    a.src = pt.buf[src_buf].get();
    a.dst = pt.buf[dst_buf].get();
    a.flags = pt.flags.get();
    a.tmask = pt.tmask.get();
    a.nx = nx_;
    a.ny = ny_;
    a.nzl = pt.nzl;
    a.zoff = pt.zoff;
    a.zwrap = nparts_ == 1;
    a.P = static_cast<uint32_t>(P_);
    a.fdx = FastDiv(nx_);
    a.fdP = FastDiv(static_cast<uint32_t>(P_));
    a.node0 = node0;
    a.count = count;
    a.trt = t;
    a.geom = geom_.kind;
    a.gny = ny_;
    a.gnz = nz_;
    a.z0 = pt.z0;
    a.period = geom_.block + geom_.spacing;
    a.spacing = geom_.spacing;
    const long long D = geom_.pipe_diameter > 0 ? geom_.pipe_diameter
                                                : (long long)std::min(ny_, nz_) - 2;
    a.d2 = D * D;
    a.band = 0;
    for (int d = 0; d < kQ; ++d) {
      const long long dn = -(long long)cz(d) * (long long)P_ - (long long)cy(d) * nx_ - cx(d);
      a.odd_off[d] = desc_.soa
                         ? (-(long long)cz(d) * kQ + dslot(opp(d))) * (long long)P_ +
                               (-(long long)cy(d) * nx_ - cx(d))
                         : dn * kQ + dslot(opp(d));
    }
    return a;
  }

  // Grid of the AoS 3-D tile kernels and their traversal (tile_origin,
  // direct_aos.cuh): blocks of tile_by_ y tiles when that is a power of two
  // dividing the y tile count (and the grid's y extent fits), else plain.
  template <int TY, int TZ>
  dim3 tile_grid(DirectArgs& at) const {
    const unsigned tx = static_cast<unsigned>(nx_ / kPtX), ty = static_cast<unsigned>(ny_ / TY),
                   tz = static_cast<unsigned>(nz_ / TZ);
    const unsigned by = tile_by_;
    if (by > 1 && (by & (by - 1)) == 0 && ty % by == 0 && uint64_t(by) * tz <= 65535u) {
      at.band = by;
      return dim3(tx, by * tz, ty / by);
    }
    at.band = 0;
    return dim3(tx, ty, tz);
  }

  template <int TY, int TZ>
  void aa_odd_aos_tile3d(const DirectArgs& a) {
    auto kern = k_full_aa_odd_aos_tile3d<TY, TZ, false>;
    constexpr size_t smem = pt_smem<TY, TZ, false>();
    LBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    const int tok = stats_.begin("full_aa_odd_aos", stream_);
    DirectArgs at = a;
    const dim3 grid = tile_grid<TY, TZ>(at);
    kern<<<grid, kPtX * TY * TZ, smem, stream_>>>(at);
    LBM_CHECK_LAUNCH();
    stats_.end(tok, stream_);
  }

  template <int TY, int TZ>
  void pull_aos_tile3d(const DirectArgs& a, bool last, const char* name) {
    auto kern = last ? k_full_pull_aos_tile3d<false, TY, TZ, false>
                     : k_full_pull_aos_tile3d<true, TY, TZ, false>;
    constexpr size_t smem = pt_smem<TY, TZ, false>();
    LBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    const int tok = stats_.begin(name, stream_);
    DirectArgs at = a;
    const dim3 grid = tile_grid<TY, TZ>(at);
    kern<<<grid, kPtX * TY * TZ, smem, stream_>>>(at);
    LBM_CHECK_LAUNCH();
    stats_.end(tok, stream_);
  }

  // AoS gather/scatter sweep over a whole part in y-band order (see
  // DirectArgs::band); plain order when ny has no suitable divisor
  DirectArgs banded(DirectArgs a) const {
    if (a.node0 != 0 || a.count != a.nzl * a.P) return a;
    for (int b : {16, 8, 4, 2})
      if (ny_ % b == 0) {
        a.band = static_cast<uint32_t>(b);
        break;
      }
    return a;
  }

  template <class K>
  void launch(const char* name, K kern, const DirectArgs& a, cudaStream_t s,
              int threads = 256) {
    if (a.count == 0) return;
    const int tok = stats_.begin(name, s);
    kern<<<static_cast<unsigned>(ceil_div(a.count, threads)), threads, 0, s>>>(a);
    LBM_CHECK_LAUNCH();
    stats_.end(tok, s);
  }

  // One SoA AA sub-step over a node range, one node per thread, 128-thread
  // CTAs.  minb_ = min CTAs/SM of the launch bounds, i.e. the register cap
  // (2 at 256: 128 registers, 16 warps/SM; DESIGN.md §4 has the sweep).
  void aa_sub(bool odd, const DirectArgs& a, const char* name) {
    if (a.count == 0) return;
    switch (minb_) {
      case 3:
        odd ? launch(name, k_full_aa_odd<true, false, 128, 3>, a, stream_, 128)
            : launch(name, k_full_aa_even<true, false, 128, 3>, a, stream_, 128);
        break;
      case 5:
        odd ? launch(name, k_full_aa_odd<true, false, 128, 5>, a, stream_, 128)
            : launch(name, k_full_aa_even<true, false, 128, 5>, a, stream_, 128);
        break;
      case 6:
        odd ? launch(name, k_full_aa_odd<true, false, 128, 6>, a, stream_, 128)
            : launch(name, k_full_aa_even<true, false, 128, 6>, a, stream_, 128);
        break;
      default:
        odd ? launch(name, k_full_aa_odd<true, false, 128, 4>, a, stream_, 128)
            : launch(name, k_full_aa_even<true, false, 128, 4>, a, stream_, 128);
    }
  }

  // Whether advance() runs as one cooperative multi-sweep launch: single
  // slab, lattice small enough to live in L2 (<= fused_bytes_, default
  // 96 MiB of PDF buffers), at least two sweeps.
  bool use_fused(long steps) const {
    if (nparts_ != 1 || steps < 2 || fused_bytes_ == 0) return false;
    // AoS with 3-D halo tiles: the per-sweep tile kernels beat the fused
    // per-node launch even on the L2-resident cfg-1 box (B200, cfg 1:
    // blk-push-aos 5,786 -> 8,386, blk-pull-aos 4,988 -> 8,465, aa-aos
    // 4,921 -> 8,931 MFLUP/s)
    if (!desc_.soa && aos_tiles()) return false;
    const Part& pt = parts_[0];
    const uint64_t bufs = desc_.prop == Prop::Aa ? 1 : 2;
    // (the fused bodies index with 32-bit arithmetic: fewer than 2^32
    // elements per buffer whatever LBMGPU_FUSED_MB says)
    const uint64_t elems = uint64_t(pt.nzs) * P_ * kQ;
    return elems * 8 * bufs <= fused_bytes_ && elems < (1ull << 32);
  }

  template <bool SOA, int KIND>
  void launch_fused(const DirectArgs& a, double* other, long steps, const char* name,
                    long sweeps) {
    // block shape, measured on cfg 1 (B200, cooperative-groups grid sync,
    // 20 sweeps per launch): push (160, 4) 18.1k MFLUP/s [(320, 2) 17.4k],
    // pull (160, 4) 19.6k, AA SoA (256, 2) 24.6k [(160, 4) 19.6k], AA AoS
    // (160, 4); the unconstrained (256, 1) compile lands at 132-146
    // registers, one block per SM
    if (KIND == kFusedAA && SOA)
      launch_fused_as<SOA, KIND, 256, 2>(a, other, steps, name, sweeps);
    else
      launch_fused_as<SOA, KIND, 160, 4>(a, other, steps, name, sweeps);
  }

  template <bool SOA, int KIND, int TPB, int MINB>
  void launch_fused_as(const DirectArgs& a, double* other, long steps, const char* name,
                       long sweeps) {
    auto kern = k_full_fused<SOA, KIND, TPB, MINB>;
    int per_sm = 0;
    per_sm = occupancy_blocks(reinterpret_cast<const void*>(kern), TPB);
    const uint64_t want = ceil_div(a.count, TPB);
    const int grid = static_cast<int>(
        std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(std::max(per_sm, 1)) * sm_count_)));
    DirectArgs aa = a;
    void* params[] = {&aa, &other, &steps};
    const int tok = stats_.begin(name, stream_, sweeps);
    LBM_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), grid, TPB, params, 0,
                                         stream_));
    stats_.end(tok, stream_);
  }

  bool advance_fused(const TrtArgs& t, long steps) {
    if (!use_fused(steps)) return false;
    const Part& pt = parts_[0];
    const uint32_t N = pt.nzl * static_cast<uint32_t>(P_);
    const bool soa = desc_.soa;
    if (desc_.prop == Prop::Aa) {
      DirectArgs a = args(pt, 0, N, t, 0, 0);
      soa ? launch_fused<true, kFusedAA>(a, nullptr, steps, "full_aa_soa_fused", steps)
          : launch_fused<false, kFusedAA>(a, nullptr, steps, "full_aa_aos_fused", steps);
      return true;
    }
    DirectArgs a = args(pt, 0, N, t, cur_, 1 - cur_);
    double* other = parts_[0].buf[1 - cur_].get();
    // SoA push in pull order (as the AoS push, os_aos_tiles): push and pull
    // realise the identical per-step mapping (reference
    // tests/test_kernels.cpp:96-126), and the fused pull -- collide pass,
    // T-1 gather + collide sweeps, one gather-only sweep -- is the faster
    // L2-resident launch (cfg 1, 100 steps: DESIGN.md section 4)
    if (desc_.prop == Prop::OsPush && soa && fused_push_as_pull_)
      launch_fused<true, kFusedPull>(a, other, steps, "full_push_soa_fused", steps + 1);
    else if (desc_.prop == Prop::OsPush)
      soa ? launch_fused<true, kFusedPush>(a, other, steps, "full_push_soa_fused", steps)
          : launch_fused<false, kFusedPush>(a, other, steps, "full_push_aos_fused", steps);
    else
      soa ? launch_fused<true, kFusedPull>(a, other, steps, "full_pull_soa_fused", steps + 1)
          : launch_fused<false, kFusedPull>(a, other, steps, "full_pull_aos_fused", steps + 1);
    if (steps & 1) cur_ ^= 1;
    return true;
  }

  // AoS 3-D halo tiles (direct_aos.cuh): single part, nx % 16, ny % 4, nz % 4
  bool aos_tiles() const {
    return nparts_ == 1 && nx_ % kPtX == 0 && ny_ % 4 == 0 && nz_ % 4 == 0;
  }

  // One-step AoS sweeps in pull order: collide pass, T-1 gather + collide
  // sweeps, one gather-only sweep (kernels_full_os.cpp:173-190), every
  // destination record assembled whole in a CTA's shared-memory tile.  The
  // push names run the same schedule: push and pull realise the identical
  // per-step mapping (reference tests/test_kernels.cpp:96-126) -- the value
  // a push stores at (x, d) [bounce-back: (x, opp d) when x is solid] is the
  // post-collision q_d of x - c_d, which is exactly what the pull gathers --
  // so the state after advance(T) is bitwise the push's, with each node
  // collided once per step and the scattered 8-byte stores of a push
  // (one 32-byte sector each) replaced by whole-record bulk stores.
  void os_aos_tiles(const TrtArgs& t, long steps, bool push) {
    const Part& pt = parts_[0];
    const uint32_t N = pt.nzl * static_cast<uint32_t>(P_);
    launch(push ? "full_push_aos_collide" : "full_collide_aos", k_full_aos_tile<false>,
           args(pt, 0, N, t, cur_, cur_), stream_, kAosTile);
    for (long s = 0; s < steps; ++s) {
      const bool last = s == steps - 1;
      const char* name = push ? (last ? "full_push_stream_aos" : "full_push_aos")
                              : (last ? "full_pull_stream_aos" : "full_pull_aos");
      const DirectArgs a = args(pt, 0, N, t, cur_, 1 - cur_);
      pull_aos_tile3d<4, 4>(a, last, name);  // (16x4x2 / 16x2x4 tiles: 4493 -> 4100 / 4326 GB/s)
      cur_ ^= 1;
    }
  }

  void advance(const TrtArgs& t, long steps) override {
    NvtxRange range(("advance " + desc_.name).c_str());
    if (peer_) peer_check();
    const bool soa = desc_.soa;
    if (advance_fused(t, steps)) return;
    if (desc_.prop != Prop::Aa && nparts_ > 1) {
      peer_ ? os_sweeps_peer(t, steps) : os_sweeps_slabs(t, steps);
      return;
    }
    if (desc_.prop != Prop::Aa && !soa && aos_tiles()) {
      os_aos_tiles(t, steps, desc_.prop == Prop::OsPush);
      return;
    }
    if (desc_.prop == Prop::OsPush) {
      const Part& pt = parts_[0];
      const uint32_t N = pt.nzl * static_cast<uint32_t>(P_);
      for (long s = 0; s < steps; ++s) {
        DirectArgs a = args(pt, 0, N, t, cur_, 1 - cur_);
        if (soa)
          launch("full_push_soa", k_full_push<true, false>, a, stream_);
        else
          launch("full_push_aos", k_full_push<false, false>, banded(a), stream_);
        cur_ ^= 1;
      }
      return;
    }
    if (desc_.prop == Prop::OsPull) {
      // collide pass, T-1 fused sweeps, one stream-only sweep
      // (kernels_full_os.cpp:173-190)
      const Part& pt = parts_[0];
      const uint32_t N = pt.nzl * static_cast<uint32_t>(P_);
      {
        DirectArgs a = args(pt, 0, N, t, cur_, cur_);
        soa ? launch("full_collide_soa", k_full_collide<true>, a, stream_)
            : launch("full_collide_aos", k_full_aos_tile<false>, a, stream_, kAosTile);
      }
      for (long s = 0; s < steps; ++s) {
        DirectArgs a = args(pt, 0, N, t, cur_, 1 - cur_);
        const bool last = s == steps - 1;
        if (soa) {
          if (last)
            launch("full_pull_stream_soa", k_full_pull<true, false, false>, a, stream_);
          else
            launch("full_pull_soa", k_full_pull<true, true, false>, a, stream_);
        } else {
          if (last)
            launch("full_pull_stream_aos", k_full_pull<false, false, false>, banded(a), stream_);
          else
            launch("full_pull_aos", k_full_pull<false, true, false>, banded(a), stream_);
        }
        cur_ ^= 1;
      }
      return;
    }
    // AA pattern: even/odd pairs, in place
    for (long s = 0; s < steps; s += 2) {
      if (nparts_ == 1) {
        const Part& pt = parts_[0];
        const uint32_t N = pt.nzl * static_cast<uint32_t>(P_);
        DirectArgs a = args(pt, 0, N, t, 0, 0);
        if (soa) {
          aa_sub(false, a, "full_aa_even_soa");
          aa_sub(true, a, "full_aa_odd_soa");
        } else {
          launch("full_aa_even_aos", k_full_aos_tile<true>, a, stream_, kAosTile);
          // (y-band order measured slower for the AA odd step: 1922 -> 1103
          // GB/s at band 16, although it halves the DRAM traffic)
          if (aos_tiles()) {
            // 16 x 4 x 4 tiles (16 x 4 x 2 / 16 x 2 x 4: 3 CTAs/SM but more
            // halo rows per node; cfg-5 box odd step 3125 -> 2810 / 2885 GB/s)
            aa_odd_aos_tile3d<4, 4>(a);
          } else {
            launch("full_aa_odd_aos", k_full_aa_odd<false, false>, a, stream_);
          }
        }
      } else {
        peer_ ? aa_pair_peer(t) : aa_pair_slabs(t);
      }
    }
  }

  // ---- pipelined job (Engine::run_job) --------------------------------------
  // load_state(host_in) + advance(T) + snapshot(host_out) with the PCIe
  // transfers overlapped with the sweeps.  The fluid planes [za, zb) are cut
  // into S compute slabs of ws planes; sub-step s of slab j touches the
  // records of slabs j-1 .. j+1 and needs sub-step s-1 of those three, so the
  // launches go out on the ONE engine stream in diagonal rounds (round L:
  // slabs j = L, L-1, .., 0 at sub-step L - j), which keeps every pair of
  // conflicting launches in the order of the plain advance -- the result is
  // bitwise the plain sequence's.  Slab j can then run ahead of slab j+1 by
  // one sub-step: while later planes are still crossing PCIe the first slabs
  // already advance, and the first slabs leave for the host while the last
  // ones finish.  Transfers move chunks of k slabs: the chunk's canonical
  // rows are a 2-D array (column-uniform geometries: every fluid (x, y)
  // column holds the same planes [za, zb)), one cudaMemcpy2DAsync + one
  // layout kernel on a copy stream each way.  Applies to SoA AA lattices of
  // one part whose z ends are not both fluid (no z ring); else false.
  bool job_plan() {
    if (job_checked_) return job_ok_;
    job_checked_ = true;
    const Part& pt = parts_[0];
    DevBuf<uint32_t> census(3 * P_);
    k_job_columns<<<grid_for(P_, 256), 256, 0, stream_>>>(pt.flags.get(), P_, nz_, census.get());
    LBM_CHECK_LAUNCH();
    std::vector<uint32_t> h(3 * P_);
    LBM_CUDA(cudaMemcpyAsync(h.data(), census.get(), h.size() * 4, cudaMemcpyDeviceToHost, stream_));
    LBM_CUDA(cudaStreamSynchronize(stream_));
    uint32_t za = 0, zb = 0;
    bool first = true;
    std::vector<uint32_t> cols;  // in-plane offsets of the fluid columns, x-major
    for (uint32_t x = 0; x < uint32_t(nx_); ++x)
      for (uint32_t y = 0; y < uint32_t(ny_); ++y) {
        const uint64_t c = uint64_t(y) * nx_ + x;
        const uint32_t cnt = h[3 * c], zmin = h[3 * c + 1], zmax = h[3 * c + 2];
        if (cnt == 0) continue;
        if (zmax - zmin + 1 != cnt) return false;  // a solid plane inside the column
        if (first) {
          za = zmin;
          zb = zmax + 1;
          first = false;
        } else if (zmin != za || zmax + 1 != zb) {
          return false;
        }
        cols.push_back(static_cast<uint32_t>(c));
      }
    if (first || (za == 0 && zb == uint32_t(nz_))) return false;
    std::vector<uint32_t> col_of(P_, 0xffffffffu);  // in-plane offset -> column rank
    for (uint32_t r = 0; r < cols.size(); ++r) col_of[cols[r]] = r;
    job_za_ = za;
    job_zb_ = zb;
    job_cols_ = cols.size();
    job_col_of_.alloc(P_);
    LBM_CUDA(cudaMemcpy(job_col_of_.get(), col_of.data(), P_ * 4, cudaMemcpyHostToDevice));
    job_ok_ = true;
    return true;
  }

  bool run_job(const TrtArgs& t, long steps, const double* host_in, double* host_out) override {
    if (nparts_ != 1 || desc_.prop != Prop::Aa || !desc_.soa || steps < 2 || use_fused(steps) ||
        !host_in || !host_out)
      return false;
    if (!job_plan()) return false;
    NvtxRange range(("run_job " + desc_.name).c_str());
    const Part& pt = parts_[0];
    const uint32_t za = job_za_, nzf = job_zb_ - job_za_;
    const uint64_t R = job_cols_;
    // S compute slabs of ws planes; loads move chunks of ki slabs, stores
    // chunks of ko slabs.  Measured on the cfg-5 job:
    // one plane per slab (the most skew: the first chunks leave earliest),
    // 16-plane loads and 32-plane stores (2-D copy rows of 2,432 / 4,864 B;
    // the device-to-host 2-D copies need the wider rows)
    int slabs = 512, ki = 16, ko = 32;
    if (const char* e = std::getenv("LBMGPU_JOB_SLABS")) slabs = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("LBMGPU_JOB_CHUNK")) ki = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("LBMGPU_JOB_CHUNK_OUT")) ko = std::max(1, std::atoi(e));
    const uint32_t ws = static_cast<uint32_t>(ceil_div(nzf, uint64_t(std::min<uint32_t>(slabs, nzf))));
    const uint32_t S = static_cast<uint32_t>(ceil_div(nzf, ws));
    // a chunk's layout tile must fit the shared memory: kJobTx x w x 19 doubles
    const uint32_t kmax = std::max<uint32_t>(1, ((200u << 10) / (kJobTx * 8) - 1) / kQ / ws);
    ki = static_cast<int>(std::min<uint32_t>(uint32_t(ki), kmax));
    ko = static_cast<int>(std::min<uint32_t>(uint32_t(ko), kmax));
    const uint32_t Ci = static_cast<uint32_t>(ceil_div(S, uint64_t(ki)));
    const uint32_t Co = static_cast<uint32_t>(ceil_div(S, uint64_t(ko)));
    const uint32_t wci = std::min<uint32_t>(ki * ws, nzf), wco = std::min<uint32_t>(ko * ws, nzf);
    try {  // no room for the staging (a lattice filling the GPU): plain sequence
      for (int bf = 0; bf < 2; ++bf) {
        if (job_in_[bf].size() < R * wci * kQ) job_in_[bf].alloc(R * wci * kQ);
        if (job_out_[bf].size() < R * wco * kQ) job_out_[bf].alloc(R * wco * kQ);
      }
    } catch (const DeviceError&) {
      for (int bf = 0; bf < 2; ++bf) {
        job_in_[bf].release();
        job_out_[bf].release();
      }
      cudaGetLastError();
      return false;
    }
    if (!job_s_in_) {
      // layout-kernel streams at the greatest priority: their CTAs take SM
      // slots ahead of the sweeps' next CTAs instead of queueing behind them
      int least = 0, greatest = 0;
      LBM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      LBM_CUDA(cudaStreamCreateWithFlags(&job_s_in_, cudaStreamNonBlocking));
      LBM_CUDA(cudaStreamCreateWithFlags(&job_s_out_, cudaStreamNonBlocking));
      LBM_CUDA(cudaStreamCreateWithPriority(&job_k_in_, cudaStreamNonBlocking, greatest));
      LBM_CUDA(cudaStreamCreateWithPriority(&job_k_out_, cudaStreamNonBlocking, greatest));
      nvtxNameCudaStreamA(job_s_in_, "lbmgpu job h2d");
      nvtxNameCudaStreamA(job_s_out_, "lbmgpu job d2h");
      nvtxNameCudaStreamA(job_k_in_, "lbmgpu job load layout");
      nvtxNameCudaStreamA(job_k_out_, "lbmgpu job store layout");
    }
    const size_t nev = 2 * size_t(Ci) + 3 * size_t(Co) + 1;
    while (job_ev_.size() < nev) {
      cudaEvent_t e;
      LBM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      job_ev_.push_back(e);
    }
    cudaEvent_t* copied = job_ev_.data();      // h2d of load chunk i done
    cudaEvent_t* loaded = copied + Ci;         // load chunk i in the lattice (staging free)
    cudaEvent_t* final_ev = loaded + Ci;       // store chunk i's planes final
    cudaEvent_t* gathered = final_ev + Co;     // store chunk i in its staging buffer
    cudaEvent_t* stored = gathered + Co;       // d2h of store chunk i done (staging free)
    cudaEvent_t start = job_ev_[nev - 1];
    // LBMGPU_JOB_TRACE=1: per-chunk timeline (ms after the job start) on stderr
    const bool trace = std::getenv("LBMGPU_JOB_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto tmark = [&](cudaStream_t st) {
      if (!trace) return;
      cudaEvent_t e;
      LBM_CUDA(cudaEventCreate(&e));
      LBM_CUDA(cudaEventRecord(e, st));
      tev.push_back(e);
    };
    tmark(stream_);
    // the side streams start after whatever the engine stream holds
    LBM_CUDA(cudaEventRecord(start, stream_));
    for (cudaStream_t st : {job_s_in_, job_s_out_, job_k_in_, job_k_out_})
      LBM_CUDA(cudaStreamWaitEvent(st, start, 0));
    double* buf = pt.buf[0].get();
    auto chunk_planes = [&](uint32_t i, int kk, uint32_t& c0, uint32_t& w) {
      c0 = za + i * kk * ws;
      w = std::min<uint32_t>(kk * ws, za + nzf - c0);
    };
    const unsigned tiles = static_cast<unsigned>(ceil_div(nx_, kJobTx) * uint64_t(ny_));
    auto smem_of = [&](uint32_t w) { return size_t(kJobTx) * (w * kQ + 1) * 8; };
    LBM_CUDA(cudaFuncSetAttribute(k_job_chunk<true, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_of(wci))));
    LBM_CUDA(cudaFuncSetAttribute(k_job_chunk<true, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_of(wco))));
    // every load up front: 2-D copy into staging buffer i % 2 (h2d stream),
    // then the layout kernel (load-layout stream)
    for (uint32_t i = 0; i < Ci; ++i) {
      uint32_t c0, w;
      chunk_planes(i, ki, c0, w);
      double* st = job_in_[i & 1].get();
      if (i >= 2) LBM_CUDA(cudaStreamWaitEvent(job_s_in_, loaded[i - 2], 0));
      LBM_CUDA(cudaMemcpy2DAsync(st, size_t(w) * kQ * 8, host_in + uint64_t(c0 - za) * kQ,
                                 size_t(nzf) * kQ * 8, size_t(w) * kQ * 8, R, cudaMemcpyHostToDevice,
                                 job_s_in_));
      LBM_CUDA(cudaEventRecord(copied[i], job_s_in_));
      tmark(job_s_in_);
      LBM_CUDA(cudaStreamWaitEvent(job_k_in_, copied[i], 0));
      k_job_chunk<true, false><<<tiles, 256, smem_of(w), job_k_in_>>>(
          buf, job_col_of_.get(), w, c0, nx_, ny_, st);
      LBM_CHECK_LAUNCH();
      LBM_CUDA(cudaEventRecord(loaded[i], job_k_in_));
      tmark(job_k_in_);
    }
    // store chunk i leaves: layout kernel into staging buffer i % 2
    // (store-layout stream), then the 2-D copy (d2h stream)
    auto store_chunk = [&](uint32_t i) {
      LBM_CUDA(cudaEventRecord(final_ev[i], stream_));
      tmark(stream_);
      LBM_CUDA(cudaStreamWaitEvent(job_k_out_, final_ev[i], 0));
      if (i >= 2) LBM_CUDA(cudaStreamWaitEvent(job_k_out_, stored[i - 2], 0));
      uint32_t c0, w;
      chunk_planes(i, ko, c0, w);
      double* st = job_out_[i & 1].get();
      k_job_chunk<true, true><<<tiles, 256, smem_of(w), job_k_out_>>>(
          buf, job_col_of_.get(), w, c0, nx_, ny_, st);
      LBM_CHECK_LAUNCH();
      LBM_CUDA(cudaEventRecord(gathered[i], job_k_out_));
      tmark(job_k_out_);
      LBM_CUDA(cudaStreamWaitEvent(job_s_out_, gathered[i], 0));
      LBM_CUDA(cudaMemcpy2DAsync(host_out + uint64_t(c0 - za) * kQ, size_t(nzf) * kQ * 8, st,
                                 size_t(w) * kQ * 8, size_t(w) * kQ * 8, R,
                                 cudaMemcpyDeviceToHost, job_s_out_));
      LBM_CUDA(cudaEventRecord(stored[i], job_s_out_));
      tmark(job_s_out_);
    };
    // the sweeps in diagonal rounds on the engine stream; programmatic
    // dependent launches (pdl_enter) hide the launch gap between slab
    // launches (LBMGPU_JOB_PDL=0: plain launches)
    const long T = steps;
    bool pdl = minb_ == 4 && !stats_.enabled();
    if (const char* e = std::getenv("LBMGPU_JOB_PDL")) pdl = pdl && std::atoi(e) != 0;
    for (long L = 0; L < T + long(S) - 1; ++L) {
      for (long j = std::min<long>(L, long(S) - 1); j >= 0; --j) {
        const long s = L - j;
        if (s >= T) continue;
        if (s == 0 && j % ki == 0) LBM_CUDA(cudaStreamWaitEvent(stream_, loaded[j / ki], 0));
        const uint32_t z0 = za + uint32_t(j) * ws, z1 = std::min<uint32_t>(z0 + ws, za + nzf);
        DirectArgs a = args(pt, z0 * static_cast<uint32_t>(P_), (z1 - z0) * static_cast<uint32_t>(P_),
                            t, 0, 0);
        if (pdl) {
          auto kern = (s & 1) ? k_full_aa_odd<true, false, 128, 4> : k_full_aa_even<true, false, 128, 4>;
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(static_cast<unsigned>(ceil_div(a.count, 128)));
          cfg.blockDim = dim3(128);
          cfg.stream = stream_;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          LBM_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
          stats_.count_launch();
        } else {
          aa_sub(s & 1, a, (s & 1) ? "full_aa_odd_soa" : "full_aa_even_soa");
        }
        if (s != T - 1) continue;
        // store chunk i is final once slab (i+1)*ko (its upper neighbour) has
        // done its last sub-step; the last chunk after the last slab
        if (j % ko == 0 && j > 0) store_chunk(static_cast<uint32_t>(j / ko - 1));
        if (j == long(S) - 1) store_chunk(Co - 1);
      }
    }
    stats_.add_launches(long(Ci) + long(Co));
    for (cudaStream_t st : {job_s_in_, job_k_in_, stream_, job_k_out_, job_s_out_})
      LBM_CUDA(cudaStreamSynchronize(st));
    if (trace) {
      auto ms = [&](size_t i) {
        float f = 0;
        cudaEventElapsedTime(&f, tev[0], tev[i]);
        return f;
      };
      fprintf(stderr, "run_job: S=%u slabs x %u planes, loads %u x %u planes, stores %u x %u planes, "
              "T=%ld\n", S, ws, Ci, wci, Co, wco, T);
      for (uint32_t i = 0; i < Ci; ++i)
        fprintf(stderr, "  load  %2u copied %8.2f loaded %8.2f ms\n", i, ms(1 + 2 * i), ms(2 + 2 * i));
      for (uint32_t i = 0; i < Co; ++i)
        fprintf(stderr, "  store %2u final %8.2f gathered %8.2f stored %8.2f ms\n", i,
                ms(1 + 2 * Ci + 3 * i), ms(2 + 2 * Ci + 3 * i), ms(3 + 2 * Ci + 3 * i));
      for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    return true;
  }

  // One-step sweeps over z-slabs (halo.hpp phases 2 / 3), per lattice step:
  //   pull: [exchange 2 (source ghost planes) || pull(interior)] -> pull(boundary)
  //   push: push(boundary) -> [exchange 3 (ghosts -> staging) || push(interior)]
  //         -> merge the staging planes into the boundary planes
  // Interior sweeps never touch a ghost plane (pull reads, push writes own
  // planes only), and the merge writes exactly the boundary-plane slots only
  // the neighbour pushes into, so nothing races.  The pull's collide pass
  // (kernels_full_os.cpp:173-190) is local to each slab.
  void os_sweeps_slabs(const TrtArgs& t, long steps) {
    const uint32_t P = static_cast<uint32_t>(P_);
    auto each = [&](bool boundary, auto&& fn) {
      for (Part& pt : parts_) {
        const uint32_t last = (pt.nzl - 1) * P;
        if (boundary) {
          fn(pt, 0u, P);
          if (pt.nzl > 1) fn(pt, last, P);
        } else if (pt.nzl > 2) {
          fn(pt, P, last - P);
        }
      }
    };
    const bool push = desc_.prop == Prop::OsPush;
    ensure_bstream();
    if (!push)
      for (Part& pt : parts_)
        launch("full_collide_soa", k_full_collide<true>,
               args(pt, 0, pt.nzl * P, t, cur_, cur_), stream_);
    for (long s = 0; s < steps; ++s) {
      const int src = cur_, dst = 1 - cur_;
      if (push) {
        auto sweep = [&](const char* name) {
          return [&, name](Part& pt, uint32_t n0, uint32_t cnt) {
            launch(name, k_full_push<true, false>, args(pt, n0, cnt, t, src, dst), stream_);
          };
        };
        // boundary stream: push(boundary) -> exchange 3 -> merge, beside
        // push(interior) (each destination slot has one writer per sweep)
        LBM_CUDA(cudaEventRecord(pev_[0], stream_));
        {
          StreamSwap on_b(stream_, bstream_);
          LBM_CUDA(cudaStreamWaitEvent(stream_, pev_[0], 0));
          each(true, sweep("full_push_soa_halo"));
          tr_->exchange(3, parts_, P_, stream_, dst);
          tr_->wait(3, stream_);
          const int g = grid_for(P_, 256);
          for (Part& pt : parts_) {
            const DirectArgs a = args(pt, 0, 0, t, src, dst);
            for (int face = 0; face < 2; ++face) {
              const int tok = stats_.begin("push_halo_merge", stream_);
              k_push_halo_merge<<<g, 256, 0, stream_>>>(
                  a, pt.stage.get() + uint64_t(face) * kQ * P_, face ? pt.nzl - 1 : 0, face == 0);
              LBM_CHECK_LAUNCH();
              stats_.end(tok, stream_);
            }
          }
          LBM_CUDA(cudaEventRecord(pev_[1], stream_));
        }
        each(false, sweep("full_push_soa"));
        LBM_CUDA(cudaStreamWaitEvent(stream_, pev_[1], 0));
      } else {
        const bool collide = s + 1 < steps;
        auto sweep = [&](const char* name) {
          return [&, name](Part& pt, uint32_t n0, uint32_t cnt) {
            const DirectArgs a = args(pt, n0, cnt, t, src, dst);
            collide ? launch(name, k_full_pull<true, true, false>, a, stream_)
                    : launch(name, k_full_pull<true, false, false>, a, stream_);
          };
        };
        // boundary stream: exchange 2 (source ghosts) -> pull(boundary),
        // beside pull(interior) (disjoint destination planes, no ghost reads)
        LBM_CUDA(cudaEventRecord(pev_[0], stream_));
        {
          StreamSwap on_b(stream_, bstream_);
          LBM_CUDA(cudaStreamWaitEvent(stream_, pev_[0], 0));
          tr_->exchange(2, parts_, P_, stream_, src);
          tr_->wait(2, stream_);
          each(true, sweep(collide ? "full_pull_soa_halo" : "full_pull_stream_soa_halo"));
          LBM_CUDA(cudaEventRecord(pev_[1], stream_));
        }
        each(false, sweep(collide ? "full_pull_soa" : "full_pull_stream_soa"));
        LBM_CUDA(cudaStreamWaitEvent(stream_, pev_[1], 0));
      }
      cur_ ^= 1;
    }
  }

  // One AA pair over z-slabs (SURVEY.md 8(e) overlap schedule):
  //   even(boundary planes) -> [exchange 0 || even(interior)] ->
  //   odd(boundary planes)  -> [exchange 1 || odd(interior)]
  // odd(boundary) reads interior slots written by even(interior), so it
  // follows it on the compute stream; the exchanged slot sets are touched by
  // no interior node, so the transfers never race with the interior sweeps.
  void aa_pair_slabs(const TrtArgs& t) {
    const uint32_t P = static_cast<uint32_t>(P_);
    auto sweep = [&](bool odd, bool boundary) {
      for (Part& pt : parts_) {
        const uint32_t last = (pt.nzl - 1) * P;
        auto run = [&](uint32_t n0, uint32_t cnt) {
          DirectArgs a = args(pt, n0, cnt, t, 0, 0);
          if (odd)
            aa_sub(true, a, boundary ? "full_aa_odd_soa_halo" : "full_aa_odd_soa");
          else
            aa_sub(false, a, boundary ? "full_aa_even_soa_halo" : "full_aa_even_soa");
        };
        if (boundary) {
          run(0, P);
          if (pt.nzl > 1) run(last, P);
        } else if (pt.nzl > 2) {
          run(P, last - P);
        }
      }
    };
    // boundary sweeps and the exchanges on the boundary stream, beside the
    // interior sweeps (the same dependencies as the peer path, aa_pair_peer;
    // the exchanged slot sets are touched by no interior node)
    ensure_bstream();
    cudaEvent_t ev_prev = pev_[0], ev_be = pev_[1], ev_ie = pev_[2], ev_bx = pev_[3];
    LBM_CUDA(cudaEventRecord(ev_prev, stream_));
    {
      NvtxRange r("aa even boundary + pre-odd exchange [boundary stream]");
      StreamSwap on_b(stream_, bstream_);
      LBM_CUDA(cudaStreamWaitEvent(stream_, ev_prev, 0));
      sweep(false, true);
      LBM_CUDA(cudaEventRecord(ev_be, stream_));
      tr_->exchange(0, parts_, P_, stream_);
    }
    {
      NvtxRange r("aa even interior [interior stream]");
      sweep(false, false);
      LBM_CUDA(cudaEventRecord(ev_ie, stream_));
    }
    {
      NvtxRange r("aa odd boundary + post-odd exchange [boundary stream]");
      StreamSwap on_b(stream_, bstream_);
      LBM_CUDA(cudaStreamWaitEvent(stream_, ev_ie, 0));
      tr_->wait(0, stream_);
      sweep(true, true);
      tr_->exchange(1, parts_, P_, stream_);
      tr_->wait(1, stream_);
      LBM_CUDA(cudaEventRecord(ev_bx, stream_));
    }
    NvtxRange r("aa odd interior [interior stream]");
    LBM_CUDA(cudaStreamWaitEvent(stream_, ev_be, 0));
    sweep(true, false);
    LBM_CUDA(cudaStreamWaitEvent(stream_, ev_bx, 0));
  }

  // ---- peer-memory transport (direct_peer.cuh) --------------
  // Per AA pair, epoch e:
  //   even(boundary) -> signal(even) -> even(interior) -> wait(even) ->
  //   odd(boundary, peer loads/stores) -> signal(odd) -> odd(interior) ->
  //   wait(odd)
  // The slots a neighbour's odd(boundary) touches in this slab (the top
  // plane's down-slots, the bottom plane's up-slots) are written by this
  // slab's even(boundary) and by nothing else in the pair, so:
  //  * wait(even) before odd(boundary): the neighbour's even(boundary) has
  //    written the slots this odd step reads from its planes;
  //  * wait(odd) before the next even(boundary): the neighbour's
  //    odd(boundary) has finished with this slab's slots (and its scatters
  //    into them are visible).
  // The two odd(boundary) steps of a face touch disjoint slot sets (down-
  // slots of the lower plane, up-slots of the upper plane), and interior
  // sweeps touch no boundary slot of another slab.
  struct PeerLink {
    double* lo[2] = {nullptr, nullptr};  // lower neighbour's grids (storage plane lo_plane = global z0-1)
    double* hi[2] = {nullptr, nullptr};  // upper neighbour's grids (storage plane hi_plane = global z1)
    uint32_t lo_plane = 0, hi_plane = 0;
    unsigned long long* lo_flags = nullptr;  // the neighbours' epoch flags (4 each)
    unsigned long long* hi_flags = nullptr;
  };
  // CUDA IPC record one rank exports (lbmgpu_peer_export)
  struct PeerRecord {
    uint32_t magic, rank, nzl, zoff, nbuf, pad;
    uint64_t buf_off[2], flag_off;
    cudaIpcMemHandle_t buf[2], flag;
  };
  static constexpr uint32_t kPeerMagic = 0x4c424d50u;  // "LBMP"

  void neighbours(int p, int& lo, int& hi) const {
    lo = p > 0 ? p - 1 : (ring_ ? nparts_ - 1 : -1);
    hi = p + 1 < nparts_ ? p + 1 : (ring_ ? 0 : -1);
  }

  void setup_peer() {
    peer_ = true;
    if (const char* e = std::getenv("LBMGPU_PEER_TIMEOUT_MS"))
      peer_timeout_ns_ = 1000000ull * std::strtoull(e, nullptr, 10);
    LBM_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&peer_err_), sizeof(int),
                           cudaHostAllocMapped));
    *peer_err_ = 0;
    LBM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&peer_err_dev_), peer_err_, 0));
    peer_abort_.alloc(1);
    LBM_CUDA(cudaMemsetAsync(peer_abort_.get(), 0, sizeof(int), stream_));
    for (Part& pt : parts_) {
      pt.pflag.alloc(4);
      LBM_CUDA(cudaMemsetAsync(pt.pflag.get(), 0, 4 * sizeof(unsigned long long), stream_));
    }
    LBM_CUDA(cudaStreamSynchronize(stream_));
    if (nranks_ > 1) return;  // lbmgpu_peer_attach links the neighbours
    // all slabs in this process: the neighbours' device pointers directly
    links_.assign(parts_.size(), PeerLink{});
    for (size_t i = 0; i < parts_.size(); ++i) {
      int lo, hi;
      neighbours(parts_[i].index, lo, hi);
      PeerLink& L = links_[i];
      if (lo >= 0) {
        const Part& q = parts_[lo];
        for (int b = 0; b < 2; ++b) L.lo[b] = q.buf[b].get();
        L.lo_plane = q.zoff + q.nzl - 1;
        L.lo_flags = q.pflag.get();
      }
      if (hi >= 0) {
        const Part& q = parts_[hi];
        for (int b = 0; b < 2; ++b) L.hi[b] = q.buf[b].get();
        L.hi_plane = q.zoff;
        L.hi_flags = q.pflag.get();
      }
    }
    peer_ready_ = true;
  }

  void peer_export(std::vector<uint8_t>& rec) override {
    if (!peer_ || nranks_ < 2)
      throw ConfigError("peer transport: export needs nranks > 1 and transport = 1");
    const Part& pt = parts_[0];
    PeerRecord r;
    std::memset(&r, 0, sizeof r);
    r.magic = kPeerMagic;
    r.rank = static_cast<uint32_t>(rank_);
    r.nzl = pt.nzl;
    r.zoff = pt.zoff;
    r.nbuf = desc_.prop == Prop::Aa ? 1 : 2;
    for (uint32_t b = 0; b < r.nbuf; ++b) {
      r.buf_off[b] = pt.buf[b].alloc_offset();
      LBM_CUDA(cudaIpcGetMemHandle(&r.buf[b],
                                   reinterpret_cast<char*>(pt.buf[b].get()) - r.buf_off[b]));
    }
    r.flag_off = pt.pflag.alloc_offset();
    LBM_CUDA(cudaIpcGetMemHandle(&r.flag, reinterpret_cast<char*>(pt.pflag.get()) - r.flag_off));
    const uint8_t* b = reinterpret_cast<const uint8_t*>(&r);
    rec.assign(b, b + sizeof r);
  }

  void peer_attach(const uint8_t* recs, size_t rec_len, int n) override {
    if (!peer_ || nranks_ < 2)
      throw ConfigError("peer transport: attach needs nranks > 1 and transport = 1");
    if (peer_ready_) throw ConfigError("peer transport: already attached");
    if (rec_len != sizeof(PeerRecord) || n != nranks_)
      throw ConfigError("peer transport: expected " + std::to_string(nranks_) +
                        " records of " + std::to_string(sizeof(PeerRecord)) + " bytes");
    auto record = [&](int r) {
      PeerRecord x;
      std::memcpy(&x, recs + size_t(r) * rec_len, sizeof x);
      if (x.magic != kPeerMagic || x.rank != static_cast<uint32_t>(r))
        throw ConfigError("peer transport: bad record for rank " + std::to_string(r));
      return x;
    };
    struct Mapped { char* buf[2]; char* flag; };
    std::vector<std::pair<int, Mapped>> opened;
    auto map = [&](int r) -> Mapped {
      for (auto& o : opened)
        if (o.first == r) return o.second;  // two ranks with the z ring: lo == hi
      const PeerRecord x = record(r);
      Mapped m{{nullptr, nullptr}, nullptr};
      for (uint32_t b = 0; b < x.nbuf && b < 2; ++b) {
        void* p = nullptr;
        LBM_CUDA(cudaIpcOpenMemHandle(&p, x.buf[b], cudaIpcMemLazyEnablePeerAccess));
        ipc_open_.push_back(p);
        m.buf[b] = static_cast<char*>(p) + x.buf_off[b];
      }
      void* f = nullptr;
      LBM_CUDA(cudaIpcOpenMemHandle(&f, x.flag, cudaIpcMemLazyEnablePeerAccess));
      ipc_open_.push_back(f);
      m.flag = static_cast<char*>(f) + x.flag_off;
      opened.emplace_back(r, m);
      return m;
    };
    int lo, hi;
    neighbours(rank_, lo, hi);
    links_.assign(1, PeerLink{});
    PeerLink& L = links_[0];
    if (lo >= 0) {
      const PeerRecord x = record(lo);
      const Mapped m = map(lo);
      for (int b = 0; b < 2; ++b) L.lo[b] = reinterpret_cast<double*>(m.buf[b]);
      L.lo_plane = x.zoff + x.nzl - 1;
      L.lo_flags = reinterpret_cast<unsigned long long*>(m.flag);
    }
    if (hi >= 0) {
      const PeerRecord x = record(hi);
      const Mapped m = map(hi);
      for (int b = 0; b < 2; ++b) L.hi[b] = reinterpret_cast<double*>(m.buf[b]);
      L.hi_plane = x.zoff;
      L.hi_flags = reinterpret_cast<unsigned long long*>(m.flag);
    }
    peer_ready_ = true;
  }

  // Copy of a boundary plane (19 slots x P, device layout) for the IPC
  // plumbing test: which = 0 lower neighbour's top plane, 1 upper
  // neighbour's bottom plane (both through the peer mapping), 2 own bottom
  // plane, 3 own top plane (first local part).
  void peer_probe(int which, std::vector<double>& out) override {
    if (!peer_ready_) throw ConfigError("peer transport: not attached");
    const Part& pt = parts_[0];
    const PeerLink& L = links_[0];
    const uint64_t plane = uint64_t(kQ) * P_;
    const double* src = nullptr;
    if (which == 0 && L.lo[0]) src = L.lo[0] + L.lo_plane * plane;
    if (which == 1 && L.hi[0]) src = L.hi[0] + L.hi_plane * plane;
    if (which == 2) src = pt.buf[0].get() + uint64_t(pt.zoff) * plane;
    if (which == 3) src = pt.buf[0].get() + uint64_t(pt.zoff + pt.nzl - 1) * plane;
    if (!src) throw ConfigError("peer transport: no such plane");
    out.resize(plane);
    LBM_CUDA(cudaStreamSynchronize(stream_));
    LBM_CUDA(cudaMemcpy(out.data(), src, plane * sizeof(double), cudaMemcpyDefault));
  }

  void peer_check() const {
    if (!peer_ready_)
      throw ConfigError("peer transport: lbmgpu_peer_attach has not been called");
    if (*static_cast<volatile int*>(peer_err_))
      throw DeviceError("peer transport: a neighbour's sub-step signal timed out (ranks must "
                        "call advance collectively within LBMGPU_PEER_TIMEOUT_MS); the slab "
                        "state is no longer consistent");
  }

  // After the stream work of a host call: a wait that timed out inside it
  // is reported by that call (and by every later one).
  void check_health() override {
    if (!peer_) return;
    LBM_CUDA(cudaStreamSynchronize(stream_));
    if (bstream_) LBM_CUDA(cudaStreamSynchronize(bstream_));
    peer_check();
  }

  void peer_signal(int kind, unsigned long long e) {
    for (const PeerLink& L : links_) {
      const int tok = stats_.begin("peer_signal", stream_);
      k_peer_signal<<<1, 32, 0, stream_>>>(L.lo_flags ? L.lo_flags + 2 * kind + 1 : nullptr,
                                           L.hi_flags ? L.hi_flags + 2 * kind : nullptr, e);
      LBM_CHECK_LAUNCH();
      stats_.end(tok, stream_);
    }
  }

  void peer_wait(int kind, unsigned long long e) {
    for (size_t i = 0; i < parts_.size(); ++i) {
      const PeerLink& L = links_[i];
      unsigned long long* own = parts_[i].pflag.get();
      const int tok = stats_.begin("peer_wait", stream_);
      k_peer_wait<<<1, 32, 0, stream_>>>(L.lo_flags ? own + 2 * kind : nullptr,
                                         L.hi_flags ? own + 2 * kind + 1 : nullptr, e,
                                         peer_err_dev_, peer_abort_.get(), peer_timeout_ns_);
      LBM_CHECK_LAUNCH();
      stats_.end(tok, stream_);
    }
  }

  // Boundary work of the peer AA path runs on its own high-priority stream
  // beside the interior sweeps (helpers launch on stream_, so it is swapped
  // for the scope).
  struct StreamSwap {
    cudaStream_t& x;
    cudaStream_t& y;
    StreamSwap(cudaStream_t& a, cudaStream_t& b) : x(a), y(b) { std::swap(x, y); }
    ~StreamSwap() { std::swap(x, y); }
  };

  void ensure_bstream() {
    if (bstream_) return;
    int least = 0, greatest = 0;
    LBM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    LBM_CUDA(cudaStreamCreateWithPriority(&bstream_, cudaStreamNonBlocking, greatest));
    nvtxNameCudaStreamA(bstream_, "lbmgpu boundary");
    for (cudaEvent_t& e : pev_) LBM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }

  // One AA pair, epoch e; boundary stream B, interior stream I:
  //   B: [I's previous work] even(b) signal(even)                wait(ev_ie) wait(even) odd(b) signal(odd) wait(odd)
  //   I:                     even(i) --ev_ie-->     [ev_be] odd(i) [ev_bo]
  // even(b) and even(i) touch disjoint own slots, and so do odd(b) and
  // odd(i) (the bottom plane's odd step uses plane 1's up-slots, plane 1's
  // uses plane 0's down-slots): each sub-step's boundary work -- with the
  // neighbour traffic and the flag waits -- overlaps the interior sweep.
  // odd(b) follows even(i) (it reads planes 1 / nzl-2), odd(i) follows
  // even(b); the next pair's even(b) follows odd(i) and the neighbours'
  // odd(b) (wait(odd)), its even(i) follows odd(b) (ev_bo).
  void aa_pair_peer(const TrtArgs& t) {
    const uint32_t P = static_cast<uint32_t>(P_);
    const unsigned long long e = ++epoch_;
    ensure_bstream();
    cudaEvent_t ev_prev = pev_[0], ev_be = pev_[1], ev_ie = pev_[2], ev_bo = pev_[3];
    auto sweep = [&](bool odd, bool boundary) {
      for (size_t i = 0; i < parts_.size(); ++i) {
        Part& pt = parts_[i];
        const uint32_t last = (pt.nzl - 1) * P;
        auto run = [&](uint32_t n0, uint32_t cnt) {
          DirectArgs a = args(pt, n0, cnt, t, 0, 0);
          if (!boundary) {
            aa_sub(odd, a, odd ? "full_aa_odd_soa" : "full_aa_even_soa");
          } else if (!odd) {
            aa_sub(false, a, "full_aa_even_soa_halo");
          } else {
            const PeerLink& L = links_[i];
            const PeerArgs pa{L.lo[0], L.hi[0], L.lo_plane, L.hi_plane, peer_abort_.get()};
            const int tok = stats_.begin("full_aa_odd_soa_peer", stream_);
            k_full_aa_odd_peer<<<static_cast<unsigned>(ceil_div(cnt, 128)), 128, 0, stream_>>>(
                a, pa);
            LBM_CHECK_LAUNCH();
            stats_.end(tok, stream_);
          }
        };
        if (boundary) {
          run(0, P);
          if (pt.nzl > 1) run(last, P);
        } else if (pt.nzl > 2) {
          run(P, last - P);
        }
      }
    };
    LBM_CUDA(cudaEventRecord(ev_prev, stream_));
    {
      NvtxRange r("aa even boundary + signal [boundary stream]");
      StreamSwap on_b(stream_, bstream_);
      LBM_CUDA(cudaStreamWaitEvent(stream_, ev_prev, 0));
      sweep(false, true);
      peer_signal(0, e);
      LBM_CUDA(cudaEventRecord(ev_be, stream_));
    }
    {
      NvtxRange r("aa even interior [interior stream]");
      sweep(false, false);
      LBM_CUDA(cudaEventRecord(ev_ie, stream_));
    }
    {
      NvtxRange r("aa odd boundary: wait, peer sweep, signal, wait [boundary stream]");
      StreamSwap on_b(stream_, bstream_);
      LBM_CUDA(cudaStreamWaitEvent(stream_, ev_ie, 0));
      peer_wait(0, e);
      sweep(true, true);
      peer_signal(1, e);
      peer_wait(1, e);
      LBM_CUDA(cudaEventRecord(ev_bo, stream_));
    }
    NvtxRange r("aa odd interior [interior stream]");
    LBM_CUDA(cudaStreamWaitEvent(stream_, ev_be, 0));
    sweep(true, false);
    LBM_CUDA(cudaStreamWaitEvent(stream_, ev_bo, 0));
  }

  // One-step sweeps with the peer transport.  Every op (the pull's collide
  // pass, each sweep) touching boundary planes runs as
  //   wait(neighbours' op e-1) -> op(boundary planes) -> signal(e) -> op(interior)
  // A neighbour's op e+1 touches only this slab's boundary planes of the grid
  // this op does not write (pull: reads our source of e+1 = destination of
  // e, written by our boundary sweep before the signal; push: writes our
  // destination of e+1 = source of e, read by our boundary sweep before the
  // signal) and each slot has one writer per sweep, so one flag per op
  // orders everything.
  void os_sweeps_peer(const TrtArgs& t, long steps) {
    const uint32_t P = static_cast<uint32_t>(P_);
    const bool push = desc_.prop == Prop::OsPush;
    auto each = [&](bool boundary, auto&& fn) {
      for (size_t i = 0; i < parts_.size(); ++i) {
        Part& pt = parts_[i];
        const uint32_t last = (pt.nzl - 1) * P;
        if (boundary) {
          fn(i, pt, 0u, P);
          if (pt.nzl > 1) fn(i, pt, last, P);
        } else if (pt.nzl > 2) {
          fn(i, pt, P, last - P);
        }
      }
    };
    // boundary part on the boundary stream beside the interior part (the two
    // write disjoint slots and only read the source grid); each op joins both
    ensure_bstream();
    auto op = [&](auto&& boundary_fn, auto&& interior_fn) {
      const unsigned long long e = ++epoch_;
      LBM_CUDA(cudaEventRecord(pev_[0], stream_));
      {
        StreamSwap on_b(stream_, bstream_);
        LBM_CUDA(cudaStreamWaitEvent(stream_, pev_[0], 0));
        peer_wait(0, e - 1);
        each(true, boundary_fn);
        peer_signal(0, e);
        LBM_CUDA(cudaEventRecord(pev_[1], stream_));
      }
      each(false, interior_fn);
      LBM_CUDA(cudaStreamWaitEvent(stream_, pev_[1], 0));
    };
    if (!push) {
      auto coll = [&](size_t, Part& pt, uint32_t n0, uint32_t cnt) {
        launch("full_collide_soa", k_full_collide<true>, args(pt, n0, cnt, t, cur_, cur_),
               stream_);
      };
      op(coll, coll);
    }
    for (long s = 0; s < steps; ++s) {
      const int src = cur_, dst = 1 - cur_;
      const bool collide = push || s + 1 < steps;
      auto interior = [&](size_t, Part& pt, uint32_t n0, uint32_t cnt) {
        const DirectArgs a = args(pt, n0, cnt, t, src, dst);
        if (push)
          launch("full_push_soa", k_full_push<true, false>, a, stream_);
        else if (collide)
          launch("full_pull_soa", k_full_pull<true, true, false>, a, stream_);
        else
          launch("full_pull_stream_soa", k_full_pull<true, false, false>, a, stream_);
      };
      auto boundary = [&](size_t i, Part& pt, uint32_t n0, uint32_t cnt) {
        const DirectArgs a = args(pt, n0, cnt, t, src, dst);
        const PeerLink& L = links_[i];
        const int g = push ? dst : src;  // the neighbour grid the boundary touches
        const PeerArgs pa{L.lo[g], L.hi[g], L.lo_plane, L.hi_plane, peer_abort_.get()};
        const unsigned grid = static_cast<unsigned>(ceil_div(cnt, 256));
        const int tok = stats_.begin(push ? "full_push_soa_peer"
                                     : collide ? "full_pull_soa_peer"
                                               : "full_pull_stream_soa_peer",
                                     stream_);
        if (push)
          k_full_push_peer<<<grid, 256, 0, stream_>>>(a, pa);
        else if (collide)
          k_full_pull_peer<true><<<grid, 256, 0, stream_>>>(a, pa);
        else
          k_full_pull_peer<false><<<grid, 256, 0, stream_>>>(a, pa);
        LBM_CHECK_LAUNCH();
        stats_.end(tok, stream_);
      };
      op(boundary, interior);
      cur_ ^= 1;
    }
    // the last op's neighbours must be done with this slab before the host
    // touches it (snapshot / load_state) or the next advance starts
    peer_wait(0, epoch_);
  }

  CanonArgs canon_args(const Part& pt, int buf) const {
    CanonArgs c;
    c.buf = const_cast<double*>(pt.buf[buf].get());
    c.node_of = pt.node_of.get();
    c.canon = nparts_ > 1 ? pt.canon.get() : nullptr;
    c.kbase = 0;
    c.k0 = 0;
    c.k1 = pt.n_fluid;
    c.c0 = 0;
    c.nx = nx_;
    c.ny = ny_;
    c.zoff = pt.zoff;
    c.P = P_;
    return c;
  }

  // restrict the part's k-range to canonical indices [c0, c0+count)
  bool clip(const Part& pt, uint64_t c0, uint64_t count, CanonArgs& c) const {
    if (nparts_ == 1) {
      c.k0 = c0;
      c.k1 = std::min<uint64_t>(c0 + count, pt.n_fluid);
    } else {
      const auto& h = pt.canon_host;
      c.k0 = std::lower_bound(h.begin(), h.end(), c0) - h.begin();
      c.k1 = std::lower_bound(h.begin(), h.end(), c0 + count) - h.begin();
    }
    c.c0 = c0;
    return c.k1 > c.k0;
  }

  void gather_canonical(uint64_t c0, uint64_t count, double* out) override {
    for (const Part& pt : parts_) {
      CanonArgs c = canon_args(pt, cur_);
      if (!clip(pt, c0, count, c)) continue;
      const int g = grid_for(c.k1 - c.k0, 256);
      desc_.soa ? k_full_canon<true, true><<<g, 256, 0, stream_>>>(c, out)
                : k_full_canon<false, true><<<g, 256, 0, stream_>>>(c, out);
      LBM_CHECK_LAUNCH();
    }
  }

  void scatter_canonical(uint64_t c0, uint64_t count, const double* in) override {
    for (const Part& pt : parts_) {
      CanonArgs c = canon_args(pt, cur_);
      if (!clip(pt, c0, count, c)) continue;
      const int g = grid_for(c.k1 - c.k0, 256);
      desc_.soa ? k_full_canon<true, false><<<g, 256, 0, stream_>>>(
                      c, const_cast<double*>(in))
                : k_full_canon<false, false><<<g, 256, 0, stream_>>>(
                      c, const_cast<double*>(in));
      LBM_CHECK_LAUNCH();
    }
  }

  // Process-local rows (multi-process): rows k in [k0, k0+count) of this
  // process's slab in canonical order, staged contiguously.
  uint64_t local_rows() const override {
    uint64_t n = 0;
    for (const Part& pt : parts_) n += pt.n_fluid;
    return n;
  }
  void local_canonical_index(uint64_t* out) const override {
    uint64_t off = 0;
    for (const Part& pt : parts_) {
      if (nparts_ == 1)
        for (uint64_t k = 0; k < pt.n_fluid; ++k) out[off + k] = k;
      else
        std::copy(pt.canon_host.begin(), pt.canon_host.end(), out + off);
      off += pt.n_fluid;
    }
  }
  void gather_local(uint64_t k0, uint64_t count, double* out, bool to_staging) override {
    // local rows are the concatenation of the parts' k-ranges
    uint64_t base = 0;
    for (const Part& pt : parts_) {
      const uint64_t a = std::max(k0, base), b = std::min(k0 + count, base + pt.n_fluid);
      if (a < b) {
        CanonArgs c = canon_args(pt, cur_);
        c.canon = nullptr;       // staging row = k - k0 (+ offset)
        c.kbase = 0;
        c.k0 = a - base;
        c.k1 = b - base;
        c.c0 = c.k0;
        double* dst = out + (a - k0) * kQ;
        const int g = grid_for(b - a, 256);
        if (to_staging)
          desc_.soa ? k_full_canon<true, true><<<g, 256, 0, stream_>>>(c, dst)
                    : k_full_canon<false, true><<<g, 256, 0, stream_>>>(c, dst);
        else
          desc_.soa ? k_full_canon<true, false><<<g, 256, 0, stream_>>>(c, dst)
                    : k_full_canon<false, false><<<g, 256, 0, stream_>>>(c, dst);
        LBM_CHECK_LAUNCH();
      }
      base += pt.n_fluid;
    }
  }

  void load_perturbed(uint64_t seed, double amp) override {
    for (const Part& pt : parts_) {
      CanonArgs c = canon_args(pt, cur_);
      if (c.k1 == 0) continue;
      const int g = grid_for(c.k1, 256);
      desc_.soa ? k_full_perturb<true><<<g, 256, 0, stream_>>>(c, seed, amp)
                : k_full_perturb<false><<<g, 256, 0, stream_>>>(c, seed, amp);
      LBM_CHECK_LAUNCH();
    }
  }

  void macro_fields(double* rho, double* u) override {
    if (nranks_ > 1)
      throw ConfigError("macro_fields: the field is split across processes");
    for (const Part& pt : parts_) {
      CanonArgs c = canon_args(pt, cur_);
      if (c.k1 == 0) continue;
      const int g = grid_for(c.k1, 256);
      desc_.soa ? k_full_macro<true><<<g, 256, 0, stream_>>>(c, rho, u)
                : k_full_macro<false><<<g, 256, 0, stream_>>>(c, rho, u);
      LBM_CHECK_LAUNCH();
    }
  }

  // Mass over fluid and solid nodes of the current buffer (full_lattice.cpp:
  // 72-87), own planes only, compensated device sum; summed over processes.
  double total_mass() override {
    double m = 0.0;
    for (const Part& pt : parts_) {
      const uint64_t per_plane = P_ * kQ;
      m += device_sum(pt.buf[cur_].get() + uint64_t(pt.zoff) * per_plane,
                      uint64_t(pt.nzl) * per_plane, stream_);
    }
    if (nranks_ > 1 && !tr_)
      throw ConfigError("total_mass over several processes needs the NCCL id (mass reduction)");
    return tr_ && nranks_ > 1 ? tr_->sum(m) : m;
  }

 private:
  int nx_ = 0, ny_ = 0, nz_ = 0;
  uint64_t P_ = 0;
  int nparts_ = 1, rank_ = 0, nranks_ = 1;
  int cur_ = 0;
  // min CTAs/SM of the 128-thread register AA kernels: 4 caps them at 128
  // registers, i.e. 16 resident warps/SM (DESIGN.md §4 has the sweep; one
  // 256-thread CTA at 140 registers, 8 warps, ran 33% slower).  128-thread
  // CTAs retire and refill warps in smaller groups than 2 x 8 warps:
  // measured cfg 5 odd 6443 -> 6650 GB/s, even 6793 -> 6830.
  int minb_ = 4;
  uint32_t tile_by_ = 8;  // AoS 3-D tiles: y tiles per traversal block (tile_origin)
  bool fused_push_as_pull_ = true;  // SoA push's fused launch in pull order
  // pipelined job (run_job): column plan, staging, copy streams, events
  bool job_checked_ = false, job_ok_ = false;
  uint32_t job_za_ = 0, job_zb_ = 0;
  uint64_t job_cols_ = 0;
  DevBuf<uint32_t> job_col_of_;
  DevBuf<double> job_in_[2], job_out_[2];
  cudaStream_t job_s_in_ = nullptr, job_s_out_ = nullptr;    // PCIe copies
  cudaStream_t job_k_in_ = nullptr, job_k_out_ = nullptr;    // layout kernels
  std::vector<cudaEvent_t> job_ev_;
  uint64_t fused_bytes_ = 96ull << 20;  // fused multi-sweep launch threshold
  int sm_count_ = 148;
  std::vector<Part> parts_;
  std::unique_ptr<Transport> tr_;
  bool ring_ = false;                   // the halo plan includes the z ring
  bool peer_ = false, peer_ready_ = false;
  unsigned long long epoch_ = 0;        // AA pairs run with the peer transport
  unsigned long long peer_timeout_ns_ = 30000000000ull;
  std::vector<PeerLink> links_;         // per local part
  int* peer_err_ = nullptr;             // host-mapped wait-timeout flag
  int* peer_err_dev_ = nullptr;
  DevBuf<int> peer_abort_;              // device copy of the timeout flag (PeerArgs::abort)
  std::vector<void*> ipc_open_;         // CUDA IPC mappings to close
  cudaStream_t bstream_ = nullptr;      // peer AA path: boundary stream (aa_pair_peer)
  cudaEvent_t pev_[4] = {nullptr, nullptr, nullptr, nullptr};
  GeomSpec geom_;  // kind/parameters for the analytic solid test (custom: flags)
};

}  // namespace

std::unique_ptr<Engine> make_direct_engine(const Descriptor& d,
                                           const GeomSpec& g,
                                           const DistSpec& dist) {
  return std::make_unique<DirectEngine>(d, g, dist);
}

}  // namespace lbmgpu
