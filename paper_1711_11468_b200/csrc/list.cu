// Indirect (list / adjacency) addressing: list-push-*, list-pull-*,
// list-pull-split-nt-*, list-aa-*, list-aa-ria-soa, list-aa-pv-soa.
//
// Reference: ListLattice / build_structure (src/list_lattice.cpp:123-310),
// ListOsKernel (src/kernels_list_os.cpp:9-97), ListNtKernel
// (src/kernels_list_nt.cpp:77-167), ListAaKernel / ListAaRiaKernel
// (src/kernels_list_aa.cpp:8-251).
//
// The structure is built ON THE DEVICE and is bit-exact with the reference:
//  * node order (order_nodes, :123-141): a bijective traversal position t(i)
//    per box node (blk = 0: canonical x,y,z; blk > 0: the y-z tile order),
//    an exclusive scan of the fluid flags in t order gives the list rank;
//  * SoA slot map: starts[d] + n with the reference's padding_offsets;
//    AoS: 19n + d (list_lattice.hpp:66-75);
//  * adjacency entry (n, d) (:177-191): neighbour at n + c_look (look = d for
//    Scatter, opp(d) for Gather; periodic wrap, else Outside) -> slot(m, d)
//    if fluid else slot(n, opp d) (half-way bounce-back baked in).
// The PDF arrays keep the reference slot numbering exactly (the adjacency
// values ARE slot numbers); only the adjacency ARRAY is stored d-major,
// adj[(d-1)*N + n], so the 18 index loads of a warp are coalesced.  The
// canonical [n*18 + d-1] order is produced on export.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <tuple>
#include <unordered_map>

#include "halo.hpp"
#include "tma.cuh"
#include "lbm.hpp"

#include "list_sweeps.cuh"
#include "list_build.cuh"
#include "list_ria.cuh"
#include "list_parts.cuh"
#include "list_aos_tile.cuh"

namespace lbmgpu {

// ------------------------------------------------------------------ engine
namespace {

int grid_for(uint64_t n, int threads) {
  return static_cast<int>(std::min<uint64_t>(ceil_div(n, threads), 148ull * 64));
}

class ListEngine final : public Engine {
 public:
  // node-range part of a decomposed list lattice (local numbering, see
  // list_parts.cuh): 19 * nloc own slots + nghost ghost slots
  struct LPart {
    int index = 0;
    uint64_t n0 = 0, n1 = 0, nloc = 0, nghost = 0, head = 0, tail = 0;
    DevBuf<double> own;
    DevBuf<uint32_t> adj;  // local d-major adjacency [(d-1) * nloc + j]
    double* buf = nullptr;
    ListArgs args(const TrtArgs& t, bool soa) const {
      ListArgs a{};
      a.src = a.dst = buf;
      a.adj = adj.get();
      a.N = nloc;
      for (int q = 0; q < kQ; ++q) a.starts[q] = soa ? uint64_t(q) * nloc : 0;
      a.trt = t;
      a.nb = 0;
      a.ne = nloc;
      return a;
    }
  };
  struct LLink {
    int r = 0, s = 0;      // slots of s's nodes referenced by r's nodes
    uint64_t count = 0;
    uint64_t ghost0 = 0;   // first ghost index of these slots on r (local)
    DevBuf<uint32_t> sidx; // local own index of each slot on s
    DevBuf<double> stage;  // NCCL staging of the gathered (s side) values
  };

  ListEngine(const Descriptor& d, const GeomSpec& g, const Padding& pad,
             const DistSpec& dist) {
    desc_ = d;
    LBM_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    nvtxNameCudaStreamA(stream_, "lbmgpu interior");
    DeviceGeometry geo = build_geometry_device(g, stream_);
    nx_ = geo.nx;
    ny_ = geo.ny;
    nz_ = geo.nz;
    per_ = geo.periodic;
    const uint64_t V = geo.volume();
    n_fluid_ = static_cast<uint64_t>(geo.n_fluid);
    if (n_fluid_ >= (1ull << 32))
      throw ConfigError("list lattice: more than 2^32 fluid nodes");

    // slot map (list_lattice.cpp:166-173)
    uint64_t total = 0;
    std::array<uint64_t, kQ> st{};
    if (d.soa) {
      st = padding_offsets(n_fluid_, pad, &total);
    } else {
      total = n_fluid_ * kQ;
    }
    if (total >= (1ull << 32))
      throw ConfigError("list lattice: " + std::to_string(total) +
                        " PDF slots exceed the 32-bit adjacency range");
    total_slots_ = total;
    for (int q = 0; q < kQ; ++q) starts_[q] = st[q];

    // ranks in traversal order and canonical order
    // the AoS AA odd step's staging tiles keep the box-order scan (V + 1
    // entries: crank[V] = N closes the last row)
    // (their grid is (z tiles, y tiles, x tiles): boxes beyond 65535 tiles in
    // y or x -- ny, nx > 131070 at the narrowest tile shape -- take the
    // per-node kernel)
    const bool aos_tiles = !d.soa && d.prop == Prop::Aa && d.blk == 0 && !d.ria &&
                           ny_ <= 131070 && nx_ <= 131070;
    DevBuf<uint32_t> crank(V + 1);
    scan_fluid(geo.flags.get(), crank.get(), V, stream_);
    DevBuf<uint32_t> trank;
    if (d.blk > 0) {
      DevBuf<uint8_t> ft(V);
      k_trav_flags<<<grid_for(V, 256), 256, 0, stream_>>>(geo.flags.get(), nx_,
                                                          ny_, nz_, d.blk,
                                                          ft.get());
      LBM_CHECK_LAUNCH();
      trank.alloc(V);
      scan_fluid(ft.get(), trank.get(), V, stream_);
      list_of_canon_.alloc(n_fluid_);
    }
    DevBuf<uint32_t> rank(V);
    nodes_.alloc(3 * n_fluid_);
    k_rank_nodes<<<grid_for(V, 256), 256, 0, stream_>>>(
        geo.flags.get(), trank.get(), crank.get(), nx_, ny_, nz_, d.blk,
        rank.get(), nodes_.get(), d.blk > 0 ? list_of_canon_.get() : nullptr);
    LBM_CHECK_LAUNCH();

    // adjacency: Gather for pull, Scatter for push and AA
    // (kernels_list_os.cpp:19-20, kernels_list_aa.cpp:40)
    scatter_ = d.prop != Prop::OsPull;
    adj_.alloc(18 * n_fluid_);
    AdjBuild b{};
    b.flags = geo.flags.get();
    b.rank = rank.get();
    b.nodes = nodes_.get();
    b.adj = adj_.get();
    b.N = n_fluid_;
    b.nx = nx_;
    b.ny = ny_;
    b.nz = nz_;
    for (int a = 0; a < 3; ++a) b.per[a] = per_[a];
    b.soa = d.soa;
    b.scatter = scatter_;
    for (int q = 0; q < kQ; ++q) b.starts[q] = starts_[q];
    k_build_adj<<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(b);
    LBM_CHECK_LAUNCH();

    // PDF buffers initialised to the weights (list_lattice.cpp:248-264);
    // pad slots are zeroed (the reference leaves them untouched).
    const int nbuf = d.prop == Prop::Aa ? 1 : 2;
    for (int q = 0; q < nbuf; ++q) {
      buf_[q].alloc(total_slots_);
      LBM_CUDA(cudaMemsetAsync(buf_[q].get(), 0, buf_[q].bytes(), stream_));
      ListArgs a = base_args();
      d.soa ? k_list_init<true><<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(buf_[q].get(), a)
            : k_list_init<false><<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(buf_[q].get(), a);
      LBM_CHECK_LAUNCH();
    }
    LBM_CUDA(cudaStreamSynchronize(stream_));
    if (aos_tiles) {
      const uint32_t nf = static_cast<uint32_t>(n_fluid_);
      LBM_CUDA(cudaMemcpy(crank.get() + V, &nf, 4, cudaMemcpyHostToDevice));
      crank_ = std::move(crank);
      if (const char* e = std::getenv("LBMGPU_LTILE")) ltile_ = std::atoi(e);
    }
    // streaming stores for the nt names and for lattices far beyond L2
    cs_nt_ = d.nt_streams > 0;
    if (d.ria) build_ria();
    if (const char* e = std::getenv("LBMGPU_PULL_PID"))
      if (std::atoi(e) != 0 && !d.ria && d.prop == Prop::OsPull && d.soa) {
        build_ria();  // pattern ids of the Gather table
        pull_pid_ = ria_npat_ > 0;
      }
    {
      int dev = 0;
      LBM_CUDA(cudaGetDevice(&dev));
      LBM_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, dev));
      if (const char* e = std::getenv("LBMGPU_RIA_MODE")) ria_mode_ = std::atoi(e);
      if (const char* e = std::getenv("LBMGPU_FUSED_MB"))
        fused_bytes_ = uint64_t(std::atoll(e)) << 20;
      // adjacency L2 prefetch distance, in resident-grid waves (0 = off)
      // one wave: measured best on B200 (cfg 2 list-aa odd: 5946 -> 6530 GB/s)
      pf_ = uint64_t(sm_count_) * 2 * 256;
    }
    const int parts = dist.nranks > 1 ? dist.nranks : std::max(1, dist.virtual_parts);
    if (parts > 1) setup_parts(dist, parts);
  }

  ~ListEngine() override {
    if (stream_) cudaStreamSynchronize(stream_);
    if (bstream_) {
      cudaStreamSynchronize(bstream_);
      cudaStreamDestroy(bstream_);
    }
    for (cudaEvent_t e : bev_)
      if (e) cudaEventDestroy(e);
    if (lnccl_) nccl_destroy(lnccl_);
    if (stream_) cudaStreamDestroy(stream_);
  }

  // ---- node-range decomposition -------------------------------------------
  // Links and local structures are derived from the global adjacency, which
  // (with the global PDF array) is released afterwards: each part keeps
  // 19 * nloc + nghost doubles and 18 * nloc indices.
  void setup_parts(const DistSpec& dist, int parts) {
    if (desc_.prop != Prop::Aa || desc_.ria)
      throw ConfigError("list decomposition is implemented for list-aa-soa / list-aa-aos "
                        "(kernel '" + desc_.name + "')");
    if (desc_.blk != 0)
      throw ConfigError("list decomposition needs blk = 0 (node ranges = x-slabs)");
    if (uint64_t(parts) > n_fluid_) throw ConfigError("more parts than fluid nodes");
    if (dist.nranks > 1 && !dist.have_id)
      throw ConfigError("dist: nranks > 1 needs the NCCL unique id");
    lnparts_ = parts;
    lrank_ = dist.rank;
    lnranks_ = dist.nranks;
    const bool multi_process = dist.nranks > 1;
    const int soa = desc_.soa ? 1 : 0;
    auto range = [&](int p) {
      return std::pair<uint64_t, uint64_t>(n_fluid_ * uint64_t(p) / parts,
                                           n_fluid_ * uint64_t(p + 1) / parts);
    };
    auto is_local = [&](int p) { return !multi_process || p == lrank_; };
    const ListArgs g = base_args();
    // links (r <- s) this process takes part in: sorted global slot lists
    std::vector<DevBuf<uint32_t>> slots;  // parallel to links_
    for (int r = 0; r < parts; ++r)
      for (int s = 0; s < parts; ++s) {
        if (r == s || !(is_local(r) || is_local(s))) continue;
        const auto [rn0, rn1] = range(r);
        const auto [sn0, sn1] = range(s);
        const uint64_t cnt = (rn1 - rn0) * 18;
        DevBuf<uint8_t> flags(cnt);
        DevBuf<uint32_t> vals(cnt);
        k_link_flags<<<grid_for(cnt, 256), 256, 0, stream_>>>(g, soa, rn0, rn1, sn0, sn1,
                                                              flags.get(), vals.get());
        LBM_CHECK_LAUNCH();
        DevBuf<uint32_t> sel(cnt);
        DevBuf<unsigned long long> nsel(1);
        size_t tmp = 0;
        LBM_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, vals.get(), flags.get(), sel.get(),
                                            nsel.get(), static_cast<int64_t>(cnt), stream_));
        DevBuf<uint8_t> t(tmp);
        LBM_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, vals.get(), flags.get(), sel.get(),
                                            nsel.get(), static_cast<int64_t>(cnt), stream_));
        unsigned long long k = 0;
        LBM_CUDA(cudaMemcpyAsync(&k, nsel.get(), 8, cudaMemcpyDeviceToHost, stream_));
        LBM_CUDA(cudaStreamSynchronize(stream_));
        if (k == 0) continue;
        DevBuf<uint32_t> sorted(k);
        tmp = 0;
        LBM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, sel.get(), sorted.get(),
                                                static_cast<int64_t>(k), 0, 32, stream_));
        DevBuf<uint8_t> t2(tmp);
        LBM_CUDA(cub::DeviceRadixSort::SortKeys(t2.get(), tmp, sel.get(), sorted.get(),
                                                static_cast<int64_t>(k), 0, 32, stream_));
        LLink l;
        l.r = r;
        l.s = s;
        l.count = k;
        links_.push_back(std::move(l));
        slots.push_back(std::move(sorted));
      }
    // parts living in this process
    for (int p = 0; p < parts; ++p) {
      if (!is_local(p)) continue;
      LPart lp;
      lp.index = p;
      std::tie(lp.n0, lp.n1) = range(p);
      lp.nloc = lp.n1 - lp.n0;
      // ghost list = the sorted link lists (p <- s) concatenated in s order
      std::vector<uint64_t> gofs(parts, 0), gcnt(parts, 0);
      for (size_t i = 0; i < links_.size(); ++i)
        if (links_[i].r == p) {
          links_[i].ghost0 = lp.nloc * kQ + lp.nghost;
          gofs[links_[i].s] = lp.nghost;
          gcnt[links_[i].s] = links_[i].count;
          lp.nghost += links_[i].count;
        }
      const uint64_t nslots = lp.nloc * kQ + lp.nghost;
      if (nslots >= (1ull << 32))
        throw ConfigError("list decomposition: more than 2^32 local slots in one part");
      DevBuf<uint32_t> gslots(std::max<uint64_t>(lp.nghost, 1));
      for (size_t i = 0; i < links_.size(); ++i)
        if (links_[i].r == p)
          LBM_CUDA(cudaMemcpyAsync(gslots.get() + gofs[links_[i].s], slots[i].get(),
                                   links_[i].count * 4, cudaMemcpyDeviceToDevice, stream_));
      DevBuf<uint64_t> dofs(parts), dcnt(parts);
      LBM_CUDA(cudaMemcpyAsync(dofs.get(), gofs.data(), parts * 8, cudaMemcpyHostToDevice,
                               stream_));
      LBM_CUDA(cudaMemcpyAsync(dcnt.get(), gcnt.data(), parts * 8, cudaMemcpyHostToDevice,
                               stream_));
      lp.adj.alloc(18 * lp.nloc);
      k_local_adj<<<grid_for(18 * lp.nloc, 256), 256, 0, stream_>>>(
          g, soa, lp.n0, lp.nloc, parts, gslots.get(), dofs.get(), dcnt.get(), lp.adj.get());
      LBM_CHECK_LAUNCH();
      lp.own.alloc(nslots);
      lp.buf = lp.own.get();
      k_local_init<<<grid_for(nslots, 256), 256, 0, stream_>>>(
          g, soa, buf_[0].get(), lp.n0, lp.nloc, gslots.get(), lp.nghost, lp.buf);
      LBM_CHECK_LAUNCH();
      // boundary nodes (any ghost entry) -> head / tail spans (x-slab ends)
      DevBuf<uint8_t> mask(lp.nloc);
      k_ghost_mask<<<grid_for(lp.nloc, 256), 256, 0, stream_>>>(lp.adj.get(), lp.nloc,
                                                                 mask.get());
      LBM_CHECK_LAUNCH();
      std::vector<uint8_t> h(lp.nloc);
      LBM_CUDA(cudaMemcpyAsync(h.data(), mask.get(), lp.nloc, cudaMemcpyDeviceToHost, stream_));
      LBM_CUDA(cudaStreamSynchronize(stream_));
      const uint64_t cnt = lp.nloc;
      uint64_t head = 0, tail = 0;
      for (uint64_t i = 0; i < cnt / 2; ++i)
        if (h[i]) head = i + 1;
      for (uint64_t i = cnt / 2; i < cnt; ++i)
        if (h[i]) {
          tail = cnt - i;
          break;
        }
      lp.head = head;
      lp.tail = std::min(tail, cnt - head);
      lparts_.push_back(std::move(lp));
    }
    // sender-side local indices; NCCL staging
    for (size_t i = 0; i < links_.size(); ++i) {
      LLink& l = links_[i];
      if (is_local(l.s)) {
        const auto [sn0, sn1] = range(l.s);
        l.sidx.alloc(l.count);
        k_own_local_idx<<<grid_for(l.count, 256), 256, 0, stream_>>>(
            g, soa, sn0, sn1 - sn0, slots[i].get(), l.count, l.sidx.get());
        LBM_CHECK_LAUNCH();
      }
      if (multi_process || dist.have_id) l.stage.alloc(l.count);
    }
    if (multi_process || dist.have_id)
      lnccl_ = nccl_create({}, multi_process ? lrank_ : 0, multi_process ? lnranks_ : 1,
                           dist.nccl_id.data());
    LBM_CUDA(cudaStreamSynchronize(stream_));
    // memory scaling: the global arrays are not needed any more
    buf_[0].release();
    adj_.release();
  }

  LPart* part_of(int index) {
    for (LPart& p : lparts_)
      if (p.index == index) return &p;
    return nullptr;
  }

  // phase 0 (after even): slots flow s -> r (s's own slots -> r's ghosts);
  // phase 1 (after odd): r -> s.  r's ghosts of one link are contiguous.
  void list_exchange(int phase) {
    if (!lnccl_) {  // all parts in this process: indexed device copies
      for (LLink& l : links_) {
        LPart* sp = part_of(l.s);
        LPart* rp = part_of(l.r);
        if (phase == 0)
          k_slots_pack<<<grid_for(l.count, 256), 256, 0, stream_>>>(
              l.sidx.get(), l.count, sp->buf, rp->buf + l.ghost0);
        else
          k_slots_unpack<<<grid_for(l.count, 256), 256, 0, stream_>>>(
              l.sidx.get(), l.count, rp->buf + l.ghost0, sp->buf);
        LBM_CHECK_LAUNCH();
      }
      return;
    }
    // phase 0: s packs its slots into the staging buffer, sends it, r
    // receives straight into its ghost range.  phase 1: r sends its ghost
    // range, s receives into staging and scatters.
    for (LLink& l : links_)
      if (phase == 0 && part_of(l.s)) {
        k_slots_pack<<<grid_for(l.count, 256), 256, 0, stream_>>>(
            l.sidx.get(), l.count, part_of(l.s)->buf, l.stage.get());
        LBM_CHECK_LAUNCH();
      }
    nccl_begin(lnccl_, phase, stream_);
    std::vector<NcclP2P> ops;
    for (LLink& l : links_) {  // global link order on every rank -> matched pairs
      LPart* sp = part_of(l.s);
      LPart* rp = part_of(l.r);
      if (phase == 0) {
        if (sp) ops.push_back({l.r, l.stage.get(), nullptr, l.count});
        if (rp) ops.push_back({l.s, nullptr, rp->buf + l.ghost0, l.count});
      } else {
        if (rp) ops.push_back({l.s, rp->buf + l.ghost0, nullptr, l.count});
        if (sp) ops.push_back({l.r, nullptr, l.stage.get(), l.count});
      }
    }
    nccl_p2p(lnccl_, ops);
    cudaStream_t cs = nccl_comm_stream(lnccl_);
    if (phase == 1)
      for (LLink& l : links_)
        if (LPart* sp = part_of(l.s)) {
          k_slots_unpack<<<grid_for(l.count, 256), 256, 0, cs>>>(l.sidx.get(), l.count,
                                                                 l.stage.get(), sp->buf);
          LBM_CHECK_LAUNCH();
        }
    nccl_end(lnccl_, phase);
  }

  void list_wait(int phase) {
    if (lnccl_) nccl_wait(lnccl_, phase, stream_);
  }

  // one AA pair over node-range parts: even(boundary) -> [exchange 0 ||
  // even(interior)] -> odd(boundary) -> [exchange 1 || odd(interior)]
  void aa_pair_parts(const TrtArgs& t) {
    const bool soa = desc_.soa;
    auto sweep = [&](bool odd, bool boundary) {
      for (LPart& p : lparts_) {
        ListArgs a = p.args(t, soa);
        auto run = [&](uint64_t b0, uint64_t b1) {
          a.nb = b0;
          a.ne = b1;
          // boundary launches carry "_halo" (stream role in the stats)
          if (odd)
            soa ? launch(boundary ? "list_aa_odd_soa_halo" : "list_aa_odd_soa",
                         k_list_aa_odd<true, false>, a, pf_)
                : launch(boundary ? "list_aa_odd_aos_halo" : "list_aa_odd_aos",
                         k_list_aa_odd<false, false>, a, pf_);
          else
            soa ? launch(boundary ? "list_aa_even_soa_halo" : "list_aa_even_soa",
                         k_list_aa_even<true, false>, a)
                : launch_tile(boundary ? "list_aa_even_aos_halo" : "list_aa_even_aos",
                              k_list_aos_tile<true>, a);
        };
        if (boundary) {
          run(0, p.head);
          run(p.nloc - p.tail, p.nloc);
        } else {
          run(p.head, p.nloc - p.tail);
        }
      }
    };
    // boundary sweeps and exchanges on a boundary stream beside the interior
    // sweeps, as in the direct z-slab paths (direct.cu aa_pair_peer): each
    // slot is touched by one node per sub-step, and the exchanged slots
    // belong to boundary nodes only
    if (!bstream_) {
      int least = 0, greatest = 0;
      LBM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      LBM_CUDA(cudaStreamCreateWithPriority(&bstream_, cudaStreamNonBlocking, greatest));
      nvtxNameCudaStreamA(bstream_, "lbmgpu boundary");
      for (cudaEvent_t& e : bev_) LBM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    struct Swap {
      cudaStream_t& x;
      cudaStream_t& y;
      Swap(cudaStream_t& a, cudaStream_t& b) : x(a), y(b) { std::swap(x, y); }
      ~Swap() { std::swap(x, y); }
    };
    LBM_CUDA(cudaEventRecord(bev_[0], stream_));
    {
      NvtxRange r("list aa even boundary + pre-odd exchange [boundary stream]");
      Swap on_b(stream_, bstream_);
      LBM_CUDA(cudaStreamWaitEvent(stream_, bev_[0], 0));
      sweep(false, true);
      LBM_CUDA(cudaEventRecord(bev_[1], stream_));
      list_exchange(0);
    }
    {
      NvtxRange r("list aa even interior [interior stream]");
      sweep(false, false);
      LBM_CUDA(cudaEventRecord(bev_[2], stream_));
    }
    {
      NvtxRange r("list aa odd boundary + post-odd exchange [boundary stream]");
      Swap on_b(stream_, bstream_);
      LBM_CUDA(cudaStreamWaitEvent(stream_, bev_[2], 0));
      list_wait(0);
      sweep(true, true);
      list_exchange(1);
      list_wait(1);
      LBM_CUDA(cudaEventRecord(bev_[3], stream_));
    }
    LBM_CUDA(cudaStreamWaitEvent(stream_, bev_[1], 0));
    sweep(true, false);
    LBM_CUDA(cudaStreamWaitEvent(stream_, bev_[3], 0));
  }

  int parts() const override { return lparts_.empty() ? 1 : static_cast<int>(lparts_.size()); }
  void part_info(int p, int* z0, int* z1, uint64_t* nf) const override {
    if (lparts_.empty()) {
      *z0 = 0;
      *z1 = nz_;
      *nf = n_fluid_;
      return;
    }
    const LPart& lp = lparts_.at(p);
    *z0 = static_cast<int>(lp.n0);  // node range for list parts
    *z1 = static_cast<int>(lp.n1);
    *nf = lp.n1 - lp.n0;
  }
  bool holds_all() const override { return lnranks_ == 1; }
  uint64_t local_rows() const override {
    if (lparts_.empty() || lnranks_ == 1) return n_fluid_;
    return lparts_[0].n1 - lparts_[0].n0;
  }
  void local_canonical_index(uint64_t* out) const override {
    if (lparts_.empty() || lnranks_ == 1) {
      for (uint64_t k = 0; k < n_fluid_; ++k) out[k] = k;
      return;
    }
    for (uint64_t k = lparts_[0].n0; k < lparts_[0].n1; ++k) out[k - lparts_[0].n0] = k;
  }
  void gather_local(uint64_t k0, uint64_t count, double* d, bool to_staging) override {
    const uint64_t base = (lparts_.empty() || lnranks_ == 1) ? 0 : lparts_[0].n0;
    if (to_staging)
      gather_canonical(base + k0, count, d);
    else
      scatter_canonical(base + k0, count, d);
  }

  ListArgs base_args() const {
    ListArgs a{};
    a.adj = adj_.get();
    a.N = n_fluid_;
    for (int q = 0; q < kQ; ++q) a.starts[q] = starts_[q];
    a.nb = 0;
    a.ne = n_fluid_;
    return a;
  }

  // AoS own-record tile kernels: kLAosTile-node blocks over [nb, ne).
  // gathers = the kernel also gathers 18 scattered values per node from
  // global memory: those hit L1 only if the shared-memory carve-out leaves
  // it room (at the default carve-out 11 CTAs x 19.5 KB of tiles leave
  // ~40 KB of L1).  A 33 % carve-out (5 CTAs/SM) measured best on cfg 2:
  // list-push-aos 8,854 -> 10,824 MFLUP/s, its stream pass 1,580 -> 4,105
  // GB/s (50 %: 10,409; 20 %: 10,207); the own-record tiles keep the default.
  template <class K>
  void launch_tile(const char* name, K kern, const ListArgs& a, bool gathers = false) {
    if (a.ne <= a.nb) return;
    if (gathers)
      LBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 33));
    const int tok = stats_.begin(name, stream_);
    kern<<<static_cast<unsigned>(ceil_div(a.ne - a.nb, kLAosTile)), kLAosTile, 0, stream_>>>(a);
    LBM_CHECK_LAUNCH();
    stats_.end(tok, stream_);
  }

  // AoS AA odd step through 3-D staging tiles (list_aos_tile.cuh)
  template <int TX, int TY, int TZ, bool EDGES = true>
  void launch_aos_odd_tile_shape(const ListArgs& a) {
    using S = LTileShape<TX, TY, TZ, EDGES>;
    static_assert(TZ % 2 == 0, "staged rows must stay 16-byte aligned");
    auto kern = k_list_aa_odd_aos_tile<TX, TY, TZ, EDGES>;
    LBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(S::kSmem)));
    LTileGeom g{};
    g.crank = crank_.get();
    g.nx = nx_;
    g.ny = ny_;
    g.nz = nz_;
    g.tiles_y = static_cast<uint32_t>(ceil_div(ny_, TY));
    g.tiles_z = static_cast<uint32_t>(ceil_div(nz_, TZ));
    const dim3 tiles(g.tiles_z, g.tiles_y, static_cast<unsigned>(ceil_div(nx_, TX)));
    const int tok = stats_.begin("list_aa_odd_aos", stream_);
    kern<<<tiles, S::kT, S::kSmem, stream_>>>(a, g);
    LBM_CHECK_LAUNCH();
    stats_.end(tok, stream_);
  }
  // Tile shape (measured on cfg 2 / cfg 4): 4 x 4 x 16
  // with only the tile's own rows staged (256 threads, 2 CTAs/SM).
  // LBMGPU_LTILE selects the other instantiated shapes for the tests: 1 =
  // 4 x 4 x 16 with the edge halo rows staged too, 5 = 2 x 2 x 32 (halo
  // rows, every wrap case), 12 = 4 x 4 x 8 (own rows, 128 threads).
  void launch_aos_odd_tiles(const ListArgs& a) {
    switch (ltile_) {
      case 1: launch_aos_odd_tile_shape<4, 4, 16, true>(a); break;
      case 5: launch_aos_odd_tile_shape<2, 2, 32, true>(a); break;
      case 12: launch_aos_odd_tile_shape<4, 4, 8, false>(a); break;
      default: launch_aos_odd_tile_shape<4, 4, 16, false>(a); break;
    }
  }

  template <class K, class... Extra>
  void launch(const char* name, K kern, const ListArgs& a, Extra... extra) {
    const int threads = threads_;
    if (a.ne <= a.nb) return;
    const int tok = stats_.begin(name, stream_);
    kern<<<static_cast<unsigned>(ceil_div(a.ne - a.nb, threads)), threads, 0, stream_>>>(
        a, extra...);
    LBM_CHECK_LAUNCH();
    stats_.end(tok, stream_);
  }

  // One cooperative launch for all sweeps when the PDFs and the adjacency
  // live in L2 (<= fused_bytes_), a single part, no run coding.
  template <bool SOA, int KIND>
  void launch_list_fused(ListArgs a, double* other, long sweeps, const char* name) {
    constexpr int TPB = 256, MINB = 2;
    auto kern = k_list_fused<SOA, KIND, TPB, MINB>;
    int per_sm = 0;
    per_sm = occupancy_blocks(reinterpret_cast<const void*>(kern), TPB);
    const int grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>(ceil_div(a.N, TPB), uint64_t(std::max(per_sm, 1)) * sm_count_)));
    void* params[] = {&a, &other, &sweeps};
    const int tok = stats_.begin(name, stream_, sweeps);
    LBM_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), grid, TPB, params, 0,
                                         stream_));
    stats_.end(tok, stream_);
  }

  bool advance_fused(const TrtArgs& t, long steps) {
    if (!lparts_.empty() || desc_.ria || pull_pid_ || steps < 2 || fused_bytes_ == 0) return false;
    const uint64_t nbuf = desc_.prop == Prop::Aa ? 1 : 2;
    if (nbuf * total_slots_ * 8 + 72 * n_fluid_ > fused_bytes_) return false;
    ListArgs a = base_args();
    a.trt = t;
    const bool soa = desc_.soa;
    if (desc_.prop == Prop::Aa) {
      a.src = a.dst = buf_[0].get();
      soa ? launch_list_fused<true, kListFusedAA>(a, nullptr, steps, "list_aa_soa_fused")
          : launch_list_fused<false, kListFusedAA>(a, nullptr, steps, "list_aa_aos_fused");
      return true;
    }
    a.src = a.dst = buf_[cur_].get();
    double* other = buf_[1 - cur_].get();
    if (desc_.prop == Prop::OsPush)
      soa ? launch_list_fused<true, kListFusedPush>(a, other, steps, "list_push_soa_fused")
          : launch_list_fused<false, kListFusedPush>(a, other, steps, "list_push_aos_fused");
    else
      soa ? launch_list_fused<true, kListFusedPull>(a, other, steps + 1, "list_pull_soa_fused")
          : launch_list_fused<false, kListFusedPull>(a, other, steps + 1, "list_pull_aos_fused");
    if (steps & 1) cur_ ^= 1;
    return true;
  }

  void advance(const TrtArgs& t, long steps) override {
    NvtxRange range(("advance " + desc_.name).c_str());
    if (advance_fused(t, steps)) return;
    ListArgs a = base_args();
    a.trt = t;
    const bool soa = desc_.soa;
    if (desc_.prop == Prop::Aa && !lparts_.empty()) {
      for (long s = 0; s < steps; s += 2) aa_pair_parts(t);
      return;
    }
    if (desc_.prop == Prop::Aa) {
      a.src = a.dst = buf_[0].get();
      for (long s = 0; s < steps; s += 2) {
        soa ? launch("list_aa_even_soa", k_list_aa_even<true, false>, a)
            : launch_tile("list_aa_even_aos", k_list_aos_tile<true>, a);
        if (desc_.ria && soa) {
          const int mode = ria_mode_ >= 0 ? ria_mode_ : (ria_npat_ > 0 ? 2 : 0);
          const int tok = stats_.begin(mode == 2 && ria_npat_ > 65536 ? "list_aa_odd_ria_pid32_soa"
                                       : mode == 2 && ria_npat_ > 256 ? "list_aa_odd_ria_pid16_soa"
                                       : mode == 2 && ria_npat_ > 0 ? "list_aa_odd_ria_pid_soa"
                                                                    : "list_aa_odd_ria_soa",
                                       stream_);
          // 128-thread CTAs: cfg 2 RIA odd 5228 -> 5431 GB/s (the indexed
          // sweeps measured equal or better at 256)
          const int rt = 128;
          const unsigned g = static_cast<unsigned>(ceil_div(a.N, rt));
          if (mode == 2 && ria_npat_ > 65536)
            launch_pid(g, rt, a, ria_nid32_.get());
          else if (mode == 2 && ria_npat_ > 256)
            launch_pid(g, rt, a, ria_nid16_.get());
          else if (mode == 2 && ria_npat_ > 0)
            launch_pid(g, rt, a, ria_nid_.get());
          else if (mode == 1)
            k_list_aa_odd_gpat<false><<<g, rt, 0, stream_>>>(a, ria_gpat_.get(), pf_);
          else
            k_list_aa_odd_ria<false><<<g, rt, 0, stream_>>>(
                a, ria_pat_.get(), ria_run0_.get(), ria_mask_.get(), pf_);
          LBM_CHECK_LAUNCH();
          stats_.end(tok, stream_);
        } else if (!soa && crank_.get()) {
          launch_aos_odd_tiles(a);
        } else {
          soa ? launch("list_aa_odd_soa", k_list_aa_odd<true, false>, a, pf_)
              : launch("list_aa_odd_aos", k_list_aa_odd<false, false>, a, pf_);
        }
      }
      return;
    }
    if (desc_.prop == Prop::OsPush && !soa) {
      // AoS push in pull order (as the direct AoS push, direct.cu
      // os_aos_tiles): collide pass, T-1 gather + collide sweeps, one
      // gather-only sweep, gathering through the Scatter table read
      // backwards (aos_gather_slot) -- push and pull realise the identical
      // per-step mapping (reference tests/test_kernels.cpp:96-126), so the
      // state is bitwise the push's, with whole own records stored through
      // the tile instead of 18 scattered 8-byte stores per node.
      a.src = a.dst = buf_[cur_].get();
      launch_tile("list_push_aos_collide", k_list_aos_tile<false>, a);
      for (long s = 0; s < steps; ++s) {
        a.src = buf_[cur_].get();
        a.dst = buf_[1 - cur_].get();
        if (s + 1 < steps)
          launch_tile("list_push_aos", k_list_pull_aos_tile<true, true>, a, true);
        else
          launch_tile("list_push_stream_aos", k_list_pull_aos_tile<false, true>, a, true);
        cur_ ^= 1;
      }
      return;
    }
    if (desc_.prop == Prop::OsPush) {
      for (long s = 0; s < steps; ++s) {
        a.src = buf_[cur_].get();
        a.dst = buf_[1 - cur_].get();
        soa ? launch("list_push_soa", k_list_push<true>, a)
            : launch("list_push_aos", k_list_push<false>, a);
        cur_ ^= 1;
      }
      return;
    }
    // pull: collide pass, T-1 fused sweeps, one stream-only sweep
    // (kernels_list_os.cpp:74-91, kernels_list_nt.cpp:146-158)
    a.src = a.dst = buf_[cur_].get();
    soa ? launch("list_collide_soa", k_list_collide<true>, a)
        : launch_tile("list_collide_aos", k_list_aos_tile<false>, a);
    for (long s = 0; s < steps; ++s) {
      a.src = buf_[cur_].get();
      a.dst = buf_[1 - cur_].get();
      const bool last = s == steps - 1;
      if (soa && pull_pid_) {
        launch_pull_pid(a, !last);
      } else if (soa) {
        if (last)
          launch("list_pull_stream_soa", k_list_pull<true, false, false>, a);
        else if (cs_nt_)
          launch("list_pull_soa", k_list_pull<true, true, true>, a);
        else
          launch("list_pull_soa", k_list_pull<true, true, false>, a);
      } else {
        if (last)
          launch_tile("list_pull_stream_aos", k_list_pull_aos_tile<false>, a, true);
        else
          launch_tile("list_pull_aos", k_list_pull_aos_tile<true>, a, true);
      }
      cur_ ^= 1;
    }
  }

  template <int MODE>
  void canon(uint64_t c0, uint64_t c1, double* stage, uint64_t seed = 0,
             double amp = 0, double* rho = nullptr, double* u = nullptr) {
    if (c1 <= c0) return;
    ListArgs a = base_args();
    const uint32_t* loc = desc_.blk > 0 ? list_of_canon_.get() : nullptr;
    auto run = [&](double* buf, uint64_t b0, uint64_t b1) {
      if (b1 <= b0) return;
      const int g = grid_for(b1 - b0, 256);
      // the kernels index stage relative to c0; pass an offset pointer
      double* st = stage ? stage + (b0 - c0) * kQ : nullptr;
      if (desc_.soa)
        k_list_canon<true, MODE><<<g, 256, 0, stream_>>>(a, buf, loc, b0, b1, st, seed, amp,
                                                         rho, u);
      else
        k_list_canon<false, MODE><<<g, 256, 0, stream_>>>(a, buf, loc, b0, b1, st, seed, amp,
                                                          rho, u);
      LBM_CHECK_LAUNCH();
    };
    if (lparts_.empty()) {
      run(buf_[cur_].get(), c0, c1);
      return;
    }
    // node-range parts (blk = 0: canonical index == list index): each node's
    // PDFs live in its owner part's local array (node n is local n - n0)
    for (LPart& p : lparts_) {
      a = p.args(TrtArgs{}, desc_.soa);
      a.node_base = p.n0;
      run(p.buf, std::max(c0, p.n0), std::min(c1, p.n1));
    }
  }

  void gather_canonical(uint64_t c0, uint64_t count, double* out) override {
    canon<0>(c0, std::min(c0 + count, n_fluid_), out);
  }
  void scatter_canonical(uint64_t c0, uint64_t count, const double* in) override {
    canon<1>(c0, std::min(c0 + count, n_fluid_), const_cast<double*>(in));
  }
  void load_perturbed(uint64_t seed, double amp) override {
    canon<2>(0, n_fluid_, nullptr, seed, amp);
  }
  void macro_fields(double* rho, double* u) override {
    canon<3>(0, n_fluid_, nullptr, 0, 0, rho, u);
  }

  double total_mass() override {
    auto part_mass = [&](double* buf, uint64_t b0, uint64_t b1, const LPart* p) {
      if (b1 <= b0) return 0.0;
      DevBuf<double> tmp((b1 - b0) * kQ);
      ListArgs a = base_args();
      if (p) {
        a = p->args(TrtArgs{}, desc_.soa);
        a.node_base = p->n0;
      }
      a.nb = b0;
      a.ne = b1;
      desc_.soa ? k_list_mass_terms<true><<<grid_for(b1 - b0, 256), 256, 0, stream_>>>(
                      a, buf, tmp.get())
                : k_list_mass_terms<false><<<grid_for(b1 - b0, 256), 256, 0, stream_>>>(
                      a, buf, tmp.get());
      LBM_CHECK_LAUNCH();
      return device_sum(tmp.get(), tmp.size(), stream_);
    };
    if (lparts_.empty()) return part_mass(buf_[cur_].get(), 0, n_fluid_, nullptr);
    double m = 0.0;
    for (LPart& p : lparts_) m += part_mass(p.buf, p.n0, p.n1, &p);
    return lnccl_ && lnranks_ > 1 ? nccl_sum(lnccl_, m) : m;
  }

  void export_structure(int32_t* nodes, uint32_t* adj, uint64_t* starts,
                        uint64_t* total) override {
    if (nodes)
      LBM_CUDA(cudaMemcpyAsync(nodes, nodes_.get(), nodes_.bytes(),
                               cudaMemcpyDeviceToHost, stream_));
    if (adj) {
      if (!lparts_.empty())
        throw ConfigError("export_structure: the adjacency of a decomposed list lattice "
                          "lives in per-part local numbering");
      DevBuf<uint32_t> canon(18 * n_fluid_);
      k_adj_canonical<<<grid_for(18 * n_fluid_, 256), 256, 0, stream_>>>(
          adj_.get(), n_fluid_, canon.get());
      LBM_CHECK_LAUNCH();
      LBM_CUDA(cudaMemcpyAsync(adj, canon.get(), canon.bytes(),
                               cudaMemcpyDeviceToHost, stream_));
      LBM_CUDA(cudaStreamSynchronize(stream_));
    }
    if (starts)
      for (int q = 0; q < kQ; ++q) starts[q] = desc_.soa ? starts_[q] : 0;
    if (total) *total = total_slots_;
    LBM_CUDA(cudaStreamSynchronize(stream_));
  }

  void launch_pull_pid(const ListArgs& a, bool collide) {
    const unsigned g = static_cast<unsigned>(ceil_div(a.N, 256));
    const char* w = ria_npat_ > 65536 ? "32" : ria_npat_ > 256 ? "16" : "";
    const std::string nm = std::string(collide ? "list_pull_pid" : "list_pull_stream_pid") + w + "_soa";
    const int tok = stats_.begin(nm.c_str(), stream_);
    auto go = [&](auto* nid) {
      using ID = std::remove_const_t<std::remove_pointer_t<decltype(nid)>>;
      if (collide)
        k_list_pull_pid<true, false, ID><<<g, 256, 0, stream_>>>(a, ria_ptab_.get(), nid, pf_);
      else
        k_list_pull_pid<false, false, ID><<<g, 256, 0, stream_>>>(a, ria_ptab_.get(), nid, pf_);
    };
    if (ria_npat_ > 65536)
      go(ria_nid32_.get());
    else if (ria_npat_ > 256)
      go(ria_nid16_.get());
    else
      go(ria_nid_.get());
    LBM_CHECK_LAUNCH();
    stats_.end(tok, stream_);
  }

  template <typename ID>
  void launch_pid(unsigned g, int rt, const ListArgs& a, const ID* nid) {
    k_list_aa_odd_pid<false, ID><<<g, rt, 0, stream_>>>(a, ria_ptab_.get(), nid, pf_);
  }

  // ria_stats / vector_fraction (kernels_list_aa.cpp:95-140) for the ria/pv
  // names; computed from the run starts of the kernel's own structure.
  // Run coding of the scatter table (build_ria, list_lattice.cpp:206-226) and
  // the device tables of the run-coded odd step.
  void build_ria() {
    DevBuf<uint8_t> is_start(n_fluid_);
    ListArgs a = base_args();
    k_ria_starts<<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(
        adj_.get(), n_fluid_, desc_.soa, a, is_start.get());
    LBM_CHECK_LAUNCH();
    DevBuf<uint32_t> incl(n_fluid_);
    {
      cub::TransformInputIterator<uint32_t, IsStart, const uint8_t*> it(is_start.get(), IsStart{});
      size_t tmp = 0;
      LBM_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, it, incl.get(),
                                             static_cast<int64_t>(n_fluid_), stream_));
      DevBuf<uint8_t> t(tmp);
      LBM_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tmp, it, incl.get(),
                                             static_cast<int64_t>(n_fluid_), stream_));
    }
    uint32_t R = 0;
    LBM_CUDA(cudaMemcpyAsync(&R, incl.get() + n_fluid_ - 1, 4, cudaMemcpyDeviceToHost, stream_));
    LBM_CUDA(cudaStreamSynchronize(stream_));
    ria_R_ = R;
    DevBuf<uint32_t> run_start(R);
    const uint64_t warps = ceil_div(n_fluid_, 32);
    ria_run0_.alloc(warps);
    ria_mask_.alloc(warps);
    k_ria_tables<<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, stream_>>>(
        is_start.get(), incl.get(), n_fluid_, run_start.get(), ria_run0_.get(), ria_mask_.get());
    LBM_CHECK_LAUNCH();
    ria_pat_.alloc(uint64_t(R) * 18);
    k_ria_patterns<<<grid_for(uint64_t(R) * 18, 256), 256, 0, stream_>>>(
        adj_.get(), run_start.get(), R, a, ria_pat_.get());
    LBM_CHECK_LAUNCH();
    ria_gpat_.alloc(warps * 18);
    k_ria_group_patterns<<<grid_for(warps * 18, 256), 256, 0, stream_>>>(
        ria_pat_.get(), ria_run0_.get(), ria_mask_.get(), n_fluid_, ria_gpat_.get());
    LBM_CHECK_LAUNCH();
    // distinct run patterns (host dedup, stops above kMaxPatterns): pattern
    // ids of 8 / 16 / 32 bits for <= 256 / 65,536 / kMaxPatterns rows
    {
      constexpr uint32_t kMaxPatterns = 1u << 20;  // table <= 72 MiB (L2-sized)
      std::vector<int32_t> hp(uint64_t(R) * 18);
      LBM_CUDA(cudaMemcpyAsync(hp.data(), ria_pat_.get(), hp.size() * 4, cudaMemcpyDeviceToHost,
                               stream_));
      LBM_CUDA(cudaStreamSynchronize(stream_));
      std::unordered_map<std::string, uint32_t> ids;
      std::vector<uint32_t> run_pid(R);
      std::vector<int32_t> tab;
      bool ok = true;
      for (uint32_t r = 0; r < R && ok; ++r) {
        std::string key(reinterpret_cast<const char*>(hp.data() + uint64_t(r) * 18), 72);
        auto it = ids.find(key);
        if (it == ids.end()) {
          if (ids.size() == kMaxPatterns) {
            ok = false;
            break;
          }
          it = ids.emplace(key, static_cast<uint32_t>(ids.size())).first;
          tab.insert(tab.end(), hp.begin() + uint64_t(r) * 18, hp.begin() + uint64_t(r) * 18 + 18);
        }
        run_pid[r] = it->second;
      }
      ria_npat_ = ok ? static_cast<int>(ids.size()) : -1;
      if (ok) {
        ria_ptab_.alloc(tab.size());
        LBM_CUDA(cudaMemcpyAsync(ria_ptab_.get(), tab.data(), tab.size() * 4,
                                 cudaMemcpyHostToDevice, stream_));
        auto node_ids = [&](auto tag, auto& out) {
          using ID = decltype(tag);
          std::vector<ID> p(run_pid.begin(), run_pid.end());
          DevBuf<ID> dpid(R);
          LBM_CUDA(cudaMemcpyAsync(dpid.get(), p.data(), uint64_t(R) * sizeof(ID),
                                   cudaMemcpyHostToDevice, stream_));
          out.alloc(n_fluid_);
          k_ria_node_ids<ID><<<grid_for(n_fluid_, 256), 256, 0, stream_>>>(
              ria_run0_.get(), ria_mask_.get(), dpid.get(), n_fluid_, out.get());
          LBM_CHECK_LAUNCH();
          LBM_CUDA(cudaStreamSynchronize(stream_));
        };
        if (ria_npat_ <= 256)
          node_ids(uint8_t{}, ria_nid_);
        else if (ria_npat_ <= 65536)
          node_ids(uint16_t{}, ria_nid16_);
        else
          node_ids(uint32_t{}, ria_nid32_);
      }
    }
    // run lengths -> vectorizable fraction (list_lattice.cpp:228-236)
    std::vector<uint32_t> h(R);
    LBM_CUDA(cudaMemcpyAsync(h.data(), run_start.get(), uint64_t(R) * 4,
                             cudaMemcpyDeviceToHost, stream_));
    LBM_CUDA(cudaStreamSynchronize(stream_));
    ria_runs_ = R;
    ria_run_start_h_ = std::move(h);
    ria_vfrac_ = vector_fraction(desc_.vector_width);
  }

  // vectorizable_fraction (list_lattice.cpp:228-236): nodes covered by whole
  // groups of W inside their run, over all fluid nodes
  double vector_fraction(int w) const {
    const uint64_t W = static_cast<uint64_t>(w), R = ria_run_start_h_.size();
    uint64_t covered = 0;
    for (uint64_t r = 0; r < R; ++r) {
      const uint64_t end = r + 1 < R ? ria_run_start_h_[r + 1] : n_fluid_;
      covered += (end - ria_run_start_h_[r]) / W * W;
    }
    return static_cast<double>(covered) / static_cast<double>(n_fluid_);
  }

  bool ria_vector_fraction(int w, double* v) override {
    if (!desc_.ria) return false;
    if (w < 1) throw ConfigError("vectorizable_fraction: W must be >= 1");
    *v = vector_fraction(w);
    return true;
  }

  // run starts of the coding (RiaRun::start, list_lattice.hpp:52-58), in
  // node order; run r ends where run r+1 starts (the last at n_fluid)
  bool ria_run_starts(std::vector<uint32_t>& out) override {
    if (!desc_.ria) return false;
    out = ria_run_start_h_;
    return true;
  }

  bool ria_stats(int64_t* runs, double* vfrac) override {
    if (!desc_.ria) return false;
    *runs = ria_runs_;
    *vfrac = ria_vfrac_;
    return true;
  }

 private:
  int nx_ = 0, ny_ = 0, nz_ = 0;
  std::array<bool, 3> per_{};
  uint64_t starts_[kQ] = {};
  uint64_t total_slots_ = 0;
  bool scatter_ = false;
  bool cs_nt_ = false;
  int sm_count_ = 148;
  int cur_ = 0;
  DevBuf<int32_t> nodes_;
  DevBuf<uint32_t> adj_;
  DevBuf<uint32_t> list_of_canon_;
  DevBuf<uint32_t> crank_;      // box-order fluid scan (AoS AA staging tiles), V + 1 entries
  int ltile_ = 0;               // staging tile shape of the AoS AA odd step (LBMGPU_LTILE)
  DevBuf<double> buf_[2];
  // node-range decomposition (list AA over several GPUs / emulated parts)
  std::vector<LPart> lparts_;
  std::vector<LLink> links_;
  int lnparts_ = 1, lrank_ = 0, lnranks_ = 1;
  NcclTransportImpl* lnccl_ = nullptr;
  int64_t ria_runs_ = -1;
  double ria_vfrac_ = 0.0;
  std::vector<uint32_t> ria_run_start_h_;  // host copy of the run starts
  uint64_t ria_R_ = 0;
  DevBuf<int32_t> ria_pat_;     // [run][18] relative offsets
  DevBuf<uint32_t> ria_run0_;   // run id of node 32w
  DevBuf<uint32_t> ria_mask_;   // run starts within nodes 32w .. 32w+31
  DevBuf<int32_t> ria_gpat_;    // [group][18] inline pattern or kMixedGroup
  // odd-step coding: -1 auto (pattern ids when <= 256 distinct run
  // patterns, else the run table), 0 run table, 1 group patterns, 2 pattern
  // ids (LBMGPU_RIA_MODE)
  int ria_mode_ = -1;
  cudaStream_t bstream_ = nullptr;  // node-range parts: boundary stream (aa_pair_parts)
  cudaEvent_t bev_[4] = {nullptr, nullptr, nullptr, nullptr};
  bool pull_pid_ = false;       // one-step pull through Gather-table pattern ids (LBMGPU_PULL_PID)
  int ria_npat_ = -1;           // distinct run patterns (-1: more than 2^20)
  DevBuf<int32_t> ria_ptab_;    // [pattern id][18]
  DevBuf<uint8_t> ria_nid_;     // pattern id of every node (<= 256 patterns)
  DevBuf<uint16_t> ria_nid16_;  // pattern id of every node (257 .. 65,536 patterns)
  DevBuf<uint32_t> ria_nid32_;  // pattern id of every node (more than 65,536 patterns)
  int threads_ = 256;           // CTA size of the sweeps
  uint64_t fused_bytes_ = 96ull << 20;  // fused multi-sweep launch threshold (PDFs + adjacency)
  uint64_t pf_ = 0;             // adjacency L2 prefetch distance in nodes (AA odd)
};

}  // namespace

std::unique_ptr<Engine> make_list_engine(const Descriptor& d,
                                         const GeomSpec& g,
                                         const Padding& pad,
                                         const DistSpec& dist) {
  return std::make_unique<ListEngine>(d, g, pad, dist);
}

}  // namespace lbmgpu
