// NCCL point-to-point halo transport for the multi-GPU z-slab AA sweep.
//
// One process per GPU; rank r owns slab r.  Each phase of the halo plan
// (halo.hpp) is one ncclGroupStart/End with a send for every row whose source
// is this rank and a recv for every row whose destination is this rank, issued
// in the plan's global row order on every rank, so the per-peer FIFO matching
// of NCCL pairs each send with its recv.  The group runs on a dedicated comm
// stream that waits for the boundary sweep (event), overlapping the interior
// sweep on the compute stream; wait() joins it back before the next boundary
// sweep.  NCCL is loaded with dlopen so the library has no link-time NCCL
// dependency (torch's bundled libnccl.so.2 or the system one, whichever is
// already loaded, is used).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "halo.hpp"
#include "lbm.hpp"

namespace lbmgpu {

namespace {

struct NcclApi {
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t,
                            ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static const NcclApi& get() {
    static NcclApi api = load();
    return api;
  }

 private:
  template <class F>
  static void sym(void* h, const char* name, F& f) {
    f = reinterpret_cast<F>(dlsym(h, name));
    if (!f) throw DeviceError(std::string("libnccl.so.2 lacks ") + name);
  }
  static NcclApi load() {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw DeviceError(std::string("cannot load libnccl.so.2: ") + dlerror());
    NcclApi a;
    sym(h, "ncclCommInitRank", a.CommInitRank);
    sym(h, "ncclCommDestroy", a.CommDestroy);
    sym(h, "ncclGroupStart", a.GroupStart);
    sym(h, "ncclGroupEnd", a.GroupEnd);
    sym(h, "ncclSend", a.Send);
    sym(h, "ncclRecv", a.Recv);
    sym(h, "ncclAllReduce", a.AllReduce);
    sym(h, "ncclGetErrorString", a.GetErrorString);
    return a;
  }
};

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(std::string(what) + ": " + NcclApi::get().GetErrorString(r));
}

}  // namespace

class NcclTransportImpl {
 public:
  NcclTransportImpl(std::vector<HaloRow> plan, int rank, int nranks,
                    const uint8_t* id128)
      : plan_(std::move(plan)), rank_(rank), nranks_(nranks) {
    const NcclApi& api = NcclApi::get();
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(&id, id128, sizeof(id));
    nccl_check(api.CommInitRank(&comm_, nranks, id, rank), "ncclCommInitRank");
    LBM_CUDA(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking));
    for (int i = 0; i < kPhases; ++i) {
      LBM_CUDA(cudaEventCreateWithFlags(&ready_[i], cudaEventDisableTiming));
      LBM_CUDA(cudaEventCreateWithFlags(&done_[i], cudaEventDisableTiming));
    }
    LBM_CUDA(cudaMalloc(&dsum_, sizeof(double)));
  }
  ~NcclTransportImpl() {
    if (comm_) NcclApi::get().CommDestroy(comm_);
    if (comm_stream_) cudaStreamDestroy(comm_stream_);
    for (int i = 0; i < kPhases; ++i) {
      if (ready_[i]) cudaEventDestroy(ready_[i]);
      if (done_[i]) cudaEventDestroy(done_[i]);
    }
    if (dsum_) cudaFree(dsum_);
  }

  // bases[p]: storage (planes x 19 slots x P doubles) of slab p if it lives
  // in this process, else nullptr.  Slab p belongs to rank p, or to rank 0
  // when the communicator has a single rank (self send/recv: the NCCL code
  // path exercised on one GPU by the tests).
  void exchange(int phase, const std::vector<double*>& bases,
                const std::vector<double*>& stages, uint64_t P, cudaStream_t s) {
    const NcclApi& api = NcclApi::get();
    LBM_CUDA(cudaEventRecord(ready_[phase], s));
    LBM_CUDA(cudaStreamWaitEvent(comm_stream_, ready_[phase], 0));
    const size_t count = size_t(kHaloSlots) * P;
    auto peer = [&](int part) { return nranks_ == 1 ? 0 : part; };
    // storage plane >= 0 of the grid, or one of the two staging planes
    auto at = [&](int part, int plane, int slot0) -> double* {
      if (plane >= 0)
        return bases[part] ? bases[part] + (uint64_t(plane) * kQ + slot0) * P : nullptr;
      return stages[part] ? stages[part] + (uint64_t(-plane - 1) * kQ + slot0) * P : nullptr;
    };
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const HaloRow& r : plan_) {
      if (r.phase != phase) continue;
      if (double* b = at(r.src_part, r.src_plane, r.slot0))
        nccl_check(api.Send(b, count, ncclFloat64, peer(r.dst_part), comm_, comm_stream_),
                   "ncclSend");
      if (double* b = at(r.dst_part, r.dst_plane, r.slot0))
        nccl_check(api.Recv(b, count, ncclFloat64, peer(r.src_part), comm_, comm_stream_),
                   "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    LBM_CUDA(cudaEventRecord(done_[phase], comm_stream_));
  }

  void wait(int phase, cudaStream_t s) {
    LBM_CUDA(cudaStreamWaitEvent(s, done_[phase], 0));
  }

  // Generic grouped point-to-point for index-list halos (list lattices):
  // begin() hands the compute stream's work over to the comm stream, p2p()
  // issues one NCCL group, end() marks the phase done on the comm stream
  // (after any unpack kernels the caller queued there).
  void begin(int phase, cudaStream_t s) {
    LBM_CUDA(cudaEventRecord(ready_[phase], s));
    LBM_CUDA(cudaStreamWaitEvent(comm_stream_, ready_[phase], 0));
  }
  void p2p(const std::vector<NcclP2P>& ops) {
    const NcclApi& api = NcclApi::get();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const NcclP2P& o : ops) {
      const int peer = nranks_ == 1 ? 0 : o.peer;
      if (o.send)
        nccl_check(api.Send(o.send, o.count, ncclFloat64, peer, comm_, comm_stream_), "ncclSend");
      if (o.recv)
        nccl_check(api.Recv(o.recv, o.count, ncclFloat64, peer, comm_, comm_stream_), "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  }
  void end(int phase) { LBM_CUDA(cudaEventRecord(done_[phase], comm_stream_)); }
  cudaStream_t comm_stream() const { return comm_stream_; }

  double sum(double v) {
    const NcclApi& api = NcclApi::get();
    LBM_CUDA(cudaMemcpyAsync(dsum_, &v, sizeof(double), cudaMemcpyHostToDevice,
                             comm_stream_));
    nccl_check(api.AllReduce(dsum_, dsum_, 1, ncclFloat64, ncclSum, comm_,
                             comm_stream_),
               "ncclAllReduce");
    double out = 0;
    LBM_CUDA(cudaMemcpyAsync(&out, dsum_, sizeof(double), cudaMemcpyDeviceToHost,
                             comm_stream_));
    LBM_CUDA(cudaStreamSynchronize(comm_stream_));
    return out;
  }

 private:
  std::vector<HaloRow> plan_;
  int rank_, nranks_;
  ncclComm_t comm_ = nullptr;
  cudaStream_t comm_stream_ = nullptr;
  static constexpr int kPhases = 4;  // halo.hpp phases 0-3
  cudaEvent_t ready_[kPhases] = {}, done_[kPhases] = {};
  double* dsum_ = nullptr;
};

NcclTransportImpl* nccl_create(std::vector<HaloRow> plan, int rank, int nranks,
                               const uint8_t* id128) {
  return new NcclTransportImpl(std::move(plan), rank, nranks, id128);
}
void nccl_exchange(NcclTransportImpl* t, int phase, const std::vector<double*>& bases,
                   const std::vector<double*>& stages,
                   uint64_t P, cudaStream_t s) {
  t->exchange(phase, bases, stages, P, s);
}
void nccl_wait(NcclTransportImpl* t, int phase, cudaStream_t s) { t->wait(phase, s); }
void nccl_begin(NcclTransportImpl* t, int phase, cudaStream_t s) { t->begin(phase, s); }
void nccl_p2p(NcclTransportImpl* t, const std::vector<NcclP2P>& ops) { t->p2p(ops); }
void nccl_end(NcclTransportImpl* t, int phase) { t->end(phase); }
cudaStream_t nccl_comm_stream(NcclTransportImpl* t) { return t->comm_stream(); }
double nccl_sum(NcclTransportImpl* t, double v) { return t->sum(v); }
void nccl_destroy(NcclTransportImpl* t) { delete t; }

}  // namespace lbmgpu
