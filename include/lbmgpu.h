/*
 * lbmgpu.h -- C ABI of the B200-native D3Q19 TRT stream-collide sweep.
 *
 * This is the drop-in boundary for the reference lbmbench kernel/geometry
 * surface (paths relative to /root/reference/proj).  Every entry point names
 * the reference interface it replaces.  All functions return an lbmgpu_status;
 * the message of the last failure on the calling thread is available from
 * lbmgpu_last_error().  Status codes keep the reference's exception classes
 * and CLI exit codes (include/lbm/errors.hpp:9-18, src/cli.cpp:566-572):
 *   1 = ConfigError, 2 = NumericalError, 3 = verification failed,
 *   4 = CUDA/device failure (no reference equivalent; never a CPU fallback).
 *
 * Threading: thread-compatible, not thread-safe (one host thread per context,
 * like the reference's single orchestrating thread, src/workers.cpp:50-60).
 * Memory: the caller owns every host buffer; the library owns device memory.
 * Plain pointers and sizes only; no CUDA or torch types cross this boundary.
 */
#ifndef LBMGPU_H
#define LBMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The library is built with -fvisibility=hidden: only these entry points are
 * exported, so the internal C++ namespace can never be interposed by a host
 * program that happens to define the same symbols. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LBMGPU_ABI_VERSION 2
#define LBMGPU_Q 19

typedef enum {
  LBMGPU_OK = 0,
  LBMGPU_ECONFIG = 1,    /* lbm::ConfigError */
  LBMGPU_ENUMERICAL = 2, /* lbm::NumericalError */
  LBMGPU_EVERIFY = 3,    /* verification did not pass (cli.cpp:330) */
  LBMGPU_EDEVICE = 4     /* CUDA / NCCL failure */
} lbmgpu_status;

/* Geometry kinds in the order of lbm::GeometryKind (geometry.hpp:31). */
typedef enum {
  LBMGPU_CHANNEL = 0,
  LBMGPU_SLIT = 1,
  LBMGPU_PIPE = 2,
  LBMGPU_BLOCKS = 3,
  LBMGPU_CUSTOM = 4 /* host-supplied FlagField (kernels.hpp:102-105 takes any) */
} lbmgpu_geometry_kind;

/* lbm::GeometrySpec (geometry.hpp:36-42) + the FlagField fields a custom
 * geometry needs (geometry.hpp:16-29).  pipe_diameter extends the pipe
 * generator (geometry.cpp:68-84): 0 = the reference's D = min(ny,nz)-2,
 * D > 0 = the same staircase test 4((y-cy)^2+(z-cz)^2) > D^2. */
typedef struct {
  int kind;
  int nx, ny, nz;
  int block, spacing;
  int pipe_diameter;
  const uint8_t* flags; /* CUSTOM only: nx*ny*nz bytes, (x*ny+y)*nz+z, 1=solid */
  int periodic[3];      /* CUSTOM only */
} lbmgpu_geometry;

/* lbm::PaddingPolicy (list_lattice.hpp:25-39): 0 none, 1 auto, 2 thrash,
 * 3 explicit (pads[19]). */
typedef struct {
  int mode;
  int64_t pads[LBMGPU_Q];
} lbmgpu_padding;

/* lbm::KernelDescriptor as make_descriptor parses it (kernels.cpp:50-82). */
typedef struct {
  int prop;       /* 0 os-push, 1 os-pull, 2 aa (lbm::Propagation) */
  int layout_soa; /* 1 SoA, 0 AoS */
  int indirect;   /* 1 list addressing */
  int blk;
  int nt_streams;
  int ria, pv, vec;
  int vector_width;
} lbmgpu_descriptor;

/* Multi-GPU decomposition (new; the reference has no distributed path):
 * z slabs for the direct SoA kernels (AA: halo phases 0/1; blk-push /
 * blk-pull: phases 2/3), contiguous node ranges for list-aa-soa/aos with
 * blk = 0.  nranks == 1 and virtual_parts <= 1: one part.
 * virtual_parts > 1 (nranks == 1): the box is cut into that many z-slabs on
 * ONE device and the halo exchange runs as device copies -- the same plan and
 * kernels as the NCCL path, used for single-GPU parity tests.  nranks > 1:
 * one process per GPU, NCCL point-to-point over NVLink; nccl_id is the
 * 128-byte id from lbmgpu_nccl_unique_id() broadcast by rank 0.
 * transport = 1 (direct SoA z slabs): no halo copies -- the boundary planes'
 * sweeps (AA odd, pull, push) load / store the neighbour slab in peer memory
 * (CUDA IPC over NVLink between processes: lbmgpu_peer_export / _attach
 * before the first advance; device pointers with virtual_parts), with
 * per-sub-step epoch flags in peer memory as the only synchronisation.
 * With transport = 1 the nccl_id is optional; without it total_mass over
 * several processes is a ConfigError (NCCL does the mass reduction). */
typedef struct {
  int rank, nranks;
  int device;        /* CUDA ordinal; -1 = current */
  int virtual_parts; /* >1: emulate that many slabs on one device */
  const void* nccl_id;
  int transport;     /* 0: halo copies (NCCL / device copies), 1: peer memory */
} lbmgpu_dist;

typedef struct lbmgpu_ctx lbmgpu_ctx;

/* ---------------------------------------------------------------- registry */

/* kernel_names() (kernels.cpp:22-43): newline-separated, NUL-terminated. */
int lbmgpu_kernel_names(char* buf, size_t cap);
/* make_descriptor(name, blk, W) (kernels.cpp:50-82); ConfigError lists the
 * valid names exactly like the reference. */
int lbmgpu_make_descriptor(const char* name, int blk, int vector_width,
                           lbmgpu_descriptor* out);
/* padding_offsets (list_lattice.cpp:84-121). */
int lbmgpu_padding_offsets(uint64_t n_fluid, const lbmgpu_padding* pad,
                           uint64_t* starts19, uint64_t* total_slots);
/* loop_balance (perfmodel.cpp:10-47): the reference B_l (CPU, with write
 * allocate) and the GPU algorithmic bytes per fluid update (no write
 * allocate; 304 direct, 340 list AA, 376 list one-step, 304.5 for the RIA
 * names: a one-byte pattern id per node and odd sub-step). */
int lbmgpu_loop_balance(const char* name, double* ref_bl_min,
                        double* ref_bl_max, double* gpu_bytes_per_flup);
/* loop_balance with geometry statistics (perfmodel.cpp:21-31): for the RIA
 * names the index bytes become 76 B of run metadata amortised over the run
 * and the even/odd pair, 76 * total_runs / (2 * n_fluid), clamped to
 * [0, 38] (total_runs < 0 or n_fluid <= 0: no statistics, as above); other
 * names ignore the statistics.  lbmgpu_ria_stats supplies them. */
int lbmgpu_loop_balance_stats(const char* name, int64_t total_runs,
                              int64_t n_fluid, double* ref_bl_min,
                              double* ref_bl_max, double* gpu_bytes_per_flup);
/* roofline (perfmodel.cpp:73-87): P_max [MFLUP/s] = GB/s * 1000 / B_l; the
 * lower prediction from the larger balance.  ConfigError when the bandwidth
 * or a balance is not positive. */
int lbmgpu_roofline(double gbps, double bl_min, double bl_max,
                    double* pmax_min_mflups, double* pmax_max_mflups);
/* omega_minus from (omega_plus, magic Lambda) (d3q19.hpp:70-73). */
double lbmgpu_omega_minus(double omega_plus, double magic_lambda);

/* ------------------------------------------------------------- geometry */

/* build_geometry + fluid_count (geometry.cpp:40-117), generated on the
 * device.  flags_out (nullable, V bytes) receives the canonical FlagField. */
int lbmgpu_geometry_build(const lbmgpu_geometry* g, uint8_t* flags_out,
                          int64_t* n_fluid, int* periodic_out);

/* ---------------------------------------------------------------- kernel */

/* make_kernel(desc, ff, padding, pool, row_pad) (kernels.hpp:102-105).
 * The geometry is built on the device; the lattice is initialised to the
 * weights (full_lattice.cpp:21-40, list_lattice.cpp:259-264).  dist may be
 * NULL.  row_pad is accepted and ignored (it never changes results,
 * tests/test_kernels.cpp:197-215; the device layout is our own). */
int lbmgpu_create(const char* kernel_name, int blk, int vector_width,
                  const lbmgpu_geometry* geom, const lbmgpu_padding* pad,
                  int row_pad, const lbmgpu_dist* dist, lbmgpu_ctx** out);
int lbmgpu_destroy(lbmgpu_ctx* ctx);

/* Kernel::advance(TrtParams, BodyForce, steps) (kernels.cpp:84-93): rejects
 * steps < 0, omega_plus outside (0,2), lambda <= 0 and odd AA step counts
 * with ConfigError before touching state. */
int lbmgpu_advance(lbmgpu_ctx* ctx, double omega_plus, double magic_lambda,
                   const double* g3, long steps);
/* Same, bracketed by CUDA events on the context's stream; *ms = device time.
 * With kernel_stats enabled, per-kernel event pairs are recorded too. */
int lbmgpu_time_advance(lbmgpu_ctx* ctx, double omega_plus,
                        double magic_lambda, const double* g3, long steps,
                        double* ms);

int lbmgpu_n_fluid(lbmgpu_ctx* ctx, uint64_t* out);
/* Kernel::snapshot / load_state (kernels.hpp:71-73): canonical N*19 doubles,
 * fluid nodes in x,y,z order (full_lattice.cpp:58-70, list_lattice.cpp:266-310).
 * count must equal N*19 (ConfigError otherwise). */
int lbmgpu_snapshot(lbmgpu_ctx* ctx, double* host, uint64_t count);
int lbmgpu_load_state(lbmgpu_ctx* ctx, const double* host, uint64_t count);
/* One job: load_state(host_in) + advance(steps) + snapshot(host_out) -- the
 * reference harness's load / advance / snapshot-for-the-fingerprint sequence
 * (harness.cpp:94-130) in one call.  Same validation and errors as the three
 * calls; the result is bitwise theirs.  Where the engine supports it (direct
 * SoA AA lattice of one part whose fluid (x, y) columns all hold the same
 * planes, e.g. the channel and slit geometries) and both buffers are
 * page-locked (lbmgpu_host_alloc), the host transfers are pipelined with the
 * sweeps; otherwise the three calls run in sequence.
 * *pipelined (may be NULL) = 1 when the pipelined schedule ran. */
int lbmgpu_run(lbmgpu_ctx* ctx, double omega_plus, double magic_lambda, const double* g3,
               long steps, const double* host_in, uint64_t in_count, double* host_out,
               uint64_t out_count, int* pipelined);
/* load_state(perturbed_equilibrium(N, seed, amplitude)) generated on the
 * device (harness.cpp:50-62); bitwise identical to the host formula. */
int lbmgpu_load_perturbed(lbmgpu_ctx* ctx, uint64_t seed, double amplitude);
/* Kernel::total_mass (full_lattice.cpp:72-87, list_lattice.cpp:282-294):
 * compensated device reduction (not bitwise equal to the sequential Kahan). */
int lbmgpu_total_mass(lbmgpu_ctx* ctx, double* out);
/* state_fingerprint(snapshot()) (harness.cpp:27-39), snapshot streamed in
 * chunks so the full-size host copy is never materialised. */
int lbmgpu_fingerprint(lbmgpu_ctx* ctx, uint64_t* out);
/* Kernel::capabilities (kernels.hpp:47-51).  nt_streams_effective reports the
 * streaming-store (st.global.cs) variant for the nt names. */
int lbmgpu_capabilities(lbmgpu_ctx* ctx, int* nt_stores_available,
                        int* nt_streams_effective, int* huge_pages_advised);
/* ria_stats / vector_fraction / pv_chunk_fraction (kernels.hpp:79-88);
 * values < 0 mean "not applicable" (std::nullopt). */
int lbmgpu_ria_stats(lbmgpu_ctx* ctx, int64_t* total_runs, int64_t* n_fluid,
                     double* vector_fraction, double* pv_chunk_fraction);
/* vectorizable_fraction(coding, W) (list_lattice.cpp:228-236) of a run-coded
 * kernel's own coding at any width W >= 1; -1 for the other names. */
int lbmgpu_vectorizable_fraction(lbmgpu_ctx* ctx, int width, double* v);
/* The run coding's run starts (RiaRun::start, build_ria,
 * list_lattice.cpp:206-226) in node order: run r covers nodes
 * [start[r], start[r+1]) (the last up to n_fluid).  *count = number of runs,
 * -1 for names without a coding; run_starts may be null to query the count. */
int lbmgpu_export_runs(lbmgpu_ctx* ctx, uint32_t* run_starts, uint64_t cap,
                       int64_t* count);
int lbmgpu_descriptor_of(lbmgpu_ctx* ctx, lbmgpu_descriptor* out);

/* List structure export for the bit-exact checks (list_lattice.hpp:86-99):
 * nodes (3 x int32 per node), adjacency in the reference's canonical
 * [n*18 + d-1] order, the 19 starts and the total slot count.  Any pointer may
 * be NULL.  ConfigError for direct kernels. */
int lbmgpu_export_structure(lbmgpu_ctx* ctx, int32_t* nodes,
                            uint32_t* adjacency, uint64_t* starts19,
                            uint64_t* total_slots);

/* ------------------------------------------------------- harness/verify */

/* steady_state_run (harness.cpp:141-174) with device-side macro fields and
 * max|du| / max|u| reductions. */
int lbmgpu_steady_state_run(lbmgpu_ctx* ctx, double omega_plus,
                            double magic_lambda, const double* g3,
                            long check_interval, double rel_tol,
                            long max_steps, long* steps, int* converged,
                            double* final_delta);
/* Layer-averaged u_x over z (verification.cpp:75-85 ordering), unshifted. */
int lbmgpu_layer_ux(lbmgpu_ctx* ctx, double* out_nz);

typedef struct {
  double linf_rel, l2_rel, half_force_shift;
  long steps;
  int converged, passed;
} lbmgpu_verify_report;
/* verify_kernel (verification.cpp:31-100): slit Poiseuille case.
 * simulated/analytic (nullable) receive nz-2 values.  Returns LBMGPU_OK
 * whether or not it passed; see report->passed. */
int lbmgpu_verify(const char* kernel_name, int nx, int ny, int nz, double g,
                  double tau, double magic_lambda, long check_interval,
                  double rel_tol, long max_steps, lbmgpu_verify_report* report,
                  double* simulated, double* analytic);

/* ---------------------------------------------------- instrumentation */

/* Record CUDA events around every sweep launch on the launching stream;
 * query per-kernel launch counts and summed device ms. */
int lbmgpu_kernel_stats_enable(lbmgpu_ctx* ctx, int enable);
/* Fills up to cap entries: names (each < 48 chars, NUL-terminated, stride 48),
 * launch counts, total ms.  *n gets the number of distinct kernels. */
int lbmgpu_kernel_stats(lbmgpu_ctx* ctx, char* names48, long* launches,
                        double* total_ms, int cap, int* n);
/* Per-launch device intervals of the launches recorded while kernel stats
 * were on (ms after the first of them; every stream shares the clock), in
 * record order; at most 65,536 are kept per period.  *n = total. */
int lbmgpu_kernel_timeline(lbmgpu_ctx* ctx, char* names48, double* t0, double* t1, int cap,
                           int* n);
int lbmgpu_kernel_stats_reset(lbmgpu_ctx* ctx);
/* Device sweep launches issued since creation (all streams). */
int lbmgpu_launch_count(lbmgpu_ctx* ctx, long* out);
/* Page-locked host allocation helpers for end-to-end timing. */
int lbmgpu_host_alloc(size_t bytes, void** out);
int lbmgpu_host_free(void* p);
/* Device bandwidth micro-benchmarks (reference run_microbench,
 * microbench.cpp:57-175): kind = "copy" | "copy-19" | "copy-19-nt-sl" |
 * "update-19"; median GB/s of `reps` passes over `working_set_bytes`
 * (>= 4x L2), GPU accounting without write allocate (16 B per element and
 * stream). */
int lbmgpu_microbench(const char* kind, uint64_t working_set_bytes, int reps,
                      double* gbps);
/* Accounting of one pass of that micro-benchmark (host only, no device):
 * elements per stream, bytes this library counts (16 B per element and
 * stream) and bytes the reference counts for the same pass
 * (microbench.cpp:92-99: copy / copy-19 add 8 B write allocate). */
int lbmgpu_microbench_accounting(const char* kind, uint64_t working_set_bytes,
                                 uint64_t* elems, uint64_t* bytes_gpu, uint64_t* bytes_ref);
/* Device properties for reports. */
int lbmgpu_device_info(int device, char* name64, int* sm_count,
                       size_t* total_mem, int* l2_bytes);
int lbmgpu_synchronize(lbmgpu_ctx* ctx);

/* ------------------------------------------------------------ multi-GPU */

/* 128-byte ncclUniqueId (NCCL loaded lazily with dlopen). */
int lbmgpu_nccl_unique_id(void* out128);
/* Process-local state access for split domains (nranks > 1): this process's
 * fluid nodes in canonical order ("local rows"), their global canonical
 * indices, and snapshot/load of exactly those rows (count = rows*19).  With
 * one process the local rows are all N canonical nodes.  lbmgpu_snapshot /
 * lbmgpu_load_state on a split domain touch only this process's rows of the
 * full-size canonical buffer. */
int lbmgpu_local_rows(lbmgpu_ctx* ctx, uint64_t* rows);
int lbmgpu_local_canonical_index(lbmgpu_ctx* ctx, uint64_t* out_rows);
int lbmgpu_snapshot_local(lbmgpu_ctx* ctx, double* host, uint64_t count);
int lbmgpu_load_state_local(lbmgpu_ctx* ctx, const double* host,
                            uint64_t count);
/* Peer-memory transport (dist.transport = 1, nranks > 1): this rank's
 * record (CUDA IPC handles of its lattice and epoch flags; *len bytes, at
 * most cap), and the attach of all ranks' records concatenated in rank order
 * (every rank calls both, export before any attach; the caller moves the
 * records, e.g. an all-gather).  advance() before attach is a ConfigError. */
int lbmgpu_peer_export(lbmgpu_ctx* ctx, void* out, size_t cap, size_t* len);
int lbmgpu_peer_attach(lbmgpu_ctx* ctx, const void* records, size_t record_len,
                       int nranks);
/* Peer-transport plumbing check (no sweep): one boundary plane, 19 x nx*ny
 * doubles in device layout ([slot][y][x]) -- which = 0 lower neighbour's top
 * plane, 1 upper neighbour's bottom plane (read through the peer mapping),
 * 2 own bottom plane, 3 own top plane. */
int lbmgpu_peer_probe(lbmgpu_ctx* ctx, int which, double* out, uint64_t count);
/* This process's slab(s): part index < number of local parts. */
int lbmgpu_part_info(lbmgpu_ctx* ctx, int part, int* z0, int* z1,
                     uint64_t* n_fluid_part);
/* Halo exchange plan as (phase, src part, dst part, src plane, dst plane,
 * group, elements) rows, 7 int64 per row; see DESIGN.md §multi-GPU.
 * z_wrap: 0 = AA plan (phases 0/1), 1 = AA plan with the z ring,
 * 2 = one-step push/pull plan (phases 2/3, always with the ring; dst plane
 * -1 / -2 = the receiver's bottom / top staging plane). */
int lbmgpu_halo_plan(int nz, int parts, int z_wrap, int64_t* rows, int cap,
                     int* n_rows);

/* FNV-1a 64 over raw bytes (state_fingerprint, harness.cpp:27-39, applied to
 * a host canonical snapshot). */
uint64_t lbmgpu_fnv1a(const void* data, uint64_t nbytes);

const char* lbmgpu_last_error(void);
int lbmgpu_abi_version(void);

/* Debug aid (no reference equivalent): with LBMGPU_GUARD=1 in the
 * environment when buffers are allocated, every device buffer carries 4 KiB
 * guard zones of a fixed byte pattern on both sides; this counts the live
 * buffers whose guards were overwritten (out-of-bounds device writes).  The
 * description of the first corruptions is left in lbmgpu_last_error(). */
int lbmgpu_guard_check(int* corrupted);
/* Negative control: writes 8 bytes past a fresh guarded buffer and reports
 * how many corrupted buffers lbmgpu_guard_check would see (1 expected). */
int lbmgpu_guard_selftest(int* detected);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* LBMGPU_H */
