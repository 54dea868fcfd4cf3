#!/usr/bin/env python3
"""Benchmark driver (contract in the task statement; numbers in DESIGN.md).

Default workload = BASELINE config 5: channel 1024x512x512 fp64 D3Q19 TRT,
direct addressing, AA pattern (aa-soa), omega+ = 1, Lambda = 3/16,
g = (1e-5, 0, 0), initial state = weights; z-slab decomposed over the
ranks (1 GPU = the whole box).  One bench "step" = one AA pair = two lattice
updates of every fluid node (AA needs even counts, reference
kernels.cpp:87-91).  MFLUP/s = N_fluid * lattice_steps / s / 1e6
(reference harness.cpp:115-116).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config 1..5]

--impl reference times the reference's own CPU implementation
(oracle/_ref/liblbm_ref.so = lbmbench compiled from its sources) on the
host cores (pinned pool, one worker per core), on the full BASELINE
workload: W warm-up and K timed bench steps on the whole box.  The b200
arm's `cpu_baseline` is the same library on a bounded sample box.

--gpus N outside torchrun re-executes under torch.distributed.run with N
ranks; N > visible GPUs or WORLD_SIZE != N exits non-zero.  At N > 1 a
bitwise pre-flight of the decomposition runs before anything is timed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (kernel, kind, dims, extra, baseline steps, cpu sample dims)
    1: ("blk-push-soa", "channel", (64, 64, 64), {}, 100, (64, 64, 64)),
    2: ("list-aa-soa", "channel", (256, 256, 256), {}, 1000, (32, 256, 256)),
    3: ("list-pull-soa", "pipe", (512, 256, 256), {"pipe_diameter": 250}, 500, (32, 256, 256)),
    4: ("list-aa-soa", "blocks", (400, 400, 400), {"block": 8, "spacing": 8}, 500, (64, 400, 400)),
    5: ("aa-soa", "channel", (1024, 512, 512), {}, 200, (128, 512, 512)),
}
OMEGA_PLUS, LAMBDA, G = 1.0, 3.0 / 16.0, (1e-5, 0.0, 0.0)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def csrc_sha16():
    """Content hash of the CUDA/C++ sources (paper_1711_11468_b200/csrc):
    what a committed ncu capture was taken of.  Content, not git, because the
    GPU box receives the tree without .git."""
    import hashlib
    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_1711_11468_b200", "csrc")
    for name in sorted(os.listdir(d)):
        if name.endswith((".cu", ".cuh", ".cpp", ".hpp", ".h")):
            h.update(name.encode())
            with open(os.path.join(d, name), "rb") as f:
                h.update(f.read())
    return h.hexdigest()[:16]


def ncu_traffic(kernel_name, cid=5, dims=None):
    """(dram bytes per launch, note) for `kernel_name` on BASELINE config
    `cid` from the committed ncu summary (profiles/ncu_summary.json: cfg 5
    under "kernels", the list configs under "configs").  None when the
    summary was captured from other kernel sources than these (its
    csrc_sha16 differs) or for other boxes."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if dims is not None:
        return None, "box differs from the captured one"
    try:
        with open(p) as f:
            d = json.load(f)
    except Exception:
        return None, "no profiles/ncu_summary.json"
    if d.get("csrc_sha16") != csrc_sha16():
        return None, (f"stale: ncu summary of csrc {d.get('csrc_sha16')}, "
                      f"running csrc {csrc_sha16()}")
    table = d.get("kernels", {}) if cid == 5 else d.get("configs", {}).get(str(cid), {})
    v = table.get(kernel_name, {}).get("dram_bytes_per_launch")
    return v, (f"ncu dram__bytes_read+write per launch, {d.get('source', '')}" if v is not None
               else "kernel not in the ncu summary")


# --------------------------------------------------------------- CPU legs
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores():
    """Cores this process may run on (sorted), i.e. the reference's --pin
    list for a pool of all of them."""
    try:
        return sorted(os.sched_getaffinity(0))
    except AttributeError:
        return list(range(os.cpu_count() or 1))


def cpu_reference_run(cid, steps_per_sample, samples, warmup_samples, full=False):
    """The reference lbmbench (oracle/_ref) on the host cores: every sample is
    `steps_per_sample` lattice steps of the reference kernel, on the full
    BASELINE box (full=True) or the bounded sample box.  The WorkerPool has
    one worker per available core, worker w pinned to core w (reference
    --pin semantics, workers.cpp:26-39).  Returns (MFLUP/s, cores,
    description, kind, seconds per sample)."""
    kernel, kind, dims, extra, _, sdims = CONFIGS[cid]
    box = dims if full else sdims
    cores = host_cores()
    threads = len(cores)
    from oracle.oracle import Ref, Port  # test/baseline infrastructure only
    try:
        ref = Ref()
    except FileNotFoundError:
        ref = None
    if ref is not None:
        k = ref.kernel(kernel, kind, *box, threads=threads, block=extra.get("block", 4),
                       spacing=extra.get("spacing", 4), pipe_diameter=extra.get("pipe_diameter", 0),
                       pin=cores)
        pinned = k.pinned()
        for _ in range(warmup_samples):
            k.advance(OMEGA_PLUS, LAMBDA, G, steps_per_sample)
        secs = [k.advance(OMEGA_PLUS, LAMBDA, G, steps_per_sample) for _ in range(samples)]
        n = k.n_fluid
        tot = sum(secs)
        desc = (f"reference lbmbench {kernel} (oracle/_ref, -O3 -ffp-contract=off -march=x86-64-v4, "
                f"WorkerPool({threads}) pinned to cores {cores[0]}..{cores[-1]} ({pinned} bound)) "
                f"on {cpu_model()}; {kind} {'x'.join(map(str, box))} "
                f"({'the full BASELINE box' if full else 'bounded sample box'}, {n} fluid nodes), "
                f"{warmup_samples} x {steps_per_sample} steps warm-up, "
                f"{samples} x {steps_per_sample} steps timed (Kernel::advance wall clock)")
        return n * steps_per_sample * samples / tot / 1e6, threads, desc, "reference", tot / samples
    # fallback: our C restatement, textbook stepper, single thread
    port = Port()
    fam = "half" if kernel.startswith("list-") else "full"
    t0 = time.perf_counter()
    port.run(fam, kind, *box, steps_per_sample * samples, OMEGA_PLUS, g=G,
             block=extra.get("block", 4), spacing=extra.get("spacing", 4),
             pipe_diameter=extra.get("pipe_diameter", 0))
    dt = time.perf_counter() - t0
    _, _, nf = port.geometry(kind, *box, extra.get("block", 4), extra.get("spacing", 4),
                             extra.get("pipe_diameter", 0))
    return (nf * steps_per_sample * samples / dt / 1e6, 1,
            f"port oracle textbook stepper on {cpu_model()}; {kind} {'x'.join(map(str, box))}",
            "port", dt / samples)


def base_line(cid, n_gpus, steps, warmup, lattice_per_step):
    kernel, kind, dims, extra, bsteps, _ = CONFIGS[cid]
    return {
        "metric": "MFLUP/s (fp64 D3Q19 TRT)",
        "unit": "MFLUP/s",
        "n_gpus": n_gpus,
        "steps": steps,
        "warmup": warmup,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE config: initial state = D3Q19 weights, rho=1, u=0)",
        "config": {
            "workload": f"cfg{cid}: {kind} {'x'.join(map(str, dims))} {kernel}"
                        + (f" {extra}" if extra else ""),
            "kernel": kernel, "geometry": kind, "dims": list(dims), **extra,
            "omega_plus": OMEGA_PLUS, "magic_lambda": LAMBDA, "g": list(G),
            "lattice_updates_per_step": lattice_per_step,
            "baseline_steps": bsteps,
            "parallelism": f"z-slab x{n_gpus}" if n_gpus > 1 else "single GPU",
            "l2": "inputs larger than L2" if cid != 1 else
                  "lattice (2 x 40 MB) fits the 126 MB L2; no flush (reported as is)",
        },
    }


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation on the host cores, on the FULL
    BASELINE workload: W warm-up and K timed bench steps of the config's
    kernel on its whole box (cfg 5: 1024x512x512, 41 GB, one AA pair per
    step), pinned pool, measured ms per step.  Rank 0 only."""
    if rank != 0:
        return
    cid = args.config
    kernel = CONFIGS[cid][0]
    per = 2 if "aa" in kernel.split("-") else 1
    mflups, cores, desc, kind, sec = cpu_reference_run(cid, per, args.steps, args.warmup,
                                                       full=True)
    line = base_line(cid, args.gpus or world, args.steps, args.warmup, per)
    line.update({"impl": "reference", "value": mflups,
                 "ms_per_step": sec * 1e3,
                 "cpu_baseline": {"value": mflups, "unit": "MFLUP/s", "cores": cores,
                                  "kind": kind, "sample": desc, "cpu_model": cpu_model()},
                 "e2e": {"value": mflups, "unit": "MFLUP/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def visible_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def relaunch(n, launch_check):
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with N ranks (one per GPU), same arguments; the
    exit code is the launcher's.  Refuses (exit 2) when N exceeds the
    visible GPUs instead of silently measuring one."""
    if not launch_check:
        have = visible_gpus()
        if n > have:
            print(f"bench.py: --gpus {n} but only {have} GPU(s) visible; refusing to run "
                  f"(no silent single-GPU line)", file=sys.stderr, flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def preflight(lbm, dist, rank, world, local, desc, transport):
    """Bitwise pre-flight of the decomposition before anything is timed:
    every rank advances its part of a small lattice (channel 64 x 32 x 6N,
    perturbed init, 10 steps) with the chosen transport; rank 0 assembles the
    local rows and compares them with its own single-GPU run of the same
    kernel (the invariance of reference tests/test_kernels.cpp:177-195
    across decompositions).  Every stage ends in a collective flag, so a rank
    that fails (e.g. a CUDA IPC error on the peer path) cannot leave the
    others blocked.  Returns (ok, detail)."""
    import numpy as np
    import torch

    def all_ok(flag):
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    spec = lbm.GeometrySpec("channel", 64, 32, 6 * world)
    params, force = lbm.TrtParams.from_tau(0.9), lbm.BodyForce((1e-5, 2e-6, -3e-6))
    err = ""
    k = None
    obj = [lbm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    try:
        k = lbm.make_kernel(desc, spec, dist={"rank": rank, "nranks": world, "device": local,
                                              "nccl_id": obj[0], "transport": transport})
        ok = True
    except Exception as e:  # noqa: BLE001 -- reported, then the flag decides
        ok, err = False, f"create: {e}"
    if not all_ok(ok):
        return False, err or "create failed on another rank"
    if transport == "peer":
        recs = [None] * world
        try:
            rec = k.peer_export()
        except Exception as e:  # noqa: BLE001
            rec, err = b"", f"peer_export: {e}"
        dist.all_gather_object(recs, rec)
        try:
            if err or any(not r for r in recs):
                raise RuntimeError(err or "peer_export failed on another rank")
            k.peer_attach(recs)
            ok = True
        except Exception as e:  # noqa: BLE001
            ok, err = False, f"peer_attach: {e}"
        if not all_ok(ok):
            return False, err or "peer_attach failed on another rank"
    try:
        k.load_perturbed(4242)
        k.advance(params, force, 10)
        rows = (k.local_canonical_index(), k.snapshot_local())
        ok = True
    except Exception as e:  # noqa: BLE001
        rows, ok, err = None, False, f"advance: {e}"
    if not all_ok(ok):
        return False, err or "advance failed on another rank"
    out = [None] * world
    dist.gather_object(rows, out if rank == 0 else None, dst=0)
    ok = True
    if rank == 0:
        ref = lbm.make_kernel(desc, spec)
        ref.load_perturbed(4242)
        ref.advance(params, force, 10)
        expect = ref.snapshot().reshape(-1, 19)
        got = np.full_like(expect, np.nan)
        for idx, snap in out:
            got[idx.astype(np.int64)] = snap.reshape(-1, 19)
        ok = bool(np.array_equal(got, expect))
        err = "" if ok else "decomposed state differs from the single-GPU run"
        del ref
    ok = all_ok(ok)
    del k
    return ok, (f"bitwise equal to 1 GPU: {desc.name} channel 64x32x{6 * world}, "
                f"{world} parts, 10 steps, transport {transport}" if ok else err)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="number of GPUs (ranks); outside torchrun, N > 1 re-executes this "
                         "script under torch.distributed.run with N ranks")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true",
                    help="skip the device update-19/copy-19 micro-benchmark ceiling")
    ap.add_argument("--transport", default="auto", choices=["auto", "copy", "peer"],
                    help="z-slab halo transport: copy = NCCL send/recv of the halo slots "
                         "(device copies with --virtual-parts); peer = boundary sweeps "
                         "load/store the neighbour slab in peer memory (CUDA IPC), epoch "
                         "flags (opt-in: falls back to copy if its pre-flight fails); "
                         "auto = copy at N > 1, peer for --virtual-parts emulation")
    ap.add_argument("--decompose", action="store_true",
                    help="at N>1: z-slab decomposition of direct push/pull and node-range "
                         "decomposition of list AA instead of replicas")
    ap.add_argument("--virtual-parts", type=int, default=1,
                    help="1 GPU: emulate the multi-GPU decomposition with this many parts "
                         "(device-copy halos) -- an overhead probe, not a bench line")
    ap.add_argument("--nccl-self", action="store_true",
                    help="with --virtual-parts: halos through the NCCL transport (one rank "
                         "owning every part, self send/recv) instead of device copies")
    ap.add_argument("--kernel", default=None,
                    help="run another kernel name on the config's geometry (extra lines)")
    ap.add_argument("--dims", default=None,
                    help="override the box (NXxNYxNZ) -- profiling only, not a bench line")
    ap.add_argument("--launch-check", action="store_true",
                    help="test hook: after the (re-)launch every rank reports its rank / world "
                         "and rank 0 prints one line; no GPU work")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        sys.exit(relaunch(args.gpus, args.launch_check))
    if args.gpus is not None and args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to run",
              file=sys.stderr, flush=True)
        sys.exit(2)
    if args.launch_check:
        import torch.distributed as tdist
        if world > 1:
            tdist.init_process_group("gloo")
            ranks = [None] * world
            tdist.all_gather_object(ranks, rank)
            tdist.destroy_process_group()
        else:
            ranks = [0]
        if rank == 0:
            print(json.dumps({"launch_check": True, "n_gpus": world, "ranks": ranks}), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist

    import paper_1711_11468_b200 as lbm

    cid = args.config
    kernel, kind, dims, extra, _, _ = CONFIGS[cid]
    if args.dims or args.kernel:
        if args.dims:
            dims = tuple(int(v) for v in args.dims.split("x"))
        if args.kernel:
            kernel = args.kernel
        CONFIGS[cid] = (kernel, kind, dims, extra, CONFIGS[cid][4], CONFIGS[cid][5])
    desc = lbm.make_descriptor(kernel)
    aa = desc.prop == "aa"
    per = 2 if aa else 1
    spec = lbm.GeometrySpec(kind, *dims, extra.get("block", 4), extra.get("spacing", 4),
                            extra.get("pipe_diameter", 0))
    dspec = None
    # direct AA (cfg 5) is z-slab decomposed over the ranks (strong scaling);
    # every other kernel runs as independent replicas, one lattice per GPU
    # (the list configs are replicas only) -> weak scaling.
    # --decompose also splits direct push/pull (z slabs) and list AA (node
    # ranges) instead of replicating them.
    decomposable = (aa and desc.addr == "direct") or (
        args.decompose and not desc.ria and (desc.addr == "direct" or aa))
    replicas = world > 1 and not decomposable
    if args.transport == "auto":
        # emulation on one GPU: the peer schedule (boundary stream, epoch
        # flags) on device pointers; several GPUs: NCCL halo copies unless
        # --transport peer asks for the peer-memory path
        args.transport = "peer" if desc.addr == "direct" and world == 1 else "copy"
    if world == 1 and args.virtual_parts > 1:
        dspec = {"virtual_parts": args.virtual_parts, "transport": args.transport}
        if args.nccl_self:
            dspec["nccl_id"] = lbm.nccl_unique_id()
            dspec["transport"] = "copy"  # NCCL self send/recv halos
    pre = None
    if world > 1 and not replicas:
        if args.transport == "peer" and desc.addr != "direct":
            args.transport = "copy"
        # bitwise pre-flight of the decomposition with the chosen transport;
        # the peer path falls back to NCCL copies, a failing copy path stops
        # the run (no number from a wrong decomposition)
        ok, detail = preflight(lbm, dist, rank, world, local, desc, args.transport)
        pre = {"transport": args.transport, "ok": ok, "detail": detail}
        if not ok and args.transport == "peer":
            args.transport = "copy"
            ok, detail = preflight(lbm, dist, rank, world, local, desc, "copy")
            pre = {"transport": "copy", "ok": ok, "detail": detail,
                   "peer_failed": pre["detail"]}
        if not ok:
            if rank == 0:
                print(f"bench.py: multi-GPU pre-flight failed: {detail}", file=sys.stderr,
                      flush=True)
            dist.destroy_process_group()
            sys.exit(3)
        obj = [lbm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        dspec = {"rank": rank, "nranks": world, "device": local, "nccl_id": obj[0],
                 "transport": args.transport}
    k = lbm.make_kernel(desc, spec, lbm.PaddingPolicy.automatic(), dist=dspec)
    if dspec and dspec.get("transport") == "peer" and world > 1:
        recs = [None] * world
        dist.all_gather_object(recs, k.peer_export())
        k.peer_attach(recs)
        dist.barrier()
    N = k.n_fluid() * (world if replicas else 1)  # fluid updates per lattice step, all ranks
    params = lbm.TrtParams(OMEGA_PLUS, LAMBDA)
    force = lbm.BodyForce(G)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        k.synchronize()

    # clock sampler first, then the warm-up right before the timed region (an
    # idle gap in between lets the GPU drop out of its boost state)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if args.warmup:
        k.advance(params, force, per * args.warmup)
    barrier()
    k.kernel_stats_reset()
    k.kernel_stats_enable(True)
    launches0 = k.launch_count()
    barrier()
    ms = k.time_advance(params, force, per * args.steps)
    barrier()
    launches = k.launch_count() - launches0
    k.kernel_stats_enable(False)
    stats = k.kernel_stats()
    overlap = None
    if dspec is not None:
        # decomposed paths: how much of the boundary-stream work (boundary
        # sweeps, halo exchanges / peer waits) ran beside interior sweeps
        overlap = lbm.lbmgpu.stream_overlap(k.kernel_timeline())
    clk = clocks.stop()
    clk_ranks = [clk]
    if dist is not None:
        # every rank sampled its own GPU: the line carries all of them, and
        # the headline clocks are the worst rank's (lowest median, union of
        # the throttle reasons)
        clk_ranks = [None] * world
        dist.all_gather_object(clk_ranks, clk)
        meds = [c["sm_mhz"] for c in clk_ranks if c.get("sm_mhz")]
        maxs = [c["sm_max_mhz"] for c in clk_ranks if c.get("sm_max_mhz")]
        clk = {"sm_mhz": min(meds) if meds else None, "sm_max_mhz": max(maxs) if maxs else None,
               "reasons": sorted({r for c in clk_ranks for r in c.get("reasons", [])}),
               "samples": sum(c.get("samples", 0) for c in clk_ranks),
               "of": "worst rank (lowest median SM clock; union of reasons)"}
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    mflups = N * per * args.steps / (ms / 1e3) / 1e6

    # roofline of the dominant kernel (largest share of the timed region)
    hbm, peak_src = peaks()
    _, _, gpu_b = lbm.loop_balance(kernel)
    local_nf = k.local_rows()  # fluid nodes this rank updates per lattice step
    rows = sorted(stats.items(), key=lambda kv: -kv[1]["ms"])
    roof = None
    kernels_out = {}
    for name, st in rows:
        if st["launches"] == 0:
            continue
        avg_ms = st["ms"] / st["launches"]
        # every sweep launch of the timed region touches each fluid node once:
        # 19 reads + 19 writes of 8 B (+ 72 B of adjacency for list one-step,
        # 72 B for the odd AA list sub-step only)
        if "ria_pid" in name or "pull_pid" in name or "pull_stream_pid" in name:
            # pattern-id coding: 304 B of PDFs + a 1/2/4-byte pattern id per
            # node (the pattern table stays in L1 / L2)
            per_node = 304 + (4 if "pid32" in name else 2 if "pid16" in name else 1)
        elif "ria" in name:
            # run-coded odd step: 304 B of PDFs + 8 B of run table per 32
            # nodes (the pattern rows are L1/L2 resident)
            per_node = 304 + 0.25
        elif "list_aa_odd" in name or ("list_pull" in name) or ("list_push" in name):
            per_node = 304 + 72
        else:
            per_node = 304
        alg = local_nf * per_node
        ach = alg / (avg_ms / 1e3) / 1e9
        kernels_out[name] = {"launches": st["launches"], "avg_ms": avg_ms,
                             "share": st["ms"] / ms if ms else None,
                             "alg_bytes_per_launch": alg, "achieved_GBps": ach}
        if roof is None:
            # the committed ncu numbers are whole-box launches on one GPU
            whole = world == 1 and args.virtual_parts <= 1
            traffic, tnote = (ncu_traffic(name, cid, args.dims) if whole
                              else (None, "decomposed run: no whole-box capture"))
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": traffic, "traffic_source": tnote,
                    "kernel": name,
                    "alg_bytes_per_launch": alg, "peak_source": peak_src,
                    "bytes_per_node": per_node}

    # the paper's second ceiling: the matching device micro-benchmark
    # (update-19 for AA, copy-19 for one-step, perfmodel.cpp:68-72), measured
    # live on this GPU after the timed region
    step_gbps = N * per * gpu_b / (ms / args.steps / 1e3) / 1e9 / max(world, 1)
    if roof is not None and not args.no_micro:
        try:
            mname = lbm.lbmgpu.micro_for(desc)
            # 32 GiB working set: the 19-stream kernels only reach their
            # plateau with streams GBs apart (8 GiB: update-19 5.5 TB/s,
            # 32-40 GiB: 6.6 TB/s on B200)
            mbw = lbm.lbmgpu.microbench(mname, 32 << 30, 3)
            roof["adjusted"] = {"micro": mname, "peak": mbw, "unit": "GB/s",
                                "frac": roof["achieved"] / mbw,
                                "step_frac": step_gbps / mbw}
        except Exception as e:  # never lose the bench line over the extra ceiling
            roof["adjusted"] = {"error": str(e)}

    line = base_line(cid, world, args.steps, args.warmup, per)
    if replicas:
        line["scaling"] = "weak"
        line["config"]["parallelism"] = f"{world} independent replicas (list kernels do not shard)"
    elif world > 1 and args.transport == "peer":
        line["config"]["parallelism"] = (f"z-slab x{world}, peer-memory boundary sweeps "
                                         "(CUDA IPC over NVLink, epoch flags)")
    elif world > 1 and desc.addr == "direct":
        line["config"]["parallelism"] = (f"z-slab x{world}, NCCL send/recv halo slots "
                                         "overlapped with the interior sweeps")
    elif world > 1 and desc.addr == "indirect":
        line["config"]["parallelism"] = f"node-range (x-slab) decomposition x{world}, NCCL index-list halos"
    if world == 1 and args.virtual_parts > 1:
        line["config"]["parallelism"] = (f"EMULATED {args.virtual_parts}-part decomposition on 1 GPU "
                                         + ("(NCCL self send/recv halos" if args.nccl_self
                                            else "(peer-memory boundary sweeps, epoch flags"
                                            if args.transport == "peer"
                                            else "(device-copy halos")
                                         + "; overhead probe)")
    line.update({
        "value": mflups,
        "ms_per_step": ms / args.steps,
        "n_fluid": N,
        "roofline": roof,
        "kernels": kernels_out,
        "gpu_launches": launches,
        "clocks": clk,
        "achieved_hbm_GBps_step": step_gbps,
        "step_roofline_frac": step_gbps / hbm,
        "gpu_bytes_per_flup": gpu_b,
    })
    if overlap is not None:
        line["overlap"] = overlap
    if world > 1:
        line["clocks_per_rank"] = clk_ranks
        line["config"]["transport"] = args.transport if not replicas else None
        line["preflight"] = pre

    # ---- end to end through the public API with host buffers: the initial
    # state is loaded from pinned host memory, the job's steps run, the final
    # state is read back to pinned host memory -- all inside the timed region.
    # The e2e job is the BASELINE run itself (cfg 5: 200 lattice steps,
    # harness.cpp:97-131) or K bench steps if that is longer: load the initial
    # state from the host, advance, read the final state back.
    if not args.no_e2e:
        job_steps = max(args.steps, CONFIGS[cid][4] // per)
        try:
            e2e = run_e2e(lbm, k, params, force, per, job_steps, world, dist, torch, N)
            e2e["job_lattice_steps"] = per * job_steps
        except Exception as e:  # report, never lose the device-timed line
            if world > 1:
                raise
            e2e = {"value": None, "error": str(e)}
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, sdesc, skind, _ = cpu_reference_run(cid, per, 3 if cid != 1 else 20, 1)
            line["cpu_baseline"] = {"value": v, "unit": "MFLUP/s", "cores": cores,
                                    "kind": skind, "sample": sdesc, "cpu_model": cpu_model()}
        except Exception as e:  # report, never fail the GPU line
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(lbm, k, params, force, per, steps, world, dist, torch, N):
    n_local = k.local_state_size() if world > 1 else k.n_fluid() * 19
    buf = lbm.PinnedBuffer(n_local)
    # initial state = weights (the BASELINE init), prepared on the host
    w = [1 / 3] + [1 / 18] * 6 + [1 / 36] * 12
    import numpy as np
    arr = buf.array
    arr.reshape(-1, 19)[:] = np.asarray(w)
    # warm-up of the transfer path (staging buffers, copy streams, events and
    # the pipelined job's column plan are created on first use), untimed
    # like the sweeps' warm-up; one process: a 2-step job through the same
    # call (the timed job then starts from that state -- same cost)
    if world > 1:
        k.load_state_local(arr)
    else:
        k.run(arr, params, force, 2, out=arr)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipelined = False
    if world > 1:
        k.load_state_local(arr)
        k.advance(params, force, per * steps)
        k.snapshot_local(arr)
    else:
        # lbmgpu_run: load_state + advance + snapshot, bitwise the three
        # calls, host transfers pipelined with the sweeps where supported
        _, pipelined = k.run(arr, params, force, per * steps, out=arr)
    k.synchronize()
    dt = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    buf.free()
    return {"value": N * per * steps / dt / 1e6, "unit": "MFLUP/s",
            "h2d_bytes_per_step": N * 19 * 8 / steps, "d2h_bytes_per_step": N * 19 * 8 / steps,
            "seconds": dt, "pipelined": pipelined,
            "what": ("lbmgpu_run: load_state(pinned host) + advance + snapshot(pinned host) in "
                     "one C-ABI call" + (", transfers pipelined with the sweeps" if pipelined
                                         else "") if world == 1 else
                     "load_state_local(pinned host) + advance + snapshot_local(pinned host) "
                     "through the C ABI") + ", wall clock, max over ranks"}


if __name__ == "__main__":
    main()
