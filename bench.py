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
host cores, on a bounded sample of the same workload.
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


def ncu_traffic(kernel_name, cid=5, dims=None):
    """dram bytes per launch for `kernel_name` on BASELINE config `cid` from
    the committed ncu summary (profiles/ncu_summary.json: cfg 5 under
    "kernels", the list configs under "configs"); None for other boxes."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if dims is not None:
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        table = d.get("kernels", {}) if cid == 5 else d.get("configs", {}).get(str(cid), {})
        return table.get(kernel_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# --------------------------------------------------------------- CPU legs
def cpu_reference_run(cid, steps_per_sample, samples, warmup_samples):
    """The reference lbmbench (oracle/_ref) on the host cores: every sample is
    `steps_per_sample` lattice steps of the reference kernel on the bounded
    sample box.  Returns (MFLUP/s, cores, description, kind)."""
    kernel, kind, dims, extra, _, sdims = CONFIGS[cid]
    threads = os.cpu_count() or 1
    from oracle.oracle import Ref, Port  # test/baseline infrastructure only
    try:
        ref = Ref()
    except FileNotFoundError:
        ref = None
    if ref is not None:
        k = ref.kernel(kernel, kind, *sdims, threads=threads, block=extra.get("block", 4),
                       spacing=extra.get("spacing", 4), pipe_diameter=extra.get("pipe_diameter", 0))
        for _ in range(warmup_samples):
            k.advance(OMEGA_PLUS, LAMBDA, G, steps_per_sample)
        secs = [k.advance(OMEGA_PLUS, LAMBDA, G, steps_per_sample) for _ in range(samples)]
        n = k.n_fluid
        tot = sum(secs)
        desc = (f"reference lbmbench {kernel} (oracle/_ref, -O3 -ffp-contract=off -march=x86-64-v4, "
                f"WorkerPool({threads})) on {kind} {'x'.join(map(str, sdims))} "
                f"({n} fluid nodes), {samples} x {steps_per_sample} steps timed")
        return n * steps_per_sample * samples / tot / 1e6, threads, desc, "reference"
    # fallback: our C restatement, textbook stepper, single thread
    port = Port()
    fam = "half" if kernel.startswith("list-") else "full"
    t0 = time.perf_counter()
    port.run(fam, kind, *sdims, steps_per_sample * samples, OMEGA_PLUS, g=G,
             block=extra.get("block", 4), spacing=extra.get("spacing", 4),
             pipe_diameter=extra.get("pipe_diameter", 0))
    dt = time.perf_counter() - t0
    _, _, nf = port.geometry(kind, *sdims, extra.get("block", 4), extra.get("spacing", 4),
                             extra.get("pipe_diameter", 0))
    return (nf * steps_per_sample * samples / dt / 1e6, 1,
            f"port oracle textbook stepper on {kind} {'x'.join(map(str, sdims))}", "port")


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
    if rank != 0:
        return
    cid = args.config
    kernel = CONFIGS[cid][0]
    per = 2 if "aa" in kernel.split("-") else 1
    mflups, cores, desc, kind = cpu_reference_run(cid, per, args.steps, args.warmup)
    line = base_line(cid, args.gpus, args.steps, args.warmup, per)
    # ms per bench step of the FULL workload at the measured CPU rate (the
    # timed samples run on the bounded sample box, see cpu_baseline.sample)
    n_full = {1: 246016, 2: 16516096, 3: 25128960, 4: 56000000, 5: 266342400}[cid]
    line.update({"impl": "reference", "value": mflups,
                 "ms_per_step": n_full * per / (mflups * 1e6) * 1e3,
                 "cpu_baseline": {"value": mflups, "unit": "MFLUP/s", "cores": cores,
                                  "kind": kind, "sample": desc},
                 "e2e": {"value": mflups, "unit": "MFLUP/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true",
                    help="skip the device update-19/copy-19 micro-benchmark ceiling")
    ap.add_argument("--transport", default="auto", choices=["auto", "copy", "peer"],
                    help="z-slab halo transport: peer = boundary sweeps load/store the "
                         "neighbour slab in peer memory (CUDA IPC), epoch flags, boundary "
                         "work on its own stream; copy = NCCL send/recv (device copies with "
                         "--virtual-parts); auto = peer for the direct SoA z slabs, copy for "
                         "the list node ranges")
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
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
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
        args.transport = "peer" if desc.addr == "direct" else "copy"
    if world == 1 and args.virtual_parts > 1:
        dspec = {"virtual_parts": args.virtual_parts, "transport": args.transport}
        if args.nccl_self:
            dspec["nccl_id"] = lbm.nccl_unique_id()
            dspec["transport"] = "copy"  # NCCL self send/recv halos
    if world > 1 and not replicas:
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
    clk = clocks.stop()
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
            traffic = ncu_traffic(name, cid, args.dims) if whole else None
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": traffic, "kernel": name,
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

    # ---- end to end through the public API with host buffers: the initial
    # state is loaded from pinned host memory, the job's steps run, the final
    # state is read back to pinned host memory -- all inside the timed region.
    # The e2e job is the BASELINE run itself (cfg 5: 200 lattice steps,
    # harness.cpp:97-131) or K bench steps if that is longer: load the initial
    # state from the host, advance, read the final state back.
    if not args.no_e2e:
        job_steps = max(args.steps, CONFIGS[cid][4] // per)
        e2e = run_e2e(lbm, k, params, force, per, job_steps, world, dist, torch, N)
        e2e["job_lattice_steps"] = per * job_steps
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, sdesc, skind = cpu_reference_run(cid, per, 3 if cid != 1 else 20, 1)
            line["cpu_baseline"] = {"value": v, "unit": "MFLUP/s", "cores": cores,
                                    "kind": skind, "sample": sdesc}
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
    # warm-up of the transfer path (staging buffers, copy stream, events are
    # created on first use), untimed like the sweeps' warm-up
    if world > 1:
        k.load_state_local(arr)
    else:
        k.load_state(arr)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if world > 1:
        k.load_state_local(arr)
        k.advance(params, force, per * steps)
        k.snapshot_local(arr)
    else:
        k.load_state(arr)
        k.advance(params, force, per * steps)
        k.snapshot(arr)
    k.synchronize()
    dt = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    buf.free()
    return {"value": N * per * steps / dt / 1e6, "unit": "MFLUP/s",
            "h2d_bytes_per_step": N * 19 * 8 / steps, "d2h_bytes_per_step": N * 19 * 8 / steps,
            "seconds": dt, "what": "load_state(pinned host) + advance + snapshot(pinned host) "
                                   "through the C ABI, wall clock, max over ranks"}


if __name__ == "__main__":
    main()
