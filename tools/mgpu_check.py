"""Multi-GPU parity check for the z-slab / node-range paths (NCCL halo copies,
or transport "peer": CUDA IPC peer memory for direct AA) (run under torchrun,
one process per GPU):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/mgpu_check.py [nx ny nz steps kind name transport]

Every rank advances its slab; rank 0 gathers the local rows (canonical
indices + PDFs) and compares the assembled state with a single-GPU run of the
same kernel.  Prints PASS/FAIL and exits non-zero on mismatch."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1711_11468_b200 as lbm  # noqa: E402


def main():
    nx, ny, nz, steps = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (64, 32, 48, 10)))
    kind = sys.argv[5] if len(sys.argv) > 5 else "channel"
    name = sys.argv[6] if len(sys.argv) > 6 else "aa-soa"
    transport = sys.argv[7] if len(sys.argv) > 7 else "copy"  # "peer": CUDA IPC peer memory
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [lbm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    spec = lbm.GeometrySpec(kind, nx, ny, nz)
    params, force = lbm.TrtParams.from_tau(0.9), lbm.BodyForce((1e-5, 2e-6, -3e-6))
    k = lbm.make_kernel(lbm.make_descriptor(name), spec,
                        dist={"rank": rank, "nranks": world, "device": local, "nccl_id": obj[0],
                              "transport": transport})
    if transport == "peer":
        recs = [None] * world
        dist.all_gather_object(recs, k.peer_export())
        k.peer_attach(recs)
        dist.barrier()
    k.load_perturbed(4242)
    k.advance(params, force, steps)
    mass = k.total_mass()
    rows = (k.local_canonical_index(), k.snapshot_local())
    out = [None] * world
    dist.gather_object(rows, out if rank == 0 else None, dst=0)
    ok = True
    if rank == 0:
        ref = lbm.make_kernel(lbm.make_descriptor(name), spec)
        ref.load_perturbed(4242)
        ref.advance(params, force, steps)
        expect = ref.snapshot().reshape(-1, 19)
        got = np.full_like(expect, np.nan)
        for idx, snap in out:
            got[idx.astype(np.int64)] = snap.reshape(-1, 19)
        ok = bool(np.array_equal(got, expect))
        ok = ok and abs(mass - ref.total_mass()) <= 1e-12 * abs(ref.total_mass())
        print(("PASS" if ok else "FAIL"),
              f"world={world} {name} {transport} {kind} {nx}x{ny}x{nz} steps={steps}",
              flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
