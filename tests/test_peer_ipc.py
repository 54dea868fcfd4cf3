"""CUDA IPC plumbing of the peer-memory transport on ONE GPU: two processes
(ranks of a 2-slab aa-soa lattice) export their records, all-gather them
over gloo and attach -- then each reads its neighbour's boundary plane
through the mapping (lbmgpu_peer_probe) and compares it with the plane the
neighbour reads from its own memory.  No sweep runs, so no kernel ever waits
on the other process (B200_PROFILING.md: ranks whose kernels wait on one
another must not share a GPU); the sweeps themselves are covered by the
emulated-slab tests (test_gpu_parity.py) and the CPU protocol tests
(test_halo_gloo.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, name, kind, dims, q, guard=False):
    import sys
    sys.path.insert(0, ROOT)
    if guard:  # guard-zone allocator: lattice pointers sit 4 KiB into their allocation
        os.environ["LBMGPU_GUARD"] = "1"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1711_11468_b200 as lbm
        k = lbm.make_kernel(lbm.make_descriptor(name), lbm.GeometrySpec(kind, *dims),
                            dist={"rank": rank, "nranks": world, "device": 0,
                                  "transport": "peer"})
        k.load_perturbed(4242)
        plane = 19 * dims[0] * dims[1]
        try:
            k.total_mass()
            mass_raised = False
        except lbm.ConfigError:
            mass_raised = True  # no NCCL id: no cross-process mass reduction
        recs = [None] * world
        dist.all_gather_object(recs, k.peer_export())
        k.peer_attach(recs)
        own = {2: k.peer_probe(2, plane), 3: k.peer_probe(3, plane)}
        seen = {}
        for which in (0, 1):
            try:
                seen[which] = k.peer_probe(which, plane)
            except lbm.ConfigError:
                pass
        allp = [None] * world
        dist.all_gather_object(allp, (own, seen))
        ok = True
        for r, (o, sn) in enumerate(allp):
            lo, hi = r - 1, r + 1
            if 1 in sn:  # upper neighbour's bottom plane == its own view
                ok &= bool(np.array_equal(sn[1], allp[hi % world][0][2]))
            if 0 in sn:
                ok &= bool(np.array_equal(sn[0], allp[lo % world][0][3]))
            rg = ring(kind) or name != "aa-soa"  # one-step plans always carry the ring
            ok &= (1 in sn) == (hi < world or rg) and (0 in sn) == (lo >= 0 or rg)
        q.put((rank, bool(ok), mass_raised))
        del k
    finally:
        dist.destroy_process_group()


def ring(kind):
    return kind == "blocks"  # fluid on z = 0 / nz - 1: the z ring is exchanged


@pytest.mark.parametrize("name,kind,dims,guard", [("aa-soa", "channel", (16, 12, 24), False),
                                                  ("aa-soa", "blocks", (16, 16, 16), False),
                                                  ("blk-push-soa", "channel", (16, 12, 24), False),
                                                  ("aa-soa", "blocks", (16, 16, 16), True)])
def test_peer_ipc_export_attach_two_processes(name, kind, dims, guard):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, name, kind, dims, q, guard))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok, _ in res), res
    assert all(raised for _, _, raised in res)


def _timeout_rank(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["LBMGPU_PEER_TIMEOUT_MS"] = "1500"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1711_11468_b200 as lbm
        dims = (16, 12, 24)
        k = lbm.make_kernel(lbm.make_descriptor("aa-soa"), lbm.GeometrySpec("channel", *dims),
                            dist={"rank": rank, "nranks": world, "device": 0,
                                  "transport": "peer"})
        k.load_perturbed(4242)
        recs = [None] * world
        dist.all_gather_object(recs, k.peer_export())
        k.peer_attach(recs)
        plane = 19 * dims[0] * dims[1]
        before = {w: k.peer_probe(w, plane) for w in (2, 3)}
        dist.barrier()
        res = {}
        if rank == 0:
            # rank 1 never advances: the even-step wait times out
            try:
                k.advance(lbm.TrtParams.from_tau(0.9), lbm.BodyForce((1e-5, 0, 0)), 2)
                res["advance_raised"] = False
            except lbm.DeviceError as e:
                res["advance_raised"] = "timed out" in str(e)
            try:
                k.snapshot_local()
                res["snapshot_raised"] = False
            except lbm.DeviceError:
                res["snapshot_raised"] = True
        dist.barrier()
        if rank == 1:
            # the healthy neighbour's boundary planes were not written
            res["untouched"] = all(np.array_equal(k.peer_probe(w, plane), before[w])
                                   for w in (2, 3))
        q.put((rank, res))
        dist.barrier()
        del k
    finally:
        dist.destroy_process_group()


def test_peer_timeout_raises_and_spares_the_neighbour():
    """a rank whose neighbour never signals gets DeviceError from
    the advance() call that timed out (after its stream sync) and from every
    later call, and its boundary sweeps behind the failed wait skip their
    peer stores, so the neighbour's slab is left bitwise untouched.  Only
    rank 0 launches kernels that wait (bounded at 1.5 s); rank 1 runs no
    sweep, so no kernel waits on a kernel of the other process."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeout_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert res[0] == {"advance_raised": True, "snapshot_raised": True}, res
    assert res[1] == {"untouched": True}, res
