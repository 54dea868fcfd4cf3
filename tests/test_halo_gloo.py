"""CPU, world_size 2 (gloo): the multi-GPU decomposition protocols end to end
(z-slab AA, z-slab push/pull, list node ranges with local numbering).

Each rank holds its slab in the device layout the CUDA path uses
([storage plane][slot][y][x], one ghost plane per side, slots grouped by c_z),
runs the AA even/odd sub-steps over its own fluid nodes with the oracle's
collision, and exchanges exactly the rows of the library's halo plan
(lbmgpu_halo_plan, the same plan the NCCL path executes) with
torch.distributed send/recv.  The gathered result must equal the full-domain
oracle bit for bit -- for a channel (no z wrap) and for z-periodic blocks
(ring exchange)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

Q = 19
CX = [0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0]
CY = [0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1]
CZ = [0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1]
OPP = [0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17]
SLOT = [5, 6, 7, 8, 9, 14, 0, 10, 11, 12, 13, 15, 1, 2, 16, 17, 3, 4, 18]  # common.cuh dslot
TAU, G = 0.8, (1e-5, -2e-6, 3e-6)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port_no, kind, dims, steps, q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port
        from paper_1711_11468_b200 import lbmgpu as L
        port = Port()
        nx, ny, nz = dims
        flags, per, nf = port.geometry(kind, nx, ny, nz)
        solid = flags.reshape(nx, ny, nz)
        z0, z1 = nz * rank // world, nz * (rank + 1) // world
        nzl = z1 - z0
        ring = bool(solid[:, :, 0].min() == 0 or solid[:, :, nz - 1].min() == 0)
        plan = L.halo_plan(nz, world, ring)
        wp = 1.0 / TAU
        wm = port.omega_minus(wp)
        buf = np.empty((nzl + 2, Q, ny, nx))
        init = port.perturbed(nf, 77)
        # canonical -> slab (weights on solids, perturbed state on fluid nodes)
        w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
        for d in range(Q):
            buf[:, SLOT[d]] = w[d]
        k = 0
        for x in range(nx):
            for y in range(ny):
                for z in range(nz):
                    if solid[x, y, z]:
                        continue
                    if z0 <= z < z1:
                        for d in range(Q):
                            buf[z - z0 + 1, SLOT[d], y, x] = init[k * Q + d]
                    k += 1
        own = [(x, y, z) for z in range(nzl) for y in range(ny) for x in range(nx)
               if not solid[x, y, z + z0]]

        def exchange(phase):
            reqs = []
            for i, (ph, src, dst, sp, dp, s0, ns) in enumerate(plan):
                if ph != phase:
                    continue
                if src == rank:
                    t = torch.from_numpy(np.ascontiguousarray(buf[sp, s0:s0 + ns]))
                    reqs.append(("s", dist.isend(t, dst, tag=i), None, None))
                if dst == rank:
                    t = torch.empty((ns, ny, nx), dtype=torch.float64)
                    reqs.append(("r", dist.irecv(t, src, tag=i), t, (dp, s0, ns)))
            for kind_, r, t, where in reqs:
                r.wait()
                if kind_ == "r":
                    dp, s0, ns = where
                    buf[dp, s0:s0 + ns] = t.numpy()

        for _ in range(steps // 2):
            for (x, y, z) in own:          # even: own slots -> opposite slots
                zs = z + 1
                f = np.array([buf[zs, SLOT[d], y, x] for d in range(Q)])
                f = port.collide(f, wp, wm, G)
                for d in range(Q):
                    buf[zs, SLOT[OPP[d]], y, x] = f[d]
            exchange(0)
            for (x, y, z) in own:          # odd: gather (x-c, opp d), scatter (x+c, d)
                zs = z + 1
                f = np.empty(Q)
                f[0] = buf[zs, SLOT[0], y, x]
                for d in range(1, Q):
                    f[d] = buf[zs - CZ[d], SLOT[OPP[d]], (y - CY[d]) % ny, (x - CX[d]) % nx]
                f = port.collide(f, wp, wm, G)
                buf[zs, SLOT[0], y, x] = f[0]
                for d in range(1, Q):
                    buf[zs + CZ[d], SLOT[d], (y + CY[d]) % ny, (x + CX[d]) % nx] = f[d]
            exchange(1)
        # gather own fluid rows in canonical order to rank 0
        rows = {}
        k = 0
        for x in range(nx):
            for y in range(ny):
                for z in range(nz):
                    if solid[x, y, z]:
                        continue
                    if z0 <= z < z1:
                        rows[k] = [buf[z - z0 + 1, SLOT[d], y, x] for d in range(Q)]
                    k += 1
        out = [None] * world
        dist.all_gather_object(out, rows)
        if rank == 0:
            full = np.zeros(nf * Q)
            for part in out:
                for kk, v in part.items():
                    full[kk * Q:(kk + 1) * Q] = v
            expect, _ = port.run("full", kind, nx, ny, nz, steps, wp, g=G, init=init)
            q.put((bool(np.array_equal(full, expect)), float(port.max_rel_diff(full, expect))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,dims", [("channel", (6, 5, 8)), ("blocks", (8, 8, 8))])
def test_two_rank_zslab_protocol_gloo(kind, dims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port_no, kind, dims, 4, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    equal, rel = q.get(timeout=5)
    assert equal, rel


def _rank_main_one_step(rank, world, port_no, kind, dims, steps, push, q):
    """blk-push / blk-pull over z slabs with the one-step plan (halo.hpp
    phases 2/3): pull fills the source ghost planes before every sweep; push
    ships its ghost planes into the neighbour's staging planes after every
    sweep and the receiver merges them by its own node flags.  Every node
    streams (solid ones too), so the plan always carries the z ring."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port
        from paper_1711_11468_b200 import lbmgpu as L
        port = Port()
        nx, ny, nz = dims
        flags, per, nf = port.geometry(kind, nx, ny, nz)
        solid = flags.reshape(nx, ny, nz).astype(bool)
        z0, z1 = nz * rank // world, nz * (rank + 1) // world
        nzl = z1 - z0
        plan = L.halo_plan(nz, world, True, one_step=True)
        wp = 1.0 / TAU
        wm = port.omega_minus(wp)
        w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
        bufs = [np.empty((nzl + 2, Q, ny, nx)) for _ in range(2)]
        stage = np.zeros((2, Q, ny, nx))
        for d in range(Q):
            bufs[0][:, SLOT[d]] = w[d]
            bufs[1][:, SLOT[d]] = w[d]
        init = port.perturbed(nf, 78)
        k = 0
        for x in range(nx):
            for y in range(ny):
                for z in range(nz):
                    if solid[x, y, z]:
                        continue
                    if z0 <= z < z1:
                        for d in range(Q):
                            bufs[0][z - z0 + 1, SLOT[d], y, x] = init[k * Q + d]
                    k += 1
        nodes = [(x, y, z) for z in range(nzl) for y in range(ny) for x in range(nx)]

        def exchange(phase, buf):
            reqs = []
            for i, (ph, src, dst, sp, dp, s0, ns) in enumerate(plan):
                if ph != phase:
                    continue
                if src == rank:
                    t = torch.from_numpy(np.ascontiguousarray(buf[sp, s0:s0 + ns]))
                    reqs.append(("s", dist.isend(t, int(dst), tag=i), None, None))
                if dst == rank:
                    t = torch.empty((ns, ny, nx), dtype=torch.float64)
                    reqs.append(("r", dist.irecv(t, int(src), tag=i), t, (dp, s0, ns)))
            for kind_, r, t, where in reqs:
                r.wait()
                if kind_ == "r":
                    dp, s0, ns = where
                    target = buf[dp] if dp >= 0 else stage[-dp - 1]
                    target[s0:s0 + ns] = t.numpy()

        def merge(buf):
            # staging plane 0 (from below, c_z=+1 crossings) -> own plane 0,
            # staging plane 1 (from above, c_z=-1 crossings) -> own plane nzl-1
            for face, zo in ((0, 0), (1, nzl - 1)):
                for y in range(ny):
                    for x in range(nx):
                        sol = solid[x, y, zo + z0]
                        for d in range(1, Q):
                            if CZ[d] != (1 if face == 0 else -1):
                                continue
                            s = SLOT[OPP[d]] if sol else SLOT[d]
                            buf[zo + 1, s, y, x] = stage[face, s, y, x]

        cur = 0
        if not push:  # collide pass (kernels_full_os.cpp:173-190)
            for (x, y, z) in nodes:
                if not solid[x, y, z + z0]:
                    f = np.array([bufs[0][z + 1, SLOT[d], y, x] for d in range(Q)])
                    f = port.collide(f, wp, wm, G)
                    for d in range(Q):
                        bufs[0][z + 1, SLOT[d], y, x] = f[d]
        for s in range(steps):
            src, dst = bufs[cur], bufs[1 - cur]
            if push:
                for (x, y, z) in nodes:
                    zs = z + 1
                    f = np.array([src[zs, SLOT[d], y, x] for d in range(Q)])
                    if not solid[x, y, z + z0]:
                        f = port.collide(f, wp, wm, G)
                    dst[zs, SLOT[0], y, x] = f[0]
                    for d in range(1, Q):
                        tx, ty = (x + CX[d]) % nx, (y + CY[d]) % ny
                        tzg = (z + z0 + CZ[d]) % nz
                        sl = SLOT[OPP[d]] if solid[tx, ty, tzg] else SLOT[d]
                        dst[zs + CZ[d], sl, ty, tx] = f[d]
                exchange(3, dst)
                merge(dst)
            else:
                exchange(2, src)
                for (x, y, z) in nodes:
                    zs = z + 1
                    f = np.empty(Q)
                    f[0] = src[zs, SLOT[0], y, x]
                    for d in range(1, Q):
                        f[d] = src[zs - CZ[d], SLOT[d], (y - CY[d]) % ny, (x - CX[d]) % nx]
                    sol = solid[x, y, z + z0]
                    if s + 1 < steps and not sol:
                        f = port.collide(f, wp, wm, G)
                    dst[zs, SLOT[0], y, x] = f[0]
                    for d in range(1, Q):
                        dst[zs, SLOT[OPP[d]] if sol else SLOT[d], y, x] = f[d]
            cur ^= 1
        buf = bufs[cur]
        rows = {}
        k = 0
        for x in range(nx):
            for y in range(ny):
                for z in range(nz):
                    if solid[x, y, z]:
                        continue
                    if z0 <= z < z1:
                        rows[k] = [buf[z - z0 + 1, SLOT[d], y, x] for d in range(Q)]
                    k += 1
        mass = float(sum(buf[zs, s].sum() for zs in range(1, nzl + 1) for s in range(Q)))
        out = [None] * world
        dist.all_gather_object(out, (rows, mass))
        if rank == 0:
            full = np.zeros(nf * Q)
            for part, _ in out:
                for kk, v in part.items():
                    full[kk * Q:(kk + 1) * Q] = v
            expect, emass = port.run("full", kind, nx, ny, nz, steps, wp, g=G, init=init)
            q.put((bool(np.array_equal(full, expect)), float(port.max_rel_diff(full, expect)),
                   sum(m for _, m in out), emass))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("push", [True, False])
@pytest.mark.parametrize("kind,dims", [("channel", (6, 5, 8)), ("blocks", (8, 8, 8))])
def test_two_rank_one_step_protocol_gloo(kind, dims, push):
    """The push / pull halo protocol on 2 gloo ranks, bitwise equal to the
    full-domain textbook full-way stepper (odd step count: result on the
    second grid)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_rank_main_one_step,
                         args=(r, 2, port_no, kind, dims, 3, push, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    equal, rel, mass, emass = q.get(timeout=5)
    assert equal, rel
    assert abs(mass - emass) <= 1e-12 * abs(emass)


def _rank_main_list(rank, world, port_no, kind, dims, steps, q):
    """list-aa-soa over node ranges with the per-part local numbering the
    CUDA path uses (list.cu, 'node-range decomposition'): own slots
    d * nloc + j, ghost copies of the incoming links' sorted slot lists, the
    scatter table remapped to local indices; per AA pair phase 0 (after
    even) s's link slots -> r's ghosts, phase 1 (after odd) back."""
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port
        port = Port()
        nx, ny, nz = dims
        st = port.structure(kind, nx, ny, nz, scatter=True)
        N = st["n_fluid"]
        starts = np.asarray(st["starts"], np.int64)
        adj = st["adj"].reshape(N, 18).astype(np.int64)
        rng = [(N * p // world, N * (p + 1) // world) for p in range(world)]
        wp = 1.0 / TAU
        wm = port.omega_minus(wp)

        def owner(n, d, e):  # entry_owner
            s0 = starts[d]
            return e - s0 if s0 <= e < s0 + N else n

        def slot_node(e):
            dd = max(d for d in range(Q) if e >= starts[d])
            return e - starts[dd], dd

        def part_of(m):
            return next(p for p, (a, b) in enumerate(rng) if a <= m < b)

        links = {}  # (r, s) -> sorted global slots
        for r in range(world):
            a, b = rng[r]
            for n in range(a, b):
                for d in range(1, Q):
                    e = int(adj[n, d - 1])
                    s = part_of(owner(n, d, e))
                    if s != r:
                        links.setdefault((r, s), set()).add(e)
        links = {k: sorted(v) for k, v in links.items()}
        n0, n1 = rng[rank]
        nloc = n1 - n0
        gofs, ghosts = {}, []
        for (r, s), sl in sorted(links.items()):
            if r == rank:
                gofs[s] = len(ghosts)
                ghosts += sl

        def local(e, n):
            mm, dd = slot_node(e)
            if n0 <= mm < n1:
                return dd * nloc + (mm - n0)
            s = part_of(mm)
            return Q * nloc + gofs[s] + links[(rank, s)].index(e)

        ladj = np.array([[local(int(adj[n, d - 1]), n) for d in range(1, Q)]
                         for n in range(n0, n1)], np.int64).reshape(nloc, 18)
        init = port.perturbed(N, 55)
        gbuf = np.zeros(int(st["total_slots"]))
        for n in range(N):
            for d in range(Q):
                gbuf[starts[d] + n] = init[n * Q + d]
        buf = np.zeros(Q * nloc + len(ghosts))
        for j in range(nloc):
            for d in range(Q):
                buf[d * nloc + j] = gbuf[starts[d] + n0 + j]
        buf[Q * nloc:] = gbuf[np.asarray(ghosts, np.int64)] if ghosts else 0
        sidx = {k: [slot_node(e)[1] * nloc + (slot_node(e)[0] - n0) for e in sl]
                for k, sl in links.items() if k[1] == rank}

        def exchange(phase):
            reqs = []
            for i, ((r, s), sl) in enumerate(sorted(links.items())):
                if phase == 0 and s == rank:
                    t = torch.from_numpy(buf[np.asarray(sidx[(r, s)])].copy())
                    reqs.append(("s", dist.isend(t, r, tag=i), None, None))
                if phase == 0 and r == rank:
                    t = torch.empty(len(sl), dtype=torch.float64)
                    reqs.append(("r", dist.irecv(t, s, tag=i), t, Q * nloc + gofs[s]))
                if phase == 1 and r == rank:
                    g0 = Q * nloc + gofs[s]
                    t = torch.from_numpy(buf[g0:g0 + len(sl)].copy())
                    reqs.append(("s", dist.isend(t, s, tag=i), None, None))
                if phase == 1 and s == rank:
                    t = torch.empty(len(sl), dtype=torch.float64)
                    reqs.append(("r", dist.irecv(t, r, tag=i), t, ("scatter", (r, s))))
            for kind_, rq, t, where in reqs:
                rq.wait()
                if kind_ == "r":
                    if isinstance(where, tuple):
                        buf[np.asarray(sidx[where[1]])] = t.numpy()
                    else:
                        buf[where:where + len(t)] = t.numpy()

        for _ in range(steps // 2):
            for j in range(nloc):  # even: own slots -> opposite slots
                f = np.array([buf[d * nloc + j] for d in range(Q)])
                f = port.collide(f, wp, wm, G)
                for d in range(Q):
                    buf[OPP[d] * nloc + j] = f[d]
            exchange(0)
            for j in range(nloc):  # odd: gather column opp(d), scatter column d
                f = np.empty(Q)
                f[0] = buf[j]
                for d in range(1, Q):
                    f[d] = buf[ladj[j, OPP[d] - 1]]
                f = port.collide(f, wp, wm, G)
                buf[j] = f[0]
                for d in range(1, Q):
                    buf[ladj[j, d - 1]] = f[d]
            exchange(1)
        rows = {n0 + j: [buf[d * nloc + j] for d in range(Q)] for j in range(nloc)}
        out = [None] * world
        dist.all_gather_object(out, rows)
        if rank == 0:
            full = np.zeros(N * Q)
            for part in out:
                for kk, v in part.items():
                    full[kk * Q:(kk + 1) * Q] = v
            expect, _ = port.run("half", kind, nx, ny, nz, steps, wp, g=G, init=init)
            q.put((bool(np.array_equal(full, expect)), float(port.max_rel_diff(full, expect))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,dims", [("channel", (6, 5, 8)), ("blocks", (8, 8, 8))])
def test_two_rank_list_node_range_protocol_gloo(kind, dims):
    """list-aa-soa node-range decomposition with local numbering on 2 gloo
    ranks (blocks: the x wrap makes both part boundaries active), bitwise
    equal to the oracle's full-domain half-way stepper."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_rank_main_list, args=(r, 2, port_no, kind, dims, 4, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    equal, rel = q.get(timeout=5)
    assert equal, rel


def _rank_main_peer(rank, world, kind, dims, steps, shared, flags, q):
    """The peer-memory transport's protocol (direct_peer.cuh, DirectEngine::
    aa_pair_peer) with real concurrency: every slab lives in shared memory
    (the stand-in for CUDA-IPC-mapped peer memory), the boundary planes' odd
    sub-step gathers from and scatters into the NEIGHBOUR's slab directly,
    and the only synchronisation is the epoch flags written into the
    neighbour's flag row (signal) and spun on in one's own (wait).  Random
    delays between the stages shuffle the interleavings; the result must
    equal the full-domain oracle bit for bit."""
    import random
    import time
    from oracle.oracle import Port
    port = Port()
    rng = random.Random(1000 + rank)
    nx, ny, nz = dims
    flags_g, per, nf = port.geometry(kind, nx, ny, nz)
    solid = flags_g.reshape(nx, ny, nz)
    zr = [nz * r // world for r in range(world + 1)]
    z0, z1 = zr[rank], zr[rank + 1]
    nzl = z1 - z0
    ring = bool(solid[:, :, 0].min() == 0 or solid[:, :, nz - 1].min() == 0)
    lo = rank - 1 if rank > 0 else (world - 1 if ring else -1)
    hi = rank + 1 if rank + 1 < world else (0 if ring else -1)
    bufs = [t.numpy() for t in shared]   # every slab: (nzl_r + 2, Q, ny, nx)
    fl = flags.numpy()                   # (world, 4): even from lo / hi, odd from lo / hi
    buf = bufs[rank]
    wp = 1.0 / TAU
    wm = port.omega_minus(wp)
    own = [(x, y, z) for z in range(nzl) for y in range(ny) for x in range(nx)
           if not solid[x, y, z + z0]]
    boundary = [n for n in own if n[2] == 0 or n[2] == nzl - 1]
    interior = [n for n in own if 0 < n[2] < nzl - 1]

    def at(zs):  # storage plane zs of this slab -> (array, plane), peer planes resolved
        if zs == 0 and lo >= 0:
            return bufs[lo], zr[lo + 1] - zr[lo]        # lower neighbour's top own plane
        if zs == nzl + 1 and hi >= 0:
            return bufs[hi], 1                          # upper neighbour's bottom own plane
        return buf, zs

    def even(nodes):
        for (x, y, z) in nodes:
            zs = z + 1
            f = np.array([buf[zs, SLOT[d], y, x] for d in range(Q)])
            f = port.collide(f, wp, wm, G)
            for d in range(Q):
                buf[zs, SLOT[OPP[d]], y, x] = f[d]

    def odd(nodes):
        for (x, y, z) in nodes:
            zs = z + 1
            f = np.empty(Q)
            for d in range(Q):
                a, p = at(zs - CZ[d])
                f[d] = a[p, SLOT[OPP[d]], (y - CY[d]) % ny, (x - CX[d]) % nx]
            f = port.collide(f, wp, wm, G)
            for d in range(Q):  # scatter written independently of the gather address
                a, p = at(zs + CZ[d])
                a[p, SLOT[d], (y + CY[d]) % ny, (x + CX[d]) % nx] = f[d]

    def signal(kind_, e):
        if lo >= 0:
            fl[lo, 2 * kind_ + 1] = e   # I am the lower neighbour's upper neighbour
        if hi >= 0:
            fl[hi, 2 * kind_] = e

    def wait(kind_, e):
        t0 = time.time()
        for j, nb in ((2 * kind_, lo), (2 * kind_ + 1, hi)):
            while nb >= 0 and fl[rank, j] < e:
                assert time.time() - t0 < 120, "peer wait timed out"
                time.sleep(0.0005)

    def jitter():
        time.sleep(rng.random() * 0.01)

    for e in range(1, steps // 2 + 1):
        jitter(); even(boundary); signal(0, e)
        jitter(); even(interior); wait(0, e)
        jitter(); odd(boundary); signal(1, e)
        jitter(); odd(interior); wait(1, e)
    q.put(rank)


@pytest.mark.parametrize("kind,dims,world", [("channel", (6, 5, 8), 2), ("blocks", (8, 8, 8), 2),
                                             ("blocks", (8, 8, 9), 3), ("channel", (5, 4, 6), 3)])
def test_peer_transport_protocol_shared_memory(kind, dims, world):
    import torch
    from oracle.oracle import Port
    port = Port()
    nx, ny, nz = dims
    flags_g, per, nf = port.geometry(kind, nx, ny, nz)
    solid = flags_g.reshape(nx, ny, nz)
    init = port.perturbed(nf, 91)
    zr = [nz * r // world for r in range(world + 1)]
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    shared = []
    for r in range(world):
        b = np.empty((zr[r + 1] - zr[r] + 2, Q, ny, nx))
        for d in range(Q):
            b[:, SLOT[d]] = w[d]
        shared.append(b)
    k = 0
    for x in range(nx):
        for y in range(ny):
            for z in range(nz):
                if solid[x, y, z]:
                    continue
                r = max(i for i in range(world) if zr[i] <= z)
                for d in range(Q):
                    shared[r][z - zr[r] + 1, SLOT[d], y, x] = init[k * Q + d]
                k += 1
    shared = [torch.from_numpy(b).share_memory_() for b in shared]
    flags = torch.zeros((world, 4), dtype=torch.int64).share_memory_()
    steps = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main_peer,
                         args=(r, world, kind, dims, steps, shared, flags, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    full = np.zeros(nf * Q)
    k = 0
    for x in range(nx):
        for y in range(ny):
            for z in range(nz):
                if solid[x, y, z]:
                    continue
                r = max(i for i in range(world) if zr[i] <= z)
                full[k * Q:(k + 1) * Q] = [shared[r][z - zr[r] + 1, SLOT[d], y, x].item()
                                           for d in range(Q)]
                k += 1
    expect, _ = port.run("full", kind, nx, ny, nz, steps, 1.0 / TAU, g=G, init=init)
    assert np.array_equal(full, expect), port.max_rel_diff(full, expect)


def _rank_main_peer_one_step(rank, world, kind, dims, steps, push, shared, flags, q):
    """The one-step peer protocol (DirectEngine::os_sweeps_peer) run
    concurrently: every op (the pull's collide pass, each sweep) is
    wait(neighbours' op e-1) -> op(boundary planes) -> signal(e) ->
    op(interior planes); pull boundary nodes gather from the neighbour's
    source grid, push boundary nodes store into the neighbour's destination
    grid (slot by the target's global solid flag).  Slabs in shared memory,
    random delays, flags as the only synchronisation."""
    import random
    import time
    from oracle.oracle import Port
    port = Port()
    rng = random.Random(2000 + rank)
    nx, ny, nz = dims
    flags_g, per, nf = port.geometry(kind, nx, ny, nz)
    solid = flags_g.reshape(nx, ny, nz).astype(bool)
    zr = [nz * r // world for r in range(world + 1)]
    z0, z1 = zr[rank], zr[rank + 1]
    nzl = z1 - z0
    lo, hi = (rank - 1) % world, (rank + 1) % world  # one-step plans always carry the ring
    bufs = [[t.numpy() for t in pair] for pair in shared]  # [slab][grid]: (nzl_r + 2, Q, ny, nx)
    fl = flags.numpy()
    wp = 1.0 / TAU
    wm = port.omega_minus(wp)
    nodes = [(x, y, z) for z in range(nzl) for y in range(ny) for x in range(nx)]
    boundary = [n for n in nodes if n[2] == 0 or n[2] == nzl - 1]
    interior = [n for n in nodes if 0 < n[2] < nzl - 1]

    def at(g, zs):  # storage plane of this slab's grid g -> (array, plane); ghosts -> peer
        if zs == 0:
            return bufs[lo][g], zr[lo + 1] - zr[lo]
        if zs == nzl + 1:
            return bufs[hi][g], 1
        return bufs[rank][g], zs

    def signal(e):
        fl[lo, 1] = e   # I am the lower neighbour's upper neighbour
        fl[hi, 0] = e

    def wait(e):
        t0 = time.time()
        for j in (0, 1):
            while fl[rank, j] < e:
                assert time.time() - t0 < 120, "peer wait timed out"
                time.sleep(0.0005)

    def op(e, fn):
        wait(e - 1)
        time.sleep(rng.random() * 0.01)
        fn(boundary)
        signal(e)
        time.sleep(rng.random() * 0.01)
        fn(interior)

    cur = 0
    e = 0
    if not push:
        def coll(ns):
            b = bufs[rank][0]
            for (x, y, z) in ns:
                if not solid[x, y, z + z0]:
                    f = np.array([b[z + 1, SLOT[d], y, x] for d in range(Q)])
                    f = port.collide(f, wp, wm, G)
                    for d in range(Q):
                        b[z + 1, SLOT[d], y, x] = f[d]
        e += 1
        op(e, coll)
    for s in range(steps):
        src, dst = cur, 1 - cur

        def sweep(ns):
            for (x, y, z) in ns:
                zs = z + 1
                if push:
                    b = bufs[rank][src]
                    f = np.array([b[zs, SLOT[d], y, x] for d in range(Q)])
                    if not solid[x, y, z + z0]:
                        f = port.collide(f, wp, wm, G)
                    bufs[rank][dst][zs, SLOT[0], y, x] = f[0]
                    for d in range(1, Q):
                        tx, ty = (x + CX[d]) % nx, (y + CY[d]) % ny
                        tzg = (z + z0 + CZ[d]) % nz
                        a, p = at(dst, zs + CZ[d])
                        a[p, SLOT[OPP[d]] if solid[tx, ty, tzg] else SLOT[d], ty, tx] = f[d]
                else:
                    f = np.empty(Q)
                    f[0] = bufs[rank][src][zs, SLOT[0], y, x]
                    for d in range(1, Q):
                        a, p = at(src, zs - CZ[d])
                        f[d] = a[p, SLOT[d], (y - CY[d]) % ny, (x - CX[d]) % nx]
                    sol = solid[x, y, z + z0]
                    if s + 1 < steps and not sol:
                        f = port.collide(f, wp, wm, G)
                    b = bufs[rank][dst]
                    b[zs, SLOT[0], y, x] = f[0]
                    for d in range(1, Q):
                        b[zs, SLOT[OPP[d]] if sol else SLOT[d], y, x] = f[d]
        e += 1
        op(e, sweep)
        cur ^= 1
    wait(e)
    q.put((rank, cur))


@pytest.mark.parametrize("push", [True, False])
@pytest.mark.parametrize("kind,dims,world", [("channel", (6, 5, 8), 2), ("blocks", (8, 8, 9), 3)])
def test_peer_transport_one_step_protocol_shared_memory(kind, dims, world, push):
    import torch
    from oracle.oracle import Port
    port = Port()
    nx, ny, nz = dims
    flags_g, per, nf = port.geometry(kind, nx, ny, nz)
    solid = flags_g.reshape(nx, ny, nz)
    init = port.perturbed(nf, 92)
    zr = [nz * r // world for r in range(world + 1)]
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    shared = []
    for r in range(world):
        pair = []
        for g in range(2):
            b = np.empty((zr[r + 1] - zr[r] + 2, Q, ny, nx))
            for d in range(Q):
                b[:, SLOT[d]] = w[d]
            pair.append(b)
        shared.append(pair)
    k = 0
    for x in range(nx):
        for y in range(ny):
            for z in range(nz):
                if solid[x, y, z]:
                    continue
                r = max(i for i in range(world) if zr[i] <= z)
                for d in range(Q):
                    shared[r][0][z - zr[r] + 1, SLOT[d], y, x] = init[k * Q + d]
                k += 1
    shared = [[torch.from_numpy(b).share_memory_() for b in pair] for pair in shared]
    flags = torch.zeros((world, 2), dtype=torch.int64).share_memory_()
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main_peer_one_step,
                         args=(r, world, kind, dims, steps, push, shared, flags, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    cur = q.get(timeout=5)[1]
    full = np.zeros(nf * Q)
    mass = 0.0
    k = 0
    for x in range(nx):
        for y in range(ny):
            for z in range(nz):
                r = max(i for i in range(world) if zr[i] <= z)
                vals = [shared[r][cur][z - zr[r] + 1, SLOT[d], y, x].item() for d in range(Q)]
                if not solid[x, y, z]:
                    full[k * Q:(k + 1) * Q] = vals
                    k += 1
    mass = float(sum(shared[r][cur][1:-1].sum().item() for r in range(world)))
    expect, emass = port.run("full", kind, nx, ny, nz, steps, 1.0 / TAU, g=G, init=init)
    assert np.array_equal(full, expect), port.max_rel_diff(full, expect)
    assert abs(mass - emass) <= 1e-12 * abs(emass)
