"""Multi-rank host logic of the element-partitioned SEM path, on CPU with the
gloo backend (world_size 2, 4 and 8; at 8 every rank holds one element layer, Ezl = 1).  Each rank builds its z-slab maps through the
C-ABI host entry points; the ranks exchange them with torch.distributed and
check that (1) every canonical unknown is owned by exactly one (rank, slot),
(2) the input-face halo a rank receives (the top c=N-1 owned layer of the rank
below) is exactly the set of nodes its first element layer gathers at k=0, and
(3) the bottom-face contributions a rank sends down land on nodes the rank
below owns in its top layer -- the NCCL exchange pattern of csrc/sem.cpp."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N, EX, EY, EZ = 3, 3, 2, 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _canon(gx, gy, gz):
    Mx, My, Mz = N * EX - 1, N * EY - 1, N * EZ - 1
    if not (1 <= gx <= Mx and 1 <= gy <= My and 1 <= gz <= Mz):
        return -1
    return ((gz - 1) * My + (gy - 1)) * Mx + (gx - 1)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_03179_b200 import sem

        d = sem.SemDesc(N, EX, EY, EZ, rank=rank, nranks=world)
        z0, z1 = d.partition()
        smap = sem.slot_map(d)
        owned = smap[smap >= 0]
        # (1) ownership: gather all owned canonical indices
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([owned.size]))
        mx = int(max(s.item() for s in sizes))
        buf = torch.full((mx,), -1, dtype=torch.int64)
        buf[: owned.size] = torch.from_numpy(owned)
        allb = [torch.empty(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, buf)
        ok1 = True
        if rank == 0:
            allm = np.concatenate([b.numpy()[b.numpy() >= 0] for b in allb])
            n = (N * EX - 1) * (N * EY - 1) * (N * EZ - 1)
            ok1 = allm.size == n and np.array_equal(np.sort(allm), np.arange(n))
        # (2) halo: what I send up = canonical ids of my top-layer c=N-1 slots (pack order ex,ey,a,b)
        Lz = z1 - z0
        send = []
        for ey in range(EY):
            for ex in range(EX):
                e = ex + EX * (ey + EY * (Lz - 1))
                for b in range(N):
                    for a in range(N):
                        send.append(smap[e * sem.slots_per_element(N) + sem.slot_pos(N, a, b, N - 1)])
        send = torch.tensor(send, dtype=torch.int64)
        recv = torch.empty_like(send)
        ops = []
        if rank + 1 < world:
            ops.append(dist.P2POp(dist.isend, send, rank + 1))
        if rank > 0:
            ops.append(dist.P2POp(dist.irecv, recv, rank - 1))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        ok2 = True
        if rank > 0:
            # what my k=0 gather of layer 0 needs, in the kernel's halo index (ex', ey', a, b)
            need = np.full(EX * EY * N * N, -2, dtype=np.int64)
            gz = z0 * N
            for ey in range(EY):
                for ex in range(EX):
                    for j in range(N + 1):
                        for i in range(N + 1):
                            gx, gy = ex * N + i, ey * N + j
                            c = _canon(gx, gy, gz)
                            if c < 0:
                                continue
                            oex, ax = (gx - 1) // N, (gx - 1) % N
                            oey, ay = (gy - 1) // N, (gy - 1) % N
                            need[(oex + EX * oey) * N * N + ax + N * ay] = c
            got = recv.numpy()
            sel = need >= 0
            ok2 = np.array_equal(got[sel], need[sel])
        # (3) contributions I send down (k=0 face of my layer 0, index (ex, ey, i, j)) are owned by rank-1's top layer
        ok3 = True
        if rank > 0:
            lower = sem.SemDesc(N, EX, EY, EZ, rank=rank - 1, nranks=world)
            lm = sem.slot_map(lower)
            lz0, lz1 = lower.partition()
            top = lm[(EX * EY * (lz1 - lz0 - 1)) * sem.slots_per_element(N):]
            top_ids = set(top[top >= 0])
            for ey in range(EY):
                for ex in range(EX):
                    for j in range(N + 1):
                        for i in range(N + 1):
                            c = _canon(ex * N + i, ey * N + j, z0 * N)
                            if c >= 0 and c not in top_ids:
                                ok3 = False
        res = torch.tensor([int(ok1), int(ok2), int(ok3)])
        dist.all_reduce(res, op=dist.ReduceOp.MIN)
        if rank == 0:
            q.put(res.tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_slab_partition_halo_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) == [1, 1, 1]
