"""World-size-2/3 CPU test (gloo) of the multi-rank host logic: the library's partition
(ptyger_partition), the band rule used by the runtime (band with rank-1 = [ext_me.lo,
ext_{me-1}.hi), with rank+1 = [ext_{me+1}.lo, ext_me.hi)), and the exchange protocol
(send own band partial, receive the neighbour's, add) reproduce the single-worker gradient on
every rank's storage rows, and the allreduced partial objectives equal the global F
(P:493-503)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ptycho as O
        from oracle.partition import local_gradient
        from paper_2106_07575_b200 import _lib as L
        from paper_2106_07575_b200 import inputs as I

        w = I.WORKLOADS["mid"]
        H, N = 256, 32
        psi_true = I.make_object(I.siemens_star(H, H))
        p = I.make_probe(N)
        scan = I.make_scan(H, H, N, 15, 14, 2, 7)
        d = np.abs(O.forward_G(psi_true, p, scan)) ** 2 * 3.0
        psi = np.ones_like(psi_true) * (0.95 + 0.05j)
        frame_rank, rows = L.partition(scan, H, N, world)
        rows_t = [tuple(int(x) for x in r) for r in rows]
        st_lo, st_hi = rows_t[rank][4], rows_t[rank][5]
        gl = local_gradient(psi, p, scan, d, frame_rank, rows_t, rank)
        # band exchange, exactly the runtime's rule
        bands = []
        if rank > 0:
            lo, hi = rows_t[rank][2], rows_t[rank - 1][3]
            if hi > lo:
                bands.append((rank - 1, lo, hi))
        if rank + 1 < world:
            lo, hi = rows_t[rank + 1][2], rows_t[rank][3]
            if hi > lo:
                bands.append((rank + 1, lo, hi))
        recv = {}
        reqs = []
        for peer, lo, hi in bands:
            send = torch.from_numpy(np.ascontiguousarray(gl[lo - st_lo:hi - st_lo]))
            buf = torch.empty_like(send)
            reqs.append(dist.isend(send, peer))
            reqs.append(dist.irecv(buf, peer))
            recv[peer] = (lo, hi, buf)
        for r in reqs:
            r.wait()
        out = gl.copy()
        for peer, (lo, hi, buf) in recv.items():
            out[lo - st_lo:hi - st_lo] += buf.numpy()
        g, far = O.gradient(psi, p, scan, d)
        err = float(np.max(np.abs(out - g[st_lo:st_hi])) / np.max(np.abs(g)))
        mine = frame_rank == rank
        fpart = torch.tensor([O.objective_F(far[mine], d[mine])], dtype=torch.float64)
        dist.all_reduce(fpart)
        ferr = abs(float(fpart.item()) - O.objective_F(far, d)) / abs(O.objective_F(far, d))
        own = g[rows_t[rank][0]:rows_t[rank][1]]
        q.put((rank, err, ferr, float(np.sum(np.abs(own) ** 2)), len(bands)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_band_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    res.sort()
    assert all(r[1] < 1e-12 for r in res), res
    assert all(r[2] < 1e-12 for r in res), res
    assert sum(r[4] for r in res) == 2 * (world - 1)      # every boundary exchanged both ways
