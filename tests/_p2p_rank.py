"""Worker for the multi-rank GPU tests: one rank of a world-P reconstruction.

    python tests/_p2p_rank.py <rank> <world> <dir> [transport p2p|nccl] [device]

transport p2p: peer-memory windows (CUDA IPC), handles exchanged through files in <dir>; ranks may
share one GPU.  transport nccl: rank 0 writes the NCCL unique id to <dir>; one GPU per rank.
device: CUDA ordinal of this rank (default 0)."""
import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.p2p_fixture import fixture  # noqa: E402
from paper_2106_07575_b200 import _lib as L  # noqa: E402


def wait_file(path, rank, what):
    t0 = time.time()
    while not os.path.exists(path):
        if time.time() - t0 > 120:
            raise RuntimeError(f"rank {rank}: no {what}")
        time.sleep(0.01)
    with open(path, "rb") as f:
        return f.read()


def put_file(path, data):
    with open(path + ".tmp", "wb") as f:
        f.write(data)
    os.replace(path + ".tmp", path)


def main():
    rank, world, d = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    transport = sys.argv[4] if len(sys.argv) > 4 else "p2p"
    device = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    psi0, p, scan, inten = fixture(world)
    psi0 = np.load(os.path.join(d, "psi0.npy"))   # warm start written by the test
    if transport == "nccl":
        try:
            import nvidia  # type: ignore
            for pth in nvidia.__path__:
                cand = os.path.join(pth, "nccl", "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ.setdefault("PTYGER_NCCL_LIB", cand)
        except Exception:
            pass
        if rank == 0:
            put_file(os.path.join(d, "ncclid"), L.nccl_unique_id())
        uid = wait_file(os.path.join(d, "ncclid"), rank, "NCCL id")
        idbuf = ctypes.create_string_buffer(uid, 128)
        cfg = L.default_config(world=world, rank=rank, transport=L.TRANSPORT_NCCL, device=device,
                               nccl_id=ctypes.cast(idbuf, ctypes.c_void_p))
        pt = L.Ptyger(psi0, p, scan, inten, config=cfg)
    else:
        cfg = L.default_config(world=world, rank=rank, transport=L.TRANSPORT_P2P, device=device)
        pt = L.Ptyger(psi0, p, scan, inten, config=cfg)
        put_file(os.path.join(d, f"h{rank}"), pt.ipc_handle())
        pt.ipc_connect([wait_file(os.path.join(d, f"h{r}"), rank, f"handle of rank {r}") for r in range(world)])
    tr1 = pt.iterate(1)
    g1 = pt.get_gradient()
    trs = tr1 + pt.iterate(3)
    obj = pt.get_object()
    np.savez(os.path.join(d, f"out{rank}.npz"), g1=g1, obj=obj, shrinks=np.array([t["shrinks"] for t in trs]),
             F=np.array([t["F"] for t in trs]), step=np.array([t["step_norm"] for t in trs]),
             alpha=np.array([complex(t["alpha_re"], t["alpha_im"]) for t in trs]))
    pt.close()


if __name__ == "__main__":
    main()
