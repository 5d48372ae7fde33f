"""Worker for tests/test_gpu_p2p_ranks.py: one rank of a world-P reconstruction over the peer-memory
transport (both ranks may share one GPU).  Usage: python tests/_p2p_rank.py <rank> <world> <dir>."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.p2p_fixture import fixture  # noqa: E402
from paper_2106_07575_b200 import _lib as L  # noqa: E402


def main():
    rank, world, d = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    psi0, p, scan, inten = fixture(world)
    psi0 = np.load(os.path.join(d, "psi0.npy"))   # warm start written by the test
    cfg = L.default_config(world=world, rank=rank, transport=L.TRANSPORT_P2P, device=0)
    pt = L.Ptyger(psi0, p, scan, inten, config=cfg)
    h = pt.ipc_handle()
    with open(os.path.join(d, f"h{rank}.tmp"), "wb") as f:
        f.write(h)
    os.replace(os.path.join(d, f"h{rank}.tmp"), os.path.join(d, f"h{rank}"))
    hs = []
    for r in range(world):
        path = os.path.join(d, f"h{r}")
        t0 = time.time()
        while not os.path.exists(path):
            if time.time() - t0 > 120:
                raise RuntimeError(f"rank {rank}: no handle from rank {r}")
            time.sleep(0.01)
        with open(path, "rb") as f:
            hs.append(f.read())
    pt.ipc_connect(hs)
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
