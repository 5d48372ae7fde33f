import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench as B
from paper_2106_07575_b200 import inputs as I, _lib as L
for name in ("small", "paper"):
    w = I.WORKLOADS[name]
    dev = torch.device("cuda", 0)
    psi_true, p, scan, d = B.synth_device(w, dev)
    pt = L.Ptyger(torch.ones((w.H, w.W), dtype=torch.complex64, device=dev), torch.from_numpy(p.astype(np.complex64)).to(dev), scan, d)
    tr = pt.iterate(40)
    sh = [t["shrinks"] for t in tr]
    prev = None; extra = 0
    for k in sh:
        keff = 16 if prev is None else min(max(prev + 3, 4), 16)
        if k >= keff: extra += 1
        prev = k
    print(name, sh, "extra passes:", extra)
    pt.close(); del d; torch.cuda.empty_cache()
