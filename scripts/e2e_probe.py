"""Where does the end-to-end (init + 1 iteration + get_object) time go at the paper config?"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench as B
from paper_2106_07575_b200 import inputs as I, _lib as L
w = I.WORKLOADS["paper"]
dev = torch.device("cuda", 0)
psi_true, p, scan, d = B.synth_device(w, dev)
d_host = d.cpu().pin_memory()
psi_h = torch.ones((w.H, w.W), dtype=torch.complex64).pin_memory()
p_h = torch.from_numpy(p.astype(np.complex64)).pin_memory()
obj_pin = torch.empty((w.H, w.W), dtype=torch.complex64).pin_memory().numpy()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dd = d_host.to(dev, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter()
    q = L.Ptyger(psi_h, p_h, scan, d_host, config=L.default_config(device=0))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    q.iterate(1, traces=False); torch.cuda.synchronize(); t3 = time.perf_counter()
    out = q.get_object(obj_pin); t4 = time.perf_counter()
    q.close(); torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"rep {rep}: raw H2D of d {1e3*(t1-t0):.1f} ms ({d_host.numel()*4/(t1-t0)/1e9:.1f} GB/s); init {1e3*(t2-t1):.1f} ms; "
          f"iterate(1) {1e3*(t3-t2):.1f} ms; get_object {1e3*(t4-t3):.1f} ms; close {1e3*(t5-t4):.1f} ms")
    del dd
