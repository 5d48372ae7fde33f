#!/usr/bin/env python
"""Benchmark: diffraction frames/sec per CG iteration (BASELINE.json metric) through libptyger.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config paper] [--impl ours|reference]

One "step" = one CG iteration of the whole hot path (GRAD -> DIR -> LS -> Update, all SURVEY
8(a) rows) over every frame of the workload.  Default workload: the paper-scale view
(4096^2 object, 128^2 detector, 158^2 = 24 964 frames), the config BASELINE.json quotes the
metric on at 1/2/4/8 B200; it fits one GPU.  Synthetic data (DESIGN.md input recipe): Siemens
star, Gaussian chirped probe, jittered raster, d = Poisson(1e3 |G psi_true|^2) generated on the
device with torch.fft (data synthesis only; the timed path is libptyger's kernels).

Multi-GPU (torchrun, one rank per GPU): the frames are partitioned into row stripes by the
library (strong scaling: the total workload is fixed), with an NCCL band exchange + scalar
allreduces per iteration.  Timing: CUDA events on the library's stream around the graph
launches, barrier + synchronize on both sides, max over ranks.  u, v, d (8.2 GB at
paper-scale) exceed the 126 MB L2, so no explicit flush is needed between iterations.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2106_07575_b200 import inputs as I  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "diffraction frames/sec per CG iteration"
UNIT = "frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="paper", choices=["tiny", "small", "paper", "mid", "large", "view3d", "l256p"])
    ap.add_argument("--views", type=int, default=0, help="view3d: number of views (default: all 64)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ls-batch", type=int, default=16)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="world > 1: peer-memory windows (CUDA IPC) or NCCL for the per-iteration exchanges")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-large", action="store_true",
                    help="skip the large-view sub-record (8192^2, 256^2, 99 856 frames) of the paper-config run")
    ap.add_argument("--large-steps", type=int, default=10)
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def frames_config(w: I.Workload, args, world: int) -> dict:
    """The JSON line's config for a single-view workload (both arms print the same one)."""
    n, N = w.n, w.N
    return {"workload": f"{w.name}: {w.H}x{w.W} object, {N}^2 probe/detector, {n} frames "
                        f"({w.k}^2 raster, step {w.step}, jitter {w.jitter}), photons {w.photons:g}, Poisson",
            "H": w.H, "W": w.W, "N": N, "frames": n, "ls_batch": args.ls_batch,
            "parallelism": f"stripes{world}",
            "transport": args.transport if world > 1 else None,
            "l2": "inputs larger than L2 (u, v, d resident in HBM: %.1f GB)" % (n * N * N * 20 / 1e9)}


def views_config(w: I.Workload, args, world: int) -> dict:
    """The JSON line's config for the 3-D view batch (both arms print the same one)."""
    nviews = args.views or w.views
    return {"workload": f"{w.name}: {nviews} views x {w.H}^2 object, {w.N}^2 detector, {w.n} frames "
                        "per view, views sharded over ranks (no communication)",
            "views": nviews, "frames": nviews * w.n, "parallelism": f"views{world}",
            "l2": "inputs larger than L2"}


def host_cpu() -> dict:
    """the CPU model and the cores available to this process (the oracle uses one)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        avail = len(os.sched_getaffinity(0))
    except AttributeError:
        avail = os.cpu_count()
    return {"cpu_model": model, "cores_available": avail}


def sm_max_mhz() -> float:
    """Max SM clock for the nominal FP32 peak: MEASURED_PEAKS.json, else the B200 boost clock."""
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return 1965.0


def lower_bound(N: int, n: int, H: int, W: int, ms_per_step: float, hbm_gbs: float, sm_mhz: float, world: int = 1,
                fp32_tflops: float | None = None):
    """SURVEY 8(d) 'report three numbers', item 3: t_min / t_measured.  t_min = min over the cache
    designs of max(HBM bytes / measured HBM bandwidth, flops / nominal FP32 peak) per frame and CG
    iteration.  Bytes per frame pixel: S (u, v cached) 64, H (u only) 24, R (nothing) 8, plus 80 B
    per object pixel; flops: 5 N^2 log2(N^2) per 2-D FFT (2 / 3 / 4 FFTs) + 124 elementwise flops per
    pixel at K = 8.  FP32 peak: MEASURED on the box (ptyger_fp32_peak, paired FFMA2, the
    form the frame kernels use) when given, else the nominal 148 SMs x 128 lanes x 2 flop x SM clock."""
    px = float(N * N)
    fft = 5.0 * px * math.log2(px)
    obj = 80.0 * H * W / n
    fp32 = fp32_tflops * 1e12 if fp32_tflops else 148 * 128 * 2 * sm_mhz * 1e6   # per GPU
    bw = hbm_gbs * 1e9
    per = {}
    for name, bpx, nfft in (("S", 64.0, 2), ("H", 24.0, 3), ("R", 8.0, 4)):
        b = bpx * px + obj
        f = nfft * fft + 124.0 * px
        per[name] = {"bytes": b, "flop": f, "ns_hbm": b / bw * 1e9, "ns_fp32": f / fp32 * 1e9,
                     "ns": max(b / bw, f / fp32) * 1e9}
    best = min(per, key=lambda k: per[k]["ns"])
    t_meas = ms_per_step * 1e6 * world / n      # ns per frame per GPU
    return {"t_min_ns_per_frame": per[best]["ns"], "design": best, "t_measured_ns_per_frame": t_meas,
            "ratio": per[best]["ns"] / t_meas, "fp32_tflops": fp32 / 1e12,
            "fp32_kind": "measured (paired FFMA2)" if fp32_tflops else "nominal", "hbm_gbs": hbm_gbs,
            "design_S_ns_per_frame": per["S"]["ns"], "per_design": per}


# ----------------------------------------------------------------------------- data

def synth_device(w: I.Workload, device, view: int | None = None):
    """psi_true, probe, scan on the host (inputs module); d on the device via torch.fft."""
    import torch
    psi_true, p, scan = I.workload_inputs(w) if view is None else I.view_inputs(w, view)
    pt = torch.from_numpy(p.astype(np.complex64)).to(device)
    ot = torch.from_numpy(psi_true.astype(np.complex64)).to(device)
    N = w.N
    d = torch.empty((len(scan), N, N), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(w.seed + (view or 0))
    rr = torch.arange(N, device=device)
    chunk = 1024
    sc = torch.from_numpy(scan.astype(np.int64)).to(device)
    for a in range(0, len(scan), chunk):
        b = min(len(scan), a + chunk)
        r = sc[a:b, 0][:, None, None] + rr[None, :, None]
        c = sc[a:b, 1][:, None, None] + rr[None, None, :]
        patch = ot[r, c] * pt[None]
        far = torch.fft.fft2(patch, norm="ortho")
        mean = w.photons * (far.real ** 2 + far.imag ** 2)
        d[a:b] = torch.poisson(mean, generator=g)
    return psi_true, p, scan, d


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML every 2 ms in a thread
    (nvidia-smi -lms 100 as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.proc = None
        self.thread = None
        self.stop_flag = False
        self.nvml = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (nv, h)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def poll():
                while not self.stop_flag:
                    try:
                        self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                             int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def rd():
            for line in self.proc.stdout:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 7 or not f[0].replace(".", "").isdigit():
                    continue
                mask = 0
                for i, nm in enumerate(names):
                    if f[3 + i].lower().startswith("active"):
                        mask |= self.REASONS[nm]
                self.samples.append((float(f[0]), mask))
                if f[1].replace(".", "").isdigit():
                    self.max_mhz = float(f[1])
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self):
        self.stop_flag = True
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(1.0)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no clock samples"], "samples": 0}
        reasons = sorted({nm for _, m in self.samples for nm, bit in self.REASONS.items() if m & bit})
        return {"sm_mhz": float(np.median([c for c, _ in self.samples])), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self.nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------- CPU oracle

def oracle_sample_run(w: I.Workload, budget_s: float, psi_true, p, scan, d_host_fn, subset: int | None = None,
                      workers: int = 1):
    """Oracle (float64 NumPy; FFTs by pocketfft on 1 thread, or scipy.fft on `workers` threads) on a
    bounded sample of the workload: the first n_s frames in raster order with the object cropped to
    their rows; one CG iteration (definition-based LS).  n_s grows until one iteration takes
    about a third of the budget, or is fixed to `subset`.  Returns (frames/s, description, shrinks, s)."""
    from oracle import ptycho as O
    N = w.N
    n_s = subset or 8
    O.set_fft_workers(workers)
    try:
        while True:
            sc = scan[:n_s].copy()
            r0 = int(sc[:, 0].min())
            r1 = int(sc[:, 0].max()) + N
            sub = sc.copy()
            sub[:, 0] -= r0
            d = d_host_fn(n_s).astype(np.float64)
            psi0 = np.ones((r1 - r0, w.W), np.complex128)
            t0 = time.perf_counter()
            st, tr, _, _ = O.cg_iterate(O.CGState(psi=psi0), p.astype(np.complex128), sub, d)
            t_one = time.perf_counter() - t0
            if subset or t_one >= budget_s / 3 or n_s >= len(scan):
                break
            n_s = min(len(scan), int(n_s * max(2.0, min(8.0, (budget_s / 3) / max(t_one, 1e-3)))))
    finally:
        O.set_fft_workers(1)
    fft = "pocketfft, 1 thread" if workers == 1 else f"scipy.fft, {workers} threads"
    desc = (f"oracle float64 NumPy ({fft}): 1 CG iteration with definition-based line search on the first "
            f"{n_s} of {len(scan)} frames (rows {r0}..{r1} of the {w.name} workload{', a fixed subset' if subset else ''}), "
            f"{tr.shrinks} shrinks; frames/s = {n_s} / {t_one:.2f} s")
    return n_s / t_one, desc, tr.shrinks, t_one


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_baselines(w, budget_s, psi_true, p, scan, d_head, subset=None, variants=("numpy", "scipy")):
    """SURVEY 8(d) CPU baselines on the GPU box's host: the oracle as-is (pocketfft, 1 thread) and with
    scipy.fft on all available cores.  The primary value is the multi-core one (cores = its threads)."""
    nc = host_cores()
    res = {}
    for var in variants:
        wk = 1 if var == "numpy" else nc
        v, desc, shr, t_one = oracle_sample_run(w, budget_s, psi_true, p, scan, lambda k: d_head[:k],
                                                subset=subset, workers=wk)
        res[var] = {"value": v, "unit": UNIT, "cores": wk, "kind": "oracle", "sample": desc}
    prim = res.get("scipy") or res["numpy"]
    out = dict(prim)
    out["variants"] = res
    out["host"] = host_cpu()
    return out


# ----------------------------------------------------------------------------- main

def stage_ms(trs) -> dict:
    """Per-stage device ms of the timed iterations (ptyger_trace ms_* fields: GPU timestamps between
    the stages of the graph-launched iteration), mean over the iterations."""
    keys = ["ms_grad", "ms_dir", "ms_ls", "ms_update", "ms_comm"]
    return {k[3:]: float(np.mean([t[k] for t in trs])) for k in keys} if trs else None


def max_over_ranks(vals, world, coll_dev):
    if world == 1:
        return vals
    import torch
    import torch.distributed as dist
    tt = torch.tensor(vals, dtype=torch.float64, device=coll_dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return [float(x) for x in tt.tolist()]


def time_frames(args, w, world, rank, local, dev, coll_dev, steps, warmup, with_e2e):
    """One single-view workload on this rank: init from device-resident data, `warmup` untimed then
    `steps` timed CG iterations (CUDA events on the library stream, barrier + synchronize on both
    sides, max over ranks), the frame kernels' own device timers, optional e2e leg.  Returns the
    JSON fields (rank 0 prints them) and what the CPU baseline needs."""
    import torch
    import torch.distributed as dist
    from paper_2106_07575_b200 import _lib as L
    psi_true, p, scan, d = synth_device(w, dev)
    n = len(scan)
    cfg = L.default_config(ls_batch=args.ls_batch, device=local, rank=rank, world=world,
                           transport=L.TRANSPORT_P2P if args.transport == "p2p" else L.TRANSPORT_NCCL)
    idbuf = None
    if world > 1 and args.transport == "nccl":
        obj = [L.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        import ctypes
        idbuf = ctypes.create_string_buffer(obj[0], 128)
        cfg.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    psi0 = torch.ones((w.H, w.W), dtype=torch.complex64, device=dev)
    pdev = torch.from_numpy(p.astype(np.complex64)).to(dev)
    pt = L.Ptyger(psi0, pdev, scan, d, config=cfg)
    del psi0
    if world > 1 and args.transport == "p2p":
        handles = [None] * world
        dist.all_gather_object(handles, pt.ipc_handle())
        pt.ipc_connect(handles)
    d_head = d[:min(n, 4096)].cpu().numpy() if rank == 0 else None   # CPU-baseline sample data
    if not with_e2e:
        del d
        torch.cuda.empty_cache()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    pt.iterate(warmup, traces=False)
    barrier()
    pt.kernel_times(reset=True)
    clk = ClockSampler(local)
    clk.start()
    t_host0 = time.perf_counter()
    trs = pt.iterate(steps)
    ms = pt.last_iterate_ms()
    t_host = time.perf_counter() - t_host0
    barrier()
    clocks = clk.stop()
    # per-launch durations of the two frame kernels over the timed region, measured on the GPU by
    # the kernels themselves (global ns timer; graph launches on the library stream)
    ktimes = pt.kernel_times(reset=True)
    launches = pt.kernel_launches()
    kt = {k: (v[0] / v[1] if v[1] else float("nan")) for k, v in ktimes.items()}
    ms, kt_grad, kt_ls = max_over_ranks([ms, kt["k_grad"], kt["k_ls"]], world, coll_dev)
    kt = {"k_grad": kt_grad, "k_ls": kt_ls}
    shrinks = [t["shrinks"] for t in trs]
    value = n * steps / (ms / 1e3)
    N = w.N
    n_local_bytes_grad = 36.0 * n * N * N / world      # u r/w 16, v r 8, d r 4, y w 8
    n_local_bytes_ls = 20.0 * n * N * N / world + 8.0 * w.H * w.W / world  # v w, u r, d r + eta once
    pk, pk_kind = peaks()
    cand = {"k_grad": (kt["k_grad"], n_local_bytes_grad), "k_ls": (kt["k_ls"], n_local_bytes_ls)}
    # + 92 B per object pixel: DY reads, eta, eta gather, update, and the object-grid LS moments (psi, I)
    it_bytes = (64.0 * n * N * N + 92.0 * w.H * w.W) / world
    dom = max(cand, key=lambda k: cand[k][0])
    dur_ms, algo_bytes = cand[dom]
    achieved = algo_bytes / (dur_ms / 1e3) / 1e9
    # the kernel that actually runs for this role at this N (default paths; the env toggles of
    # DESIGN.md 7 select the single-group LS kernels)
    if dom == "k_ls":
        if N == 256:
            kname = "k_ls_c256" if os.environ.get("PTYGER_C256_WS") == "0" else "k_ls_c256ws"
            if kname == "k_ls_c256ws" and os.environ.get("PTYGER_C256_SIDE", "110") != "0":
                # + the side kernel on the SMs the four-CTA clusters leave idle (one launch span)
                kname = "k_ls_c256ws+k_ls256_side"
        elif N == 128:
            kname = "k_ls" if os.environ.get("PTYGER_LS_WS") == "0" else "k_ls_ws"
        else:
            kname = "k_ls"
    else:
        kname = "k_grad256" if N == 256 else "k_grad"
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_json):
        try:
            with open(prof_json) as f:
                traffic = json.load(f).get(w.name, {}).get(kname)
        except Exception:
            traffic = None

    # end-to-end through the public API from pinned HOST buffers (H2D + 1 iteration + D2H)
    e2e = None
    if with_e2e and d.numel() * 4 < 8e9 and (world == 1 or args.transport == "p2p"):
        # every rank passes the same full host arrays; the library uploads its stripe only
        d_host = d.cpu().pin_memory()
        psi_h = torch.ones((w.H, w.W), dtype=torch.complex64).pin_memory()
        p_h = torch.from_numpy(p.astype(np.complex64)).pin_memory()
        pt.close()
        del d
        torch.cuda.empty_cache()
        obj_pin = torch.empty((w.H, w.W), dtype=torch.complex64).pin_memory().numpy()
        torch.cuda.synchronize()
        t_list = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            q = L.Ptyger(psi_h, p_h, scan, d_host,
                         config=L.default_config(ls_batch=args.ls_batch, device=local, rank=rank, world=world,
                                                 transport=L.TRANSPORT_P2P))
            if world > 1:
                hs = [None] * world
                dist.all_gather_object(hs, q.ipc_handle())
                q.ipc_connect(hs)
            q.iterate(1, traces=False)
            out = q.get_object(obj_pin)      # collective when world > 1: every rank gets the object
            t_list.append(time.perf_counter() - t0)
            q.close()
        tm = max_over_ranks([float(np.median(t_list))], world, coll_dev)[0]
        e2e = {"value": n / tm, "unit": UNIT, "h2d_bytes_per_step": int(d_host.numel() * 4 + psi_h.numel() * 8
                                                                          + p_h.numel() * 8 + scan.size * 4),
               "d2h_bytes_per_step": int(out.nbytes), "steps": args.e2e_steps,
               "note": "ptyger_init from pinned host buffers (H2D of d, psi0, probe, scan; u0 = G psi0, F0) + 1 CG "
                       "iteration + ptyger_get_object (D2H), wall clock per step (max over ranks; per rank: the "
                       "same full host arrays, its stripe uploaded)"}
        del d_host
    else:
        pt.close()
    torch.cuda.empty_cache()
    fields = {
        "value": value, "ms_per_step": ms / steps,
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": pk, "peak_kind": pk_kind,
                     "unit": "GB/s", "frac": achieved / pk, "traffic": traffic,
                     "algorithmic_bytes_per_launch": algo_bytes, "avg_launch_ms": dur_ms,
                     "timing": "device globaltimer per launch, timed region (%d launches)" % ktimes[dom][1],
                     "k_grad_avg_ms": kt["k_grad"], "k_ls_avg_ms": kt["k_ls"]},
        # whole-iteration design-S roofline: 64 B per frame pixel (k_grad 36, k_ls 20,
        # k_adj 8) + 92 B per object pixel (DY reads, eta, eta gather, update, LS moments) per CG iteration
        "iteration_roofline": {"algorithmic_bytes": it_bytes, "achieved_GBps": it_bytes / (ms / steps) / 1e6,
                               "peak_GBps": pk, "frac": it_bytes / (ms / steps) / 1e6 / pk},
        "stage_ms": stage_ms(trs),
        "mean_shrinks": float(np.mean(shrinks)),
        "shrinks": [int(x) for x in shrinks],
        # LS passes over the cached far fields per timed iteration: [screened, exact] (1, 0 = all
        # decided in the pass fused into the LS frame kernel)
        "ls_passes": [[int(t["ls_passes"]), int(t["ls_exact_passes"])] for t in trs] if trs else None,
        "clocks": clocks,
        "gpu_launches": int(launches),
        "e2e": e2e,
        "host_wall_s": t_host,
    }
    return fields, (psi_true, p, scan, d_head)


def multi_evidence(args, w, world, rank, local, coll_dev):
    """world > 1: which device / PCI bus each rank ran on, its frames and stripe, peer access between
    neighbouring devices, and the band bytes each boundary exchanges per iteration."""
    import torch
    import torch.distributed as dist
    from paper_2106_07575_b200 import _lib as L
    props = torch.cuda.get_device_properties(local)
    mine = {"rank": rank, "device": local, "name": props.name,
            "pci_bus_id": getattr(props, "pci_bus_id", None), "local_rank": int(os.environ.get("LOCAL_RANK", "0"))}
    allr = [None] * world
    dist.all_gather_object(allr, mine)
    if rank != 0:
        return None
    psi_true, p, scan = I.workload_inputs(w)
    fr, rows = L.partition(scan, w.H, w.N, world)
    devs = [r["device"] for r in allr]
    for r in allr:
        r["frames"] = int(np.sum(fr == r["rank"]))
        r["own_rows"] = [int(rows[r["rank"], 0]), int(rows[r["rank"], 1])]
    bands = []
    for r in range(world - 1):
        lo, hi = int(rows[r + 1, 2]), int(rows[r, 3])
        bands.append({"ranks": [r, r + 1], "rows": max(0, hi - lo), "bytes_each_way": max(0, hi - lo) * w.W * 8})
    peer = [bool(torch.cuda.can_device_access_peer(devs[r], devs[r + 1])) if devs[r] != devs[r + 1] else None
            for r in range(world - 1)]
    return {"transport": args.transport, "ranks": allr, "distinct_devices": len(set(devs)),
            "peer_access_neighbours": peer, "band_exchange": bands,
            "scalars_per_iteration": "fp64 rank-ordered sums: 7 DY + ||eta||^2 + 20 per LS pass (+16 exact)",
            "nccl_debug": os.environ.get("NCCL_DEBUG")}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = I.WORKLOADS[args.config]

    if args.impl == "reference":
        return reference_arm(args, w, world, rank)

    if world > 1 and args.transport == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # INIT log: rings / NVLS / P2P channels used
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    import torch.distributed as dist
    from paper_2106_07575_b200 import _lib as L

    # one rank per GPU; more ranks than GPUs share them round-robin (functional runs only)
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # bench-level collectives (barrier, max over ranks, handle exchange) run on CPU tensors over gloo
    # with the peer-memory transport (NCCL is not needed at all), on NCCL otherwise
    coll_dev = dev if args.transport == "nccl" else torch.device("cpu")
    if world > 1:
        if args.transport == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        try:
            import nvidia  # type: ignore
            for pth in nvidia.__path__:
                cand = os.path.join(pth, "nccl", "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ.setdefault("PTYGER_NCCL_LIB", cand)
        except Exception:
            pass
    if w.views > 1:
        return run_views(args, w, world, rank, local, dev, coll_dev)
    fp32 = {"paired_ffma2_tflops": L.fp32_peak(local, True), "ffma_tflops": L.fp32_peak(local, False)}
    main_f, (psi_true, p, scan, d_head) = time_frames(args, w, world, rank, local, dev, coll_dev, args.steps,
                                                       args.warmup, args.e2e_steps > 0)
    large = None
    if args.config == "paper" and not args.no_large:
        # north_star's target view: 8192^2 object, 256^2 frames, 99 856 positions (~155 GB on 1 GPU)
        wl = I.WORKLOADS["large"]
        total = torch.cuda.get_device_properties(dev).total_memory
        if total * world >= 170e9:
            try:
                lf, (lpsi, lp, lscan, ld_head) = time_frames(args, wl, world, rank, local, dev, coll_dev,
                                                             args.large_steps, 3, False)
                large = {"config": frames_config(wl, args, world), "steps": args.large_steps, "warmup": 3,
                         "metric": METRIC, "unit": UNIT,
                         **{k: v for k, v in lf.items() if k not in ("e2e", "host_wall_s")}}
                large["lower_bound"] = lower_bound(wl.N, wl.n, wl.H, wl.W, lf["ms_per_step"], peaks()[0],
                                                   float(sm_max_mhz()), world, fp32["paired_ffma2_tflops"])
                if rank == 0 and world == 1 and not args.no_cpu_baseline:
                    large["cpu_baseline"] = oracle_baselines(wl, args.cpu_seconds, lpsi, lp, lscan, ld_head,
                                                             subset=1024, variants=("scipy",))
            except Exception as e:   # a failure here must not cost the main record
                large = {"error": f"{type(e).__name__}: {e}"[:300]}
        else:
            large = {"skipped": f"{total / 1e9:.0f} GB per GPU x {world} < 170 GB"}
    multi = multi_evidence(args, w, world, rank, local, coll_dev) if world > 1 else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = oracle_baselines(w, args.cpu_seconds, psi_true, p, scan, d_head)

    n = len(scan)
    line = {
        "metric": METRIC,
        "value": main_f["value"],
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": main_f["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": frames_config(w, args, world),
        **{k: main_f[k] for k in ("roofline", "iteration_roofline", "stage_ms")},
        "lower_bound": lower_bound(w.N, n, w.H, w.W, main_f["ms_per_step"], peaks()[0],
                                   float(sm_max_mhz()), world, fp32["paired_ffma2_tflops"]),
        "fp32_peak_measured": fp32,
        **{k: main_f[k] for k in ("mean_shrinks", "shrinks", "ls_passes", "clocks", "gpu_launches", "e2e")},
        "cpu_baseline": cpu,
        "large_view": large,
        "multi_gpu": multi,
        "host_wall_s": main_f["host_wall_s"],
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_views(args, w, world, rank, local, dev, coll_dev=None):
    """3-D ptycho-tomography batch (BASELINE config 5): independent views, sharded
    round-robin over the ranks with no communication; each view is its own libptyger context.
    One step = one CG iteration of every view."""
    import torch
    import torch.distributed as dist
    from paper_2106_07575_b200 import _lib as L
    nviews = args.views or w.views
    mine = [v for v in range(nviews) if v % world == rank]
    views = []
    for v in mine:
        _, p, scan, d = synth_device(w, dev, view=v)
        psi0 = torch.ones((w.H, w.W), dtype=torch.complex64, device=dev)
        views.append(L.Ptyger(psi0, torch.from_numpy(p.astype(np.complex64)).to(dev), scan, d,
                              config=L.default_config(ls_batch=args.ls_batch, device=local)))
        del d
    for q in views:
        q.launch(args.warmup)
    for q in views:
        q.wait(traces=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    # all views enqueued on their own streams before any is waited for (they overlap on the GPU);
    # device time of the batch = CUDA events: one start event every view stream waits on, one end
    # event per view stream, max over the views
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    ends = []
    for q in views:
        xs = torch.cuda.ExternalStream(q.stream(), device=dev)
        xs.wait_event(start)
        q.launch(args.steps)
        e = torch.cuda.Event(enable_timing=True)
        e.record(xs)
        ends.append(e)
    shr = []
    vtr = []
    for q in views:
        tq = q.wait()
        vtr.append(tq)
        shr += [t["shrinks"] for t in tq]
    torch.cuda.synchronize()
    ms = max(start.elapsed_time(e) for e in ends) if ends else 0.0
    clocks = clk.stop()
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=coll_dev if coll_dev is not None else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    launches = sum(q.kernel_launches() for q in views)
    kts = [q.kernel_times(reset=True) for q in views]
    frames = nviews * w.n
    if rank == 0:
        pk, pk_kind = peaks()
        algo = 36.0 * w.n * w.N * w.N
        kg = sum(k["k_grad"][0] for k in kts) / max(1, sum(k["k_grad"][1] for k in kts))
        line = {"metric": METRIC, "value": frames * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": views_config(w, args, world),
                "roofline": {"bound": "hbm", "kernel": "k_grad (per view)", "achieved": algo / (kg / 1e3) / 1e9,
                             "peak": pk, "peak_kind": pk_kind, "unit": "GB/s",
                             "frac": algo / (kg / 1e3) / 1e9 / pk, "traffic": None,
                             "timing": "device globaltimer per launch (views overlap on their streams)"},
                "stage_ms": stage_ms(vtr[0]) if vtr else None,
                "lower_bound": lower_bound(w.N, frames, w.H, w.W * nviews, ms / args.steps, pk,
                                           float(sm_max_mhz()), 1),
                "mean_shrinks": float(np.mean(shr)) if shr else None, "clocks": clocks,
                "gpu_launches": int(launches), "e2e": None, "cpu_baseline": None}
        print(json.dumps(line))
    for q in views:
        q.close()
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, w, world, rank):
    """--impl reference: the float64 oracle (the only reference this paper-tier run has) timed on
    the host cores on bounded samples of the same workload; rank 0 only."""
    if rank != 0:
        return
    psi_true, p, scan = I.workload_inputs(w)
    from oracle import ptycho as O

    def d_fn(k):
        mean = w.photons * np.abs(O.forward_G(psi_true, p, scan[:k])) ** 2
        return I.poisson_counts(mean, w.seed)
    per = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    vals = []
    desc = None
    nc = host_cores()
    for i in range(args.warmup + args.steps):
        v, desc, shr, t_one = oracle_sample_run(w, per, psi_true, p, scan, d_fn, workers=nc)
        if i >= args.warmup:
            vals.append(v)
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": views_config(w, args, world) if w.views > 1 else frames_config(w, args, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nc, "kind": "oracle", "sample": desc,
                             "host": host_cpu()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
