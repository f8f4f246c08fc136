"""bench.py — MG-preconditioned SQMR Stokes solve on B200 (BASELINE.json metric).

One "step" = one full MG-SQMR solve of the BASELINE config to its tolerance
(cfg 1 by default: 128^3 cube, 5-level V-cycle, iid U[-1,1] forcing seed 1,
tol 1e-6).  Metric: DOF/s = N * iterations / T_solve, plus
time-to-1e-6 (ms_per_step) and the HBM roofline of the dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1]

--impl reference times the CPU implementation of the path (the oracle port —
the reference ships no solver) on the host cores.
Under torchrun (N > 1) every rank solves its own copy of the config (replicas,
weak scaling; the z-slab decomposition is future work) and the
max over ranks of the device time is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (nx, ny, nz, h, levels, forcing kind, seed, tol, name)
    0: (32, 32, 32, 1 / 32, 3, 0, 0, 1e-6, "cfg0: 32^3 cube, 3-level V, U[-1,1] seed 0, tol 1e-6"),
    1: (128, 128, 128, 1 / 128, 5, 0, 1, 1e-6, "cfg1: 128^3 cube, 5-level V, U[-1,1] seed 1, tol 1e-6"),
    2: (256, 256, 256, 1 / 256, 6, 1, 2, 1e-6, "cfg2: 256^3 cube, 6-level V, 8 Fourier modes seed 2, tol 1e-6"),
    3: (512, 512, 512, 1 / 512, 7, 0, 3, 1e-6, "cfg3: 512^3 cube, 7-level V, U[-1,1] seed 3, tol 1e-6"),
    4: (1024, 256, 256, 1 / 256, 7, 2, 4, 1e-8, "cfg4: 1024x256x256 channel, 7-level V, 1+U[-.1,.1] seed 4, tol 1e-8"),
}


def ndof(nx, ny, nz):
    return (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1) + nx * ny * nz


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=ws)
    return ws, rank, local


def allmax(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_sample(cfg, threads, iters=2):
    """Oracle port on host cores: `iters` MG-SQMR iterations of the config (bounded sample)."""
    import oracle

    nx, ny, nz, h, lv, kind, seed, tol, _ = CONFIGS[cfg]
    oracle.set_threads(threads)
    o = oracle.Oracle(nx, ny, nz, h=h, levels=lv)
    b = oracle.forcing_box(nx, ny, nz, h, kind, seed)
    t0 = time.perf_counter()
    _, hist, _, _ = o.sqmr(b, tol=1e-300, maxit=iters)
    dt = time.perf_counter() - t0
    return o, b, len(hist), dt


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cfg = args.config
    nx, ny, nz, h, lv, kind, seed, tol, name = CONFIGS[cfg]
    n = ndof(nx, ny, nz)
    threads = os.cpu_count() or 1
    import oracle

    oracle.set_threads(threads)
    o = oracle.Oracle(nx, ny, nz, h=h, levels=lv)
    b = oracle.forcing_box(nx, ny, nz, h, kind, seed)
    iters = args.ref_iters
    for _ in range(args.warmup):
        o.sqmr(b, tol=1e-300, maxit=1)
    t0 = time.perf_counter()
    tot_it = 0
    for _ in range(args.steps):
        _, hist, _, _ = o.sqmr(b, tol=1e-300, maxit=iters)
        tot_it += len(hist)
    dt = time.perf_counter() - t0
    val = n * tot_it / dt
    line = {
        "impl": "reference", "metric": "MG-SQMR DOF/s (N x iterations / T_solve)", "value": val, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "N_dof": n, "sample": f"{iters} SQMR iterations per step"},
        "cpu_baseline": {"value": val, "unit": "DOF/s", "cores": threads, "kind": "port",
                         "sample": f"{iters} MG-SQMR iterations of {name} per step, oracle/stokes_oracle.cpp"},
        "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import paper_2312_10615_b200 as smg

    cfg = args.config
    nx, ny, nz, h, lv, kind, seed, tol, name = CONFIGS[cfg]
    n = ndof(nx, ny, nz)
    s = smg.Solver(nx, ny, nz, h=h, levels=lv, device=local)
    # host input in pinned memory (e2e path) and the same b resident in HBM
    bpin = smg.PinnedArray(n)
    smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed, out=bpin.array)
    xpin = smg.PinnedArray(n)
    s.set_rhs(bpin.array)
    for _ in range(args.warmup):
        s.solve_resident(tol, 500)
    # ---- device-resident timed region ----
    barrier(ws)
    dev_ms, iters, launches = 0.0, 0, 0
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hist, st = s.solve_resident(tol, 500)
            t = s.timing()
            dev_ms += t["solve_ms"]
            iters += t["iterations"]
            launches += t["kernel_launches"]
        wall = time.perf_counter() - t0
    barrier(ws)
    dev_ms = allmax(dev_ms, ws)
    value = ws * n * iters / (dev_ms / 1e3)
    # ---- end-to-end through the C-ABI with host buffers ----
    barrier(ws)
    t0 = time.perf_counter()
    e2e_it = 0
    for _ in range(args.steps):
        x, hh, _, st = s.sqmr(bpin.array, tol, 500, out=xpin.array)
        e2e_it += len(hh)
    e2e_s = allmax(time.perf_counter() - t0, ws)
    e2e_val = ws * n * e2e_it / e2e_s
    # ---- roofline of the dominant kernel (symmetric DGS sweep on the fine level) ----
    peak, peak_kind = measured_peak_gbs()
    roof = roofline(s, n, nx, ny, nz, peak, peak_kind)
    out = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            th = os.cpu_count() or 1
            _, _, it, dt = cpu_sample(cfg, th, args.ref_iters)
            cpu = {"value": n * it / dt, "unit": "DOF/s", "cores": th, "kind": "port",
                   "sample": f"{it} MG-SQMR iterations of {name}, oracle/stokes_oracle.cpp, {dt:.1f} s"}
        out = {
            "metric": "MG-SQMR DOF/s (N x iterations / T_solve)", "value": value, "unit": "DOF/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "N_dof": n, "iterations_per_solve": iters / args.steps,
                       "time_to_tol_ms": dev_ms / args.steps, "parallelism": "replicas" if ws > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (fine-level vectors 73 MB each, 7 live)"},
            "e2e": {"value": e2e_val, "unit": "DOF/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": 1e3 * e2e_s / args.steps},
            "roofline": roof,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "wall_s_timed": wall,
        }
        print(json.dumps(out), flush=True)
    s.close()
    return out


def roofline(s, n, nx, ny, nz, peak, peak_kind):
    """Fine-level symmetric DGS sweep (the largest V-cycle cost)."""
    reps = 5
    ms = s.time_kernel(2, reps, 0)
    # algorithmic bytes of one symmetric DGS sweep: every one of
    # the 20 phases reads the 7 fields it needs once and writes the updated one:
    # velocity phase: read u,v,w,p,bu,bv,bw (7 fields) + write u,v,w (3);
    # pressure fwd phase: read u,v,w,p,bp (5) + write u,v,w,p (4);
    # pressure rev phase: read u,v,w,p,bu,bv,bw,bp (8) + write p (1).
    cells = nx * ny * nz
    fields = 4 * (7 + 3) + 8 * (5 + 4) + 8 * (8 + 1)
    alg_bytes = fields * 8 * cells
    achieved = alg_bytes / (ms / 1e3) / 1e9
    apply_ms = s.time_kernel(0, 20, 0)
    return {"bound": "hbm", "kernel": "symmetric DGS sweep (20 phases), fine level", "achieved": achieved,
            "peak": peak, "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "algorithmic_bytes_per_launch": alg_bytes, "avg_ms": ms,
            "apply_L": {"avg_ms": apply_ms, "achieved_gbs": 16 * n / (apply_ms / 1e3) / 1e9}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--ref-iters", type=int, default=2, help="SQMR iterations per CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
