"""bench.py — MG-preconditioned SQMR Stokes solve on B200 (BASELINE.json metric).

One "step" = one full MG-SQMR solve of the BASELINE config to its tolerance
(cfg 2 by default -- the config the metric's 1/2/4/8-GPU series is quoted on:
256^3 cube, 6-level V-cycle, 8 Fourier modes seed 2, tol 1e-6).  Metric: DOF/s =
N * iterations / T_solve, plus time-to-1e-6 (ms_per_step) and
the HBM roofline of the dominant kernel.  By default the line also carries a
device-resident cfg-3 (512^3) measurement under "also".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

--impl reference times the CPU implementation of the path (the oracle port --
the reference ships no solver) on the host cores.

CPU numbers (cpu_baseline and the reference arm) time the oracle on a bounded
sample: the Alg. 4 setup (lines 1-4, one V-cycle) and two SQMR iterations,
separately, then report DOF/s for the config's whole solve, N * K / (t_init + K
t_iter), with K the iteration count of the committed golden history -- the
same quantity the GPU line reports.
Under torchrun (N > 1) every rank builds its own z-slab of the same config on
its GPU (smg_create_rank: one process per GPU, halo planes by
NCCL send/recv after every smoother phase, inner-product plane partials by one
NCCL all-reduce, coarse levels replicated) and the max over ranks of the device
time is reported (strong scaling).  --replicas runs N independent copies
instead; SMG_EMULATE_SLABS=1 puts all slabs in rank 0's process on device 0.
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
    """nvidia-smi clocks / throttle reasons streamed every 50 ms (`-lms 50`) while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._proc = None
        self._t = None

    def _reader(self):
        for line in self._proc.stdout:
            v = [x.strip() for x in line.strip().split(",")]
            if len(v) >= 7:
                self.samples.append(v)

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                           "--format=csv,noheader,nounits", "-lms", "50"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.15)  # let the first samples arrive before the timed region
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *a):
        if self._proc is not None:
            time.sleep(0.06)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        if self._t:
            self._t.join(timeout=5)

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
    if os.environ.get("SMG_BENCH_ONE_GPU"):  # tests: every rank on cuda:0 (with the NCCL stand-in, tests/fake_nccl)
        local = 0
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


def share_nccl_id(ws, rank):
    """Rank 0's NCCL unique id (smg_nccl_unique_id), broadcast over the launcher's gloo group."""
    import paper_2312_10615_b200 as smg

    if ws == 1:
        return smg.nccl_unique_id()
    import torch.distributed as dist

    obj = [smg.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def golden_iterations(cfg):
    """Iterations to tolerance of the committed oracle history (tests/golden), else None."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", f"cfg{cfg}_history.json")) as f:
            g = json.load(f)
        return int(g["iterations"]) if g.get("status") == 0 else None
    except (OSError, ValueError, KeyError):
        return None


def cpu_sample(cfg, threads, iters=2, oracle_obj=None):
    """Oracle port on `threads` host cores, bounded sample of the config: Alg. 4 lines 1-4 (the
    initial V-cycle) and `iters` SQMR iterations, timed apart (the per-iteration time excludes
    the setup).  Returns (t_init, t_iter, iterations sampled, wall seconds)."""
    import oracle

    nx, ny, nz, h, lv, kind, seed, tol, _ = CONFIGS[cfg]
    oracle.set_threads(threads)
    o = oracle_obj or oracle.Oracle(nx, ny, nz, h=h, levels=lv)
    b = oracle.forcing_box(nx, ny, nz, h, kind, seed)
    t0 = time.perf_counter()
    _, hist, secs, _ = o.sqmr(b, tol=1e-300, maxit=iters + 1)
    dt = time.perf_counter() - t0
    k = len(hist)
    t_it = (secs[-1] - secs[0]) / max(k - 1, 1)  # iterations 2..k: no setup inside
    t_init = max(secs[0] - t_it, 0.0)
    return t_init, t_it, k - 1, dt


def cpu_dofs(cfg, t_init, t_it, k_solve):
    nx, ny, nz = CONFIGS[cfg][:3]
    return ndof(nx, ny, nz) * k_solve / (t_init + k_solve * t_it)


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
    k_solve = golden_iterations(cfg) or 10
    for _ in range(args.warmup):
        cpu_sample(cfg, threads, 1, o)
    t_init = t_it = wall = 0.0
    # bounded sample per step: a step is ~9 s of CPU work per timed iteration at cfg 2, so long runs
    # (the driver's --steps 20) time one iteration per step and the whole arm stays within a few minutes
    ref_iters = args.ref_iters if args.steps <= 6 else 1
    for _ in range(args.steps):
        ti, tt, _, dt = cpu_sample(cfg, threads, ref_iters, o)
        t_init += ti / args.steps
        t_it += tt / args.steps
        wall += dt
    val = cpu_dofs(cfg, t_init, t_it, k_solve)
    sample = (f"per step: Alg. 4 setup (1 V-cycle) + {ref_iters} MG-SQMR iterations of {name}, timed apart; "
              f"value = N K / (t_setup + K t_iter) with K = {k_solve} (committed golden), "
              f"oracle/stokes_oracle.cpp on {threads} threads, {cpu_model()}")
    line = {
        "impl": "reference", "metric": "MG-SQMR DOF/s (N x iterations / T_solve)", "value": val, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "N_dof": n, "sample": sample, "t_setup_s": t_init, "t_iter_s": t_it,
                   "iterations_per_solve": k_solve, "time_to_tol_ms": 1e3 * (t_init + k_solve * t_it)},
        "cpu_baseline": {"value": val, "unit": "DOF/s", "cores": threads, "kind": "port", "cpu": cpu_model(),
                         "sample": sample},
        "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import paper_2312_10615_b200 as smg

    cfg = args.config
    nx, ny, nz, h, lv, kind, seed, tol, name = CONFIGS[cfg]
    n = ndof(nx, ny, nz)
    slabs = ws > 1 and not args.replicas
    emulate = slabs and os.environ.get("SMG_EMULATE_SLABS")  # 1-GPU box: rank 0 holds all slabs on device 0
    if emulate and rank != 0:
        barrier(ws)  # mirror rank 0's collective sequence: B, B, max, B, max
        barrier(ws)
        allmax(0.0, ws)
        barrier(ws)
        allmax(0.0, ws)
        return None
    if emulate:
        s = smg.Solver(nx, ny, nz, h=h, levels=lv, devices=[0] * ws)
    elif slabs:  # one process per GPU: this rank's z-slab, NCCL halos / reductions (smg_create_rank)
        s = smg.Solver.for_rank(rank, ws, share_nccl_id(ws, rank), nx, ny, nz, h=h, levels=lv, device=local)
    else:
        s = smg.Solver(nx, ny, nz, h=h, levels=lv, device=local)
    wsum = 1 if slabs else ws  # problem copies solved (replicas) -> aggregate DOF/s
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
    statuses = []
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            hist, st = s.solve_resident(tol, 500)
            statuses.append(st)
            t = s.timing()
            dev_ms += t["solve_ms"]
            iters += t["iterations"]
            launches += t["kernel_launches"]
        wall = time.perf_counter() - t0
    barrier(ws)
    dev_ms = allmax(dev_ms, ws)
    value = wsum * n * iters / (dev_ms / 1e3)
    # ---- end-to-end through the C-ABI with host buffers ----
    barrier(ws)
    t0 = time.perf_counter()
    e2e_it = 0
    for _ in range(args.steps):
        x, hh, _, st = s.sqmr(bpin.array, tol, 500, out=xpin.array)
        e2e_it += len(hh)
    e2e_s = allmax(time.perf_counter() - t0, ws)
    e2e_val = wsum * n * e2e_it / e2e_s
    # ---- roofline of the dominant component (fine-level smooth) + whole iteration ----
    peak, peak_kind = measured_peak_gbs()
    roof = roofline(s, lv, peak, peak_kind, dev_ms / max(iters, 1), f"cfg{args.config}",
                    share=1.0 / ws if slabs and not emulate else 1.0)
    out = None
    also = {}
    if ws == 1 and args.also:
        for c in [int(v) for v in args.also.split(",") if v.strip()]:
            if c != args.config:
                also[f"cfg{c}"] = measure_resident(smg, c, 2)
        if not args.no_labelled:
            also["labelled_cylinder"] = measure_labelled(smg, 2)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            th = os.cpu_count() or 1
            k_solve = iters / args.steps
            ti, tt, it, dt = cpu_sample(cfg, th, args.ref_iters)
            cpu = {"value": cpu_dofs(cfg, ti, tt, k_solve), "unit": "DOF/s", "cores": th, "kind": "port",
                   "cpu": cpu_model(),
                   "sample": f"Alg. 4 setup + {it} MG-SQMR iterations of {name} timed apart "
                             f"(setup {ti:.2f} s, {tt:.2f} s/iteration), extrapolated to this solve's "
                             f"{k_solve:g} iterations; oracle/stokes_oracle.cpp, {dt:.1f} s wall",
                   "t_setup_s": ti, "t_iter_s": tt}
            if args.cpu_1thread:  # single-thread reference point on the smaller cfg 1 (DOF/s ~ size-independent)
                ti1, tt1, it1, dt1 = cpu_sample(1, 1, 1)
                k1 = golden_iterations(1) or 8
                cpu["single_thread"] = {"value": cpu_dofs(1, ti1, tt1, k1), "unit": "DOF/s", "cores": 1,
                                        "sample": f"cfg 1 (128^3): setup {ti1:.1f} s + {it1} iteration(s) at "
                                                  f"{tt1:.1f} s, extrapolated to {k1} iterations; {dt1:.0f} s wall"}
        out = {
            "metric": "MG-SQMR DOF/s (N x iterations / T_solve)", "value": value, "unit": "DOF/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if slabs else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "N_dof": n, "iterations_per_solve": iters / args.steps,
                       "time_to_tol_ms": dev_ms / args.steps,
                       "converged": all(v == smg.SMG_CONVERGED for v in statuses),
                       "final_rel_residual": float(hist[-1]) if len(hist) else None, "tol": tol,
                       "parallelism": (f"z-slab x{ws}" if slabs else f"replicas x{ws}") if ws > 1 else "1 GPU",
                       "l2": l2_note(s)},
            "e2e": {"value": e2e_val, "unit": "DOF/s", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": 1e3 * e2e_s / args.steps},
            "roofline": roof,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "wall_s_timed": wall,
            "also": also,
        }
        print(json.dumps(out), flush=True)
    s.close()
    return out


def measure_resident(smg, cfg, steps, warmup=1):
    """Device-resident solves of another config (CUDA-event time per solve, max over steps)."""
    nx, ny, nz, h, lv, kind, seed, tol, name = CONFIGS[cfg]
    n = ndof(nx, ny, nz)
    try:
        s = smg.Solver(nx, ny, nz, h=h, levels=lv)
    except Exception as e:  # e.g. not enough device memory
        return {"workload": name, "error": str(e)}
    b = smg.forcing(nx, ny, nz, h=h, kind=kind, seed=seed)
    s.set_rhs(b)
    for _ in range(warmup):
        s.solve_resident(tol, 500)
    ms, its, hist, st = [], [], None, None
    for _ in range(steps):
        hist, st = s.solve_resident(tol, 500)
        t = s.timing()
        ms.append(t["solve_ms"])
        its.append(t["iterations"])
    s.close()
    tot_ms = sum(ms)
    return {"workload": name, "N_dof": n, "value": n * sum(its) / (tot_ms / 1e3), "unit": "DOF/s",
            "ms_per_solve": tot_ms / steps, "iterations_per_solve": sum(its) / steps, "converged": st == 0,
            "final_rel_residual": float(hist[-1]) if len(hist) else None, "steps": steps, "warmup": warmup}


def measure_labelled(smg, steps, warmup=1):
    """General labelled domain: the cylinder channel of PAPER section 6.2.2 at
    256 x 128 x 128 cells (Dirichlet cylinder, Exterior outflow column), 5 levels, channel forcing
    seed 4, tol 1e-6 -- device-resident solves through the labelled-domain kernels."""
    from paper_2312_10615_b200 import scenarios
    nx, ny, nz, lv, tol = 256, 128, 128, 5, 1e-6
    name = f"cylinder3d {nx}x{ny}x{nz}, {lv}-level V, channel forcing seed 4, tol {tol:g}"
    lab = scenarios.cylinder3d(nx, ny, nz)
    try:
        s = smg.Solver.from_labels(lab, h=1.0 / ny, levels=lv)
    except Exception as e:
        return {"workload": name, "error": str(e)}
    s.set_rhs(smg.forcing_labels(lab, 1.0 / ny, smg.FORCE_CHANNEL, 4))
    n = s.ndof(0)
    for _ in range(warmup):
        s.solve_resident(tol, 500)
    ms, its, hist, st = [], [], None, None
    for _ in range(steps):
        hist, st = s.solve_resident(tol, 500)
        t = s.timing()
        ms.append(t["solve_ms"])
        its.append(t["iterations"])
    s.close()
    tot_ms = sum(ms)
    return {"workload": name, "N_dof": n, "value": n * sum(its) / (tot_ms / 1e3), "unit": "DOF/s",
            "ms_per_solve": tot_ms / steps, "iterations_per_solve": sum(its) / steps, "converged": st == 0,
            "final_rel_residual": float(hist[-1]) if len(hist) else None, "steps": steps, "warmup": warmup}


def l2_note(s):
    """Fine-level vector size against the device L2 (inputs larger than L2, or not)."""
    vec = 8 * s.ndof()
    l2 = None
    try:
        import torch

        l2 = torch.cuda.get_device_properties(0).L2_cache_size
    except Exception:
        pass
    if not l2:
        l2 = 126 << 20
    live = 8  # x, b, r of the fine level + q, d, x_sqmr, rhs + the Vanka ping-pong copy
    rel = "larger than" if vec > l2 else "smaller than"
    return (f"fine-level vectors {vec / 1e6:.0f} MB each ({live} live, {live * vec / 1e9:.2f} GB), each "
            f"{rel} L2 ({l2 / 2**20:.0f} MiB); no explicit flush")


def level_counts(s, levels):
    out = []
    for l in range(levels):
        c = s.counts(l)
        n = c["nu"] + c["nv"] + c["nw"] + c["np"]
        out.append((n, c["V1"], n - c["V1"]))
    return out


def b_iter_model(cnt, nu=1):
    """Algorithmic bytes of one SQMR iteration, SURVEY §8(d):
    136 N0 + sum_{l<L-1} [2 (48 N_l^V2 + 96 nu N_l^V1) + 24 N_l + (8 N_l + 8 N_l+1) + (16 N_l + 8 N_l+1)]
    + 8 Nc^2 + 16 Nc."""
    b = 136 * cnt[0][0]
    for l in range(len(cnt) - 1):
        n, v1, v2 = cnt[l]
        nc = cnt[l + 1][0]
        b += 2 * (48 * v2 + 96 * nu * v1) + 24 * n + (8 * n + 8 * nc) + (16 * n + 8 * nc)
    nc = cnt[-1][0]
    return b + 8 * nc * nc + 16 * nc


def roofline(s, levels, peak, peak_kind, iter_ms, config_key=None, share=1.0):
    """Dominant kernel: the fine-level symmetric DGS sweep (~40% of the cfg-2 iteration) -- on a tiled
    level 16 launches of k_dgs_tile (8 tile colours forward, 8 reverse) after one k_dgs_cb, else 13
    per-step kernels.  Algorithmic bytes per SURVEY 8(d): 48 B per V2 DOF per symmetric sweep;
    `achieved` = those bytes / the sweep's CUDA-event time (the same ratio as bytes per launch / average
    launch duration).  Components: the whole smooth (Alg. 3, 48 B per V2 DOF + 96 nu B per V1 DOF),
    the Vanka sweep, apply L, and the whole iteration against B_iter."""
    cnt = level_counts(s, levels)
    n0, v1, v2 = cnt[0]
    if share != 1.0:  # one rank of a z-slab run: its kernels cover its share of the fine level
        v1, v2, n0 = v1 * share, v2 * share, n0 * share
    reps = 5
    # As the V-cycle runs them: the m^T b pass k_dgs_cb (on a tiled level it also writes the tile-major
    # copy of b the tiles stage from) runs ONCE per level visit and serves the visit's two smooths, so
    # a sweep / a smooth carries half of it.
    cb_ms = s.time_kernel(12, reps, 0)
    smooth_ms = s.time_kernel(14, reps, 0) + cb_ms / 2
    dgs_ms = s.time_kernel(13, reps, 0) + cb_ms / 2
    vanka_ms = s.time_kernel(4, reps, 0)
    apply_ms = s.time_kernel(0, 20, 0)
    alg_smooth = 48 * v2 + 96 * v1
    alg = 48 * v2
    achieved = alg / (dgs_ms / 1e3) / 1e9
    biter = b_iter_model(cnt)
    tiled = s.dgs_tiled(0) if hasattr(s, "dgs_tiled") else False
    # measured DRAM bytes from the committed ncu launch list of one fine-level smooth
    # (`tools/profile_kernel.py --which 5 --level 0` -> profiles/smooth_traffic.json)
    traffic = smooth_traffic = None
    tpath = os.path.join(ROOT, "profiles", "smooth_traffic.json")
    if os.path.exists(tpath):
        rec = json.load(open(tpath)).get(config_key)
        if rec:
            smooth_traffic = rec["dram_bytes"]
            div = rec.get("component_launches_in_range", 1)
            # half of k_dgs_cb: the pass serves the two smooths of a level visit (as in avg_ms)
            dgs = [v["dram_bytes"] * (0.5 if "k_dgs_cb" in k else 1.0)
                   for k, v in rec["per_kernel_in_range"].items() if "k_dgs_" in k]
            traffic = sum(dgs) / div if dgs else None
    nl = 16.5 if tiled else 13.5  # launches per sweep: the step kernels + half a k_dgs_cb
    return {
        "bound": "hbm",
        "kernel": ("k_dgs_tile: fine-level symmetric DGS sweep in tile order (16 TMA-staged launches + half of the level visit's k_dgs_cb)"
                   if tiled else "fine-level symmetric DGS sweep (13 per-step kernels + half of the level visit's k_dgs_cb)"),
        "achieved": achieved, "peak": peak, "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic,
        "traffic_source": "ncu dram__bytes_read+write of the sweep's kernels (cold caches), profiles/smooth_traffic.json",
        "algorithmic_bytes_per_launch": alg / nl, "avg_launch_ms": dgs_ms / nl, "launches_per_sweep": nl,
        "algorithmic_bytes_per_sweep": alg, "avg_ms": dgs_ms, "k_dgs_cb_ms_per_level_visit": cb_ms,
        "units": {"N_V2": v2, "N_V1": v1, "bytes_per_V2_dof": 48, "bytes_per_V1_dof": 96},
        "components": {
            "smooth_alg3": {"avg_ms": smooth_ms, "alg_bytes": alg_smooth,
                            "achieved_gbs": alg_smooth / (smooth_ms / 1e3) / 1e9,
                            "frac": alg_smooth / (smooth_ms / 1e3) / 1e9 / peak, "traffic": smooth_traffic},
            "vanka_sym_sweep": {"avg_ms": vanka_ms, "alg_bytes": 48 * v1,
                                "achieved_gbs": 48 * v1 / (vanka_ms / 1e3) / 1e9,
                                "note": "V1 shell: sector-bound gathers, 8 dependent phases per sweep"},
            "apply_L": {"avg_ms": apply_ms, "alg_bytes": 16 * n0, "achieved_gbs": 16 * n0 / (apply_ms / 1e3) / 1e9},
        },
        "iteration": {"alg_bytes": biter, "ms": iter_ms, "achieved_gbs": biter / (iter_ms / 1e3) / 1e9,
                      "frac": biter / (iter_ms / 1e3) / 1e9 / (peak / share), "model": "SURVEY 8(d) B_iter",
                      "peak_gbs_all_gpus": peak / share},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--no-labelled", action="store_true", help="skip the labelled-domain (cylinder channel) line "
                                                               "reported under also.labelled_cylinder")
    ap.add_argument("--also", default="3", help="comma list of extra configs measured device-resident "
                                                "(2 solves each) and reported under 'also'; '' for none")
    ap.add_argument("--cpu-1thread", action="store_true", help="add a single-thread CPU reference point")
    ap.add_argument("--ref-iters", type=int, default=2, help="SQMR iterations per CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent copies instead of z-slabs")
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
