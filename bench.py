#!/usr/bin/env python
"""bench.py -- LRBMS online time steps/s on one B200 (fp64), with roofline and CPU-oracle baselines.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C5]
A "step" is one pass of the whole hot path a1..a6 (mobility, assembly + projection, reduced solve,
reconstruction, fluxes + CFL step, upwind transport) over the workload BASELINE.json's metric is
quoted on at full size: C5 (128x128x64 cells, 2048 subdomains of 8x8x8, N = 32).
Multi-GPU: replicas only (BASELINE.json mandates one GPU, no collectives): every rank
runs its own C5 replica; value = total steps of all ranks / max-over-ranks device time.
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LRBMS online time steps/sec (1 B200, fp64) and achieved HBM GB/s vs roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--basis", default="pod",
                    help="local bases: pod = the paper's offline recipe (host, offline/recipe.py); poly")
    ap.add_argument("--reps", type=int, default=5, help="timed repetitions of the window (median reported)")
    ap.add_argument("--no-small", dest="small", action="store_false",
                    help="skip the C1-C4 us/step keys")
    ap.add_argument("--cpu-steps", type=int, default=3, help="oracle steps timed for cpu_baseline")
    ap.add_argument("--no-offline", dest="offline", action="store_false",
                    help="skip the GPU offline stage (NEXT-3) key")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--coarse-refresh", type=int, default=None)
    ap.add_argument("--rtol", type=float, default=None)
    ap.add_argument("--fine-steps", type=int, default=5,
                    help="steps timed in the fine-scale reference scheme (NEXT-2, Phi_E = I; 0 = skip)")
    ap.add_argument("--k1-steps", type=int, default=10,
                    help="steps of the k = 1 fine-space variant (NEXT-4) timed as an extra key (0 = skip)")
    ap.add_argument("--affine-steps", type=int, default=50,
                    help="steps timed in the paper's affine online variant (NEXT-1; 0 = skip)")
    return ap.parse_args()


def dist_setup(use_cuda):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import datetime
        dist.init_process_group("nccl" if use_cuda else "gloo", timeout=datetime.timedelta(minutes=30))
    return rank, local, world


def shared_scenario(config, basis, rank, world, device):
    """The workload's inputs on every rank.  The paper-recipe bases take ~100 s of host time on C5, so
    under torchrun rank 0 runs the recipe and broadcasts Phi (a shared INPUT, before any timed region;
    the data path has no collective); the seeded fields are generated on every rank."""
    from paper_1405_2810_b200 import inputs
    if world == 1 or basis != "pod":
        return inputs.make_scenario(config, basis=basis)
    import numpy as np
    import torch
    import torch.distributed as dist
    sc = inputs.make_scenario(config, basis="pod" if rank == 0 else "poly")
    t = torch.as_tensor(np.ascontiguousarray(sc.Phi), dtype=torch.float64, device=device)
    dist.broadcast(t, 0)
    sc.Phi = t.cpu().numpy()
    return sc


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1])); smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def stage_bytes(sc, iters_per_step):
    """Algorithmic DRAM/L2 bytes per STEP of each stage, C5: see DESIGN.md."""
    n, ns, N, nl, dim = sc.n, sc.n_s, sc.N, sc.n_loc, sc.dim
    R = ns * N
    phi = 8.0 * ns * N * nl
    iface = 8.0 * ns * N * sum(nl // s for s in (sc.sx, sc.sy, sc.sz)[:dim])  # neighbour interface rows
    blocks = 8.0 * ns * (1 + dim) * N * N
    couplings = 8.0 * ns * dim * N * N
    diagb = 8.0 * ns * N * N
    n_pad = -(-ns // 32) * 32
    # The PCG (k_pcg_tm) loads the scaled couplings once per solve into tensor memory / shared memory
    # (one warp per subdomain) and keeps the CTA's rows of the fp32 coarse inverse in shared memory:
    # its compulsory DRAM/L2 bytes per launch are one pass of the couplings, the deflation vectors and
    # the coarse rows, the history vectors of the initial guess, L^-1 for the back-transform, plus per
    # iteration the neighbour exchange through L2 (z, p written and read by the neighbours, the
    # hand-overs T, the coarse-rhs contributions: ~8 R-vectors)
    per_iter = 8.0 * 8 * R + 4.0 * 8 * n_pad
    onchip = couplings + 8.0 * 6 * R + 4.0 * n_pad * n_pad + 8.0 * R * (2 * 8 + 4) + diagb
    return {
        "project": phi + iface + 8.0 * n + 48.0 * n + blocks + 8.0 * R,
        "coarse": 20.0 * n_pad * n_pad,                   # Newton-Schulz: X -> RT, X, RT -> Xn (fp32)
        "scale": blocks + 2 * diagb + couplings + 8.0 * 6 * R,   # read B, write L, L^-1, couplings, Y
        "guess": couplings + 8.0 * R * 8 * 6,             # one multi-vector SpMV pass + history vectors
        "pcg": onchip + (iters_per_step + 1) * per_iter,
        "recon": phi + 8.0 * n + 8.0 * R,
        "flux_cfl": 8.0 * n * 4 + 48.0 * n,               # p, lambda, f, netw + static face coefficients
        "transport": 8.0 * n * 5,                         # s, netw in; s, lambda, f out
    }


def stage_flops(sc):
    """fp64 flops per STEP of the stages with dense contractions: the projection
    (Y = A_EE Phi_E^T with the (2 dim + 1)-point stencil, B_EE = Phi_E Y, the couplings over the
    interface faces), the scaling transform (two N^3 products per coupling block) and the
    reconstruction (p = Phi c)."""
    n, ns, N, nl, dim = sc.n, sc.n_s, sc.N, sc.n_loc, sc.dim
    iface_faces = ns * sum(nl // s for s in (sc.sx, sc.sy, sc.sz)[:dim])
    return {"project": ns * (2.0 * N * N * nl + 2.0 * N * (2 * dim + 1) * nl) + 2.0 * N * N * iface_faces,
            "scale": 4.0 * N ** 3 * ns * dim + 2.0 * N ** 3 / 3 * ns * 2,
            "recon": 2.0 * N * n}


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
    if os.path.exists(p):
        d, _ = json.JSONDecoder().raw_decode(open(p).read())   # the tool's output: a JSON object, then its status line
        for k in ("dmma_tflops", "DMMA_tflops", "dmma"):
            if k in d:
                return float(d[k]), "measured (profiles/r01_fp64_peaks.json, DMMA)"
    return 37.1, "fallback: the DMMA peak measured in round 1 (tools/fp64_peaks.cu)"


# measured cost of one deterministic grid-wide reduction fused with a grid barrier (147 CTAs x 448
# threads, a neighbour store + load before each; tools/mb_gridreduce.cu, release-reduction arrival)
GRID_REDUCE_US = 2.84


def sync_roofline(stages, K, iters):
    """The PCG's latency floor: three grid-wide synchronisations per iteration (two reductions and one
    barrier), each at least the measured GRID_REDUCE_US; frac = floor / measured time per iteration."""
    if "pcg" not in stages or iters <= 0:
        return None
    us_iter = 1e3 * stages["pcg"][0] / K / iters
    floor = 3 * GRID_REDUCE_US
    return {"us_per_iteration": us_iter, "floor_us_per_iteration": floor, "frac": floor / us_iter,
            "floor_source": "3 x measured grid reduction (tools/mb_gridreduce.cu, mode 3)"}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(cfg, basis, n_steps):
    """Time the CPU oracle (as it stands) on n_steps of the same workload from s0."""
    from oracle import lrbms_oracle as O
    from paper_1405_2810_b200 import inputs
    sc = inputs.make_scenario(cfg, basis=basis)
    fp = O.fprime_max(sc)
    s = sc.s0.copy()
    c_prev = None
    times = []
    for _ in range(n_steps):
        t0 = time.perf_counter()
        out = O.lrbms_step(sc, s, fpmax=fp, x0=c_prev)
        times.append(time.perf_counter() - t0)
        s, c_prev = out["s"], out["c"]
    return times


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    K = max(1, min(args.steps, 3))
    W = min(args.warmup, 1)  # one untimed step pages in NumPy/SciPy; more only lengthens a ~15 s/step run
    times = oracle_sample(args.config, args.basis, K + W)[W:]
    tot = sum(times)
    value = K / tot
    cores = cpu_threads()
    sample = (f"{K} full oracle online steps of {args.config} after {W} untimed step(s) from s0 (of --steps "
              f"{args.steps} --warmup {args.warmup}; capped so the run ends within minutes); NumPy/SciPy fp64 "
              "oracle/lrbms_oracle.py as it stands")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": 1e3 * tot / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "basis": args.basis},
            "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def timed_window(ctx, sc, W, K, world, device, profile=False):
    """One repetition of the timed window: from s0 (set_saturation resets the solver history and the
    coarse inverse, so every repetition does identical work), W untimed steps, then K steps timed with
    CUDA events on the library's stream, inputs resident in HBM.  Returns (ms max over ranks, PCG
    iterations per step, kernel launches, stage times or None)."""
    import torch
    ctx.set_saturation(sc.s0)
    ctx.run(W)
    st0 = ctx.stats()
    if profile:
        ctx.set_profiling(True)
    barrier(world)
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    ctx.run(K)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    stages = None
    if profile:
        stages = ctx.stage_times()
        ctx.set_profiling(False)
    st1 = ctx.stats()
    barrier(world)
    return max_over_ranks(ms, world, device), (st1["total_iters"] - st0["total_iters"]) / K, launches, stages


def small_configs(args, device):
    """us per step of the latency-bound configs C1-C4 (paper-recipe bases), median of 3
    repetitions of a window from s0 (3 untimed steps, then min(steps, 50) timed)."""
    from paper_1405_2810_b200 import inputs
    from paper_1405_2810_b200.lrbms import LrbmsContext
    out = {}
    for cfg in ("C1", "C2", "C3", "C4"):
        sc = inputs.make_scenario(cfg, basis=args.basis)
        ctx = LrbmsContext(sc, device=device)
        K = min(sc.n_steps, 50)
        reps = [timed_window(ctx, sc, 3, K, 1, device) for _ in range(3)]
        ms = statistics.median(r[0] for r in reps)
        out[cfg] = {"us_per_step": round(1e3 * ms / K, 2), "steps_per_s": round(1e3 * K / ms, 1), "steps": K,
                    "pcg_iters_per_step": reps[0][1], "launches_per_step": reps[0][2] / K,
                    "cells": sc.n, "reduced_dofs": sc.n_s * sc.N,
                    "pcg_launch": ("one CTA" if sc.n_s <= 16 else
                                   ("one thread-block cluster" if sc.n_s <= 224 else "cooperative grid")),
                    "ns_guard_trips": int(ctx.stats()["ns_guard_trips"])}
        ctx.close()
    return out


def run_ours(args, rank, local, world):
    import torch
    from paper_1405_2810_b200 import inputs
    from paper_1405_2810_b200.lrbms import LrbmsContext

    if not torch.cuda.is_available():
        raise SystemExit("bench.py --impl ours needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    t_inputs = time.perf_counter()
    sc = shared_scenario(args.config, args.basis, rank, world, device)
    t_inputs = time.perf_counter() - t_inputs
    solver = {}
    if args.coarse_refresh:
        solver["coarse_refresh"] = args.coarse_refresh
    if args.rtol:
        solver["rtol"] = args.rtol
    ctx = LrbmsContext(sc, device=device, solver=solver or None)
    stream = ctx.stream
    K, W = args.steps, args.warmup

    # ---- the headline: median of --reps repetitions of the same window (W untimed + K timed steps
    #      from s0), clocks sampled during them
    ctx.run(1)   # first-call costs (TMA descriptors, occupancy queries) outside every window
    clocks = ClockSampler(local)
    clocks.start()
    reps = [timed_window(ctx, sc, W, K, world, device) for _ in range(args.reps)]
    clk = clocks.stop()
    rep_ms = [r[0] for r in reps]
    ms_max = statistics.median(rep_ms)
    value = world * K / (ms_max / 1e3)
    iters = reps[0][1]
    launches = reps[0][2]
    ms = ms_max

    # ---- per-stage device times of the SAME window (CUDA events around every stage cost ~70 us per
    #      step, so this is one extra repetition, not one of the timed ones; deterministic, so the
    #      iteration count equals the headline's)
    _, iters_p, _, stages = timed_window(ctx, sc, W, K, world, device, profile=True)
    Kp = K
    diag = ctx.diagnostics()   # K6 of the window's last step (off the timed path)

    # ---- e2e: the same window through the C ABI with HOST buffers (pinned): every step copies s in
    #      and s, p out inside the timed region
    Ke = args.e2e_steps or K
    s_pin = torch.empty(sc.n, dtype=torch.float64, pin_memory=True)
    p_pin = torch.empty(sc.n, dtype=torch.float64, pin_memory=True)
    ctx.set_saturation(sc.s0)
    ctx.run(W)
    s_dev, _, _ = ctx.get_state()
    s_pin.copy_(s_dev.cpu())
    barrier(world)
    torch.cuda.synchronize()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    t_wall0 = time.perf_counter()
    for _ in range(Ke):
        ctx.run_host_ptr(1, s_pin.data_ptr(), s_pin.data_ptr(), p_pin.data_ptr())
    e3.record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    ms_e2e = max(e2.elapsed_time(e3), 1e3 * t_wall)
    ms_e2e = max_over_ranks(ms_e2e, world, device)
    e2e_value = world * Ke / (ms_e2e / 1e3)

    small = small_configs(args, device) if (world == 1 and args.small) else None

    # ---- NEXT-1: the paper's affine online variant on the same workload (theta fit + sum_q theta_q
    #      b_q instead of the direct projection); reported beside the north-star metric, not as it
    affine = None
    if args.affine_steps > 0:
        sp = inputs.profile_saturations(sc)
        ctx.set_profiles(sp)
        ctx.set_online(True)
        ctx.run(3)
        sa0 = ctx.stats()
        barrier(world)
        torch.cuda.synchronize()
        e4 = torch.cuda.Event(enable_timing=True)
        e5 = torch.cuda.Event(enable_timing=True)
        e4.record(stream)
        ctx.run(args.affine_steps)
        e5.record(stream)
        torch.cuda.synchronize()
        ms_a = max_over_ranks(e4.elapsed_time(e5), world, device)
        sa1 = ctx.stats()
        ctx.set_profiling(True)   # stage breakdown from a separate short pass
        ctx.run(min(args.affine_steps, 20))
        st_a = ctx.stage_times()
        ctx.set_profiling(False)
        ctx.set_online(False)
        affine = {"value": world * args.affine_steps / (ms_a / 1e3), "unit": "steps/s",
                  "ms_per_step": ms_a / args.affine_steps, "steps": args.affine_steps, "profiles": int(sp.shape[0]),
                  "pcg_iters_per_step": (sa1["total_iters"] - sa0["total_iters"]) / args.affine_steps,
                  "stage_us_per_step": {k: round(1e3 * v[0] / min(args.affine_steps, 20), 1) for k, v in st_a.items()},
                  "note": "the paper's online variant (eq:leastSquaresFit theta fit + eq:reducedSystem "
                          "sum_q theta_q b_q, d_q; NEXT-1), continuing the trajectory above; "
                          "the north-star metric is the direct-projection line"}

    # ---- NEXT-2: the fine-scale reference scheme (the paper's comparison run) on the
    #      same workload, continuing the trajectory: fine Jacobi-PCG pressure + the same transport
    fine = None
    if args.fine_steps > 0:
        ctx.run_fine(1, rtol=1e-12)   # workspace allocation, neighbour table, warm start
        barrier(world)
        torch.cuda.synchronize()
        e6 = torch.cuda.Event(enable_timing=True)
        e7 = torch.cuda.Event(enable_timing=True)
        e6.record(stream)
        _, fit = ctx.run_fine(args.fine_steps, rtol=1e-12)
        e7.record(stream)
        torch.cuda.synchronize()
        ms_f = max_over_ranks(e6.elapsed_time(e7), world, device)
        # algorithmic bytes of one CG iteration: per cell, phase A reads z, p, the 2-byte neighbour
        # code, 3 face weights, d and writes p_new, q (66 B), phase B reads x, p_new, q, r, d and
        # writes x, r, z (64 B), the coarse part re-reads r (8 B); plus one pass of the fp32 coarse
        # inverse (4 n_pad^2 B; the per-step Gauss-Jordan inverse is not counted)
        n_pad = -(-sc.n_s // 32) * 32
        fbytes = (138.0 * sc.n + 4.0 * n_pad * n_pad) * fit
        fine = {"value": world * args.fine_steps / (ms_f / 1e3), "unit": "steps/s",
                "ms_per_step": ms_f / args.fine_steps, "steps": args.fine_steps,
                "cg_iters_per_step": fit / args.fine_steps, "rtol": 1e-12,
                "achieved_gbs": fbytes / (ms_f / 1e3) / 1e9,
                "lrbms_speedup": value / (world * args.fine_steps / (ms_f / 1e3)),
                "note": "the fine k = 0 scheme on the GPU (alg:highDimTwoPhaseFlow at Phi_E = I; NEXT-2): "
                        "CG with a Jacobi + subdomain-coarse two-level preconditioner in one cooperative "
                        "kernel, then the same fluxes and transport; lrbms_speedup = the headline steps/s over these steps/s (the paper's "
                        "online-vs-fine comparison, P:1300-1302)"}

    # ---- NEXT-3: the offline basis recipe on the GPU (the same recipe the host ran for this workload's
    #      bases), timed and compared with the host bases
    offline = None
    if args.offline and args.basis == "pod":
        from offline import recipe as R
        mus = R.training_parameters(8, 2 * sc.N, 100 + inputs.CONFIG_INDEX[args.config])
        ctx.set_saturation(sc.s0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Phi_g, kept_g, info_g, _, _ = ctx.offline_basis(mus, M=8, horizon_steps=sc.n_steps)
        torch.cuda.synchronize()
        t_off = time.perf_counter() - t0
        Pg = torch.einsum("ekl,ekm->elm", Phi_g, Phi_g)
        Ph = torch.as_tensor(sc.Phi, device=device)
        Ph = torch.einsum("ekl,ekm->elm", Ph, Ph)
        dP = (Pg - Ph).abs().amax(dim=(1, 2)).cpu().numpy()
        offline = {"seconds": t_off, "host_recipe_seconds": t_inputs, "tof_sweeps": info_g["tof_sweeps"],
                   "fine_solves": 1 + 2 * sc.N, "fine_cg_iters": info_g["fine_cg_iters"],
                   "projector_diff_max": float(dP.max()), "projector_diff_median": float(np.median(dP)),
                   "kept_modes_histogram": np.bincount(kept_g).tolist(),
                   "note": "lrbms_offline_basis (NEXT-3): fine solve at s0, time of flight, 8 profiles, "
                           "2N fine snapshots, per-subdomain one-sided Jacobi POD, on the GPU; compared with "
                           "the host recipe's bases the headline ran on (host_recipe_seconds includes the "
                           "seeded field generation)"}
        del Pg, Ph

    # ---- NEXT-4: the online step on the k = 1 SWIP-DG fine space (P1 transport + limiter) on the same
    #      grid, medium, fluid and wells (polynomial P1 bases; its own context)
    k1 = None
    if args.k1_steps > 0:
        sc1 = inputs.make_scenario_k1(args.config)
        ctx1 = LrbmsContext(sc1, device=device, k1_only=True)
        ctx1.k1_set_basis(sc1.Phi1)
        s1_0 = np.zeros((sc1.dim + 1, sc1.n))
        s1_0[0] = sc1.s0
        ctx1.k1_set_saturation(s1_0)
        ctx1.k1_run(3)
        barrier(world)
        torch.cuda.synchronize()
        st0 = ctx1.stats()
        e8 = torch.cuda.Event(enable_timing=True)
        e9 = torch.cuda.Event(enable_timing=True)
        e8.record(stream)
        ctx1.k1_run(args.k1_steps)
        e9.record(stream)
        torch.cuda.synchronize()
        ms_1 = max_over_ranks(e8.elapsed_time(e9), world, device)
        st1 = ctx1.stats()
        ctx1.set_profiling(True)
        ctx1.k1_run(args.k1_steps)
        torch.cuda.synchronize()
        st_1 = ctx1.stage_times()
        ctx1.set_profiling(False)
        nflag = ctx1.k1_get_state()[3]
        nd = sc1.dim + 1
        # algorithmic bytes of the k = 1 projection and reconstruction: one pass of Phi1 each
        phi1_bytes = 8.0 * sc1.n_s * sc1.N * nd * sc1.n_loc
        proj_bytes = phi1_bytes + 8.0 * sc1.n_s * (1 + sc1.dim) * sc1.N ** 2 + (48.0 + 8.0) * sc1.n
        k1 = {"value": world * args.k1_steps / (ms_1 / 1e3), "unit": "steps/s", "ms_per_step": ms_1 / args.k1_steps,
              "steps": args.k1_steps, "fine_dofs": nd * sc1.n, "reduced_dofs": sc1.n_s * sc1.N,
              "pcg_iters_per_step": (st1["total_iters"] - st0["total_iters"]) / args.k1_steps,
              "stage_us_per_step": {k: round(1e3 * v[0] / args.k1_steps, 1) for k, v in st_1.items()},
              "limiter_flagged_cells_last_step": nflag,
              "project_gbs": proj_bytes / (st_1["project"][0] / args.k1_steps / 1e3) / 1e9,
              "recon_gbs": (phi1_bytes + 8.0 * nd * sc1.n) / (st_1["recon"][0] / args.k1_steps / 1e3) / 1e9,
              "note": "lrbms_k1_run (NEXT-4): eq:swipBilP projection on the P1 dofs (k1_project, DMMA), the "
                      "reduced solve with the additive two-level preconditioner, eq:velocityDG fluxes, "
                      "eq:saturationDG transport and the limiter of P:419-469; stage 'transport' = transport + "
                      "limiter; project_gbs / recon_gbs = one pass of Phi1 (+ outputs) over the stage time"}
        ctx1.close()
        del ctx1

    if rank != 0:
        return 0

    # ---- roofline of the dominant kernel (per step: every stage is one launch per step except the
    #      three small initial-guess kernels; the PCG stage is exactly the one k_pcg launch)
    peak, peak_src = measured_peaks()
    per_step = {k: v[0] / Kp for k, v in stages.items()}
    dom = max((k for k in stages if stages[k][1] > 0), key=lambda k: stages[k][0])
    dom_ms = per_step[dom]
    sb = stage_bytes(sc, iters_p)
    algo = sb.get(dom, 0.0)
    achieved = algo / (dom_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(args.config, {}).get(dom)
    # whole-step view: every stage's algorithmic bytes once per step
    step_bytes = sum(sb[k] for k in sb if k in stages)
    sf = stage_flops(sc)
    p64, p64_src = fp64_peak()
    t_roof_us = sum(max(sb[k] / (peak * 1e9), sf.get(k, 0.0) / (p64 * 1e12)) for k in sb if k in stages) * 1e6
    step_ms = ms / K
    ms_prof = sum(v[0] for v in stages.values())
    stage_share = {k: round(v[0] / max(ms_prof, 1e-9), 4) for k, v in stages.items()}
    stage_us = {k: round(1e3 * v, 1) for k, v in per_step.items()}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits
        n_cpu = max(1, args.cpu_steps)
        ts_all = oracle_sample(args.config, args.basis, n_cpu + 1)[1:]
        with threadpool_limits(1):
            ts_one = oracle_sample(args.config, args.basis, 2)[1:]
        cpu = {"value": n_cpu / sum(ts_all), "unit": "steps/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": f"{n_cpu} oracle online steps of {args.config} after 1 untimed step from s0 "
                         f"({sum(ts_all):.1f} s) on all host threads; NumPy/SciPy fp64 oracle as it stands",
               "one_thread": {"value": 1.0 / sum(ts_one), "unit": "steps/s", "cores": 1,
                              "sample": f"1 oracle step after 1 untimed step, BLAS limited to 1 thread ({sum(ts_one):.1f} s)"}}

    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded %s recipe of DESIGN.md section 4, %s bases; no dataset)" % (args.config, args.basis),
        "config": {"workload": args.config, "grid": f"{sc.nx}x{sc.ny}x{sc.nz}",
                   "subdomains": f"{sc.Sx}x{sc.Sy}x{sc.Sz} of {sc.sx}x{sc.sy}x{sc.sz}", "N": sc.N,
                   "cells": sc.n, "reduced_dofs": sc.n_s * sc.N, "basis": args.basis,
                   "l2": "inputs larger than L2 (Phi = %.0f MB > 126 MB L2), no flush" % (8e-6 * sc.n_s * sc.N * sc.n_loc),
                   "parallelism": "replicas" if world > 1 else "single GPU"},
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": 8 * sc.n,
                "d2h_bytes_per_step": 16 * sc.n, "steps": Ke,
                "note": "lrbms_run_host with pinned host buffers, one step per call (s in, s and p out), "
                        "the same window as the headline"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "k_pcg_tm" if dom == "pcg" else dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": algo, "avg_launch_ms": dom_ms,
                     "note": ("k_pcg_tm holds the scaled reduced operator on chip (tensor memory + shared memory) "
                              "for the whole solve: its compulsory DRAM/L2 bytes are one pass of the operator and "
                              "the per-iteration neighbour exchange, so it is far from the HBM roofline by "
                              "construction; it is bound by the latency of its three grid-wide synchronisations "
                              "per iteration (sync_roofline)") if dom == "pcg" else ""},
        "sync_roofline": sync_roofline(stages, Kp, iters_p),
        "reps": {"ms_per_window": [round(x, 4) for x in rep_ms], "median_ms": ms_max, "window": f"{W} untimed + {K} timed steps from s0"},
        "profiled_pass": {"steps": Kp, "pcg_iters_per_step": iters_p,
                          "note": "stage times, roofline and sync_roofline come from one more repetition of the "
                                  "same window with per-stage CUDA events (same iterations as the headline)"},
        "small_configs": small,
        "diagnostics": dict(diag, note="K6 (lrbms_diagnostics) after the window's last step: mass, s range, "
                                       "relative mass loss zeta (P:1114-1120), coarse defect, link fluxes"),
        "step_roofline": {"algorithmic_bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (step_ms / 1e3) / 1e9,
                          "frac": step_bytes / (step_ms / 1e3) / 1e9 / peak,
                          "t_roof_us": t_roof_us, "frac_time": t_roof_us / (1e3 * step_ms),
                          "fp64_peak_tflops": p64, "fp64_peak_source": p64_src,
                          "note": "t_roof = sum over stages of max(algorithmic bytes / HBM peak, fp64 flops / "
                                  "DMMA peak) (SURVEY 8(d)); frac_time = t_roof / measured step time"},
        "stage_share": stage_share,
        "stage_us_per_step": stage_us,
        "pcg_iters_per_step": iters,
        "affine_variant": affine,
        "fine_reference": fine,
        "offline_gpu": offline,
        "k1_variant": k1,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    use_cuda = args.impl == "ours"
    rank, local, world = dist_setup(use_cuda)
    try:
        if args.impl == "reference":
            return run_reference(args, rank, world)
        return run_ours(args, rank, local, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
