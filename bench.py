#!/usr/bin/env python
"""Benchmark of the B200 hot path — fine-propagator fp64 grid-point updates/s.

Workload (BASELINE.json config 5, fine-propagator-only throughput sweep): periodic 2D
grid, seeded random smooth medium c in [0.5, 1] (sum of 8 low-frequency sinusoids),
seeded random Gaussian pulses as initial states, 64 velocity-Verlet steps per slice per
step (= one coupling interval of K1).  A "step" is one batched K1 call over the
per-GPU batch; slices are sharded across ranks (weak scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--grid 4096] [--batch 64]
  python bench.py --impl reference      # the reference's propagate_coupling on host cores

One JSON line (rank 0).  Timing: CUDA events on the launching stream, barrier +
synchronize on both sides, max over ranks.  Inputs (>= 1 GiB) exceed the 126 MB L2.
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
from pathlib import Path

import numpy as np

from workloads import cfg5_medium, cfg5_pulses, cfg5_pulses_device

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fine-propagator fp64 grid-pt updates/s"
ITER_CONFIGS = (1, 2, 3, 4)  # BASELINE configs timed for seconds per parareal iteration
FLOPS_PER_UPDATE = 17  # Laplacian 9, x c^2 1, u-update 4, udot-update 3
STEPS_PER_COUPLING = 64


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def arm_config(n, batch, mode, world):
    """The workload both arms report (bench.py's own arm and --impl reference)."""
    return {"workload": f"cfg5 fine propagator {n}x{n} periodic, {batch} slices/GPU x "
                        f"{STEPS_PER_COUPLING} velocity-Verlet steps per step ({mode} mode)",
            "grid": n, "slices_per_gpu": batch, "steps_per_slice": STEPS_PER_COUPLING,
            "parallelism": f"slice-sharded x{world}", "l2": "inputs > L2 (no flush needed)"}


def run_reference(args, rank, world):
    """The reference's propagate_coupling (propagator.cpp, compiled verbatim in oracle/_ref)
    over a bounded sample of the same workload on all host cores."""
    if rank != 0:
        return
    from oracle import refbind
    from oracle.paratime_np import Grid

    n = args.grid
    cores = os.cpu_count() or 1
    sample_slices = cores  # one slice per std::thread worker (parareal.cpp:25-47 partition)
    g = Grid((n, n), (1.0 / n, 1.0 / n))
    c = cfg5_medium(n)
    dt = 0.9 * (1.0 / n) / (math.sqrt(2.0) * float(c.max()))
    u0 = cfg5_pulses(n, sample_slices)
    v0 = np.zeros_like(u0)
    steps = max(1, args.ref_steps)
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        refbind.propagate(u0, v0, c, g, dt, steps, workers=cores)
        t1 = time.perf_counter()
        if k >= args.warmup:
            times.append(t1 - t0)
    per = float(np.mean(times))
    value = sample_slices * n * n * steps / per
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "grid-pt updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg5 medium/pulses)",
        "config": dict(arm_config(n, args.batch, args.mode, world),
                       sample=f"each step: {sample_slices} slices x {steps} steps of this workload on the host "
                              f"(bounded CPU sample; the metric is per grid-point update)"),
        "cpu_baseline": {"value": value, "unit": "grid-pt updates/s", "cores": cores, "kind": "reference",
                         "sample": f"{sample_slices} slices of {n}^2 x {steps} steps, propagate_coupling "
                                   f"(propagator.cpp verbatim, -O3, std::thread x{cores})"},
        "e2e": {"value": value, "unit": "grid-pt updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=512, help="slices per GPU")
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--ref-steps", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-batch", type=int, default=128, help="slices per e2e call (host-pinned state)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the cfg5 grid sweep")
    ap.add_argument("--no-parareal", action="store_true", help="skip the s/iteration measurement")
    ap.add_argument("--no-pml", action="store_true", help="skip the cfg4 absorbing-layer section")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference legs (parity check too)")
    args = ap.parse_args()

    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    import paratime_b200 as B

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    n, batch = args.grid, args.batch
    mode = B.FAST if args.mode == "fast" else B.EXACT
    ctx = B.Context(local)
    c = cfg5_medium(n)
    dt = 0.9 * (1.0 / n) / (math.sqrt(2.0) * float(c.max()))
    grid = B.Grid((n, n), (1.0 / n, 1.0 / n))
    prop = B.Propagator(ctx, grid, c, dt, STEPS_PER_COUPLING)
    # each rank owns its own contiguous block of slices, seeded by rank; generated on the device
    # (a 4096^2 x 512 batch is 69 GB per field)
    seed = 20261019 + 50 + 1000 * rank
    u = torch.empty((batch, n, n), dtype=torch.float64, device=f"cuda:{local}")
    cfg5_pulses_device(n, batch, u, seed)
    v = torch.zeros_like(u)
    stream = torch.cuda.current_stream()
    eb = min(args.e2e_batch, batch)
    e2e_host = None
    if not args.no_e2e:  # pinned host copies of the first e2e slices (inputs of the e2e leg)
        e2e_host = (u[:eb].cpu().pin_memory(), torch.zeros((eb, n, n), dtype=torch.float64).pin_memory())
    cpu_leg = rank == 0 and world == 1 and not args.no_cpu
    check_idx = parity_slices(batch, os.cpu_count() or 1) if cpu_leg else []
    u_check0 = u[check_idx].cpu().numpy() if cpu_leg else None

    def step():
        prop.propagate(u, v, mode=mode)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    l0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = ctx.launches() - l0
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    updates = world * batch * n * n * STEPS_PER_COUPLING * args.steps
    value = updates / (ms * 1e-3)
    ms_per_step = ms / args.steps
    finite = all(bool(torch.isfinite(f[b:b + 8]).all().item()) for f in (u, v) for b in range(0, batch, 8))

    # parity of the timed kernel plan: one more step of the SAME batch from regenerated inputs;
    # the checked slices go to the reference's propagate_coupling (cpu_baseline leg below)
    u_check1 = None
    if cpu_leg:
        cfg5_pulses_device(n, batch, u, seed)
        v.zero_()
        step()
        torch.cuda.synchronize()
        u_check1 = (u[check_idx].cpu().numpy(), v[check_idx].cpu().numpy())

    # roofline: live fp64 FMA peak on this GPU; dominant kernel = the wavefront K1 pass
    tflops_peak, _ = probe_fp64(ctx)
    per_launch_ms = ms / max(launches, 1)
    plan = prop.plan(batch, mode)
    # every launch is one wavefront pass of `fused` steps over one chunk of slices (the headline
    # batch runs in scratch chunks, PTB_SCRATCH_MIB): algorithmic work per launch = the step's
    # updates / launches per step
    fused = fused_steps(plan)
    launches_per_step = launches / args.steps
    updates_per_launch = batch * n * n * STEPS_PER_COUPLING / launches_per_step
    steps_per_launch = fused
    slices_per_launch = updates_per_launch / (n * n * fused)
    flops_per_launch = updates_per_launch * FLOPS_PER_UPDATE
    achieved = flops_per_launch / (per_launch_ms * 1e-3) / 1e12
    hbm_bytes_per_launch = updates_per_launch * 40.0 / fused  # read u, udot, coef; write u, udot (8 B each)
    traffic = ncu_traffic(n, batch, args.mode, plan)

    # achieved fraction = max(upd/s*17/FP64_peak, upd/s*40/s_f/HBM_peak), s_f the
    # steps fused per HBM round trip; the larger term names the binding roofline of this design.
    hbm_peak = None
    try:
        hbm_peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        pass
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    if hbm_peak is None:
        hbm_peak, hbm_src = 7700.0, "B200_PROFILING.md fallback"
    hbm_achieved = hbm_bytes_per_launch / (per_launch_ms * 1e-3) / 1e9
    fp64 = {"achieved": achieved, "peak": tflops_peak, "unit": "TFLOP/s",
            "frac": achieved / tflops_peak if tflops_peak else None, "flops_per_update": FLOPS_PER_UPDATE,
            "peak_source": "measured live: DFMA probe (ptb_probe_fp64_peak)"}
    hbm = {"achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_achieved / hbm_peak,
           "bytes_per_point_per_launch": 40, "peak_source": hbm_src}
    binding = "hbm" if (fp64["frac"] or 0.0) <= hbm["frac"] else "fp64"
    main_ = hbm if binding == "hbm" else fp64
    roofline = {"bound": binding, "achieved": main_["achieved"], "peak": main_["peak"], "unit": main_["unit"],
                "frac": main_["frac"], "traffic": traffic and traffic["dram_bytes_per_launch"],
                "traffic_source": traffic and traffic["source"], "kernel": plan, "per_launch_ms": per_launch_ms,
                "steps_per_launch": steps_per_launch, "slices_per_launch": slices_per_launch, "fp64": fp64,
                "hbm": hbm}
    del u, v
    torch.cuda.empty_cache()

    def guarded_section(fn):
        """Secondary measurements never cost the headline line: at N > 1 a failure in the
        sharded parareal / e2e section is reported in the JSON instead of aborting the run."""
        try:
            return fn()
        except Exception as ex:  # pragma: no cover - only on multi-GPU failures
            if world == 1:
                raise
            return {"error": f"{type(ex).__name__}: {ex}"[:300]}

    e2e = None
    if e2e_host is not None:
        e2e = guarded_section(lambda: measure_e2e(B, prop, e2e_host, mode, args.e2e_steps, local, dist, world))
        del e2e_host
    parareal = None
    if not args.no_parareal:
        parareal = guarded_section(lambda: parareal_iteration_times(B, ctx, rank, world, dist))

    pml = None
    if not args.no_pml:
        pml = guarded_section(lambda: pml_section(B, ctx, tflops_peak, hbm_peak, rank, world, dist))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "grid-pt updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg5 medium and Gaussian pulses)",
            "config": dict(arm_config(n, batch, args.mode, world), finite=finite),
            "gpu_launches": launches,
            "roofline": roofline,
            "clocks": clocks.summary(),
            "e2e": e2e,
        }
        if parareal is not None:  # compact top-level keys (the driver keeps the line's head)
            for k, r in parareal.items():
                line[f"s_per_iteration_{k}"] = round(r["s_per_iteration"], 6)
        if cpu_leg:
            base, par = cpu_baseline_and_parity(n, c, dt, check_idx, u_check0, u_check1)
            line["parity"] = par
            line["cpu_baseline"] = base
            if parareal is not None:
                line["cpu_baseline_parareal"] = {k: cpu_parareal_iteration(k) for k in ("cfg1", "cfg2", "cfg3", "cfg4r")}
                line["cpu_host"] = host_cpu_model()
        line["parareal"] = parareal
        if not args.no_sweep:
            line["cfg5_sweep"] = sweep(B, ctx, mode, tflops_peak, hbm_peak)
        if pml is not None:
            line["cfg4_pml"] = pml
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def fused_steps(plan):
    """Steps fused per HBM round trip by a plan string (wavefront depth S, or the whole
    coupling for the on-chip k_small / k_cluster)."""
    import re

    m = re.search(r"k_wave2?<(\d+),", plan)
    return int(m.group(1)) if m else STEPS_PER_COUPLING


def parity_slices(batch, cores):
    """Slices checked against the reference (first, last, evenly spread; one per host core)."""
    k = max(2, min(batch, cores))
    return sorted({int(round(i * (batch - 1) / (k - 1))) for i in range(k)})


def cpu_baseline_and_parity(n, c, dt, idx, u0, got):
    """The reference's propagate_coupling (oracle/_ref, propagator.cpp verbatim; parareal.cpp:25-47
    thread partition) on the checked slices of the headline batch: timed on all host cores (the
    `cpu_baseline`), and its outputs compared with the device's for the SAME slices under the
    SAME launch plan as the timed region (north star: <= 1e-12 relative L2 over [u; udot])."""
    from oracle import refbind
    from oracle.paratime_np import Grid

    if not refbind.LIB_PATH.exists():
        return {"value": None, "error": "oracle/_ref not built"}, {"checked": False}
    cores = os.cpu_count() or 1
    g = Grid((n, n), (1.0 / n, 1.0 / n))
    v0 = np.zeros_like(u0)
    t0 = time.perf_counter()
    ru, rv, div = refbind.propagate(u0, v0, c, g, dt, STEPS_PER_COUPLING, workers=cores)
    el = time.perf_counter() - t0
    rel = []
    for b in range(len(idx)):
        num = np.concatenate([got[0][b].ravel() - ru[b].ravel(), got[1][b].ravel() - rv[b].ravel()])
        den = np.concatenate([ru[b].ravel(), rv[b].ravel()])
        rel.append(float(np.linalg.norm(num) / np.linalg.norm(den)))
    base = {"value": len(idx) * n * n * STEPS_PER_COUPLING / el, "unit": "grid-pt updates/s", "cores": cores,
            "kind": "reference",
            "sample": f"{len(idx)} slices of the headline batch ({n}^2 x {STEPS_PER_COUPLING} steps each) through the "
                      f"reference's propagate_coupling (oracle/_ref, propagator.cpp verbatim) on std::thread x{cores}"}
    par = {"checked": True, "slices": idx, "max_rel_l2": max(rel), "tol": 1e-12, "ok": max(rel) <= 1e-12,
           "against": "oracle/_ref propagate_coupling, same inputs, device run under the timed plan"}
    return base, par


def host_cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.lower().startswith("model name"):
                return {"model": line.split(":", 1)[1].strip(), "cores": os.cpu_count()}
    except OSError:
        pass
    return {"model": None, "cores": os.cpu_count()}


def ncu_traffic(n, batch, mode, plan):
    """DRAM bytes per launch of the dominant kernel from the committed `ncu --set full` summary
    (profiles/k1_ncu.json), used only when it was captured on this exact grid/batch/mode/plan."""
    try:
        d = json.loads((ROOT / "profiles" / "k1_ncu.json").read_text())
    except Exception:
        return None
    if (d.get("grid"), d.get("batch"), d.get("mode"), d.get("plan")) != (n, batch, mode, plan):
        return None
    return {"dram_bytes_per_launch": d["dram_bytes_per_launch"], "source": d["source"]}


def parareal_iteration_times(B, ctx, rank, world, dist, cfgs=ITER_CONFIGS):
    """Seconds per theta-parareal iteration on BASELINE configs (device-timed CUDA events around
    each iteration's body: parallel F + C.R, all-gather, snapshots + update_svd, coarse sweep,
    fine combine + finalize), slices sharded over the ranks.  The one-time serial fine
    reference is excluded and reported separately."""
    import workloads as W

    comm = None
    if world > 1:
        def bcast(raw):
            obj = [raw]
            dist.broadcast_object_list(obj, src=0)
            return obj[0]

        comm = B.api.Comm(ctx, rank, world, broadcast=bcast)
    out = {}
    for cfg in cfgs:
        spec, cf, cc, u0, v0 = W.CONFIGS[cfg]()
        B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0, comm=comm)  # warm-up (all K: module loads)
        r = B.api.parareal_run(ctx, B.api.run_spec(**spec), cf, cc, u0, v0, comm=comm)
        t = r["times"]
        it = np.array(t["iteration_ms"])
        out[f"cfg{cfg}"] = {
            "s_per_iteration": float(np.median(it)) / 1e3, "iteration_ms": [round(x, 3) for x in it],
            "phase_ms_median": {k: float(np.median(t[k])) for k in ("parallel_ms", "gather_ms", "procrustes_ms",
                                                                       "sweep_ms", "finalize_ms")},
            "serial_fine_reference_ms": t["reference_ms"], "ranks": r["rank"].tolist(),
            "final_energy_error": float(r["energy_err"][-1, -1]), "tol": spec["tol"], "K": spec["iterations"],
            "N": spec["n_couplings"], "fine": spec["fine_n"][0], "coarse": spec["coarse_n"][0]}
    return out


def cpu_parareal_iteration(cfg="cfg2"):
    """The reference's theta_parareal (oracle/_ref: parareal.cpp verbatim, Procrustes on LAPACK)
    on the host cores for one BASELINE config: (wall - serial fine reference) / K.  "cfg4r" is
    config 4's first 16 couplings (workloads.cfg4_subset, K = 2): the full config 4 would take
    ~15 min per iteration here; its per-iteration cost is reported scaled by 128/16 (the fine
    stage, snapshots and sweep are linear in N)."""
    try:
        import workloads as W
        from oracle import refbind

        if not refbind.LIB_PATH.exists():
            return None
        spec, cf, cc, u0, v0 = W.cfg4_subset() if cfg == "cfg4r" else W.CONFIGS[int(cfg[3:])]()
        cores = os.cpu_count() or 1
        rs = refbind.RunSpec()
        rs.dim = 2
        for k in range(2):
            rs.fine_n[k], rs.fine_h[k] = spec["fine_n"][k], spec["fine_h"][k]
            rs.coarse_n[k], rs.coarse_h[k] = spec["coarse_n"][k], spec["coarse_h"][k]
        for k in ("dt_fine", "m_fine", "dt_coarse", "m_coarse", "T", "dt_com", "n_couplings", "interp",
                  "iterations", "variant", "scheme", "metric_scheme", "tol", "remove_leading"):
            setattr(rs, k, spec[k])
        rs.workers = cores
        from oracle.paratime_np import Grid

        g = Grid(tuple(spec["fine_n"]), tuple(spec["fine_h"]))
        t0 = time.perf_counter()  # the serial fine reference the driver computes first
        u, v = u0[None], v0[None]
        for _ in range(spec["n_couplings"]):
            u, v, _ = refbind.propagate(u, v, cf, g, spec["dt_fine"], spec["m_fine"], workers=1)
        ref_s = time.perf_counter() - t0
        r = refbind.parareal_run(rs, cf, cc, u0, v0)
        wall = r["wall_ms"] / 1e3
        out = {"value": (wall - ref_s) / spec["iterations"], "unit": "s/iteration", "cores": cores,
               "kind": "reference", "config": cfg,
               "sample": f"theta_parareal on {cfg} (K={spec['iterations']}, N={spec['n_couplings']}), "
                         f"wall {wall:.2f} s minus serial fine reference {ref_s:.2f} s, std::thread x{cores}"}
        if cfg == "cfg4r":
            out["cfg4_estimate_s_per_iteration"] = out["value"] * 128 / spec["n_couplings"]
        return out
    except Exception as e:  # pragma: no cover
        return {"value": None, "error": str(e)}


def probe_fp64(ctx):
    import ctypes

    import paratime_b200 as B

    tf, ms = ctypes.c_double(), ctypes.c_double()
    B.api.check(B.lib().ptb_probe_fp64_peak(ctx.h, ctypes.byref(tf), ctypes.byref(ms)))
    return tf.value, ms.value


def measure_e2e(B, prop, host, mode, steps, local, dist, world):
    """Same metric through the C-ABI host-buffer call (ptb_propagate_batch_host): every step
    copies the slices' state host->device, propagates, and copies it back device->host, in
    place in the pinned host buffers (the call pipelines chunks over three streams)."""
    import ctypes

    import torch

    uh, vh = host
    batch, n = uh.shape[0], uh.shape[1]
    flags = np.zeros(batch, dtype=np.int32)
    dp = ctypes.POINTER(ctypes.c_double)

    def call():
        B.api.check(B.lib().ptb_propagate_batch_host(
            prop.h, ctypes.c_size_t(batch), ctypes.cast(uh.data_ptr(), dp), ctypes.cast(vh.data_ptr(), dp),
            ctypes.cast(uh.data_ptr(), dp), ctypes.cast(vh.data_ptr(), dp),
            flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.c_int(mode)))

    call()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    el = time.perf_counter() - t0
    if dist:
        t = torch.tensor([el], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    value = world * batch * n * n * STEPS_PER_COUPLING * steps / el
    return {"value": value, "unit": "grid-pt updates/s", "h2d_bytes_per_step": int(2 * uh.numel() * 8),
            "d2h_bytes_per_step": int(2 * uh.numel() * 8 + batch * 4), "ms_per_step": el / steps * 1e3,
            "slices_per_call": batch, "grid": n,
            "api": "ptb_propagate_batch_host (pinned host buffers, in place; 3-stream chunked copies)"}


def sweep(B, ctx, mode, tflops_peak, hbm_peak):
    """cfg5 grid sweep (the >= 60 % target is judged on every cfg5 grid at batch >= 64):
    device-resident, FAST, 64 steps per slice, batch 64 (and 512 on the grids below 2048^2).  Per grid: updates/s, the launch plan,
    and the binding-roofline fraction max(upd/s*17/FP64, upd/s*(40/s_f)/HBM) with s_f the steps
    fused per HBM round trip of the plan (64 for the on-chip k_cluster, 8 per wavefront pass)."""
    import torch

    out = []
    for n, batch in ((128, 64), (128, 512), (256, 64), (512, 64), (512, 512), (1024, 64), (1024, 512), (2048, 64),
                     (4096, 64)):
        c = cfg5_medium(n)
        dt = 0.9 * (1.0 / n) / (math.sqrt(2.0) * float(c.max()))
        prop = B.Propagator(ctx, B.Grid((n, n), (1.0 / n, 1.0 / n)), c, dt, STEPS_PER_COUPLING)
        u = torch.as_tensor(cfg5_pulses(n, batch), device="cuda")
        v = torch.zeros_like(u)
        for _ in range(3):
            prop.propagate(u, v, mode=mode)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        reps = 5
        e0.record()
        for _ in range(reps):
            prop.propagate(u, v, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ups = batch * n * n * STEPS_PER_COUPLING / (ms * 1e-3)
        plan = prop.plan(batch, mode)
        s_f = fused_steps(plan)
        f_fp64 = ups * FLOPS_PER_UPDATE / (tflops_peak * 1e12) if tflops_peak else None
        f_hbm = ups * (40.0 / s_f) / (hbm_peak * 1e9)
        out.append({"grid": n, "batch": batch, "ms": round(ms, 3), "updates_per_s": ups, "plan": plan,
                    "fused_steps": s_f, "frac_fp64": f_fp64, "frac_hbm": f_hbm,
                    "frac_binding": max(f_fp64 or 0.0, f_hbm)})
        del u, v, prop
    return out

def pml_section(B, ctx, tflops_peak, hbm_peak, rank=0, world=1, dist=None):
    """BASELINE.json config 4 WITH its 32-cell absorbing layer (workloads.cfg4_pml; not in the
    reference).  (1) fine-stage throughput of the layered propagator on the
    per-GPU share of cfg4 at 8 GPUs (16 slices x 128 steps, 2048^2), device-resident, CUDA events;
    binding roofline from the super-pass traffic (interior 40 B per point per 8 steps, band frame
    2 x 72 B per point per 8 steps: ~6 B/update; the round-1/2 figure at 10 B/update beside it) and
    17 flops/update;
    (2) s/iteration of theta parareal with the layer (ptb_pml_theta_run: N = 128, K = 8, tol 1e-4;
    slices sharded over the ranks when world > 1, max over ranks).  Plain parareal is not reported:
    its iterates grow without bound on this hyperbolic problem."""
    import torch

    from workloads import cfg4_pml

    spec, c, cc, u0, v0, (zf, zc) = cfg4_pml()
    nf, nc = spec["fine_n"][0], spec["coarse_n"][0]
    gf = B.Grid((nf, nf), (1.0 / nf, 1.0 / nf))
    gc = B.Grid((nc, nc), (1.0 / nc, 1.0 / nc))
    fine = B.PmlPropagator(ctx, gf, c, zf, zf, spec["dt_fine"], spec["m_fine"])
    coarse = B.PmlPropagator(ctx, gc, cc, zc, zc, spec["dt_coarse"], spec["m_coarse"])
    batch = 16
    t = [torch.zeros((batch, nf, nf), dtype=torch.float64, device="cuda") for _ in range(4)]
    t[0].copy_(torch.as_tensor(u0, device="cuda").expand(batch, nf, nf))
    for _ in range(3):
        fine.propagate(*t)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    reps = 5
    e0.record()
    for _ in range(reps):
        fine.propagate(*t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ups = batch * nf * nf * spec["m_fine"] / (ms * 1e-3)
    del t
    torch.cuda.empty_cache()
    # algorithmic HBM bytes per update under the super-pass: the interior rectangle (SUPER_MARGIN = 10
    # cells from the damped bands) moves 40 B per point per 8 fused steps, the band frame 72 B per
    # point (u, udot, px, py read + write, coefficient read) in each of its two 4-step passes
    layer = int(np.count_nonzero(np.asarray(zf) > 0)) // 2
    fi = ((nf - 2 * (layer + 10)) / nf) ** 2
    bytes_per_update = fi * 40.0 / 8.0 + (1.0 - fi) * 2 * 72.0 / 8.0
    f_hbm = ups * bytes_per_update / (hbm_peak * 1e9)
    f_fp64 = ups * FLOPS_PER_UPDATE / (tflops_peak * 1e12) if tflops_peak else None
    tr = B.Transfer(ctx, gc, gf, spec["interp"])
    comm = None
    if world > 1:
        def bcast(raw):
            obj = [raw]
            dist.broadcast_object_list(obj, src=0)
            return obj[0]

        comm = B.api.Comm(ctx, rank, world, broadcast=bcast)
    r = B.pml_theta_run(fine, coarse, tr, spec["n_couplings"], spec["iterations"], u0, v0, tol=spec["tol"],
                        scheme=spec["scheme"], comm=comm)
    its = np.asarray(r["iteration_ms"], dtype=np.float64)
    if world > 1:  # device time of each iteration, max over ranks
        t_it = torch.as_tensor(its, device="cuda")
        dist.all_reduce(t_it, op=dist.ReduceOp.MAX)
        its = t_it.cpu().numpy()
    its = [float(x) for x in its]
    return {"workload": "cfg4 + 32-cell absorbing layer (fine 2048^2 / coarse 256^2, layered-faulted medium)",
            "fine_stage": {"per_gpu": True, "batch": batch, "steps": spec["m_fine"], "ms": round(ms, 3), "updates_per_s": ups,
                           "frac_hbm": f_hbm, "frac_fp64": f_fp64, "frac_binding": max(f_hbm, f_fp64 or 0.0),
                           "bytes_per_update": bytes_per_update,
                           "frac_hbm_at_10B_per_update": ups * 10.0 / (hbm_peak * 1e9),
                           "kernel": "super-pass of 8 steps: k_wave2<8> on the interior rectangle + k_pml<layer> band "
                                     "tiles in two 4-step passes (47/51- and 42-cell bands, halo 9 / 5 on undamped inner sides)"},
            "theta_parareal": {"N": spec["n_couplings"], "K": spec["iterations"], "tol": spec["tol"], "ranks": world,
                               "s_per_iteration": float(np.median(its)) / 1e3, "iteration_ms": [round(x, 2) for x in its],
                               "corrector_rank": [int(x) for x in r["rank"]],
                               "max_err_rel_init_per_k": [float(x) for x in np.max(r["rel_err"], axis=1)],
                               "diverged": r["diverged"]}}


if __name__ == "__main__":
    main()
