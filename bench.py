#!/usr/bin/env python
"""Benchmark of the B200 SPH density / smoothing-length pass.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

A step is one full density pass (ordering + search tree + h search + exact
K-th neighbour + density + write-back) over one synthetic particle set of
BASELINE.json config C (default 3, the largest clustered config that fits one
GPU: 16,777,216 fp32 particles, 80% in 20,000 NFW halos + 20% uniform
background, periodic box of side 252, DesNumNgb = 64).

value   : useful particle-pair interactions / s = N*K / t_pass, inputs already
          resident in HBM, t_pass = CUDA-event time on the library's stream,
          L2 flushed (256 MiB write) before every step; median over the K
          timed steps, max over ranks.
e2e     : the same metric through the public API (density_pass_soa) with
          pinned host buffers; host->device inputs and device->host results
          inside the timed region.
roofline: the dominant kernel (by device time) against the measured FP32-pipe
          FFMA rate; algorithmic ops = 6 per pair test (+10 per accepted pair
          in the density kernel), SURVEY 8(d).
cpu_baseline: the CPU oracle (a C restatement of the reference pass, OpenMP
          on all host cores) on a bounded random target sample of the same
          workload, extrapolated: t = t_tree + t_sample * N / S.
--impl reference times that CPU implementation alone (rank 0 only): the
          whole pass over the whole set per step where that fits the run
          (C1 always, C2 when the steps fit ~6 minutes), otherwise a bounded
          target sample per step, extrapolated and labelled "extrapolated".
Multi-GPU (torchrun, N > 1): weak scaling over ONE global set of N x the
1-GPU config (same generator, N x the halos and volume), each rank starting
from an interleaved slice; a step is the whole decomposed pass (key-range
ownership, NCCL all-to-all redistribution and ghost exchange, final per-rank
pass; paper_1612_06090_b200/distributed.py), timed with CUDA events, max over
ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-pair interactions/sec (device-timed)"
UNIT = "pairs/s"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ref-python", action="store_true", help="skip the reference Python/numba timing")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU sample time")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kernel", default="wendland_c6", choices=("wendland_c6", "m4"))
    ap.add_argument("--decompose", action="store_true", help="run the decomposed multi-GPU path even at N=1")
    return ap.parse_args()


def workload_config(cfg: int, seed: int | None, n_ranks: int = 1, device: int | None = None):
    """Config ``cfg``'s inputs.  Clustered configs (2-5) are generated on the
    GPU when ``device`` is given (workload.config_device; the host copy in
    ``pos`` feeds e2e and the CPU baseline), else by the numpy restatement
    of the same generator (the reference arm touches no library kernel)."""
    from paper_1612_06090_b200 import workload
    t0 = time.perf_counter()
    ranks = n_ranks if cfg in (2, 3) else 1  # 4 and 5 scale strongly
    if cfg in (2, 3, 4, 5) and device is not None:
        w = workload.config_device(cfg, seed, device=device, n_ranks=ranks, host_positions=True)
    elif cfg in (2, 3, 4, 5):
        n, box, n_halos, k, conc, x_max = workload._config_table(cfg, ranks)
        seed_ = cfg if seed is None else seed
        if cfg == 5:
            n_bg = int(round(0.05 * n))
            start = np.array([0, n - n_bg], dtype=np.int64)
            halo = np.array([[0.5 * box, 0.5 * box, 0.5 * box, 1.0, 1.0]])
        else:
            start, halo = workload.halo_table(n, box, n_halos, seed_)
        pos = workload.nfw_host_restatement(n, box, start, halo, seed_, conc, x_max).astype(np.float64)
        w = dict(pos=pos, mass=np.full(n, 1.0 / n), h0=np.full(n, workload._initial_h(box, n, k)), k=k, box=box,
                 periodic=True, fp32=True)
    else:
        w = workload.config_weak(cfg, n_ranks, seed)
    w["gen_s"] = time.perf_counter() - t0
    return w


def config_json(w, cfg, n_gpus, kernel):
    desc = {
        1: "C1: 32,768 uniform particles, fp64, K=64, m=1/N, h0=2*N^(-1/3)",
        2: "C2: 1,048,576 particles, fp32, 80% in 200 NFW halos (c=10, dN/dM~M^-1.9 on [100,5e4]) + 20% uniform, "
           "periodic box 100, K=64",
        3: "C3: 16,777,216 particles, fp32, NFW halos (20,000) + background, periodic box 252, K=64",
        4: "C4: 134,217,728 particles, fp32, NFW halos (150,000) + background, periodic box 400, K=64",
        5: "C5: 8,388,608 particles, fp32, single NFW halo c=20 r_vir=1 + 5% background, periodic box 4, K=128",
        6: "diagnostic: 1,048,576 uniform particles, fp32, periodic box 100, K=64 (not a BASELINE config)",
    }[cfg]
    if n_gpus > 1 and cfg in (2, 3, 6):
        desc = (f"{desc.split(':')[0]} weak-scaled x{n_gpus}: {int(w['pos'].shape[0]):,} particles "
                f"({n_gpus} x the 1-GPU set: same generator, {n_gpus}x halos, box side {float(w['box']):.1f})")
    elif n_gpus > 1:
        desc = f"{desc} (strong scaling: the one set over {n_gpus} GPUs)"
    return {"workload": desc, "config_index": cfg, "n_particles": int(w["pos"].shape[0]), "k_neighbors": int(w["k"]),
            "box": float(w["box"]), "periodic": bool(w["periodic"]), "positions": "f32" if w["fp32"] else "f64",
            "kernel": kernel,
            "parallelism": (f"{n_gpus} GPUs: key-range domain decomposition, NCCL all-to-all redistribution + "
                            "ghost exchange" if n_gpus > 1 else "1 GPU"),
            "l2": "flushed before every step (256 MiB device write)",
            "h0": "reference initial_smoothing_length rule" if cfg != 1 else "2*N^(-1/3)",
            "generator": ("splitmix64 counter NFW generator on the device (sph_nfw_positions_device; halo table "
                          "from the host rules)" if cfg in (2, 3, 4, 5) else
                          "reference UniformBox stream (splitmix64)" if cfg == 1 else "numpy uniform")}


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle (reference algorithm restated in C) on a bounded sample
# ---------------------------------------------------------------------------
def _prepared(w):
    """The oracle's octree over the whole set (periodic: + images within
    2 x the largest h0, as density_pass_periodic starts), built once: the
    fixed part of a CPU pass, timed."""
    import oracle
    pos = w["pos"]
    x, y, z = pos[:, 0], pos[:, 1], pos[:, 2]
    t0 = time.perf_counter()
    if w["periodic"]:
        box = float(w["box"])
        prep = oracle.Prepared(x, y, z, box=box, margin=min(0.5 * box, 2.0 * float(np.max(np.abs(w["h0"])))))
    else:
        prep = oracle.Prepared(x, y, z)
    return prep, time.perf_counter() - t0


def _sample_pass(w, prep, size, seed):
    """One timed pass of the CPU port over `size` random targets on the prebuilt tree."""
    import oracle
    n = w["pos"].shape[0]
    rng = np.random.default_rng(seed)
    tg = np.sort(rng.choice(n, size=min(size, n), replace=False))
    t0 = time.perf_counter()
    prep.density_pass(w["mass"], w["h0"], int(w["k"]), tg, threads=oracle.nthreads())
    return time.perf_counter() - t0, tg.size


def cpu_sampled(w, target_seconds: float, seed: int = 0, prep=None, fixed_s: float | None = None):
    """The CPU port on random target samples of the full set.  A pass costs a
    fixed part (periodic images + the single-threaded octree over the whole
    set, built once here and timed) plus a per-target part (search, select,
    density on all host cores, timed on a sample of S targets), so the whole
    pass is extrapolated as t = t_fixed + t_S * N / S."""
    import oracle
    n = w["pos"].shape[0]
    k = int(w["k"])
    threads = oracle.nthreads()
    if prep is None:
        prep, fixed_s = _prepared(w)
    s = min(n, 4096)
    spent = 0.0
    while True:
        t_s, size = _sample_pass(w, prep, s, seed)
        spent += t_s
        if t_s >= 0.5 * target_seconds or size >= n or spent > 4 * target_seconds:
            break
        s = min(n, int(s * max(2.0, min(16.0, 0.6 * target_seconds / max(t_s, 1e-9)))))
    t_full = fixed_s + t_s * n / size
    return {"value": n * k / t_full, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"{size} random targets of {n}: {t_s:.2f}s on the prebuilt tree, plus {fixed_s:.2f}s "
                       f"for the tree itself (images + octree over all {n}, built once); extrapolated "
                       f"t = t_fixed + t_S * N / S = {t_full:.1f}s"),
            "extrapolated": size < n, "measured_s": t_s + fixed_s, "fixed_s": fixed_s, "sample_targets": size,
            "converged_particles_per_s": n / t_full, "cpu_count": os.cpu_count()}


def cpu_full(w):
    """The CPU port over the whole set (every target): one full pass."""
    import oracle
    pos = w["pos"]
    n, k = pos.shape[0], int(w["k"])
    x, y, z = pos[:, 0], pos[:, 1], pos[:, 2]
    threads = oracle.nthreads()
    t0 = time.perf_counter()
    if w["periodic"]:
        oracle.density_pass_periodic(x, y, z, w["mass"], w["h0"], k, float(w["box"]), threads=threads)
    else:
        oracle.density_pass(x, y, z, w["mass"], w["h0"], k, threads=threads)
    t = time.perf_counter() - t0
    return {"value": n * k / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"full pass over all {n} particles ({t:.2f}s)", "extrapolated": False,
            "measured_s": t, "converged_particles_per_s": n / t, "cpu_count": os.cpu_count()}


REF_PKG = os.path.join(ROOT, "baseline", "_ref")  # pip install --target baseline/_ref (offline, git-ignored)

_REF_PY = r"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
import sphlab
n, k = 32768, 64
p = sphlab.generate(sphlab.WorkloadSpec(kind=sphlab.WorkloadKind.UNIFORM_BOX, n_particles=n, box_side=1.0, seed=1),
                    k_neighbors=k)
p["mass"] = 1.0 / n
p["smoothing_length"] = 2.0 * n ** (-1.0 / 3.0)       # BASELINE config 1: h0 = 2 x mean spacing
cores = os.cpu_count() or 1
runs = []
for preset in ("optimised", "original"):
    cfg = sphlab.preset_config(preset, k_neighbors=k)
    sphlab.compute_density_pass(p.copy(), cfg, cores)  # JIT warm-up
    for threads in sorted({1, cores}):
        best = None
        for _ in range(2):
            q = p.copy()
            t0 = time.perf_counter()
            rho, st = sphlab.compute_density_pass(q, cfg, threads)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        runs.append({"preset": preset, "threads": threads, "seconds": best, "pairs_per_s": n * k / best,
                     "iterations": int(st.iteration_count),
                     "checksum": sphlab.bench.density_checksum(rho) if hasattr(sphlab.bench, "density_checksum") else None})
print(json.dumps({"workload": "C1: 32,768 uniform particles (reference generate(UNIFORM_BOX, seed=1)), mass 1/N, "
                              "h0 = 2 N^(-1/3), open boundary (the reference has no periodic mode), K = 64",
                  "numba_version": __import__("numba").__version__, "cpu_count": cores, "runs": runs}))
"""


def reference_python():
    """The reference's own Python/numba compute_density_pass (density.py:286)
    on BASELINE config 1, presets `optimised` (fastest rung) and `original`
    (the paper's baseline), 1 and all host threads, best of 2 after a JIT
    warm-up (SURVEY 8d CPU baseline).  Needs the reference installed in
    baseline/_ref; otherwise reports why it is absent."""
    if not os.path.isdir(os.path.join(REF_PKG, "sphlab")):
        return {"unavailable": "reference package not installed in baseline/_ref"}
    env = dict(os.environ)
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    try:
        r = subprocess.run([sys.executable, "-c", _REF_PY, REF_PKG], env=env, capture_output=True, text=True,
                           timeout=900)
        if r.returncode != 0:
            return {"error": r.stderr.strip().splitlines()[-1:] or ["exit %d" % r.returncode]}
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001 - reported, not fatal
        return {"error": repr(exc)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload_config(args.config, args.seed, max(1, args.gpus))
    n, k = w["pos"].shape[0], int(w["k"])
    steps_total = args.warmup + args.steps
    # full passes when the whole run fits ~6 minutes: C1 always; C2 is
    # probed once (its full pass takes ~20 s on 16 cores)
    full = args.config == 1
    probe = None
    if args.config == 2:
        probe = cpu_full(w)
        full = probe["measured_s"] * steps_total <= 360.0
    vals, measured = [], []
    base = None
    per_step = max(0.5, min(args.cpu_seconds / 2, 120.0 / max(1, steps_total)))
    prep = fixed = None
    if not full:
        prep, fixed = _prepared(w)  # the tree is the fixed part of every pass: built and timed once
        size = None
    for step in range(steps_total):
        if full:
            base = probe if (probe is not None and step == 0) else cpu_full(w)
        elif size is None:
            base = cpu_sampled(w, target_seconds=per_step, seed=step, prep=prep, fixed_s=fixed)
            size = base["sample_targets"]  # later steps: one sample pass of this size each
        else:
            t_s, _ = _sample_pass(w, prep, size, step)
            t_full = fixed + t_s * n / size
            base = dict(base, value=n * k / t_full, measured_s=t_s + fixed,
                        converged_particles_per_s=n / t_full,
                        sample=(f"{size} random targets of {n}: {t_s:.2f}s on the prebuilt tree, plus {fixed:.2f}s "
                                f"for the tree (built once); extrapolated t = t_fixed + t_S * N / S = {t_full:.1f}s"))
        if step >= args.warmup:
            vals.append(base["value"])
            measured.append(base["measured_s"])
    value = statistics.median(vals)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": n * k / value * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(w, args.config, args.gpus, "wendland_c6"), "impl": "reference",
            "extrapolated": not full,
            "measured_ms_per_step": statistics.median(measured) * 1e3,
            "cpu_baseline": dict(base, value=value),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "converged_particles_per_s": n / (n * k / value)}
    if not full:
        line["note"] = ("each step times one pass of the CPU port over a bounded random target sample of the full "
                        "set on its octree (built and timed once: the fixed part of every pass); ms_per_step is the "
                        "extrapolated time of a whole pass t_fixed + t_S * N / S, measured_ms_per_step the sample "
                        "pass plus the tree build")
    if not args.no_ref_python:
        line["reference_python"] = reference_python()
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import ctypes

    import torch

    from paper_1612_06090_b200 import _lib
    from paper_1612_06090_b200.density import density_pass_soa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.decompose:
        return run_decomposed(args, world, rank, local)
    dist = False
    if dist:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local
    torch.cuda.set_device(device)
    seed = (args.seed if args.seed is not None else args.config) + 1000 * rank
    w = workload_config(args.config, seed, device=device)
    n, k = w["pos"].shape[0], int(w["k"])
    pos = w["pos"]
    f32 = bool(w["fp32"])
    pdt = torch.float32 if f32 else torch.float64
    if "x" in w:  # generated on the device
        dx, dy, dz = w["x"], w["y"], w["z"]
    else:
        dx = torch.from_numpy(np.ascontiguousarray(pos[:, 0])).to(device=device, dtype=pdt)
        dy = torch.from_numpy(np.ascontiguousarray(pos[:, 1])).to(device=device, dtype=pdt)
        dz = torch.from_numpy(np.ascontiguousarray(pos[:, 2])).to(device=device, dtype=pdt)
    dm = torch.from_numpy(w["mass"]).to(device)
    dh0 = torch.from_numpy(w["h0"]).to(device)
    dh = dh0.clone()
    drho = torch.empty(n, dtype=torch.float64, device=device)
    dfl = torch.empty(n, dtype=torch.uint8, device=device)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)

    L = _lib.load()
    ctx = _lib.context(device)
    stream = torch.cuda.ExternalStream(_lib.stream_handle(ctx), device=device)
    prm = _lib.SphParams(n=n, k=k, max_iterations=100, precision=_lib.PRECISION["f32" if f32 else "f64"],
                         periodic=1 if w["periodic"] else 0, box=float(w["box"]), kernel=_lib.KERNELS[args.kernel],
                         reserved=0)
    vp = ctypes.c_void_p

    def one_pass(st):
        rc = L.sph_density_pass_device(ctx, prm, vp(dx.data_ptr()), vp(dy.data_ptr()), vp(dz.data_ptr()),
                                       vp(dm.data_ptr()), vp(dh.data_ptr()), vp(drho.data_ptr()),
                                       vp(dfl.data_ptr()), st)
        if rc != _lib.SPH_OK:
            raise RuntimeError(f"density pass failed ({rc}): {_lib.last_error(ctx)}")

    st = _lib.SphStats()
    for i in range(args.warmup):
        with torch.cuda.stream(stream):
            dh.copy_(dh0)
            flush.fill_(i & 255)
        one_pass(st)
    torch.cuda.synchronize(device)
    if dist:
        tdist.barrier()
    torch.cuda.synchronize(device)

    clocks = ClockSampler(device)
    clocks.start()
    step_ms, kern = [], {"search": 0.0, "select": 0.0, "density": 0.0, "tree": 0.0}
    tests = accepted = search_tests = launches = 0
    stage_tot = {}
    last = None
    known_ms = 0.0
    for i in range(args.steps):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            dh.copy_(dh0)
            flush.fill_((i + 7) & 255)
            ev0.record(stream)
        st = _lib.SphStats()
        one_pass(st)
        with torch.cuda.stream(stream):
            ev1.record(stream)
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
        d = st.as_dict()
        for kk in kern:
            kern[kk] += d["t_kernel_ms"][kk]
        for kk, v in d["t_stage_ms"].items():
            stage_tot[kk] = stage_tot.get(kk, 0.0) + v
        tests += d["pair_tests"]
        accepted += d["accepted_pairs"]
        search_tests += d["search_pair_tests"]
        launches += d["gpu_launches"]
        known_ms += d.get("t_known_ms", 0.0)
        last = d
    torch.cuda.synchronize(device)
    clk = clocks.stop()
    ms_per_step = statistics.median(step_ms)
    t_local = torch.tensor([ms_per_step], dtype=torch.float64, device=device)
    n_total = torch.tensor([float(n)], dtype=torch.float64, device=device)
    if dist:
        tdist.all_reduce(t_local, op=tdist.ReduceOp.MAX)
        tdist.all_reduce(n_total, op=tdist.ReduceOp.SUM)
        tdist.barrier()
    ms_max = float(t_local.item())
    total_particles = float(n_total.item())
    value = total_particles * k / (ms_max * 1e-3)

    # ---- roofline of the search launches (k_target calibration sample + k_lane + k_target leftovers: 92 % of the pass) ----
    peak_ffma = float(L.sph_fp32_peak(ctx))
    t_k = kern["search"] + kern["select"] + kern["density"]
    ops = 6.0 * tests + 10.0 * accepted
    achieved = ops / (t_k * 1e-3) / 1e12 if t_k > 0 else 0.0
    peak = peak_ffma / 1e12
    traffic = None
    issue = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            # measured on one config only: attached to that config's line
            if int(pj.get("config_index", 2)) == int(args.config):
                traffic = pj.get("search_bytes_per_launch")
            issue = {"issue_slots_busy": pj.get("issue_slots_busy"), "warp_instructions": pj.get("warp_instructions")}
        except Exception:
            traffic = None

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if f32 else "f64", "data": "synthetic",
            "config": config_json(w, args.config, world, args.kernel),
            "converged_particles_per_s": total_particles / (ms_max * 1e-3),
            "gpu_launches": launches // args.steps,
            "clocks": clk,
            "roofline": {"bound": "fp32", "kernel": "search launches: k_lane (one lane per target over bundles of 32 sorted neighbours) + k_target (the calibration sample and what k_lane leaves)", "achieved": achieved, "peak": peak,
                         "unit": "Tops/s (fp32-pipe ops)", "frac": achieved / peak if peak else None,
                         "traffic": traffic,
                         "peak_source": "measured FFMA issue rate on this B200 (sph_fp32_peak); MEASURED_PEAKS.json "
                                        "has no FP32 vector figure",
                         "ops_model": "6 per executed pair test, +10 per accepted pair (density); useful_frac counts only N*K pair "
                                      "tests and N*(K+1) kernel terms",
                         "useful_frac": ((6.0 * n * k + 10.0 * n * (k + 1)) * args.steps / (t_k * 1e-3) / 1e12 / peak) if (t_k > 0 and peak) else None,
                         "traffic_unit": "DRAM bytes (read + write) of the search launches of one pass, ncu",
                         "issue_bound": issue},
            "search_efficiency": n * k / (search_tests / args.steps) if search_tests else None,
            "pair_tests_per_step": tests / args.steps,
            "kernel_ms_per_step": {kk: v / args.steps for kk, v in kern.items()},
            "known_ms_per_step": known_ms / args.steps,
            "known_fallbacks": last.get("known_fallbacks") if last else None,
            "stage_ms_per_step": {kk: v / args.steps for kk, v in stage_tot.items()},
            "todo_sizes": last["todo_sizes"] if last else None,
            "search_rounds": last["search_rounds"] if last else None,
            "select_rounds": last["select_rounds"] if last else None}

    # ---- end to end through the public API with pinned host buffers ----
    if not args.no_e2e:
        def pinned(a):
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return t, t.numpy()
        hx = pinned(pos[:, 0].astype(np.float32 if f32 else np.float64))
        hy = pinned(pos[:, 1].astype(np.float32 if f32 else np.float64))
        hz = pinned(pos[:, 2].astype(np.float32 if f32 else np.float64))
        hm = pinned(w["mass"])
        hh = pinned(w["h0"].copy())
        hrho = pinned(np.zeros(n))
        hfl = pinned(np.zeros(n, dtype=np.uint8))
        e2e_ms = []
        for i in range(args.warmup + args.steps):
            hh[1][:] = w["h0"]
            torch.cuda.synchronize(device)
            t0 = time.perf_counter()
            density_pass_soa(hx[1], hy[1], hz[1], hm[1], None, k, periodic=bool(w["periodic"]),
                             box=float(w["box"]), kernel=args.kernel, device=device, out=(hh[1], hrho[1], hfl[1]))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                e2e_ms.append(dt * 1e3)
        e2e_local = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device=device)
        if dist:
            tdist.all_reduce(e2e_local, op=tdist.ReduceOp.MAX)
        e_ms = float(e2e_local.item())
        es = 4 if f32 else 8
        line["e2e"] = {"value": total_particles * k / (e_ms * 1e-3), "unit": UNIT,
                       "h2d_bytes_per_step": int(n * (3 * es + 8 + 8)), "d2h_bytes_per_step": int(n * (8 + 8 + 1)),
                       "ms_per_step": e_ms, "api": "paper_1612_06090_b200.density_pass_soa (C ABI sph_density_pass), "
                                                   "pinned host buffers"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_sampled(w, args.cpu_seconds)
        except Exception as exc:  # the baseline is reported, never gating
            line["cpu_baseline"] = {"error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


def run_decomposed(args, world, rank, local):
    """N > 1: one global weak-scaled set (N x the 1-GPU config), each rank
    starting from an interleaved slice of it; a step is the whole decomposed
    pass (bbox all-reduce, keys, splitters, NCCL all-to-all redistribution,
    bounds, ghost exchange, the final per-rank pass)."""
    import torch
    import torch.distributed as tdist

    from paper_1612_06090_b200 import distributed as D

    # test hooks: SPH_BENCH_DEVICE pins every rank to one GPU and
    # SPH_BENCH_BACKEND=gloo replaces NCCL, so the torchrun path can be run
    # with several ranks on a one-GPU box (tests/test_gpu_distributed.py)
    if os.environ.get("SPH_BENCH_DEVICE") is not None:
        local = int(os.environ["SPH_BENCH_DEVICE"])
    backend = os.environ.get("SPH_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world == 1:  # --decompose outside torchrun
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "MASTER_PORT" not in os.environ:
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    if backend == "nccl":
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        tdist.init_process_group(backend)
    device = local

    def red(t, op=None):  # all-reduce in place (host staging for gloo)
        h = t.cpu() if backend == "gloo" else t
        tdist.all_reduce(h, op=op if op is not None else tdist.ReduceOp.SUM)
        if h is not t:
            t.copy_(h)

    w = workload_config(args.config, args.seed, world, device=local)
    n_glob, k = w["pos"].shape[0], int(w["k"])
    sel = np.arange(rank, n_glob, world)
    f32 = bool(w["fp32"])
    pdt = torch.float32 if f32 else torch.float64
    npdt = np.float32 if f32 else np.float64
    hp = [np.ascontiguousarray(w["pos"][sel, i].astype(npdt)) for i in range(3)]
    hm, hh0 = np.ascontiguousarray(w["mass"][sel]), np.ascontiguousarray(w["h0"][sel])
    dx, dy, dz = (torch.from_numpy(a).to(device) for a in hp)
    dm, dh0 = torch.from_numpy(hm).to(device), torch.from_numpy(hh0).to(device)
    dgid = torch.from_numpy(sel.astype(np.int64)).to(device)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    compute = D.LibCompute(device)
    periodic, box = bool(w["periodic"]), float(w["box"])

    def step(x, y, z, m, h0, gid):
        return D.decomposed_pass(x, y, z, m, h0, gid, k, compute, periodic=periodic, box=box)

    for i in range(args.warmup):
        flush.fill_(i & 255)
        r = step(dx, dy, dz, dm, dh0, dgid)
    torch.cuda.synchronize(device)
    tdist.barrier()
    torch.cuda.synchronize(device)
    clocks = ClockSampler(device)
    clocks.start()
    step_ms = []
    for i in range(args.steps):
        flush.fill_((i + 7) & 255)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        r = step(dx, dy, dz, dm, dh0, dgid)
        ev1.record()
        ev1.synchronize()
        step_ms.append(ev0.elapsed_time(ev1))
    torch.cuda.synchronize(device)
    tdist.barrier()
    clk = clocks.stop()
    st = compute.last_stats or {}
    t_local = torch.tensor([statistics.median(step_ms)], dtype=torch.float64, device=device)
    red(t_local, tdist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    info = torch.tensor([r.n_owned, r.n_ghosts, r.n_owned, r.n_owned], dtype=torch.float64, device=device)
    isum = info.clone()
    red(isum)
    imax = info.clone()
    red(imax, tdist.ReduceOp.MAX)
    imin = info.clone()
    red(imin, tdist.ReduceOp.MIN)
    value = n_glob * k / (ms_max * 1e-3)

    # end to end: pinned host slices in, owned (gid, h, rho) back to the host
    e2e = None
    if not args.no_e2e:
        pin = [torch.from_numpy(a).pin_memory() for a in (*hp, hm, hh0, sel.astype(np.int64))]
        e2e_ms = []
        outs = None  # pinned result buffers (the owned count is fixed for a fixed input)
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize(device)
            tdist.barrier()
            t0 = time.perf_counter()
            d = [t.to(device, non_blocking=True) for t in pin]
            rr = step(*d)
            src = (rr.gid, rr.h, rr.rho)
            if outs is None or outs[0].numel() != src[0].numel():
                outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in src]
            for o, t in zip(outs, src):
                o.copy_(t, non_blocking=True)
            torch.cuda.synchronize(device)
            out = outs
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                e2e_ms.append(dt * 1e3)
        el = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device=device)
        red(el, tdist.ReduceOp.MAX)
        es = 4 if f32 else 8
        e2e = {"value": n_glob * k / (float(el.item()) * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(len(sel) * (3 * es + 8 + 8 + 8)),
               "d2h_bytes_per_step": int(out[0].numel() * (8 + 8 + 8)), "ms_per_step": float(el.item()),
               "api": "paper_1612_06090_b200.distributed.decomposed_pass (per-rank C ABI sph_density_pass_device), "
                      "pinned host slices, max over ranks"}
    if rank == 0:
        tk = st.get("t_kernel_ms", {})
        t_k = tk.get("search", 0.0) + tk.get("select", 0.0) + tk.get("density", 0.0)
        peak = float(compute.L.sph_fp32_peak(compute.ctx)) / 1e12
        ops = 6.0 * st.get("pair_tests", 0) + 10.0 * st.get("accepted_pairs", 0)
        achieved = ops / (t_k * 1e-3) / 1e12 if t_k > 0 else 0.0
        scaling = "weak" if args.config in (2, 3, 6) else "strong"  # workload.config_weak scales 2, 3, 6
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32" if f32 else "f64", "data": "synthetic",
                "config": config_json(w, args.config, world, args.kernel),
                "converged_particles_per_s": n_glob / (ms_max * 1e-3),
                "gpu_launches": int(st.get("gpu_launches", 0)) + 1,
                "clocks": clk,
                "roofline": {"bound": "fp32", "kernel": "k_target (rank 0's final pass)", "achieved": achieved,
                             "peak": peak, "unit": "Tops/s (fp32-pipe ops)", "frac": achieved / peak if peak else None,
                             "traffic": None, "ops_model": "6 per pair test, +10 per accepted pair (density)"},
                "decomposition": {"owned_min": int(imin[0].item()), "owned_max": int(imax[0].item()),
                                  "ghosts_total": int(isum[1].item()), "ghosts_max": int(imax[1].item()),
                                  "final_pass_ms_rank0": st.get("t_stage_ms", {}).get("total")},
                "e2e": e2e}
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
