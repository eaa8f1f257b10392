#!/usr/bin/env python
"""Benchmark of the B200 e–e Coulomb collision operator (arXiv 2508.06771, step S1).

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  A "step" is one call of the whole hot path
(coulomb_collide: count -> scan -> stable scatter -> pair + TA collide ->
moments/diagnostics) on one batch of synthetic input resident in HBM.

Workload (BASELINE.json configs[3], "C4"): 64 x 64 = 4096 cells x 25,000
electrons = 1.024e8 e- per GPU, isotropic Maxwellian 2 eV.  The headline is
the steady state of a PIC loop: each step consumes the previous step's
(cell-sorted, pair-ordered) output after a stand-in drift moved 2% of the
electrons to a neighbour cell; the first step starts from a random particle
order (the paper stores particles unsorted).  "cold" (the same randomly
ordered input every step) and "warm" (sorted input, no drift) are reported
beside it.  The operator picks its binning mode on the device from the input's
order: steady -> index mode (4-byte indices), cold -> record mode
(32-byte records), warm -> sorted mode (nothing moved); the R1 whole-cell pairing
(CC_CELL_UNIFORM) is timed as a variant.  Inputs are 2.87 GB, far larger than the
126 MB L2, so no flush is needed between steps.  For N > 1 (torchrun) each rank owns a C5 shard: global
cells [4096 r, 4096 (r+1)) of a 64 x 64N grid, its own data seed; the stand-in
drift of SURVEY §8(e) moves particles of the shard's first and last cell rows
across the shard boundary (p = 0.1), and the step includes their migration to
the owning rank (NCCL) and the diagnostics reduction.  Weak scaling.

Roofline accounting: the method's algorithmic bytes are 52 per
particle (read v 24 + cell 4, write v 24); ``roofline`` divides them by the
dominant kernel's event-timed duration, ``step_hbm`` by the whole step's.  The
DRAM bytes ncu measured for the same kernels (profiles/traffic.json, stamped
with the hash of the kernel sources; a stale file is refused) are reported
beside them with their ratio to the algorithmic bytes.

``--impl reference`` times the CPU oracle (oracle/, as it stands) on the host
cores instead, on a bounded sample of the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "electron-electron pair collisions/sec (TA77 Coulomb operator step, fp64)"
UNIT = "pair-collisions/s"
# algorithmic bytes per particle: the method must read v (24 B)
# and the cell id (4 B) and write v (24 B) once per step — the per-unit figure of every roofline
ALGO_BYTES = 52
# SURVEY §8(d) design traffic per particle: cold (unsorted input) and warm (cell-sorted input)
DESIGN_BYTES = {"cold": 112, "warm": 56}
# the binning mode the device picks for each bench workload (k_count's descents) and
# what each kernel's own contract moves once per particle in it (informative, not the roofline):
#   steady -> index mode: scatter reads the cell id twice and writes a 4-byte index; the collide
#             reads the index and v (24) and writes v, cell, perm (32)
#   cold   -> record mode: scatter reads cell twice + v, writes a 32-byte record; collide reads it back
#   warm   -> sorted mode: no scatter; the collide reads v straight from the input
BIN_MODE = {"steady": "index", "steady_nomig": "index", "cold": "record", "warm": "sorted"}
STAGE_CONTRACT_BYTES = {"index": {"count": 4, "scatter": 12, "collide": 4 + 24 + 32},
                        "record": {"count": 4, "scatter": 8 + 24 + 32, "collide": 32 + 32},
                        "sorted": {"count": 4, "scatter": 0, "collide": 24 + 32}}
PIPELINE_BYTES = {m: sum(b.values()) for m, b in STAGE_CONTRACT_BYTES.items()}   # 76 / 132 / 60
KERNEL_SOURCES = ("paper_2508_06771_b200/csrc/cc_kernels.cu", "paper_2508_06771_b200/csrc/cc_device.cuh",
                  "include/coulomb.h")


def sources_sha() -> str:
    """Hash of the kernel sources: stamps profiles/traffic.json so a capture of older kernels is refused."""
    import hashlib
    h = hashlib.sha256()
    for f in KERNEL_SOURCES:
        h.update(open(os.path.join(ROOT, f), "rb").read())
    return h.hexdigest()[:16]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--per-cell", type=int, default=25_000)
    ap.add_argument("--nx", type=int, default=64)
    ap.add_argument("--ny", type=int, default=64)
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--e2e-buffers", type=int, default=2, help="streams / device buffers of the e2e pipeline")
    ap.add_argument("--drift", type=float, default=0.02, help="fraction of electrons changing cell per step")
    ap.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for N > 1 (nccl; gloo "
                    "only to smoke-test the multi-rank path when fewer GPUs than ranks are available)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pic", action="store_true", help="skip the NEXT f2 PIC-loop section")
    ap.add_argument("--cpu-cells", type=int, default=96,
                    help="cells of the C4 workload the CPU baseline processes per step")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, rank):
    import workloads as W
    if rank == 0 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        return W.c4(nx=args.nx, ny=args.ny, per_cell=args.per_cell)
    return W.c5_rank(rank, nx=args.nx, ny=args.ny, per_cell=args.per_cell)


def workload_name(args, world):
    base = f"C4 2D argon discharge {args.nx}x{args.ny} cells x {args.per_cell} e-/cell, Maxwellian 2 eV"
    if world > 1:
        return f"C5 weak scaling: {base} per GPU, cell-range sharded over {world} GPUs"
    return base


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~2 ms from a background thread; `mark()` brackets the timed region and
    `summary()` keeps the samples taken inside it.  (nvidia-smi -lms could not
    resolve a ~70 ms timed region: round-1 runs recorded 0 samples.)"""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.samples = []          # (time, sm_mhz, reasons bitmask)
        self.t0 = self.t1 = None
        self.max_mhz = None
        self.err = None
        self._stop = threading.Event()

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = self.index
            if vis:                                  # NVML indexes physical GPUs
                ids = [x.strip() for x in vis.split(",") if x.strip()]
                if idx < len(ids) and ids[idx].isdigit():
                    idx = int(ids[idx])
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception as e:                       # never let clock sampling kill the bench
            self.err = repr(e)
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.time(), float(sm), int(rs)))
            except Exception as e:
                self.err = repr(e)
                return
            time.sleep(self.period)

    def mark(self, begin: bool):
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        self._stop.set()
        if hasattr(self, "thread"):
            self.thread.join(timeout=2)

    def summary(self):
        s = self.samples
        if self.t0 is not None and self.t1 is not None:
            s = [x for x in s if self.t0 <= x[0] <= self.t1]
        if not s:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "source": "nvml", "error": self.err}
        N = self.N
        reasons = sorted({nm for _, _, rs in s for nm, attr in self.REASONS
                          if hasattr(N, attr) and rs & getattr(N, attr)})
        return {"sm_mhz": statistics.median(x[1] for x in s), "sm_min_mhz": min(x[1] for x in s),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(s),
                "source": "nvml, 2 ms period, timed region of the headline mode"}


# ---------------------------------------------------------------- CPU oracle (baseline / reference arm)


def oracle_sample(args, cells_per_step, seed_offset=4):
    """A bounded sample of the C4 workload: the first `cells_per_step` cells
    (25,000 e- each, Maxwellian 2 eV), randomly ordered like the full input."""
    import workloads as W
    w = W.c4(nx=1, ny=cells_per_step, per_cell=args.per_cell, seed_offset=seed_offset)
    return w


def time_oracle(args, steps, cells_per_step):
    import oracle
    oracle.build()
    w = oracle_sample(args, cells_per_step)
    p = w.params()
    oracle.coulomb_collide(w.v[:, :2000], np.zeros(2000, np.int32), 1, want_pairs=False, **p)  # load/warm
    t0 = time.perf_counter()
    for s in range(steps):
        r = oracle.coulomb_collide(w.v, w.cell, w.cells, step=s, want_pairs=False, **p)
    dt = time.perf_counter() - t0
    pairs = float(r.diag[2]) * steps
    return {"value": pairs / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{cells_per_step} of {args.nx * args.ny} C4 cells ({w.n:.3g} e-, "
                      f"{int(r.diag[2])} pairs) per step, {steps} step(s), {dt:.1f} s wall",
            "seconds": dt}


def time_oracle_on(w, args):
    """The oracle as it stands, on the host cores, on the SAME resident C4 input
    (one step; ~1e8 e- is 5-30 s of CPU work depending on the core count)."""
    import oracle
    oracle.build()
    p = w.params()
    t0 = time.perf_counter()
    r = oracle.coulomb_collide(w.v, w.cell, w.cells, step=0, want_pairs=False, **p)
    dt = time.perf_counter() - t0
    cores = oracle.num_threads()
    # the oracle also single-threaded on C1-C3 and on all cores on C3 (one step each)
    import workloads as W
    per_config = {}
    for name, wl, threads in (("C1_1_thread", W.c1(), 1), ("C2_1_thread", W.c2(), 1), ("C3_1_thread", W.c3(), 1),
                              (f"C3_{cores}_threads", W.c3(), cores)):
        oracle.set_num_threads(threads)
        t1 = time.perf_counter()
        rr = oracle.coulomb_collide(wl.v, wl.cell, wl.cells, step=0, want_pairs=False, **wl.params())
        s1 = time.perf_counter() - t1
        per_config[name] = {"seconds": s1, "pair_collisions_per_s": float(rr.diag[2]) / s1}
    oracle.set_num_threads(cores)
    return {"value": float(r.diag[2]) / dt, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(),
            "nproc": os.cpu_count(), "kind": "oracle",
            "sample": f"the full C4 input ({w.n:.4g} e-, {int(r.diag[2])} pairs), 1 step, {dt:.1f} s wall",
            "seconds": dt, "configs": per_config}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    steps = max(args.steps, 1)
    # bounded: each step processes a sample sized so the whole run stays within minutes
    cells = max(4, min(args.cpu_cells, int(1200 / max(steps + args.warmup, 1))))
    import oracle
    oracle.build()
    w = oracle_sample(args, cells)
    p = w.params()
    for s in range(args.warmup):
        oracle.coulomb_collide(w.v, w.cell, w.cells, step=1000 + s, want_pairs=False, **p)
    t0 = time.perf_counter()
    for s in range(steps):
        r = oracle.coulomb_collide(w.v, w.cell, w.cells, step=s, want_pairs=False, **p)
    dt = time.perf_counter() - t0
    pairs = float(r.diag[2]) * steps
    value = pairs / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_name(args, 1) + f" — CPU oracle on a {cells}-cell sample per step",
                   "cells_per_step": cells, "electrons_per_step": w.n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "cpu_model": cpu_model(),
                         "nproc": os.cpu_count(), "kind": "oracle",
                         "sample": f"{cells} of {args.nx * args.ny} C4 cells ({w.n:.3g} e-) per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm


def drift_cells(cell, nx, ny, frac, gen):
    """Stand-in pusher (workload generation, not the operator): each live
    particle moves to a random von-Neumann neighbour cell of the periodic
    nx x ny grid with probability `frac` (SURVEY §8(e)/(f2) stand-in drift)."""
    import torch
    live = cell >= 0
    r = torch.rand(cell.numel(), generator=gen, device=cell.device)
    mv = (r < frac) & live
    d = torch.clamp((r * (4.0 / frac)).to(torch.int32), max=3)
    cx = torch.remainder(cell, nx)
    cy = torch.div(cell, nx, rounding_mode="floor")
    cx = torch.where(mv & (d == 0), torch.remainder(cx + 1, nx), cx)
    cx = torch.where(mv & (d == 1), torch.remainder(cx - 1, nx), cx)
    cy = torch.where(mv & (d == 2), torch.remainder(cy + 1, ny), cy)
    cy = torch.where(mv & (d == 3), torch.remainder(cy - 1, ny), cy)
    cell.copy_(torch.where(live, cy * nx + cx, cell))


def drift_cells_global(cell, nx, ny, rank, world, frac, gen, p_boundary=0.1):
    """The C5 stand-in pusher on several ranks: LOCAL ids in, GLOBAL ids out on the
    64 x 64P grid whose rows [ny r, ny (r+1)) rank r owns.  Every live particle takes the random
    neighbour move of drift_cells (periodic over the GLOBAL grid, so the first and last local rows
    can leave the shard), and a particle in the shard's first or last row additionally moves one
    row outward, across the shard boundary, with probability p_boundary (a Philox-free torch
    draw: workload generation, not the operator)."""
    import torch
    live = cell >= 0
    g = torch.where(live, cell + rank * nx * ny, cell)
    r = torch.rand(cell.numel(), generator=gen, device=cell.device)
    rb = torch.rand(cell.numel(), generator=gen, device=cell.device)
    gy_total = ny * world
    mv = (r < frac) & live
    d = torch.clamp((r * (4.0 / frac)).to(torch.int32), max=3)
    cx = torch.remainder(g, nx)
    cy = torch.div(g, nx, rounding_mode="floor")
    cx = torch.where(mv & (d == 0), torch.remainder(cx + 1, nx), cx)
    cx = torch.where(mv & (d == 1), torch.remainder(cx - 1, nx), cx)
    cy = torch.where(mv & (d == 2), torch.remainder(cy + 1, gy_total), cy)
    cy = torch.where(mv & (d == 3), torch.remainder(cy - 1, gy_total), cy)
    ly = cy - rank * ny
    out = (rb < p_boundary) & live
    cy = torch.where(out & (ly == 0), torch.remainder(cy - 1, gy_total), cy)
    cy = torch.where(out & (ly == ny - 1), torch.remainder(cy + 1, gy_total), cy)
    cell.copy_(torch.where(live, cy * nx + cx, cell))


def hbm_peak_gbs() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def pic_section(args, dev, w, K):
    """NEXT f2: the subcycled PIC loop (PicLoop: per substep coulomb_collide + cc_push,
    every 10 substeps the Coulomb-log feedback), one GPU.  C4 grid (64 x 64 cells of
    5 mm, periodic, field-free, dt = 1e-10 s: ~1.9% of the electrons change cell per
    step) timed over whole field steps replayed from a CUDA graph; C1 / C2 (launch-
    bound, one cell) with the graph and eagerly."""
    import torch
    import workloads as W
    import paper_2508_06771_b200 as cc
    from paper_2508_06771_b200.pic import PicLoop

    def timed(loop, F):
        loop.field_step()                      # capture (graph) / warm-up; re-sorts cold input
        loop.field_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(F):
            loop.field_step()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (F * loop.k)

    out = {}
    nx, ny = args.nx, args.ny
    x = torch.from_numpy(W.positions_in_cells(w.cell, nx, ny, seed=77)).to(dev)
    grid = cc.Grid(2, (nx, ny), (W.PIC_DX, W.PIC_DX), 3)
    prm = dict(dt=w.dt, weight=w.weight, cell_volume=w.cell_volume)
    F = max(1, K // 10)
    loop = PicLoop(x, torch.from_numpy(w.v).to(dev), torch.from_numpy(w.cell).to(dev), grid, subcycles=10,
                   graph=True, fused=True, **prm)
    ms_fused = timed(loop, F)
    del loop
    loop = PicLoop(x, torch.from_numpy(w.v).to(dev), torch.from_numpy(w.cell).to(dev), grid, subcycles=10,
                   graph=True, fused=False, **prm)
    ms = timed(loop, F)
    pairs = float(loop.diag[2].item())
    # the push alone, on the loop's current state (eager, events on the stream)
    xs, vs, cs = loop.state
    perm = torch.arange(w.n, dtype=torch.int32, device=dev)
    v2, c2 = vs.clone(), cs.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xo = torch.empty_like(xs)
    cc.cc_push(xs, v2, c2, grid, dt=w.dt, perm=perm, x_out=xo)
    e0.record()
    for _ in range(3):                         # single GPU: output ids are valid input ids again
        cc.cc_push(xs, v2, c2, grid, dt=w.dt, perm=perm, x_out=xo)
    e1.record()
    torch.cuda.synchronize()
    push_ms = e0.elapsed_time(e1) / 3
    # cc_push algorithmic bytes, 2D field-free: read perm 4 + cell 4 + v 24 + x 16, write x 16 + cell 4
    push_bytes = 68 * w.n
    peak = hbm_peak_gbs()
    out["c4"] = {"ms_per_substep": ms, "pair_collisions_per_s": pairs / (ms * 1e-3),
                 "ms_per_substep_fused_push": ms_fused,
                 "push_ms": push_ms,
                 "push_roofline": {"kernel": "k_push", "bound": "hbm", "achieved": push_bytes / (push_ms * 1e-3) / 1e9,
                                   "peak": peak, "unit": "GB/s",
                                   "frac": push_bytes / (push_ms * 1e-3) / 1e9 / peak,
                                   "algorithmic_bytes_per_particle": 68},
                 "field_steps_timed": F, "subcycles": 10,
                 "cells_changed_per_step": "~1.9% (5 mm cells, 2 eV, dt 1e-10 s)",
                 "what": "PicLoop field steps replayed from one CUDA graph: per substep coulomb_collide + cc_push "
                         "(the default); ms_per_substep_fused_push: the push inside the collision call's output "
                         "stage (cc_params.push)"}
    del loop, x, xs, vs, cs, v2, c2, xo, perm
    for name, wl in (("c1", W.c1()), ("c2", W.c2())):
        g1 = cc.Grid(1, (1,), (W.PIC_DX,), 1)
        xx = torch.from_numpy(W.positions_in_cells(wl.cell, 1, 1, seed=78)).to(dev)
        r = {}
        for mode in ("graph", "eager"):
            lp = PicLoop(xx, torch.from_numpy(wl.v).to(dev), torch.from_numpy(wl.cell).to(dev), g1, subcycles=10,
                         graph=(mode == "graph"), dt=wl.dt, weight=wl.weight, cell_volume=wl.cell_volume)
            r[mode + "_ms_per_substep"] = timed(lp, 5)
        r["n"] = wl.n
        out[name] = r
    return out


def p2c_section(dev, w):
    """NEXT f4: the paper's atomic, sub-binned P2C (cc_p2c + cc_p2c_moments) on the C4 particles,
    unsorted (the paper's storage) and cell-sorted, 1 and 16 sub-bins per cell."""
    import torch
    import paper_2508_06771_b200 as cc
    v = torch.from_numpy(w.v).to(dev)
    cell = torch.from_numpy(w.cell).to(dev)
    order = torch.argsort(cell.to(torch.int64), stable=True)
    vs, cs = v[:, order].contiguous(), cell[order].contiguous()
    scratch = torch.empty(w.cells * 16 * 7, dtype=torch.float64, device=dev)
    peak = hbm_peak_gbs()
    out = {}
    for name, (vv, cc_) in (("unsorted", (v, cell)), ("sorted", (vs, cs))):
        for sub in (1, 16):
            raw = cc.cc_p2c(vv, cc_, w.cells, sub=sub, scratch=scratch)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                raw = cc.cc_p2c(vv, cc_, w.cells, sub=sub, scratch=scratch)
                cc.cc_p2c_moments(raw, weight=w.weight, cell_volume=w.cell_volume)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            # algorithmic bytes: read v 24 + cell 4 per particle
            out[f"{name}_sub{sub}_ms"] = ms
            out[f"{name}_sub{sub}_hbm_frac"] = 28 * w.n / (ms * 1e-3) / 1e9 / peak
    out["what"] = ("atomic P2C (7 fp64 red.add per particle into [cells][sub] bins) + fixed-order sub-bin "
                   "reduction + moments; algorithmic 28 B/particle")
    # NEXT f3: recombination C5 on a collision output (cell-sorted, pair order), per-cell primary probability
    res = cc.coulomb_collide(v, cell, w.cells, step=1, dt=w.dt, weight=w.weight, cell_volume=w.cell_volume)
    rec = {}
    for pr in (1e-3, 0.1):
        prob = torch.full((w.cells,), pr, dtype=torch.float64, device=dev)
        times = []
        for rep in range(3):               # each call on a fresh copy of the collision output (precondition)
            vv, ccell = res.v_out.clone(), res.cell_out.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = cc.cc_recombine(vv, ccell, prob, eps_bind=15.76 * 1.602176634e-19, step=1 + rep)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = min(times[1:])
        rec[f"prob_{pr:g}"] = {"ms": ms, "particles_per_s": w.n / (ms * 1e-3), "stats": st.tolist()}
    rec["what"] = ("cc_recombine on the C4 collision output (fresh copy per call; min of 2 after a warm-up); "
                   "one Philox draw per particle (per-warp ordered primary lists, catalytes by binary search), "
                   "no per-particle memory traffic except the matched pairs and the kill-marker pass: bound by "
                   "integer ALU, not HBM")
    return {"p2c": out, "recombination": rec}


def configs_section(dev):
    """BASELINE configs C1-C3 (parity-test sizes) and C4b (C4 with a 2D sine density profile, cells
    up to ~62,000 e-) timed through the operator: cold (the
    workload's random order every step) and warm (each step consumes the previous output),
    mean of 20 calls after 3 warm-up calls, CUDA events; C1/C2 are launch/latency-bound, so they are
    also timed as 20 chained steps replayed from one CUDA graph (graph_ms_per_step)."""
    import torch
    import workloads as W
    import paper_2508_06771_b200 as cc
    out = {}
    for name, w in (("C1", W.c1()), ("C2", W.c2()), ("C3", W.c3()), ("C4b", W.c4b())):
        v0, c0 = torch.from_numpy(w.v).to(dev), torch.from_numpy(w.cell).to(dev)
        col = cc.Collider(w.n, w.cells, dev, **w.params())
        r = {"n": w.n, "cells": w.cells}
        for mode in ("cold", "warm"):
            v, c = v0, c0
            for s in range(3):
                o = col.step(v, c, step=s)
                if mode == "warm":
                    v, c = o.v_out, o.cell_out
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in range(20):
                o = col.step(v, c, step=10 + s)
                if mode == "warm":
                    v, c = o.v_out, o.cell_out
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            r[f"{mode}_ms_per_step"] = ms
            r[f"{mode}_pair_collisions_per_s"] = float(o.diag[2].item()) / (ms * 1e-3)
        if name in ("C1", "C2"):
            # launch-bound: the operator alone from a CUDA graph of 20 chained steps (the
            # randoms advance through the device step counter, cc_params.step_dev); no roofline applies
            sd = torch.zeros(1, dtype=torch.int32, device=dev)
            ws = cc.alloc_workspace(w.n, w.cells, dev)
            outs = [cc.coulomb_collide(v0, c0, w.cells, step=0, workspace=ws, step_dev=sd, **w.params())
                    for _ in range(2)]

            def chain():
                v, c = v0, c0
                for s in range(20):
                    o = cc.coulomb_collide(v, c, w.cells, step=s, workspace=ws, step_dev=sd, out=outs[s % 2],
                                           **w.params())
                    v, c = o.v_out, o.cell_out
                cc.cc_step_advance(sd, 20)

            st = torch.cuda.Stream(dev)
            st.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(st):
                chain()                                 # warm-up outside capture
            torch.cuda.current_stream(dev).wait_stream(st)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                chain()
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            r["graph_ms_per_step"] = e0.elapsed_time(e1) / 100
            r["graph_pair_collisions_per_s"] = float(outs[1].diag[2].item()) / (r["graph_ms_per_step"] * 1e-3)
        out[name] = r
    return out


def run_ours(args):
    import ctypes as C

    import torch
    from paper_2508_06771_b200 import dist as ccd
    rank, world, local = ccd.init_from_env(args.dist_backend)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL: the library's own communicator (C ABI cc_dist_*); gloo smoke runs: torch collectives
        dist_ops = ccd.cuda_ops(ccd.NcclComm() if args.dist_backend == "nccl" else None)
    if not torch.cuda.is_available():
        sys.exit("bench.py: no CUDA device — the product path runs only on the GPU (no CPU fallback); "
                 "`--impl reference` times the CPU oracle")
    local = local % torch.cuda.device_count()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    import paper_2508_06771_b200 as cc
    from paper_2508_06771_b200 import _lib
    from paper_2508_06771_b200.coulomb import CollideOut

    w = workload(args, rank)
    n_live, M = w.n, w.cells
    v_host = torch.from_numpy(w.v)
    c_host = torch.from_numpy(w.cell)
    n = n_live
    mig = None
    if world > 1:
        # fixed, dead-padded particle slots: the device-side Migrator moves
        # leavers out and appends arrivals into the dead tail, no count ever reaches the host
        # slot capacity per peer: twice the expected leavers towards one neighbour (boundary rows
        # 2/ny x p = 0.1, plus the drift's row moves), the dead padding twice the arrivals
        cap = int(2 * n_live * (0.1 / args.ny + args.drift / 4 * 2 / args.ny)) * (2 if world == 2 else 1) + 4096
        n = n_live + 2 * cap + 4096
        bounds = ccd.owner_bounds(M * world, world)
        peers = sorted({(rank - 1) % world, (rank + 1) % world} - {rank})
        mig = ccd.Migrator(n, bounds, rank, cap, dev, comm=dist_ops.nccl, peers=peers,
                           exchange=None if dist_ops.nccl is not None else ccd.torch_exchange())
    v = torch.zeros((3, n), dtype=torch.float64, device=dev)
    v[:, :n_live].copy_(v_host.to(dev))
    cell = torch.full((n,), -1, dtype=torch.int32, device=dev)
    cell[:n_live].copy_(c_host.to(dev))
    p = w.params()
    ws = cc.alloc_workspace(n, M, dev)

    def new_out():
        return CollideOut(torch.empty((3, n), dtype=torch.float64, device=dev),
                          torch.empty(n, dtype=torch.int32, device=dev),
                          torch.empty(n, dtype=torch.int32, device=dev),
                          torch.empty((M, 7), dtype=torch.float64, device=dev),
                          torch.empty(16, dtype=torch.float64, device=dev))

    bufs = [new_out(), new_out()]
    stream = torch.cuda.current_stream(dev)
    nst = _lib.CC_NUM_STAGES
    lib = _lib.load()

    model = {"flags": 0}
    red_diag = [None]

    def call(src_v, src_cell, dst, step, events=None, post=None):
        prm = cc.make_params(weight=p["weight"], cell_volume=p["cell_volume"], ln_lambda=p["ln_lambda"],
                             flags=model["flags"])
        if events is not None:
            arr = (C.c_void_p * (nst + 1))(*[e.cuda_event for e in events])
            prm.stage_events = C.cast(arr, C.POINTER(C.c_void_p))
        rc = lib.coulomb_collide(C.c_void_p(src_v.data_ptr()), n, C.c_void_p(src_cell.data_ptr()),
                                 C.c_void_p(dst.v_out.data_ptr()), C.c_void_p(dst.cell_out.data_ptr()),
                                 C.c_void_p(dst.perm_out.data_ptr()), n, M, w.cell_base, w.dt, C.byref(prm),
                                 w.seed, step, C.c_void_p(dst.moments.data_ptr()), C.c_void_p(dst.diag.data_ptr()),
                                 C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(stream.cuda_stream))
        _lib.check(rc, "coulomb_collide")
        if world > 1:
            # NCCL all_gather + rank-ordered device sum: the GLOBAL diagnostics (pairs of all ranks)
            red_diag[0] = ccd.reduce_diag(dst.diag, dist_ops)
        if post is not None:
            post.record(stream)                      # end of the step incl. the diagnostics collective

    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def between(mode, dst, timed_mig=None):
        """After a call: the stand-in pusher (outside the timed region) and, on several ranks,
        the device-side migration (timed: events around it)."""
        if mode == "cold":
            return
        if world > 1 and mode == "steady":
            drift_cells_global(dst.cell_out, args.nx, args.ny, rank, world, args.drift, gen)
            if timed_mig is not None:
                timed_mig[0].record(stream)
            mig(dst.v_out, None, dst.cell_out, dst.diag)
            if timed_mig is not None:
                timed_mig[1].record(stream)
        elif mode in ("steady", "steady_nomig"):
            drift_cells(dst.cell_out, args.nx, args.ny, args.drift, gen)

    def run_mode(mode, K, W, step0, sampler=None):
        """K timed operator calls after W untimed ones.  cold: the same randomly
        ordered input every step; warm: each step consumes the previous step's
        (cell-sorted) output; steady: warm + the stand-in drift between steps (the
        drift is not timed); on several ranks the steady step also migrates the
        particles that crossed a shard boundary (timed) — steady_nomig drifts
        inside the shard only."""
        cur = (v, cell)
        for s in range(W):
            dst = bufs[s % 2]
            call(*cur, dst, step0 + s)
            between(mode, dst)
            if mode != "cold":
                cur = (dst.v_out, dst.cell_out)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nst + 4)] for _ in range(K)]
        for row in ev:
            for e in row:
                e.record(stream)          # materialise the cudaEvent_t handles
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.mark(True)
        t0.record(stream)
        for s in range(K):
            dst = bufs[(W + s) % 2]
            call(*cur, dst, step0 + W + s, ev[s][:nst + 1], ev[s][nst + 1])
            between(mode, dst, (ev[s][nst + 2], ev[s][nst + 3]))
            if mode != "cold":
                cur = (dst.v_out, dst.cell_out)
        t1.record(stream)
        torch.cuda.synchronize()
        if sampler:
            sampler.mark(False)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        migrating = world > 1 and mode == "steady"
        mig_ms = [ev[s][nst + 2].elapsed_time(ev[s][nst + 3]) if migrating else 0.0 for s in range(K)]
        per = [ev[s][0].elapsed_time(ev[s][nst + 1]) + mig_ms[s] for s in range(K)]
        op_ms = statistics.mean(per)
        stages = {name: statistics.mean(ev[s][i].elapsed_time(ev[s][i + 1]) for s in range(K))
                  for i, name in enumerate(_lib.STAGE_NAMES)}
        if migrating:
            stages["migrate"] = statistics.mean(mig_ms)
        assert cc.cc_device_status(ws) == 0
        last = bufs[(W + K - 1) % 2]
        # pairs: the reduced (all-rank) diagnostics on several ranks, the local ones on one
        pairs = float((red_diag[0] if world > 1 else last.diag)[2].item())
        return {"ms": op_ms, "ms_median": statistics.median(per), "ms_min": min(per), "ms_max": max(per),
                "wall_ms": t0.elapsed_time(t1) / K, "stages": stages, "pairs": pairs}

    K, W = args.steps, args.warmup
    clk = ClockSampler(local).start()
    res = {"steady": run_mode("steady", K, W, 0, clk),
           "cold": run_mode("cold", K, W, 100_000),
           "warm": run_mode("warm", K, W, 200_000)}
    clk.stop()
    if world > 1:
        res["steady_nomig"] = run_mode("steady_nomig", max(3, K // 2), W, 300_000)
        mig_status = mig.status.cpu().tolist()
        assert mig_status[:3] == [0, 0, 0], f"migration overflow {mig_status}"
    # NEXT f1 collision-model variants, steady state (shorter runs)
    variants = {}
    for name, fl in (("odd_triplet", _lib.CC_ODD_TRIPLET), ("nanbu", _lib.CC_NANBU),
                     ("preserve_order", _lib.CC_PRESERVE_ORDER)):
        model["flags"] = fl
        r = run_mode("steady", max(3, K // 4), W, 400_000 + 1000 * fl)
        variants[name] = {"flags": fl, "ms_per_step": r["ms"], "stages_ms": r["stages"],
                          "value": r["pairs"] / (r["ms"] * 1e-3)}
        if fl == _lib.CC_PRESERVE_ORDER:
            variants[name]["what"] = ("outputs in input order: the chain keeps the C4 input's random order "
                                      "(a cold-order step plus the scattered output stores)")
    # R1 over the whole cell (CC_CELL_UNIFORM: gathered records, no index modes) in all three orders
    model["flags"] = _lib.CC_CELL_UNIFORM
    for mode in ("steady", "warm", "cold"):
        r = run_mode(mode, max(3, K // 4), W, 500_000 + 1000 * len(mode))
        variants["cell_uniform_" + mode] = {"flags": _lib.CC_CELL_UNIFORM, "ms_per_step": r["ms"],
                                            "stages_ms": r["stages"], "value": r["pairs"] / (r["ms"] * 1e-3)}
    model["flags"] = 0

    # ---- end to end through the host-buffer entry coulomb_collide_host (cold input): every step
    # copies its inputs (v, cell ids) host->device and its result — the post-collision
    # velocities in the caller's own particle order (CC_PRESERVE_ORDER, so no cell ids or perm
    # need to come back) — device->host inside the library call.  Two streams and two device
    # buffers: step s+1's host->device copies overlap step s's device->host copies (PCIe is
    # full duplex); each step still moves all its bytes.
    v_pin = v_host.pin_memory()
    c_pin = c_host.pin_memory()
    NB = max(1, args.e2e_buffers)
    houts = [torch.empty((3, n_live), dtype=torch.float64).pin_memory() for _ in range(NB)]
    devbufs = [cc.alloc_host_buffer(n_live, M, dev) for _ in range(NB)]
    streams = [torch.cuda.Stream(dev) for _ in range(NB)]
    E = max(args.e2e_steps, 1)

    def e2e_call(s):
        k = s % NB
        cc.coulomb_collide_host(v_pin, c_pin, M, out_v=houts[k], dev_buffer=devbufs[k], stream=streams[k],
                                step=300_000 + s, flags=_lib.CC_PRESERVE_ORDER, **p)

    e2e_call(0)                                 # warm-up (not timed)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for st_ in streams:
        st_.wait_event(e0)
    for s in range(E):
        e2e_call(1 + s)
    for st_ in streams:
        stream.wait_stream(st_)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / E
    del devbufs

    # ---- max over ranks (times), sum over ranks (pairs)
    names = [k for k in ("steady", "cold", "warm", "steady_nomig") if k in res]
    if dist is not None:
        # time = max over ranks; pairs already come from the reduced (all-rank) diagnostics
        mx = torch.tensor([res[k]["ms"] for k in names] + [e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        for i, k in enumerate(names):
            res[k]["ms"] = float(mx[i])
        e2e_ms = float(mx[len(names)])
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"

    traffic, traffic_note = {}, None
    try:      # DRAM bytes per launch from an ncu capture of these kernels (tools/traffic_from_ncu.py)
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        if t.get("sources_sha") == sources_sha():
            traffic = t.get("kernels", {})
        else:
            traffic_note = "profiles/traffic.json was captured on other kernel sources: refused"
    except Exception:
        traffic_note = "no profiles/traffic.json"
    kernel_of = {"count": "k_count", "scatter": "k_scatter", "collide": "k_collide_large"}

    def roofline(r, mode, with_traffic=False):
        """ALGO_BYTES per particle x n over the dominant kernel's event-timed duration."""
        st = r["stages"]
        contract = STAGE_CONTRACT_BYTES[BIN_MODE[mode]]
        dom = max(("count", "scatter", "collide"), key=lambda k: st[k])
        achieved = ALGO_BYTES * n_live / (st[dom] * 1e-3) / 1e9
        tr = traffic.get(kernel_of[dom], {}).get("dram_bytes_per_launch") if (world == 1 and with_traffic) else None
        return {"kernel": kernel_of[dom], "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": tr,
                "traffic_over_algorithmic": (tr / (ALGO_BYTES * n_live)) if tr else None,
                "traffic_source": ("profiles/traffic.json (ncu --set full, same kernel sources, steady call)"
                                   if tr else traffic_note),
                "algorithmic_bytes_per_particle": ALGO_BYTES, "algorithmic_bytes_per_launch": ALGO_BYTES * n_live,
                "binning_mode": BIN_MODE[mode],
                "kernel_contract_bytes_per_particle": contract[dom],
                "kernel_contract_frac": contract[dom] * n_live / (st[dom] * 1e-3) / 1e9 / hbm_peak,
                "kernel_ms": st[dom], "peak_source": peak_src}

    STEP_KERNELS = ("k_count", "k_scan_tiles", "k_scan_cells", "k_cell_setup", "k_scatter", "k_collide_small",
                    "k_collide_large", "k_copy_dead", "k_finalize_cells", "k_finalize_diag")

    def step_hbm(ms):
        """Whole step: algorithmic 52 B/particle over the step time (SURVEY §8(d) reading 2) and the DRAM
        bytes ncu measured for every kernel of one steady call (reading 1), with SURVEY §8(d)'s
        1.15 x design-traffic guard against its cold (112 B) and warm (56 B) designs and against this
        pipeline's own index-mode design (76 B)."""
        out = {"algorithmic_bytes_per_particle": ALGO_BYTES,
               "frac": ALGO_BYTES * n_live / (ms * 1e-3) / 1e9 / hbm_peak,
               "design_bytes_per_particle": DESIGN_BYTES, "pipeline_design_bytes_per_particle": PIPELINE_BYTES}
        if world != 1 or not all(k in traffic for k in STEP_KERNELS):
            out["achieved_dram_frac"] = None
            out["traffic_note"] = traffic_note
            return out
        b = sum(traffic[k]["dram_bytes_per_launch"] for k in STEP_KERNELS)
        out.update({"achieved_dram_bytes_per_particle": b / n_live,
                    "traffic_over_algorithmic": b / (ALGO_BYTES * n_live),
                    "achieved_dram_gbs": b / (ms * 1e-3) / 1e9,
                    "achieved_dram_frac": b / (ms * 1e-3) / 1e9 / hbm_peak,
                    "guard_1.15x_cold_design": b / n_live <= 1.15 * DESIGN_BYTES["cold"],
                    "guard_1.15x_warm_design": b / n_live <= 1.15 * DESIGN_BYTES["warm"],
                    "guard_1.15x_index_mode_design": b / n_live <= 1.15 * PIPELINE_BYTES["index"],
                    "source": "profiles/traffic.json (ncu dram__bytes_read/write.sum per kernel, one steady call, "
                              "same kernel sources)"})
        return out

    def timing(r):
        return {"ms_mean": r["ms"], "ms_median": r["ms_median"], "ms_min": r["ms_min"], "ms_max": r["ms_max"]}

    def summary(r, mode):
        return {"value": r["pairs"] / (r["ms"] * 1e-3), "ms_per_step": r["ms"], "wall_ms_per_step": r["wall_ms"],
                "timing": timing(r), "stages_ms": r["stages"], "roofline": roofline(r, mode),
                "step_hbm_frac": ALGO_BYTES * n_live / (r["ms"] * 1e-3) / 1e9 / hbm_peak}

    head = res["steady"]
    line = {
        "metric": METRIC, "value": head["pairs"] / (head["ms"] * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args, world) + f"; steady-state PIC: each step consumes the previous "
                   f"step's output after a stand-in drift moves {100 * args.drift:g}% of the electrons to a "
                   f"neighbour cell (first step: randomly ordered input)"
                   + ("; on several ranks the first/last row of each shard also moves outward with p = 0.1 and the "
                      "step includes the device-side migration to the owning rank (NCCL, fixed-size slots)"
                      if world > 1 else ""),
                   "cells_per_gpu": M, "electrons_per_gpu": n_live, "pairs_per_step": head["pairs"],
                   "l2": f"inputs {(w.v.nbytes + w.cell.nbytes) / 1e9:.2f} GB/GPU >> 126 MB L2 (no flush needed)",
                   "timing": "CUDA events around each operator call (drift excluded); value = mean of K, "
                             "median/min/max in timing",
                   "parallelism": f"cell-range shards x{world}" if world > 1 else "1 GPU"},
        "roofline": roofline(head, "steady", with_traffic=True),
        "timing": timing(head),
        "stages_ms": head["stages"],
        "step_hbm": step_hbm(head["ms"]),
        "cold": dict(summary(res["cold"], "cold"), what="every step bins the same randomly ordered input"),
        "warm": dict(summary(res["warm"], "warm"), what="chained steps, no drift (input already cell-sorted)"),
        "e2e": {"value": res["cold"]["pairs"] / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": int(v_host.numel() * 8 + c_host.numel() * 4),
                "d2h_bytes_per_step": int(n_live * 24), "ms_per_step": e2e_ms,
                "what": "coulomb_collide_host (C-ABI host-buffer entry, CC_PRESERVE_ORDER) on pinned host memory: "
                        "per step H2D of v and cell ids, D2H of the post-collision v in the caller's order; "
                        f"{NB} streams / device buffers, consecutive steps' copies overlap"},
        "variants": variants,
        # our kernels per timed step: coulomb_collide 10; on several ranks + cc_diag_sum_ranks 1 and the
        # migration's k_mig_count / k_mig_scan / k_mig_pack / k_mig_unpack 4 (NCCL's own kernels not counted)
        "gpu_launches": 10 * K + (5 * K if world > 1 else 0),
        "clocks": clk.summary(),
    }
    if world > 1:
        line["multi_gpu"] = {
            "steady_without_migration": dict(summary(res["steady_nomig"], "steady_nomig"),
                                             what="drift inside the shard only, no migration step"),
            "migration": {"peers": mig.peers, "cap_per_peer": mig.cap, "slot_bytes": mig.slot,
                          "status": mig_status, "ms_per_step": res["steady"]["stages"].get("migrate"),
                          "what": "cc_mig_pack + cc_dist_mig_exchange (grouped ncclSend/ncclRecv of whole "
                                  "fixed-size slots with the two neighbour shards) + cc_mig_unpack, inside the "
                                  "timed step; status = [dropped: slot full, ids out of range, buffer full, "
                                  "arrivals] summed over all steps of this rank"},
            "diagnostics": "value's pair count from the NCCL-reduced diagnostics (cc_dist_diag_reduce)"}
    if world == 1 and not args.no_pic:
        try:
            line["pic"] = pic_section(args, dev, w, K)
        except Exception as e:  # the NEXT-row measurement must never kill the headline
            line["pic"] = {"error": repr(e)}
    if world == 1 and not args.no_pic:
        try:
            line["configs"] = configs_section(dev)
        except Exception as e:
            line["configs"] = {"error": repr(e)}
        try:
            line.update(p2c_section(dev, w))
        except Exception as e:
            line["p2c"] = {"error": repr(e)}
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = time_oracle_on(w, args)
        except Exception as e:  # the baseline must never kill the GPU number
            line["cpu_baseline"] = {"error": repr(e)}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
