#!/usr/bin/env python
"""Benchmark: cell-updates/s (fp64, 3D Sedov) of the telescoped SSP-RK2 hydro
step (BASELINE.json metric), one process per GPU.

Workload (BASELINE.json configs[3], "3D Sedov weak scaling, 4096 blocks of
16^3 cells per GPU at 1/2/4/8 B200 with NCCL halo exchange + dt allreduce"):
every rank owns a brick of 16x16x16 blocks of 16^3 cells (256^3 cells,
dx = 1/256) arranged on a GPU grid (1,1,1), (2,1,1), (2,2,1), (2,2,2); the
Sedov blast sits at the global centre.  A step is one pass
of the whole hot path: guard fill (+ halo exchange) -> CFL dt (+ allreduce)
-> telescoped RK2 advance of the packet.  Inputs (2.2 GB state per GPU) are
far larger than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BRICK_BLOCKS = (16, 16, 16)
NB = (16, 16, 16)
GPU_GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
METRIC = "cell-updates/sec (fp64, 3D Sedov)"
UNIT = "cell-updates/s"


def algorithmic_costs(nb=16, ng=4, fill_mode="gather"):
    """Per cell-update algorithmic work of the telescoped 16^3 step (DESIGN.md
    section 6): bytes of the advance (read the padded block once,
    write the interior once) and of the guard fill -- full mode: read every
    guard's source and write the guard; gather mode: stage 2 writes the
    x-guards (the y/z guard rows are read from their owners inside the
    advance's one read of the padded block); fp64-pipe instructions of the
    advance (1498 per cell-update for the box stage-1 region,
    SASS-derived)."""
    P = nb + 2 * ng
    n3 = nb ** 3
    adv_bytes = (P ** 3 + n3) * 5 * 8 / n3
    guards = P ** 3 - n3
    fill_bytes = 2 * guards * 5 * 8 / n3 if fill_mode == "full" else 2 * ng * nb * nb * 5 * 8 / n3
    return adv_bytes, fill_bytes, FP64_INSTR_PER_CU


FP64_INSTR_PER_CU = 1498.0   # the literal telescoped step (computed ring on every side), SURVEY 8(d)
# fp64-pipe work model of one step: 142 per face flux (slopes
# shared), 15 per EOS cell (A5), FP64_PER_UPDATE per updated
# cell -- the last calibrated so that the literal telescoped 16^3 step is
# SURVEY's 1498 per cell-update (its F1 row then comes out at 1026 vs 1033)
FP64_PER_FACE, FP64_PER_EOS = 142.0, 15.0
# executed thread-instructions per cell-update of the advance kernels (ncu
# source page of the current kernels) -- the issue-slot view of the same
# kernels (context beside the fp64 roofline)
EXEC_INSTR_PER_CU = 2608.7
EXEC_INSTR_SOURCE = "profiles/r02_sass_mix_ring_v13.txt"


def _stage_counts(w):
    wx, wy, wz = w
    faces = (wx + 1) * wy * wz + wx * (wy + 1) * wz + wx * wy * (wz + 1)
    return faces, (wx + 4) * (wy + 4) * (wz + 4), wx * wy * wz


def _fp64_per_update(nb=16):
    f1, e1, u1 = _stage_counts((nb + 4,) * 3)
    f2, e2, u2 = _stage_counts((nb,) * 3)
    return (FP64_INSTR_PER_CU * nb ** 3 - FP64_PER_FACE * (f1 + f2) - FP64_PER_EOS * (e1 + e2)) / (u1 + u2)


def step_fp64_model(stage1_regions, nb=16):
    """Algorithmic fp64-pipe instructions per cell-update of a step whose
    stage 1 covers the given per-block output regions (wx, wy, wz) and whose
    stage 2 covers each block's interior."""
    per_u = _fp64_per_update(nb)
    tot = 0.0
    for w in stage1_regions + [(nb,) * 3] * len(stage1_regions):
        f, e, c = _stage_counts(w)
        tot += FP64_PER_FACE * f + FP64_PER_EOS * e + per_u * c
    return tot / (len(stage1_regions) * nb ** 3)


def borrowed_ring_regions(brick, nb=16):
    """Stage-1 output region of each block of a rank's brick under the
    borrowed ring (include/orcha.h orcha_set_ring_mode): self sides are the
    brick faces (a physical boundary or another rank); blocks with an x or y
    self side run the box kernel (20 x 20 columns; 18 x 18 for 16^3 blocks
    with at most one self side per axis), the rest the interior kernel; all
    extend the planes by 2 on each self z side."""
    out = []
    for k in range(brick[2]):
        for j in range(brick[1]):
            for i in range(brick[0]):
                sx = (i == 0) + (i == brick[0] - 1)
                sy = (j == 0) + (j == brick[1] - 1)
                sz = (k == 0) + (k == brick[2] - 1)
                if not (sx or sy):
                    w = nb
                elif nb in (8, 16) and sx < 2 and sy < 2:
                    w = nb + 2
                else:
                    w = nb + 4
                out.append((w, w, nb + 2 * sz))
    return out


def measured_traffic():
    """dram read+write bytes per advance from the committed ncu --set full
    capture (profiles/traffic.json, written by scripts/traffic_from_ncu.py), or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        t = json.load(open(path))
        return t.get("advance_bytes_per_launch"), t.get("source")
    return None, None


def peaks():
    p = {"hbm_gbs": 6535.4, "source": "fallback (B200_PROFILING.md earlier pool measurement is 6650; "
                                      "MEASURED_PEAKS.json absent)"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        m = json.load(open(path))
        p = {"hbm_gbs": float(m["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)",
             "sm_max_mhz": float(m.get("sm_max_mhz", 1965.0))}
    # fp64 pipe: 148 SMs x 64 fp64 lanes x clock thread-instructions/s (B200_PROFILING.md unit counts)
    p["fp64_tinst"] = 148 * 64 * p.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/orcha_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


# ------------------------------------------------------------------ reference
def workload_config(world):
    """The workload both arms report (cfg4 at `world` GPUs)."""
    px, py, pz = GPU_GRIDS[world]
    nblk = (BRICK_BLOCKS[0] * px, BRICK_BLOCKS[1] * py, BRICK_BLOCKS[2] * pz)
    return {"workload": "cfg4: 3D Sedov, 4096 blocks of 16^3 (+4 guards) per GPU, one packet",
            "global_cells": [nblk[a] * NB[a] for a in range(3)],
            "blocks_per_gpu": BRICK_BLOCKS[0] * BRICK_BLOCKS[1] * BRICK_BLOCKS[2], "gpu_grid": list(GPU_GRIDS[world]),
            "ng": 4, "gamma": 1.4, "cfl": 0.4}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores, one
    bounded sample of the workload per step (a 64^3 sub-box of the same Sedov
    setup: ghost fill, dt, one telescoped RK2 step)."""
    if rank != 0:
        return
    import numpy as np  # noqa: F401

    import oracle
    import orcha_inputs as inp

    n = 64
    og = oracle.Grid(N=(n, n, n))
    U0 = inp.sedov((n, n, n))
    U = oracle.padded(og, U0)

    def one_step():
        oracle.fill_ghosts(og, U)
        r = oracle.compute_dt(og, U)
        oracle.step(og, U, r.dt)

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    el = time.perf_counter() - t0
    ms = el / args.steps * 1e3
    value = n ** 3 * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(world), parallelism="cpu oracle, 1 thread (each step: a 64^3 sub-box "
                                                                           "sample of the same Sedov setup)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"64^3 3D Sedov, {args.steps} timed steps (plain C oracle, -O2 -ffp-contract=off)",
                             "host": host_cpu()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def host_cpu():
    """nproc and the CPU model of this host (recorded with the CPU baseline)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    if model is None and os.path.exists("/proc/cpuinfo"):
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    return {"nproc": os.cpu_count(), "model": model}


def _oracle_rate(n, seconds_target, threads):
    import oracle
    import orcha_inputs as inp

    used = oracle.use_threads(threads)
    try:
        og = oracle.Grid(N=(n, n, n))
        U = oracle.padded(og, inp.sedov((n, n, n)))
        steps = 0
        t0 = time.perf_counter()
        while True:
            oracle.fill_ghosts(og, U)
            r = oracle.compute_dt(og, U)
            oracle.step(og, U, r.dt)
            steps += 1
            if time.perf_counter() - t0 > seconds_target:
                break
        el = time.perf_counter() - t0
    finally:
        oracle.use_threads(1)
    return n ** 3 * steps / el, steps, el, used


def cpu_baseline(seconds_target=12.0):
    """The oracle as it stands on this host (1 thread), on a bounded sample of
    the workload: a 96^3 sub-box of the 3D Sedov setup, as many steps as fit
    ~12 s (at least 1); beside it the labelled oracle-omp variant (the same
    source with -fopenmp over k-planes, bitwise the same results) on every
    core of the host for ~8 s."""
    n = 96
    v, steps, el, _ = _oracle_rate(n, seconds_target, 1)
    cpu = host_cpu()
    out = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"{n}^3 3D Sedov sub-box, {steps} steps (fill+dt+RK2), {el:.1f} s, 1 thread",
           "host": cpu}
    nthr = cpu["nproc"] or 1
    if nthr > 1:
        vo, so, elo, used = _oracle_rate(n, 8.0, nthr)
        out["omp"] = {"value": vo, "unit": UNIT, "cores": used, "kind": "oracle-omp",
                      "sample": f"{n}^3 3D Sedov sub-box, {so} steps, {elo:.1f} s, {used} OpenMP threads "
                                "(bitwise the 1-thread result: tests/test_oracle_scheme.py)"}
    return out


# ----------------------------------------------------------------- GPU arm
def streamed_loop(g, ids, N, px, py, pz, comm, stream, K, copy_priority=0, copy_streams=2):
    """The streamed time step of streamed_e2e: returns (packets, host mesh,
    step function, per-packet D2H-done events)."""
    import numpy as np
    import torch

    import orcha_inputs as inp
    from paper_2507_09337_b200 import hydro
    slabs = [a for a in np.array_split(ids, K) if len(a)]
    pks = [hydro.Packet(g, a) for a in slabs]
    mesh = [torch.from_numpy(inp.sedov_packet(N, NB, a, xmax=(float(px), float(py), float(pz)))).pin_memory()
            for a in slabs]
    # copy streams (priority < 0: their pack / unpack kernels are scheduled
    # ahead of the pending CTAs of the advance on the compute stream)
    # copy_streams > 1: packets alternate over that many H2D and D2H streams,
    # so one packet's pack / unpack kernel runs while another's copy holds the link
    h2ds = [torch.cuda.Stream(priority=copy_priority) for _ in range(copy_streams)]
    d2hs = [torch.cuda.Stream(priority=copy_priority) for _ in range(copy_streams)]
    done = [None] * len(pks)

    # one rank (lagged pipeline): the dt of a step is reduced on the device
    # at the end of the previous step, from the records its stage-2 epilogues
    # left (the values shipped out and back are bitwise the ones those
    # epilogues saw); each slab's guard fill follows the next slab's pack
    # (the brick's z faces are outflow, so a z-slab's guards read only its
    # two neighbour slabs) and its advance + unpack follow the fill of the
    # slab after it (which still reads its U^n): the first unpack of a step
    # starts three slabs into the H2D chain.  Several ranks: the set-wide
    # fill with its exchange, dt, then the advances.
    pipelined = comm is None
    clock = hydro.DevClock(0.0, math.inf)

    def advance_out(i):
        hydro.orcha_hydro_advance_devdt(pks[i], clock.dt_tensor, stream)
        e = torch.cuda.Event()
        e.record(stream)
        d2h = d2hs[i % len(d2hs)]
        d2h.wait_event(e)
        pks[i].unpack(mesh[i], d2h, sync=False)
        e2 = torch.cuda.Event()
        e2.record(d2h)
        done[i] = e2

    def prime():
        """Before the first step: upload the mesh once and reduce the first dt."""
        for i, p in enumerate(pks):
            p.pack(mesh[i], stream)
        hydro.orcha_compute_dt_device(pks, clock, comm, stream)

    def one():
        K_ = len(pks)
        ev_in = []
        for i, p in enumerate(pks):
            h2d = h2ds[i % len(h2ds)]
            if done[i] is not None:
                h2d.wait_event(done[i])
            p.pack(mesh[i], h2d)
            e = torch.cuda.Event()
            e.record(h2d)
            ev_in.append(e)
            if pipelined:
                stream.wait_event(e)
                if i >= 1:
                    hydro.orcha_fill_guardcells_packet(pks, i - 1, stream)
                if i >= 2:
                    advance_out(i - 2)
        if pipelined:
            hydro.orcha_fill_guardcells_packet(pks, K_ - 1, stream)
            for i in range(max(K_ - 2, 0), K_):
                advance_out(i)
            hydro.orcha_compute_dt_device(pks, clock, comm, stream)  # the next step's dt, on the device
            return
        for e in ev_in:
            stream.wait_event(e)
        hydro.orcha_fill_guardcells(pks, comm, stream)
        hydro.orcha_compute_dt_device(pks, clock, comm, stream)  # dt stays on the device
        for i in range(K_):
            advance_out(i)
    one.prime = prime
    return pks, mesh, one, done


def streamed_e2e(g, ids, N, px, py, pz, comm, stream, nsteps, K, world, copy_priority=0, copy_streams=2):
    """End to end with a host-resident mesh (the paper's
    execution model: every cycle each DataPacket is shipped H2D, advanced and
    shipped back): the brick is K z-slab packets whose interiors
    live in pinned host memory.  Per step: pack every packet (H2D stream;
    packet i waits for its own D2H of the previous step) -> fill + dt over
    the set -> advance packet i -> unpack it (D2H stream, no sync) while
    packet i+1 is advanced.  Step n+1 consumes step n's output from the host
    mesh: a real simulation loop, not independent replicas.  Timed with CUDA
    events on the compute stream (max over ranks)."""
    import torch
    import torch.distributed as dist

    pks, mesh, one, done = streamed_loop(g, ids, N, px, py, pz, comm, stream, K, copy_priority, copy_streams)
    if comm is None:
        one.prime()
        torch.cuda.synchronize()
    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(nsteps):
        one()
    for e in done:
        stream.wait_event(e)
    b.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / nsteps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ems = float(t.item())
    nbytes = sum(m.numel() for m in mesh) * 8
    del pks
    # the host link's own roofline: the step's H2D and D2H bytes over the
    # same pinned mesh buffers, both directions at once on two streams
    # (scripts/pcie_probe.py; best of 3), measured here on this box after the
    # timed region (the mesh contents are no longer needed)
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "scripts"))
    import pcie_probe
    lk = pcie_probe.probe_buffers(mesh, reps=3)
    floor_ms = 2 * nbytes / (lk["bidir_gbs"] * 1e9) * 1e3
    out = {"value": N[0] * N[1] * N[2] / (ems / 1e3), "unit": UNIT,   # N: the global grid (all ranks)
           "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": ems, "packets": len(mesh),
           "link": {"bound": "pcie", "h2d_gbs": lk["h2d_gbs"], "d2h_gbs": lk["d2h_gbs"],
                    "bidir_gbs": lk["bidir_gbs"], "floor_ms": floor_ms, "frac": floor_ms / ems,
                    "note": "floor = the step's H2D + D2H bytes moved concurrently at the bidirectional rate "
                            "measured over the same pinned mesh buffers; the rest is the serial part of the step (last slab's H2D, fill, "
                            "dt, first slab's advance + D2H)"},
           "note": f"host-resident mesh, {len(mesh)} z-slab packets per GPU shipped in and out every step on copy "
                   "streams overlapping the other packets' compute (one rank: each slab's guard fill as soon as its "
                   "neighbours are on the device, its advance and unpack right after the next slab's fill, the "
                   "step's dt reduced on the device at the end of the previous step from its stage-2 records); "
                   "step n+1 reads step n's output from the host"}
    return out


def other_workloads(stream):
    """cell-updates/s of BASELINE.json's other configs (single GPU, device dt,
    CUDA events around the timed steps after 3 warm-up steps): configs[0]
    (2D Sedov, 4x4 blocks of 8^2), configs[1] (Sod: 1D 64 blocks x 16 cells
    and the 2D tube of 64 x 1 blocks of 16^2), configs[2] (3D Sedov 128^3 as
    512 blocks of 16^3), and a large 2D Sedov (2048^2 as 128 x 128 blocks of
    16^2) so the 2D kernels are measured at a size that fills the GPU.  2D
    grids of 8^2 / 16^2 blocks run the one-kernel 2D step (kernels_fused2d.cu),
    1D grids the reference kernels (one thread per output cell)."""
    import numpy as np
    import torch

    import orcha_inputs as inp
    from paper_2507_09337_b200 import hydro
    P_, O_ = 1, 0
    cases = {
        "cfg1_sedov2d_32x32": dict(ndim=2, nb=(8, 8), nblk=(4, 4), ic=lambda N: inp.sedov(N), steps=200),
        "cfg2_sod1d_1024": dict(ndim=1, nb=(16,), nblk=(64,), ic=lambda N: inp.sod(N), steps=200),
        "cfg2_sod2d_tube_1024x16": dict(ndim=2, nb=(16, 16), nblk=(64, 1), bc=((O_, O_), (P_, P_), (O_, O_)),
                                        xmax=(1.0, 16.0 / 1024), ic=lambda N: inp.sod(N), steps=200),
        "cfg3_sedov3d_128": dict(ndim=3, nb=(16, 16, 16), nblk=(8, 8, 8), ic=lambda N: inp.sedov(N), steps=20),
        "sedov2d_2048": dict(ndim=2, nb=(16, 16), nblk=(128, 128), ic=lambda N: inp.sedov(N), steps=20),
    }
    out = {}
    for name, c in cases.items():
        g = hydro.Grid(c["ndim"], c["nb"], c["nblk"], bc=c.get("bc", ((0, 0),) * 3),
                       xmax=c.get("xmax", (1.0, 1.0, 1.0)))
        nd = c["ndim"]
        N = g.N[:nd]
        pk = hydro.Packet(g, np.arange(g.nblocks))
        pk.pack(inp.to_blocks(c["ic"](N), g.nb[:nd], pk.block_ids), stream)
        clock = hydro.DevClock(0.0, math.inf)

        def one():
            hydro.orcha_fill_guardcells([pk], None, stream)
            hydro.orcha_compute_dt_device([pk], clock, None, stream)
            hydro.step_devdt([pk], clock.dt_tensor, None, stream)
        for _ in range(3):
            one()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(c["steps"]):
            one()
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / c["steps"]
        cells = int(np.prod(N))
        out[name] = {"value": cells / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "cells": cells,
                     "steps": c["steps"],
                     "kernels": "fused z-marching (two stage kernels)" if nd == 3
                     else "fused 2D (both stages in one kernel, U1 in shared memory)" if nd == 2 and c["nb"][0] in (8, 16)
                     else "reference (one thread per cell)"}
        del pk, g
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="orcha", choices=["orcha", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-priority", type=int, default=-1,
                    help="streamed e2e: CUDA priority of the copy streams (-1 = high)")
    ap.add_argument("--e2e-copy-streams", type=int, default=2,
                    help="streamed e2e: H2D and D2H streams each (packets alternate over them)")
    ap.add_argument("--e2e-packets", type=int, default=16,
                    help="streamed e2e: packets (z-slabs of the brick) shipped in and out every step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the phase-timing pass, the fp64 probe and the other-config throughputs")
    ap.add_argument("--variant", type=int, default=None, help="advance kernel variant (0 ref, 1 fused)")
    ap.add_argument("--method", default="telescoped", choices=["telescoped", "per-stage"],
                    help="RK2 step: the paper's telescoped step (default) or the per-stage F1 variant")
    ap.add_argument("--dt-mode", default="device", choices=["device", "host"],
                    help="dt kept on the device (orcha_compute_dt_device, default) or returned to the host every step")
    ap.add_argument("--no-variants", action="store_true", help="skip the per-stage measurement beside the main line")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "ipc"],
                    help="N > 1: NCCL halo exchange + dt allgather (default), or the F2 peer mode over CUDA IPC "
                         "(other ranks' packets read directly, device barriers; gloo carries only the handles)")
    ap.add_argument("--fill-mode", default="gather", choices=["gather", "full"],
                    help="guard fill: gather (x-guards only, y/z rows staged from their owners; default) or full")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import orcha_inputs as inp
    from paper_2507_09337_b200 import abi, build, hydro

    if world != args.gpus:
        args.gpus = world
    if world not in GPU_GRIDS:
        raise SystemExit(f"--gpus must be one of {sorted(GPU_GRIDS)}")
    # ORCHA_BENCH_SAME_GPU=1 (functional runs on a one-GPU box): every rank on
    # GPU 0 -- only with --comm ipc (NCCL refuses two ranks on one GPU); the
    # ranks then time-slice the GPU, so the numbers are not a scaling result
    same_gpu = os.environ.get("ORCHA_BENCH_SAME_GPU") == "1" and world > 1
    if same_gpu and args.comm != "ipc":
        raise SystemExit("ORCHA_BENCH_SAME_GPU=1 needs --comm ipc")
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    backend = "gloo" if args.comm == "ipc" else "nccl"
    red_dev = "cpu" if backend == "gloo" else "cuda"   # device of the timing reductions
    if world > 1:
        if backend == "nccl":
            # NCCL's own communicator lines (ranks, channels, NVLS / P2P transport) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    if rank == 0 and not os.path.exists(abi.library_path(False)):
        build.build()
    if world > 1:
        dist.barrier()
    lib = abi.load(False)
    if args.variant is not None:
        hydro.set_kernel_variant(lib, args.variant)
    abi.call(lib, "orcha_set_fill_mode", 1 if args.fill_mode == "gather" else 0)

    px, py, pz = GPU_GRIDS[world]
    nblk = (BRICK_BLOCKS[0] * px, BRICK_BLOCKS[1] * py, BRICK_BLOCKS[2] * pz)
    N = tuple(nblk[a] * NB[a] for a in range(3))
    g = hydro.Grid(3, NB, nblk, xmin=(0.0, 0.0, 0.0), xmax=(float(px), float(py), float(pz)))
    # this rank's brick (block ids in natural order inside the brick)
    rx, ry, rz = rank % px, (rank // px) % py, rank // (px * py)
    bi = np.arange(BRICK_BLOCKS[0]) + rx * BRICK_BLOCKS[0]
    bj = np.arange(BRICK_BLOCKS[1]) + ry * BRICK_BLOCKS[1]
    bk = np.arange(BRICK_BLOCKS[2]) + rz * BRICK_BLOCKS[2]
    ids = ((bk[:, None, None] * nblk[1] + bj[None, :, None]) * nblk[0] + bi[None, None, :]).reshape(-1)
    comm = None
    owner = hydro.brick_owner(nblk, BRICK_BLOCKS, GPU_GRIDS[world])
    if world > 1 and args.comm == "nccl":
        comm = hydro.Comm.create(g, world, rank, owner)
    pk = hydro.Packet(g, ids)
    # initial Sedov state of this brick (host, closed form) -> pinned -> pack
    host = torch.from_numpy(inp.sedov_packet(N, NB, ids, xmax=(float(px), float(py), float(pz)))).pin_memory()
    stream = torch.cuda.current_stream()
    pk.pack(host, stream)
    stream.synchronize()
    if world > 1 and args.comm == "ipc":
        # F2 peer mode across processes: exchange the CUDA IPC blobs, map the
        # other ranks' packets, counters and dt buffers; tables + kernels now
        comm = hydro.Comm.create_ipc(g, world, rank, owner)
        blobs = [None] * world
        dist.all_gather_object(blobs, comm.ipc_export(pk))
        comm.ipc_attach(blobs)
        hydro.orcha_fill_prepare([pk], comm)
        torch.cuda.synchronize()

    adv_ev = []

    # dt on the device (default): orcha_compute_dt_device -> the *_devdt step
    # calls, no host synchronization inside the time loop; --dt-mode host:
    # orcha_compute_dt returns dt to the host every step (the paper's MPI model)
    clock = hydro.DevClock(0.0, math.inf) if args.dt_mode == "device" else None

    def step(record=False, method=args.method):
        if method == "per-stage":
            hydro.orcha_fill_guardcells_stage([pk], 0, comm, stream)
        else:
            hydro.orcha_fill_guardcells([pk], comm, stream)
        info = None
        if clock is None:
            info = hydro.orcha_compute_dt([pk], math.inf, comm, stream)
        else:
            hydro.orcha_compute_dt_device([pk], clock, comm, stream)
        if record:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        if clock is None:
            hydro.step([pk], info.dt, comm, stream, method)
        else:
            hydro.step_devdt([pk], clock.dt_tensor, comm, stream, method)
        if record:
            b.record(stream)
            adv_ev.append((a, b))
        return info

    def timed_variant(method, nsteps):
        """Same protocol for another step variant (reported beside the main line)."""
        for _ in range(3):
            step(method=method)
        adv_ev.clear()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        for _ in range(nsteps):
            step(record=True, method=method)
        v1.record(stream)
        torch.cuda.synchronize()
        vt = torch.tensor([v0.elapsed_time(v1) / nsteps], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(vt, op=dist.ReduceOp.MAX)
        vms = float(vt.item())
        return {"ms_per_step": vms, "value": N[0] * N[1] * N[2] / (vms / 1e3),
                "advance_ms": statistics.mean(a.elapsed_time(b) for a, b in adv_ev)}

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = lib.orcha_launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = lib.orcha_launch_count() - launches0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    cells = N[0] * N[1] * N[2]
    value = cells / (ms / 1e3)
    adv_ms = statistics.mean(a.elapsed_time(b) for a, b in adv_ev)
    # SURVEY 8(d) timing protocol: the same K-step measurement repeated (4
    # more times, after the reported one) -- median and spread, so a run's
    # variance is visible; `value` stays the first (the contract's) timing
    reps = [ms]
    if not args.no_extras:
        for _ in range(4):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record(stream)
            for _ in range(args.steps):
                step()
            r1.record(stream)
            torch.cuda.synchronize()
            rt = torch.tensor([r0.elapsed_time(r1) / args.steps], dtype=torch.float64, device=red_dev)
            if world > 1:
                dist.all_reduce(rt, op=dist.ReduceOp.MAX)
            reps.append(float(rt.item()))
    repetitions = {"ms_per_step": reps, "median_ms": statistics.median(reps),
                   "median_value": cells / (statistics.median(reps) / 1e3),
                   "spread": (max(reps) - min(reps)) / statistics.median(reps)}
    variants = {}
    if args.method == "telescoped" and not args.no_variants and args.comm != "ipc":
        # SURVEY 8(f) F1, measured beside the paper's telescoped step (same protocol)
        variants["per-stage"] = timed_variant("per-stage", args.steps)
        variants["per-stage"]["note"] = ("fill -> dt -> stage 1 (interior) -> U1 guard refill -> stage 2; "
                                         "oracle mode 'refill'; gather fill mode: no fill kernel runs (stage 1 "
                                         "writes the U1 x-guards, stage 2 stages U1 guard rows from their owners)")
        # the paper's literal telescoped step (stage-1 ring computed on every
        # side, orcha_set_ring_mode(0)) with the same kernels -- the same result
        if lib.orcha_get_ring_mode() == 1:
            lib.orcha_set_ring_mode(0)
            try:
                variants["literal-ring"] = timed_variant("telescoped", args.steps)
            finally:
                lib.orcha_set_ring_mode(1)
            variants["literal-ring"]["note"] = ("orcha_set_ring_mode(0): every block computes its whole 2-cell "
                                               "stage-1 ring (box kernel, 1498 fp64 per cell-update) -- the "
                                               "main line's result, with the ring borrowed from resident owners")
        # restore the packet to a telescoped-step history is not needed: both
        # variants advance the same Sedov state, timing only
    if args.method == "telescoped" and not args.no_variants and clock is not None and world == 1:
        # the steady-state device-dt step captured once in a CUDA graph (10
        # steps per graph) and replayed: no per-kernel host launches at all
        step()
        torch.cuda.synchronize()
        gsteps = 10
        graph = hydro.capture_steps([pk], clock, gsteps)
        graph.replay()
        torch.cuda.synchronize()
        reps = max(1, args.steps // gsteps)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(reps):
            graph.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / (reps * gsteps)
        variants["cuda-graph"] = {"ms_per_step": gms, "value": N[0] * N[1] * N[2] / (gms / 1e3),
                                  "note": f"{gsteps} steady-state device-dt steps (fill: no launch; dt reduce + "
                                          "finish; stage 1 + 2) captured in one CUDA graph, replayed"}
        del graph

    # per-phase device times (a separate pass of the same steps with the
    # library's phase events on; the timed loop above records none), per-rank
    # busy fraction, measured fp64 peak, BASELINE's other configs
    phases = None
    fp64_probe = None
    others = None
    per_rank = None
    if not args.no_extras:
        hydro.orcha_set_phase_timing(lib, True)
        hydro.orcha_phase_times(lib)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for _ in range(args.steps):
            step()
        p1.record(stream)
        torch.cuda.synchronize()
        pt = hydro.orcha_phase_times(lib)
        hydro.orcha_set_phase_timing(lib, False)
        pms = p0.elapsed_time(p1) / args.steps
        phases = {k: v[0] / args.steps for k, v in pt.items()}
        phases["step"] = pms
        phases["note"] = ("ms per step: device time between each phase's CUDA events (library-recorded, "
                          "orcha_set_phase_timing), separate pass of the same steps; fill includes the exchange, "
                          "dt includes the allgather; gather fill mode on one GPU launches no fill kernel")
        busy = (phases["fill"] + phases["dt"] + phases["stage1"] + phases["stage2"]) / pms
        mine = torch.tensor([ms, adv_ms, busy, phases["exchange"], phases["dt_allgather"]], dtype=torch.float64,
                            device=red_dev)
        if world > 1:
            allr = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(allr, mine)
        else:
            allr = [mine]
        per_rank = [{"rank": r, "ms_per_step": float(x[0]), "advance_ms": float(x[1]), "gpu_busy": float(x[2]),
                     "exchange_ms": float(x[3]), "dt_allgather_ms": float(x[4])} for r, x in enumerate(allr)]
        if rank == 0:
            tinst, pms_probe = hydro.orcha_probe_fp64(lib, 20000, stream)
            fp64_probe = {"tinst_per_s": tinst, "kernel_ms": pms_probe,
                          "note": "measured DFMA thread-instructions/s / 1e12 (orcha_probe_fp64: 8 CTAs x 256 "
                                  "threads per SM, 8 independent chains each)"}
            if world == 1:
                others = other_workloads(stream)

    # roofline of the dominant kernel (the advance): algorithmic bytes / flops
    pks = peaks()
    # (N > 1: the remote guards are exchanged into each rank's packet first;
    # the local part of the fill follows the mode)
    fill_eff = args.fill_mode
    adv_bytes, fill_bytes, fp_instr = algorithmic_costs(fill_mode=fill_eff)
    # the borrowed ring (default: gather fill, one packet, not F2 peer mode)
    # computes the stage-1 ring on the brick faces only: its own work model
    borrowed = (lib.orcha_get_ring_mode() == 1 and args.fill_mode == "gather" and args.method == "telescoped"
                and not (args.comm == "ipc" and world > 1))
    regions = borrowed_ring_regions(BRICK_BLOCKS, NB[0]) if borrowed else [(NB[0] + 4,) * 3]
    fp_instr = step_fp64_model(regions, NB[0])
    cu_local = BRICK_BLOCKS[0] * BRICK_BLOCKS[1] * BRICK_BLOCKS[2] * NB[0] * NB[1] * NB[2]
    hbm_achieved = adv_bytes * cu_local / (adv_ms / 1e3) / 1e9
    fp_achieved = fp_instr * cu_local / (adv_ms / 1e3) / 1e12
    traffic, traffic_src = measured_traffic()
    roof_hbm = {"bound": "hbm", "achieved": hbm_achieved, "peak": pks["hbm_gbs"], "unit": "GB/s",
                "frac": hbm_achieved / pks["hbm_gbs"], "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": pks["source"], "kernel": "hydro_advance (stage_fused_kernel<16,1> + <16,2>)",
                "algorithmic_bytes_per_cell_update": adv_bytes, "units_per_launch": cu_local}
    roof_fp = {"bound": "alu", "achieved": fp_achieved, "peak": pks["fp64_tinst"],
               "unit": "T fp64-pipe inst/s", "frac": fp_achieved / pks["fp64_tinst"], "traffic": traffic,
               "traffic_source": traffic_src,
               "peak_source": "derived (DESIGN.md 6): 148 SM x 64 fp64 lanes x sm_max clock",
               "peak_measured": fp64_probe["tinst_per_s"] if fp64_probe else None,
               "kernel": "hydro_advance (stage_fused_kernel<16,1> box + interior, <16,2>)",
               "algorithmic_fp64_instr_per_cell_update": fp_instr, "units_per_launch": cu_local,
               "ring": "borrowed" if borrowed else "computed",
               "work_model": "142 fp64 per face + 15 per EOS cell + 31.1 per updated cell over the step's "
                             "stage-1 / stage-2 regions (DESIGN.md 6)",
               "literal_telescoped_equivalent": {
                   "fp64_instr_per_cell_update": FP64_INSTR_PER_CU,
                   "achieved": FP64_INSTR_PER_CU * cu_local / (adv_ms / 1e3) / 1e12,
                   "frac": FP64_INSTR_PER_CU * cu_local / (adv_ms / 1e3) / 1e12 / pks["fp64_tinst"],
                   "note": "the literal step's work (ring computed on every side) per second of this advance: "
                           "context, not the kernel's own efficiency"}}
    primary, other = (roof_fp, roof_hbm) if roof_fp["frac"] >= roof_hbm["frac"] else (roof_hbm, roof_fp)
    # issue slots: 148 SMs x 4 schedulers x 1 warp-instruction per cycle
    issue_peak = 148 * 4 * pks.get("sm_max_mhz", 1965.0) * 1e6 * 32 / 1e12   # T thread-instructions/s
    issue_ach = EXEC_INSTR_PER_CU * cu_local / (adv_ms / 1e3) / 1e12
    roof_issue = {"bound": "issue", "achieved": issue_ach, "peak": issue_peak, "unit": "T thread-inst/s",
                  "frac": issue_ach / issue_peak, "executed_instr_per_cell_update": EXEC_INSTR_PER_CU,
                  "source": EXEC_INSTR_SOURCE,
                  "note": "executed (not algorithmic) instructions: the advance is issue/latency bound"}
    step_hbm = (adv_bytes + fill_bytes) * value / world / 1e9

    # end to end through the public API with host buffers (the paper's model:
    # the packet is shipped H2D, advanced and shipped back every cycle)
    e2e = None
    e2e_serial = None
    if args.comm == "ipc" and world > 1:
        args.e2e_steps = 0   # peer mode takes one packet per rank; the streamed e2e uses 16
    if args.e2e_steps > 0:
        e2e = streamed_e2e(g, ids, N, px, py, pz, comm, stream, args.e2e_steps, args.e2e_packets, world,
                             copy_priority=args.e2e_priority, copy_streams=args.e2e_copy_streams)
    if args.e2e_steps > 0:
        out = torch.empty_like(host).pin_memory()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.e2e_steps):
            pk.pack(host, stream)
            step()
            pk.unpack(out, stream)
        s1.record(stream)
        torch.cuda.synchronize()
        ems = s0.elapsed_time(s1) / args.e2e_steps
        te = torch.tensor([ems], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        nbytes = host.numel() * 8
        e2e_serial = {"value": cells / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": nbytes,
                      "d2h_bytes_per_step": nbytes + 8, "ms_per_step": ems,
                      "note": "one packet, one stream: pack (H2D, pinned) -> fill -> dt (D2H) -> advance -> "
                              "unpack (D2H, pinned)"}

    fh, bad = pk.counters(stream)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (closed-form Sedov IC)",
            "config": dict(workload_config(world), l2_flush="not needed: 2.2 GB state per GPU >> 126 MB L2",
                           kernel_variant=int(lib.orcha_get_kernel_variant()), fill_mode=fill_eff,
                           parallelism=f"blocks over {world} GPU(s)",
                           comm=(args.comm if world > 1 else None),
                           same_gpu=(True if same_gpu else None)),
            "roofline": primary, "roofline_other": other, "roofline_issue": roof_issue,
            "hbm_fraction_full_step": {"achieved_gbs": step_hbm, "frac": step_hbm / pks["hbm_gbs"],
                                       "frac_of_nominal_8tbs": step_hbm / 8000.0,
                                       "algorithmic_bytes_per_cell_update": adv_bytes + fill_bytes,
                                       "dram_bytes_per_cell_update_ncu": (traffic / cu_local) if traffic else None},
            "advance_ms": adv_ms, "method": args.method, "dt_mode": args.dt_mode, "variants": variants,
            "clocks": clk, "gpu_launches": int(launches), "e2e": e2e, "e2e_serial": e2e_serial,
            "floor_hits": fh, "nonphysical_first_cell": bad,
            "phases": phases, "per_rank": per_rank, "fp64_probe": fp64_probe, "other_configs": others,
            "repetitions": repetitions,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
