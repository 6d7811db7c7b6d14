#!/usr/bin/env python3
"""Benchmark of the B200 Tucker-ALS hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one multi-exposure stereo stack end to end on one GPU: u8 images ->
IPT coding-space tensor -> T-HOSVD -> 20 HOOI sweeps -> 10-bit core
quantisation -> reconstruction + relative error, i.e. BASELINE.json config 2
(1080x1920x3x10, ranks (270,480,3,5)). With N GPUs every rank runs its own
independent stack per step (data-parallel, no inter-GPU traffic; weak
scaling), launched one process per GPU by torchrun.

Prints ONE JSON line on rank 0. ``value`` is device-resident throughput
(stacks/s over all ranks, max-over-ranks CUDA-event time); ``e2e`` is the same
metric through the public API (``encode_stack``) with the u8 images copied
from pinned host memory and the quantised model copied back every step.
``--impl reference`` times the CPU reference path (the oracle port of the
reference algorithm, see oracle/) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2104_04726_b200.synth import CONFIGS, make_stack  # noqa: E402

WORKLOAD = "c2"
METRIC = "Tucker-ALS stacks/sec (BASELINE config 2: 1080x1920x3x10 IPT stack, ranks (270,480,3,5), 20 HOOI sweeps, 10-bit core)"
UNIT = "stacks/s"
FP64_PEAK_TFLOPS = 35.47   # torch fp64 8192^3 matmul (cuBLAS DGEMM), profiles/r01_probe_peaks.txt
FP64_PEAK_SRC = "measured: torch.float64 8192^3 matmul best of 10 on this pool's B200 (profiles/r01_probe_peaks.txt)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:  # noqa: BLE001
            pass
    return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.tmp.flush()
        rows = [r.split(",") for r in Path(self.tmp.name).read_text().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU reference
def cpu_reference_sample(cfg, images) -> dict:
    """Oracle port of the reference path on the host cores: colour + T-HOSVD +
    one HOOI sweep + quantise + reconstruct of one C2 stack, timed per phase,
    extrapolated to the full 20-sweep stack."""
    import oracle
    from threadpoolctl import threadpool_info

    t0 = time.perf_counter()
    x = oracle.coding_tensor(images, cfg.space)
    x = np.asfortranarray(x.astype(np.float32).astype(np.float64))
    t1 = time.perf_counter()
    core, factors = oracle.t_hosvd(x, cfg.ranks)
    t2 = time.perf_counter()
    core, factors = oracle.hooi_sweep(x, factors)
    t3 = time.perf_counter()
    oracle.quantize_core(core, cfg.qp)
    t4 = time.perf_counter()
    oracle.reconstruct(core, factors)
    t5 = time.perf_counter()
    stack_s = (t1 - t0) + (t2 - t1) + cfg.sweeps * (t3 - t2) + (t4 - t3) + (t5 - t4)
    threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    return {"stack_s": stack_s, "sweep_s": t3 - t2, "thosvd_s": t2 - t1, "colour_s": t1 - t0,
            "sample_s": t5 - t0, "threads": int(threads)}


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[WORKLOAD]
    images = make_stack(cfg, seed=0)
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, images)
    samples = [cpu_reference_sample(cfg, images) for _ in range(args.steps)]
    total = sum(s["stack_s"] for s in samples)
    value = args.steps / total
    sample_desc = (f"{WORKLOAD} stack: oracle-port colour + t_hosvd + 1 hooi_sweep + quantize + reconstruct "
                   f"timed per step, sweep time x{cfg.sweeps} extrapolated (mean sweep "
                   f"{statistics.mean(s['sweep_s'] for s in samples):.2f}s)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d); stands in for the paper's ZED captures)",
        "config": {"workload": f"{WORKLOAD}: 1080x1920x3x10 IPT, ranks (270,480,3,5), 20 sweeps, qp 39",
                   "global_batch": 1, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": samples[0]["threads"], "kind": "port",
                         "sample": sample_desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2104_04726_b200 as tb
    from paper_2104_04726_b200 import _lib as L
    from paper_2104_04726_b200.pipeline import encode_stack_device

    cfg = CONFIGS[WORKLOAD]
    sc = tb.SolveConfig(ranks=cfg.ranks, max_sweeps=cfg.sweeps, fit_tol=1e-300, pp_enter_tol=0.0)
    images = make_stack(cfg, seed=rank)  # one independent stack per rank
    pinned = torch.from_numpy(images).pin_memory()
    dev_images = pinned.to("cuda")
    h = L.ctx()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident throughput (value)
    bufs = None
    for _ in range(args.warmup):
        bufs, tr, step, rel = encode_stack_device(dev_images, cfg.space, cfg.ranks, sc, cfg.qp, True, bufs)
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    L.check(L.LIB.tmb_timing(h, 1), h)
    n0 = L.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        bufs, tr, step, rel = encode_stack_device(dev_images, cfg.space, cfg.ranks, sc, cfg.qp, True, bufs)
    ev1.record()
    barrier()
    launches = L.launch_count() - n0
    clk = clocks.stop()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    fam = {}
    for tag, name in ((0, "gemm_dmma"), (1, "sytrd"), (2, "tridiag_vectors"), (3, "color_u8"),
                      (4, "eig_gemm_dmma"), (5, "ttm_ozaki_i8")):
        cnt, tms, work = L.C.c_int64(), L.C.c_double(), L.C.c_double()
        L.check(L.LIB.tmb_timing_read(h, tag, L.C.byref(cnt), L.C.byref(tms), L.C.byref(work)), h)
        fam[name] = {"launches": cnt.value, "ms": tms.value, "work": work.value}
    L.check(L.LIB.tmb_timing(h, 0), h)
    value = world * args.steps / (ms / 1e3)

    # ---- HOOI sweep time: 20-sweep solve minus 0-sweep solve (same stack)
    sc0 = tb.SolveConfig(ranks=cfg.ranks, max_sweeps=0, fit_tol=1e-300, pp_enter_tol=0.0)
    def timed_solve(c):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        encode_stack_device(dev_images, cfg.space, cfg.ranks, c, cfg.qp, True, bufs)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e)
    t20 = min(timed_solve(sc) for _ in range(2))
    t0 = min(timed_solve(sc0) for _ in range(2))
    sweep_ms = max_over_ranks((t20 - t0) / cfg.sweeps)

    # ---- e2e through the public API (pinned H2D + D2H of the quantised model)
    ranks = cfg.ranks
    # warm-up as for the device-resident loop: the first calls also populate torch's
    # pinned host-block cache used for the D2H of the quantised model
    for _ in range(args.warmup):
        res = tb.encode_stack(pinned, cfg.space, ranks, cfg.sweeps, cfg.qp)
    barrier()
    ee0 = torch.cuda.Event(enable_timing=True)
    ee1 = torch.cuda.Event(enable_timing=True)
    ee0.record()
    for _ in range(args.steps):
        res = tb.encode_stack(pinned, cfg.space, ranks, cfg.sweeps, cfg.qp)
    ee1.record()
    barrier()
    e2e_ms = max_over_ranks(ee0.elapsed_time(ee1))
    h2d = int(images.nbytes)
    d2h = int(res.levels.nbytes + res.model.core.array.nbytes + sum(f.nbytes for f in res.model.factors))
    e2e = {"value": world * args.steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h}

    # ---- roofline of the dominant kernel family (live CUDA-event launch durations)
    dom_name, dom = max(fam.items(), key=lambda kv: kv[1]["ms"])
    peaks = measured_peaks()
    if dom_name == "color_u8":
        achieved = dom["work"] / (dom["ms"] / 1e3) / 1e9
        peak = float(peaks.get("hbm_gbs", 6443.8))
        roof = {"bound": "hbm", "unit": "GB/s", "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    else:
        achieved = dom["work"] / (dom["ms"] / 1e3) / 1e12 if dom["work"] > 0 else 0.0
        peak = FP64_PEAK_TFLOPS
        roof = {"bound": "tensor", "unit": "TFLOP/s", "pipe": "fp64 (DMMA / DFMA)", "peak_source": FP64_PEAK_SRC}
    traffic = None
    tf = ROOT / "profiles" / "r01_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(dom_name)
        except Exception:  # noqa: BLE001
            traffic = None
    roof.update({"kernel": dom_name, "achieved": achieved, "peak": peak, "frac": achieved / peak if peak else None,
                 "traffic": traffic, "launches_per_step": dom["launches"] / args.steps,
                 "ms_per_step": dom["ms"] / args.steps,
                 "share_of_step": dom["ms"] / (ev0.elapsed_time(ev1))})

    # the HBM-bound elementwise kernel of the step (u8 -> IPT colour, 15 B/px), same live timing
    col = fam["color_u8"]
    col_gbs = col["work"] / (col["ms"] / 1e3) / 1e9 if col["ms"] > 0 else None
    hbm_peak = float(peaks.get("hbm_gbs", 6443.8))
    roof_elem = {"bound": "hbm", "kernel": "color_u8 (IPT: 3 fp64 exp2(0.43 log2) per pixel, FP64-pipe bound)", "unit": "GB/s",
                 "achieved": col_gbs, "peak": hbm_peak, "frac": col_gbs / hbm_peak if col_gbs else None,
                 "bytes_per_launch": col["work"] / max(col["launches"], 1)}

    # the contraction kernels on the FP64 tensor pipe (TTM full passes on DMMA, Grams) and the
    # Ozaki tcgen05 TTM, same live timing, algorithmic flops (SURVEY 8(d) counting rules)
    roof_gemm = {}
    for nm in ("gemm_dmma", "ttm_ozaki_i8"):
        f = fam[nm]
        if f["ms"] > 0:
            tf = f["work"] / (f["ms"] / 1e3) / 1e12
            roof_gemm[nm] = {"achieved": tf, "unit": "TFLOP/s (fp64-equivalent)", "peak": FP64_PEAK_TFLOPS,
                             "frac": tf / FP64_PEAK_TFLOPS, "ms_per_step": f["ms"] / args.steps}
    # the tridiagonalisation is latency-bound: per-column time against the measured
    # 148-block grid-barrier floor (2.5k cycles at 1965 MHz, scripts/research/barrier_bench.cu)
    sy = fam["sytrd"]
    cols = sum(n - 1 for n in cfg.dims[:2]) * (cfg.sweeps + 1)
    per_col_us = 1e3 * sy["ms"] / args.steps / cols
    roof["latency"] = {"per_column_us": per_col_us, "grid_barrier_floor_us": 2500 / 1965.0,
                       "columns_per_step": cols,
                       "note": "one grid barrier + two block reductions + one L2 gather per column"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md 8(d); stands in for the paper's ZED captures)",
        "config": {"workload": f"{WORKLOAD}: 1080x1920x3x10 IPT stack, ranks (270,480,3,5), 20 HOOI sweeps, "
                               f"qp 39 (10-bit), reconstruction + rel. error",
                   "global_batch": world, "parallelism": f"dp{world} (independent stacks, no collectives)",
                   "l2": "no flush: per-step working set (249 MB fp32 tensor + fp64 intermediates) > 126 MB L2",
                   "stack_seed": "rank"},
        "hooi_sweep_ms": sweep_ms,
        "fit": float(tr.fit[tr.n_records - 1]), "rel_err": rel,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": roof,
        "roofline_elementwise": roof_elem,
        "roofline_contractions": roof_gemm,
        "kernel_families": {k: {"launches_per_step": v["launches"] / args.steps, "ms_per_step": v["ms"] / args.steps}
                            for k, v in fam.items()},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = cpu_reference_sample(cfg, images)
        line["cpu_baseline"] = {"value": 1.0 / ref["stack_s"], "unit": UNIT, "cores": ref["threads"], "kind": "port",
                                "sample": f"{WORKLOAD} stack on the host: oracle-port colour + t_hosvd + 1 hooi_sweep + "
                                          f"quantize + reconstruct ({ref['sample_s']:.1f}s), sweep x{cfg.sweeps} "
                                          f"extrapolated; stack {ref['stack_s']:.1f}s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
