#!/usr/bin/env python3
"""Benchmark of the B200 Tucker-ALS hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2|c3]

Workloads (BASELINE.json configs; synthetic seeded stacks):

* ``c2`` (default; the config the metric is quoted on at one GPU): one
  1080x1920x3x10 IPT stack end to end per rank per step -- u8 images -> IPT
  coding-space tensor -> T-HOSVD -> 20 HOOI sweeps -> 10-bit core quantisation
  -> reconstruction + relative error. With N GPUs every rank runs its own
  independent stack (weak scaling, "replicas only").
* ``c3``: the 64-stack batch (Y'CbCr, ranks (135,240,3,5), 10 sweeps each),
  stacks assigned round-robin to the ranks (``dist.assign_stacks``), no
  inter-GPU traffic (strong scaling: the 64 stacks are the fixed job).

Multi-GPU: one process per GPU. Under torchrun the RANK/WORLD_SIZE env is used;
``--gpus N`` without it spawns the N ranks itself (127.0.0.1 rendezvous, NCCL).

Prints ONE JSON line on rank 0. ``value`` is device-resident throughput
(stacks/s over all ranks, max-over-ranks CUDA-event time); ``e2e`` is the same
metric through the public API (``encode_stack`` / ``encode_stacks``) with the
u8 images copied from pinned host memory and the results copied back every
step. ``--impl reference`` runs the UNMODIFIED reference package (``tmcodec``,
installed into ``oracle/_ref`` by ``oracle/build_ref.py``) on the host cores
through its own public API; it never loads libtmb.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def _load_synth():
    """The seeded stack generator, loaded by file path: importing it through the
    package would run the package __init__ and map libtmb.so, which the
    reference arm must not do."""
    name = "tmb_synth"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, ROOT / "paper_2104_04726_b200" / "synth.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


synth = _load_synth()
CONFIGS, make_stack = synth.CONFIGS, synth.make_stack

UNIT = "stacks/s"
DATA = "synthetic (seeded generator, SURVEY.md 8(d); stands in for the paper's ZED captures)"
C3_STACKS = 64
FP64_PEAK_TFLOPS = 35.47   # torch fp64 8192^3 matmul (cuBLAS DGEMM), profiles/r01_probe_peaks.txt
FP64_PEAK_SRC = "measured: torch.float64 8192^3 matmul best of 10 on this pool's B200 (profiles/r01_probe_peaks.txt)"
METRICS = {
    "c2": "Tucker-ALS stacks/sec (BASELINE config 2: 1080x1920x3x10 IPT stack, ranks (270,480,3,5), 20 HOOI "
          "sweeps, 10-bit core)",
    "c3": "Tucker-ALS stacks/sec (BASELINE config 3: 64 independent 1080x1920x3x10 Y'CbCr stacks, ranks "
          "(135,240,3,5), 10 HOOI sweeps each, 8-bit core)",
}
SCALING = {"c2": "weak", "c3": "strong"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(METRICS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--lanes", type=int, default=None,
                    help="c3: concurrent solves per GPU (host threads with their own stream + context; "
                         "default pipeline.DEFAULT_LANES)")
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(workload: str, world: int) -> dict:
    """The workload description; identical for both arms (``--impl``)."""
    if workload == "c2":
        return {"workload": "c2: 1080x1920x3x10 IPT stack, ranks (270,480,3,5), 20 HOOI sweeps, qp 39 (10-bit), "
                            "reconstruction + rel. error",
                "global_batch": world, "parallelism": f"dp{world} (one independent stack per rank per step, "
                                                      f"no collectives)",
                "l2": "no flush: per-step working set (249 MB fp32 tensor + fp64 intermediates) > 126 MB L2",
                "stack_seed": "rank"}
    return {"workload": f"c3: {C3_STACKS} independent 1080x1920x3x10 Y'CbCr stacks (seeds 0..63, disparity phase "
                        f"drifting with the frame index), ranks (135,240,3,5), 10 HOOI sweeps each, qp 51 (8-bit), "
                        f"reconstruction + rel. error",
            "global_batch": C3_STACKS, "parallelism": f"dp{world} (stacks round-robin over ranks, no collectives)",
            "l2": "no flush: per-stack working set > 126 MB L2", "stack_seed": "stack index"}


def base_line(workload: str, world: int, args, value: float, ms_per_step: float) -> dict:
    return {"metric": METRICS[workload], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": SCALING[workload], "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": config_dict(workload, world)}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:  # noqa: BLE001
            pass
    return {}


def _stack_seed_frame(workload: str, i: int) -> tuple[int, int]:
    return (i, i) if workload == "c3" else (i, 0)


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


# ----------------------------------------------------------------------------- launcher
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawned(local: int, world: int, port: int, target, args) -> None:
    os.environ.update(RANK=str(local), LOCAL_RANK=str(local), WORLD_SIZE=str(world), LOCAL_WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    target(args)


def launch(args, target) -> None:
    """Run ``target(args)`` on every rank: in this process under torchrun (or
    for one GPU), else spawn ``args.gpus`` processes, one per GPU, with a
    127.0.0.1 rendezvous (RANK/LOCAL_RANK/WORLD_SIZE set as torchrun would)."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import torch.multiprocessing as mp

        mp.start_processes(_spawned, args=(args.gpus, _free_port(), target, args), nprocs=args.gpus,
                           join=True, start_method="spawn")
    else:
        target(args)


# ----------------------------------------------------------------------------- CPU reference (tmcodec)
def _ref_tensor(tm, images: np.ndarray, space: str) -> np.ndarray:
    """The reference's own colour transform per image (``to_coding_space``,
    color.py:185-194, on ``ColorImage(u8/255)`` as sceneio.read_image does),
    assembled into the (H, W, 3, V*E) tensor of the BASELINE configs in F order
    (the reference is bit-identical for C/F input, F is faster)."""
    from tmcodec.color import ColorImage, to_coding_space

    v_, e_, h, w, _ = images.shape
    t = np.empty((h, w, 3, v_ * e_), order="F")
    for v in range(v_):
        for e in range(e_):
            t[:, :, :, v * e_ + e] = to_coding_space(ColorImage(images[v, e] / 255.0), space).pixels
    return t


def reference_stack(tm, images: np.ndarray, cfg) -> dict:
    """One full stack through the reference's public API: colour -> tucker_als
    (exactly ``cfg.sweeps`` HOOI sweeps) -> quantize_core -> reconstruct +
    relative error."""
    from tmcodec.codec import quantize_core
    from tmcodec.tensor import DenseTensor
    from tmcodec.tucker import SolveConfig, reconstruct, tucker_als

    t0 = time.perf_counter()
    x = _ref_tensor(tm, images, cfg.space)
    t = DenseTensor(x)
    model, trace = tucker_als(t, SolveConfig(ranks=cfg.ranks, max_sweeps=cfg.sweeps, fit_tol=1e-300,
                                             pp_enter_tol=0.0))
    if cfg.qp is not None:
        quantize_core(model, cfg.qp)
    rec = reconstruct(model).array
    rel = float(np.linalg.norm((x - rec).ravel()) / np.linalg.norm(x.ravel()))
    return {"stack_s": time.perf_counter() - t0, "fit": trace.records[-1].fit, "rel_err": rel}


def reference_sample(tm, images: np.ndarray, cfg) -> dict:
    """Bounded sample of the same reference path: colour + t_hosvd + ONE
    hooi_sweep + quantize_core + reconstruct, each timed; the stack time is
    extrapolated to ``cfg.sweeps`` sweeps (SURVEY §8(d) CPU baseline plan)."""
    from tmcodec.codec import quantize_core
    from tmcodec.tensor import DenseTensor
    from tmcodec.tucker import hooi_sweep, reconstruct, t_hosvd

    t0 = time.perf_counter()
    x = _ref_tensor(tm, images, cfg.space)
    t = DenseTensor(x)
    t1 = time.perf_counter()
    model = t_hosvd(t, cfg.ranks)
    t2 = time.perf_counter()
    model = hooi_sweep(t, model)
    t3 = time.perf_counter()
    if cfg.qp is not None:
        quantize_core(model, cfg.qp)
    reconstruct(model)
    t4 = time.perf_counter()
    stack = (t2 - t0) + cfg.sweeps * (t3 - t2) + (t4 - t3)
    return {"stack_s": stack, "sample_s": t4 - t0, "sweep_s": t3 - t2}


def _host_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        return int(max((i.get("num_threads", 1) for i in threadpool_info()), default=1))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def run_reference(args) -> None:
    """``--impl reference``: the unmodified reference on the host cores, rank 0
    only (other ranks exit without work). Warm-up steps are bounded samples of
    the same code path (colour, t_hosvd, hooi_sweep, quantize_core,
    reconstruct -- nothing on a CPU needs more warming); each timed step is
    one FULL stack (``tucker_als`` with every sweep), no extrapolation."""
    world, rank, _ = dist_env()
    world = max(world, args.gpus)
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "oracle"))
    from build_ref import import_reference  # oracle/build_ref.py (reference installer, not the port)

    tm = import_reference()
    cfg = CONFIGS[args.workload]
    ids = [0] if args.workload == "c2" else list(range(C3_STACKS))
    seed, frame = _stack_seed_frame(args.workload, ids[0])
    images = make_stack(cfg, seed=seed, frame=frame)
    for _ in range(args.warmup):
        reference_sample(tm, images, cfg)
    times, last = [], None
    for k in range(args.steps):
        if args.workload == "c3" and k > 0:   # c3: step k solves stack k of the 64 (one stack per step)
            seed, frame = _stack_seed_frame(args.workload, ids[k % len(ids)])
            images = make_stack(cfg, seed=seed, frame=frame)
        last = reference_stack(tm, images, cfg)
        times.append(last["stack_s"])
    total = sum(times)
    value = args.steps / total
    cores = _host_threads()
    line = base_line(args.workload, world, args, value, 1e3 * total / args.steps)
    sample = (f"{args.workload}: one full stack per timed step through tmcodec's public API (to_coding_space per "
              f"image, tucker_als with {cfg.sweeps} sweeps, quantize_core, reconstruct), no extrapolation; "
              f"{cores} BLAS threads; fit {last['fit']:.10f}")
    line.update({"impl": "reference",
                 "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                                  "sample": sample},
                 "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                 "reference": {"package": "tmcodec (oracle/_ref, installed unmodified by oracle/build_ref.py)",
                               "rank": "rank 0 only (host CPU); other ranks exit without work",
                               "warmup": "bounded samples of the same path (t_hosvd + 1 hooi_sweep)"}})
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def _gen(args):
    wl, i = args
    seed, frame = _stack_seed_frame(wl, i)
    return make_stack(CONFIGS[wl], seed=seed, frame=frame)


def generate_stacks(wl: str, cfg, ids) -> list:
    """This rank's seeded u8 stacks (host side, before the timed regions); a
    fork pool when there are several (4-5 s of numpy per 1080p stack)."""
    if len(ids) <= 1:
        return [_gen((wl, i)) for i in ids]
    import concurrent.futures as cf
    import multiprocessing as mp

    workers = max(1, min(len(ids), (os.cpu_count() or 2) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))))
    with cf.ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
        return list(ex.map(_gen, [(wl, i) for i in ids]))


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2104_04726_b200 as tb
    from paper_2104_04726_b200 import _lib as L
    from paper_2104_04726_b200.dist import assign_stacks
    from paper_2104_04726_b200 import pipeline as P
    from paper_2104_04726_b200.pipeline import encode_stack_device, encode_stacks_device, stream_lanes

    wl = args.workload
    cfg = CONFIGS[wl]
    sc = tb.SolveConfig(ranks=cfg.ranks, max_sweeps=cfg.sweeps, fit_tol=1e-300, pp_enter_tol=0.0)
    ids = [rank] if wl == "c2" else assign_stacks(C3_STACKS, rank, world)
    host_stacks = generate_stacks(wl, cfg, ids)
    pinned = [torch.from_numpy(s).pin_memory() for s in host_stacks]
    dev_stacks = [p.to("cuda") for p in pinned]
    h = L.ctx()
    units_total = world if wl == "c2" else C3_STACKS

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

    nl = 1 if wl == "c2" else max(1, min(P.DEFAULT_LANES if args.lanes is None else args.lanes, len(dev_stacks)))
    ctxs = [h] + ([ln.ctx for ln in stream_lanes(nl)] if nl > 1 else [])

    def device_step(bufs):
        if nl > 1:   # c3: stacks spread over concurrent lanes (pipeline.encode_stacks_device)
            res = encode_stacks_device(dev_stacks, cfg.space, cfg.ranks, sc, cfg.qp, True, nl)
            return bufs, (res[-1][0].records[-1].fit, res[-1][2])
        out = None
        for d in dev_stacks:
            bufs, tr, step, rel = encode_stack_device(d, cfg.space, cfg.ranks, sc, cfg.qp, True, bufs)
            out = (float(tr.fit[tr.n_records - 1]), rel)
        return bufs, out

    def launches_all() -> int:
        return sum(int(L.LIB.tmb_launch_count(c)) for c in ctxs)

    # ---- device-resident throughput (value): inputs already in HBM
    bufs = None
    for _ in range(args.warmup):
        bufs, last = device_step(bufs)
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    for c in ctxs:
        L.check(L.LIB.tmb_timing(c, 1), c)
    n0 = launches_all()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        bufs, last = device_step(bufs)
    ev1.record()
    barrier()
    launches = launches_all() - n0
    clk = clocks.stop()
    my_ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(my_ms)
    fam = {}
    for tag, name in ((0, "gemm_dmma"), (1, "sytrd"), (2, "tridiag_vectors"), (3, "color_u8"),
                      (4, "eig_gemm_dmma"), (5, "ttm_ozaki_i8")):
        fam[name] = {"launches": 0, "ms": 0.0, "work": 0.0}
        for c in ctxs:
            cnt, tms, work = L.C.c_int64(), L.C.c_double(), L.C.c_double()
            L.check(L.LIB.tmb_timing_read(c, tag, L.C.byref(cnt), L.C.byref(tms), L.C.byref(work)), c)
            fam[name]["launches"] += cnt.value
            fam[name]["ms"] += tms.value
            fam[name]["work"] += work.value
    for c in ctxs:
        L.check(L.LIB.tmb_timing(c, 0), c)
    value = units_total * args.steps / (ms / 1e3)
    fit_last, rel = last

    # ---- HOOI sweep time: K-sweep solve minus 0-sweep solve (same stack)
    sc0 = tb.SolveConfig(ranks=cfg.ranks, max_sweeps=0, fit_tol=1e-300, pp_enter_tol=0.0)

    def timed_solve(c):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        encode_stack_device(dev_stacks[0], cfg.space, cfg.ranks, c, cfg.qp, True, bufs)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e)
    tk = min(timed_solve(sc) for _ in range(2))
    t0 = min(timed_solve(sc0) for _ in range(2))
    sweep_ms = max_over_ranks((tk - t0) / cfg.sweeps)

    # ---- e2e through the public API: pinned H2D of the u8 images + D2H of the results, every step
    def e2e_step():
        if wl == "c2":
            r = tb.encode_stack(pinned[0], cfg.space, cfg.ranks, cfg.sweeps, cfg.qp)
            return [r]
        return tb.encode_stacks(pinned, cfg.space, cfg.ranks, cfg.sweeps, cfg.qp, lanes=nl)
    for _ in range(args.warmup):      # also populates torch's pinned host-block cache used by the D2H
        res = e2e_step()
    barrier()
    ee0 = torch.cuda.Event(enable_timing=True)
    ee1 = torch.cuda.Event(enable_timing=True)
    ee0.record()
    for _ in range(args.steps):
        res = e2e_step()
    ee1.record()
    barrier()
    e2e_ms = max_over_ranks(ee0.elapsed_time(ee1))
    h2d = int(sum(s.nbytes for s in host_stacks))
    d2h = 0
    for r in res:
        d2h += int(r.levels.nbytes)
        if r.model is not None:
            d2h += int(r.model.core.array.nbytes + sum(f.nbytes for f in r.model.factors))
    e2e = {"value": units_total * args.steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "path": "encode_stack" if wl == "c2" else
           f"encode_stacks ({nl} lanes; per lane the H2D of its next stack on a copy stream overlaps its current solve)"}

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
    for tf in (ROOT / "profiles" / "r02_traffic.json", ROOT / "profiles" / "r01_traffic.json"):
        if traffic is None and tf.exists():
            try:
                traffic = json.loads(tf.read_text()).get(dom_name)
            except Exception:  # noqa: BLE001
                traffic = None
    roof.update({"kernel": dom_name, "achieved": achieved, "peak": peak, "frac": achieved / peak if peak else None,
                 "traffic": traffic, "launches_per_step": dom["launches"] / args.steps,
                 "ms_per_step": dom["ms"] / args.steps, "share_of_step": dom["ms"] / my_ms})

    # the HBM-bound elementwise kernel of the step (u8 -> coding space, 15 B/px), same live timing
    col = fam["color_u8"]
    col_gbs = col["work"] / (col["ms"] / 1e3) / 1e9 if col["ms"] > 0 else None
    hbm_peak = float(peaks.get("hbm_gbs", 6443.8))
    roof_elem = {"bound": "hbm", "kernel": f"color_u8 ({cfg.space})", "unit": "GB/s",
                 "achieved": col_gbs, "peak": hbm_peak, "frac": col_gbs / hbm_peak if col_gbs else None,
                 "bytes_per_launch": col["work"] / max(col["launches"], 1)}

    # the contraction kernels (TTM full passes, Grams) against the FP64 pipe, algorithmic flops
    roof_gemm = {}
    for nm in ("gemm_dmma", "ttm_ozaki_i8"):
        f = fam[nm]
        if f["ms"] > 0:
            tfl = f["work"] / (f["ms"] / 1e3) / 1e12
            roof_gemm[nm] = {"achieved": tfl, "unit": "TFLOP/s (fp64-equivalent)", "peak": FP64_PEAK_TFLOPS,
                             "frac": tfl / FP64_PEAK_TFLOPS, "ms_per_step": f["ms"] / args.steps}
    sy = fam["sytrd"]
    if sy["ms"] > 0:
        cols = sum(n - 1 for n in cfg.dims[:2]) * (cfg.sweeps + 1) * len(dev_stacks)
        roof["latency"] = {"per_column_us": 1e3 * sy["ms"] / args.steps / cols,
                           "grid_barrier_floor_us": 2500 / 1965.0, "columns_per_step": cols}

    line = base_line(wl, world, args, value, ms / args.steps)
    line.update({
        "hooi_sweep_ms": sweep_ms,
        "fit": fit_last, "rel_err": rel,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": roof,
        "roofline_elementwise": roof_elem,
        "roofline_contractions": roof_gemm,
        "kernel_families": {k: {"launches_per_step": v["launches"] / args.steps, "ms_per_step": v["ms"] / args.steps}
                            for k, v in fam.items()},
        "clocks": clk,
        "stacks_per_rank": len(ids),
        "lanes": nl,
    })
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, host_stacks[0])
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(cfg, images) -> dict:
    """The reference itself (oracle/_ref) on a bounded sample of the workload,
    in a subprocess so this process never imports the reference package."""
    code = ("import sys, json; sys.path.insert(0, %r); import bench; from build_ref import import_reference; "
            "tm = import_reference(); import numpy as np; "
            "cfg = bench.CONFIGS[%r]; im = np.load(sys.argv[1]); "
            "r = bench.reference_sample(tm, im, cfg); r['threads'] = bench._host_threads(); print(json.dumps(r))"
            % (str(ROOT / "oracle"), cfg.name))
    with tempfile.NamedTemporaryFile(suffix=".npy", delete=False) as f:
        np.save(f, images)
    try:
        out = subprocess.run([sys.executable, "-c", code, f.name], capture_output=True, text=True, cwd=str(ROOT),
                             timeout=900)
        r = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "cores": None, "kind": "reference", "sample": f"failed: {exc}"}
    finally:
        os.unlink(f.name)
    return {"value": 1.0 / r["stack_s"], "unit": UNIT, "cores": r["threads"], "kind": "reference",
            "sample": f"{cfg.name} stack through tmcodec (oracle/_ref): to_coding_space + t_hosvd + 1 hooi_sweep + "
                      f"quantize_core + reconstruct ({r['sample_s']:.1f}s), sweep x{cfg.sweeps} extrapolated; "
                      f"stack {r['stack_s']:.1f}s"}


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        run_reference(args)
    else:
        launch(args, run_ours)


if __name__ == "__main__":
    main()
