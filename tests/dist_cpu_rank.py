"""A CPU rank body for the data-parallel launcher test (tests/test_dist.py).

bench.py's launcher spawns one process per rank; on the GPU box each rank runs
``bench.run_ours`` (the libtmb device path). Here the same launcher and the
same data-parallel bookkeeping (``dist.assign_stacks`` round-robin sharding,
gloo max-over-ranks timing, ``bench.base_line``'s JSON line) run with the CPU
oracle solving real small stacks -- test infrastructure only.
"""

from __future__ import annotations

import hashlib
import json
import os
import time

import numpy as np

N_STACKS = 6
RANKS = (6, 8, 3, 3)
SWEEPS = 3
QP = 51


def solve_stack(i: int) -> str:
    import bench
    import oracle

    images = bench.make_stack(bench.CONFIGS["c3"], seed=i, frame=i, height=24, width=32)
    x = np.asfortranarray(oracle.coding_tensor(images, "ycbcr").astype(np.float32).astype(np.float64))
    core, factors, _ = oracle.tucker_als(x, RANKS, max_sweeps=SWEEPS, fit_tol=1e-300, pp_enter_tol=0.0)
    levels, step = oracle.quantize_core(core, QP)
    return hashlib.sha256(np.ascontiguousarray(levels).tobytes()).hexdigest()[:16]


def cpu_rank(args) -> None:
    import torch.distributed as dist

    import bench
    from paper_2104_04726_b200.dist import assign_stacks, reduce_max

    world, rank, _ = bench.dist_env()
    dist.init_process_group("gloo")
    assert dist.get_world_size() == world
    ids = assign_stacks(N_STACKS, rank, world)
    dist.barrier()
    t0 = time.perf_counter()
    mine = {i: solve_stack(i) for i in ids}
    dt = reduce_max(time.perf_counter() - t0)
    gathered = [None] * world
    dist.all_gather_object(gathered, {"rank": rank, "pid": os.getpid(), "levels": mine})
    if rank == 0:
        line = bench.base_line("c3", world, args, N_STACKS * args.steps / dt, 1e3 * dt / args.steps)
        line["ranks"] = gathered
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
