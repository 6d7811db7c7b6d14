"""Multi-process (world_size 2, gloo, CPU) coverage of the data-parallel path:
stack sharding, max-over-ranks timing and the aggregate throughput formula."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2104_04726_b200.dist import aggregate_throughput, assign_stacks, reduce_max, run_stacks


def test_assign_covers_disjoint_balanced():
    for n, world in [(64, 1), (64, 2), (64, 8), (10, 4), (3, 8)]:
        parts = [assign_stacks(n, r, world) for r in range(world)]
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(n))
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        assign_stacks(4, 2, 2)


def test_aggregate_throughput():
    assert aggregate_throughput([32, 32], 4.0) == 16.0
    with pytest.raises(ValueError):
        aggregate_throughput([1], 0.0)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_launcher_spawns_ranks_and_solves_real_stacks():
    """bench.launch (the `--gpus N` path without torchrun) spawns N ranks with a
    127.0.0.1 rendezvous; each solves its round-robin share of real (small)
    stacks; rank 0 prints one JSON line with n_gpus == N, and every stack's
    quantised levels equal a single-process solve of the same stack."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = ("import sys; sys.path[:0] = [%r, %r]; import bench, dist_cpu_rank; "
            "bench.launch(bench.parse(['--gpus', '2', '--steps', '1']), dist_cpu_rank.cpu_rank)"
            % (str(root), str(root / "tests")))
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["config"]["global_batch"] == 64
    ranks = sorted(line["ranks"], key=lambda r: r["rank"])
    assert [r["rank"] for r in ranks] == [0, 1] and ranks[0]["pid"] != ranks[1]["pid"]
    got = {int(k): v for r in ranks for k, v in r["levels"].items()}
    assert sorted(got) == list(range(6))
    assert sorted(int(k) for k in ranks[1]["levels"]) == [1, 3, 5]
    sys.path[:0] = [str(root), str(root / "tests")]
    import dist_cpu_rank

    for i in (0, 5):
        assert got[i] == dist_cpu_rank.solve_stack(i)


def _worker(rank: int, world: int, port: int, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = assign_stacks(64, rank, world)
    done = run_stacks(mine, lambda i: i * i)          # bookkeeping only; real solves: test above
    elapsed = 1.0 + rank                              # rank 1 is the slow one
    slowest = reduce_max(elapsed)
    total = reduce_max(float(len(done)))               # every rank holds 32 stacks
    q.put((rank, mine[:3], len(done), slowest, total))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, ids0, n0, slow0, tot0), (r1, ids1, n1, slow1, tot1) = res
    assert ids0 == [0, 2, 4] and ids1 == [1, 3, 5]
    assert n0 == n1 == 32
    assert slow0 == slow1 == 2.0                       # max over ranks, identical everywhere
    assert aggregate_throughput([n0, n1], slow0) == 32.0
