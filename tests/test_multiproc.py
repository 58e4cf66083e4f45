"""N > 1 host logic on CPU with gloo (world size 2): image sharding covers
the batch exactly once and the step time is reduced as the max over ranks,
as bench.py does over NCCL on GPUs."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_03617_b200.scheduler import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(1000, world, rank)
    covered = torch.zeros(1000)
    covered[lo:hi] = 1
    dist.all_reduce(covered)  # every image exactly once
    t = torch.tensor([1.0 + rank])  # a fake per-rank step time
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out.put((covered.min().item(), covered.max().item(), t.item()))
    dist.destroy_process_group()


def test_gloo_sharding_and_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == (1.0, 1.0, 2.0)


def test_shard_range_edges():
    assert shard_range(128, 8, 7) == (112, 128)
    assert [shard_range(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]


def test_bench_gpus_flag_relaunches_one_process_per_rank():
    """``bench.py --gpus 2`` without a launcher re-executes itself under
    torch.distributed.run (2 ranks); the reference arm runs on rank 0 only
    and prints exactly one JSON line."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WL_REF_WORKERS="2")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
    from oracle.reference_net import load_reference

    # "reference" when baseline/_ref holds the installed reference, else the oracle port
    want = "reference" if load_reference() is not None else "port"
    assert lines[0]["cpu_baseline"]["kind"] == want and lines[0]["cpu_baseline"]["cores"] == 2
