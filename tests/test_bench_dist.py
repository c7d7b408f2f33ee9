"""bench.py's multi-GPU plumbing on CPU: `--gpus N` re-executes the script under torchrun with one
rank per GPU (127.0.0.1 rendezvous), a mismatched WORLD_SIZE is refused, and the two collectives of
the run's plumbing -- the NCCL unique-id broadcast and the max-over-ranks timing -- is exercised with
a world-size-2 gloo group.  (The histogram reduction itself is the library's NCCL call,
tapt_allreduce_observables, tested on the GPU box.)"""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_launcher_command_spawns_one_rank_per_gpu():
    cmd = bench.launcher_cmd(["--gpus", "4", "--steps", "2"], 4, port=29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29555"
    assert os.path.samefile(cmd[cmd.index("--master-port") + 2], os.path.join(ROOT, "bench.py"))
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_world_size_must_match_gpus(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    args = type("A", (), {"gpus": 4})()
    with pytest.raises(SystemExit):
        bench.check_world(args)
    args.gpus = 2
    assert bench.check_world(args) == 2
    monkeypatch.delenv("WORLD_SIZE")
    args.gpus = 1
    assert bench.check_world(args) == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist = bench.init_dist(world, rank, backend="gloo")
    from paper_2509_23043_b200 import sharding
    off, cnt = sharding.shard(4096, world, rank)
    uid = bench.share_unique_id(lambda: bytes(range(128)), rank)
    ms, ranks = bench.max_over_ranks(10.0 * (rank + 1), world, "cpu")
    q.put((rank, off, cnt, uid == bytes(range(128)), ms, ranks))
    dist.destroy_process_group()


def test_gloo_world2_unique_id_broadcast_and_timing_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, off, cnt, uid_ok, ms, ranks in out:
        assert (off, cnt) == ((0, 2048) if rank == 0 else (2048, 2048))
        assert uid_ok
        assert ms == 20.0 and ranks == 2
