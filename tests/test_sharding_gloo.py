"""World-size-2 gloo tests (CPU) of the multi-GPU path's host logic: instance sharding by
global id, per-rank compute, and the end-of-run reductions.  The per-rank compute here is
the oracle restatement standing in for the device (no GPU in this container); the device
side of sharding (streams keyed by global id) is covered by the GPU test
test_cfg5_full_size_energy_consistency_and_determinism."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_23043_b200 import sharding


def test_shard_covers_every_instance_once():
    for total in (1, 7, 128, 4096):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                off, cnt = sharding.shard(total, world, r)
                got.extend(range(off, off + cnt))
            assert got == list(range(total))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_instances(gids, L=6, R=8, sweeps=30):
    """Per-instance PT on the oracle: returns per-slot observables, histograms, best energies."""
    from oracle import oracle as O
    betas = np.linspace(0.3, 2.0, R)
    cols = O.checkerboard_colours((L,))
    obs = np.zeros((len(gids), R, 5), np.int64)
    hist = np.zeros((R, 16), np.int64)
    best = np.zeros(len(gids), np.int64)
    for k, gid in enumerate(gids):
        g = O.ea_graph((L,), 5, gid)
        pt = O.PT(g, betas, 11, gid, g.colour_order(cols))
        pt.run(sweeps, 1, 0, 0, None, 0, 5, 0, -3 * L ** 3, 3 * L ** 3 // 8 + 1, 16)
        m = pt.meas
        obs[k] = np.stack([m["cnt"], m["sumE"], m["sumE2"], m["sumAbsM"], m["sumM2"]], axis=1)
        hist += pt.hist
        best[k] = pt.best
    return obs, hist, best


def _worker(rank, world, port, total, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    off, cnt = sharding.shard(total, world, rank)
    obs, hist, best = _oracle_instances(list(range(off, off + cnt)))
    red = sharding.reduce_observables(obs, hist)
    allbest = sharding.gather_instances(best, total)
    tmax = sharding.reduce_max(float(rank))
    if rank == 0:
        q.put((red["obs"], red["hist"], allbest, tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_reduction_equals_single_process():
    total = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    obs, hist, best, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_obs, ref_hist, ref_best = _oracle_instances(list(range(total)))
    assert np.array_equal(obs, ref_obs.sum(axis=0))
    assert np.array_equal(hist, ref_hist)
    assert np.array_equal(best, ref_best)
    assert tmax == 1.0
