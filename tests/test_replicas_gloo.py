"""The multi-GPU contract of bench.py ("replicas only"): N independent
replicas, whole-job throughput timed by the slowest rank.  Exercised on CPU with the
gloo backend, world size 2."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms_local = 10.0 + 5.0 * rank  # rank 1 is the slow one
    ms = bench.max_over_ranks(ms_local, device="cpu")
    out[rank] = (ms, bench.replica_throughput(50, ms, world), bench._dist())
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        ms, value, (ws, r, local) = res[rank]
        assert ms == 15.0  # both ranks agree on the slowest rank's time
        assert abs(value - world * 50 / 0.015) < 1e-6
        assert ws == world and r == rank and local == rank


def test_single_process_identity():
    assert bench.max_over_ranks(3.5, device="cpu") == 3.5
    assert bench.replica_throughput(10, 1000.0, 1) == 10.0
