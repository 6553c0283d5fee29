"""CPU coverage of bench.py's N>1 path (independent replicas): max-over-ranks time, summed work,
with a world_size-2 gloo process group (the GPU run uses NCCL; the aggregation is the same)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms, its = bench.aggregate_replicas(100.0 + 50.0 * rank, 10 + rank, world, device="cpu")
    out[rank] = (ms, its)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        assert out[r] == (150.0, 21.0)       # max time, summed iterations on every rank


def test_replica_aggregation_single():
    import bench
    assert bench.aggregate_replicas(12.5, 7, 1) == (12.5, 7.0)
