"""world_size-2 gloo test of the replica (data-parallel) host path on CPU."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_18813_b200.replicas import max_over_ranks, shard_requests, sum_over_ranks
from paper_2310_18813_b200.traffic import Request


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    reqs = [Request(id=i, arrival=0.1 * i) for i in range(11)]
    mine = shard_requests(reqs, rank, world)
    local_ms = 10.0 + rank  # rank 1 is slower
    job_ms = max_over_ranks(local_ms)
    tokens = sum_over_ranks(len(mine) * 128)
    out[rank] = (tuple(r.id for r in mine), job_ms, tokens)
    dist.destroy_process_group()


def test_replicas_two_ranks():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    ids0, ms0, tok0 = out[0]
    ids1, ms1, tok1 = out[1]
    assert sorted(ids0 + ids1) == list(range(11)) and not set(ids0) & set(ids1)
    assert ms0 == ms1 == 11.0  # max over ranks
    assert tok0 == tok1 == 11 * 128
