"""Multi-process (world size 2, gloo, CPU) check of the frame-sharding host
logic bench.py uses: disjoint shards keyed by global frame id, plane tables
gathered to rank 0, identical to a single-process run over all frames."""
import os
import socket
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import scenegen

B_PER_RANK, W, H, R, HYP = 2, 96, 72, 8, 16


def _tables(first, n):
    d, lab, K = scenegen.stair_stream(first, n, W, H, R)
    rows = []
    for i in range(n):
        res = oracle.ransac(d[i].numpy(), lab[i].numpy(), K, R, HYP, 0.01, 0x1919, frame_id=first + i)
        rows.append(np.concatenate([res["best_hyp"], res["inliers"], res["status"], res["n_points"]]))
    return torch.from_numpy(np.stack(rows).astype(np.int64))


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, n = bench.shard(rank, B_PER_RANK)
    t = _tables(first, n)
    full = bench.gather_tables(t, world, rank)
    if rank == 0:
        torch.save(full, out_path)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_sharding_matches_single_process():
    oracle.build()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "gathered.pt")
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        gathered = torch.load(out)
    single = _tables(0, 2 * B_PER_RANK)
    assert torch.equal(gathered, single)
    assert bench.shard(1, 512) == (512, 512)
