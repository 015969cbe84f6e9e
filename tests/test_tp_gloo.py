"""Multi-process (world size 2, gloo, CPU) test of the tensor-parallel host
logic: head ownership from the C ABI, the rank-local W^vo slice and the
all-reduce of paper_2505_21487_b200/tp.py reproduce the unsharded output
projection, checked against oracle.sharding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, h_c, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_21487_b200 import tp

    T, H, d_c, D = 3, 16, 8, 12
    g = torch.Generator().manual_seed(0)
    o_lat = torch.randn(T, H, d_c, generator=g, dtype=torch.float64)  # same on every rank
    w_vo = torch.randn(H * d_c, D, generator=g, dtype=torch.float64)
    kb, ke, qb, qe = tp.shard(H, h_c, world, rank)
    y = tp.oproj_allreduce(o_lat[:, qb:qe].contiguous(), tp.wvo_slice(w_vo, H, h_c, world, rank, d_c))
    if rank == 0:
        np.save(out_path, y.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("h_c", [2, 8, 1])
def test_tp2_oproj_allreduce_matches_unsharded(tmp_path, h_c):
    world = 2
    out = str(tmp_path / "y.npy")
    mp.start_processes(_worker, args=(world, _free_port(), h_c, out), nprocs=world, join=True,
                       start_method="spawn")
    from oracle import sharding as SH
    g = torch.Generator().manual_seed(0)
    o_lat = torch.randn(3, 16, 8, generator=g, dtype=torch.float64)
    w_vo = torch.randn(16 * 8, 12, generator=g, dtype=torch.float64)
    ref = SH.tp_oproj_allreduce(o_lat.numpy(), w_vo.numpy().reshape(16, 8, 12), world, h_c)
    np.testing.assert_allclose(np.load(out), ref, atol=1e-10)


def _worker_lse(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_21487_b200 import tp
    g = torch.Generator().manual_seed(7)
    lse = torch.randn(world, 3, 2, 5, generator=g)
    lse[0, 1, 1, 2] = -float("inf")  # an empty range on rank 0
    gathered = tp.gather_lse(lse[rank].clone())
    if rank == 0:
        np.save(out_path, gathered.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_seq_split_lse_allgather(tmp_path):
    """Sequence split host plumbing over gloo, world size 2:
    the LSE all-gather returns every rank's lse in rank order (the input of
    glad_seq_split_rescale)."""
    world = 2
    out = str(tmp_path / "g.npy")
    mp.start_processes(_worker_lse, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    g = torch.Generator().manual_seed(7)
    lse = torch.randn(world, 3, 2, 5, generator=g)
    lse[0, 1, 1, 2] = -float("inf")
    np.testing.assert_array_equal(np.load(out), lse.numpy())
