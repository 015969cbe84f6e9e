"""§8(a) row a10 on the GPU: the tensor-parallel GLA step through
the product function tp.oproj_allreduce — each rank's decode on its latent
heads (libglad), its row-parallel W^vo slice (cuBLAS GEMM) and the
all-reduce — against the oracle's unsharded output projection
(oracle.sharding.tp_oproj_allreduce over the fp64 oracle attention),
element by element at the north-star tolerance.

One GPU only: (1) N ranks emulated in one process (the all-reduce is the
sum of the rank-local products, formed here in fp32); (2) two real
processes sharing cuda:0 over a gloo process group, so dist.all_reduce
inside tp.oproj_allreduce runs on CUDA tensors (NCCL refuses two ranks on
one device; the NCCL path is the same call with backend "nccl")."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import attention as OA
from oracle import sharding as OS

from gpu_side import DEV, build_paged, max_abs, rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

B, Lq, H, h_c, d_c, d_R, D_MODEL = 2, 2, 32, 8, 256, 64, 320
SL = np.array([700, 333])
SCALE = 1.0 / math.sqrt(192)


def _inputs():
    q, c, kr = synth.latent_kernel_inputs(B, Lq, H, h_c, d_c, d_R, int(SL.max()), seed=31)
    w_vo = synth.normal_bf16((H * d_c, D_MODEL), seed=32, std=1.0 / math.sqrt(H * d_c))
    return q, c, kr, w_vo


def _rank_step(rank, N, q, c, kr, w_vo):
    """What rank r of a TP-N job runs: decode on its shard, then
    tp.oproj_allreduce (the all-reduce is a no-op without a process group)."""
    from paper_2505_21487_b200 import glad, tp
    kb, ke, qb, qe = tp.shard(H, h_c, N, rank)
    L = int(SL.max())
    rows = torch.cat([c[:, :, kb:ke].reshape(B, L, -1), kr], -1).contiguous()
    layout, pool, bt = build_paged(rows, SL, 64, ke - kb, d_c, d_R, seed=rank)
    out, _ = glad.gla_decode(q[:, :, qb:qe].contiguous().to(DEV), pool, layout, bt,
                             torch.from_numpy(SL.astype(np.int32)).to(DEV), SCALE)
    w_loc = tp.wvo_slice(w_vo.to(DEV), H, h_c, N, rank, d_c)
    return tp.oproj_allreduce(out.view(B * Lq, qe - qb, d_c), w_loc)


def _reference(q, c, kr, w_vo, N):
    o_ref, _ = OA.latent_decode(q.double().numpy(), c.double().numpy(), kr.double().numpy(), SL, SCALE)
    return OS.tp_oproj_allreduce(o_ref.reshape(B * Lq, H, d_c), w_vo.double().numpy().reshape(H, d_c, D_MODEL),
                                 N, h_c)


def _check(y, y_ref, what):
    ma, rl = max_abs(y, y_ref), rel_l2(y, y_ref)
    assert ma <= 1e-2 and rl <= 5e-3, f"{what}: max_abs={ma:.3e} rel_l2={rl:.3e}"


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_oproj_allreduce_emulated_ranks(N):
    q, c, kr, w_vo = _inputs()
    y = torch.zeros(B * Lq, D_MODEL, dtype=torch.float32, device=DEV)
    for r in range(N):
        y_r = _rank_step(r, N, q, c, kr, w_vo)
        assert y_r.dtype == torch.bfloat16 and y_r.shape == (B * Lq, D_MODEL)
        y += y_r.float()
    torch.cuda.synchronize()
    _check(y.cpu(), _reference(q, c, kr, w_vo, N), f"TP{N} emulated")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q, c, kr, w_vo = _inputs()
    y = _rank_step(rank, world, q, c, kr, w_vo)  # all-reduce over the group inside
    torch.cuda.synchronize()
    if rank == 0:
        np.save(out_path, y.float().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_oproj_allreduce_two_processes(tmp_path):
    out = str(tmp_path / "y.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    q, c, kr, w_vo = _inputs()
    _check(np.load(out), _reference(q, c, kr, w_vo, 2), "TP2 two processes (gloo on CUDA tensors)")


def _worker_seq(rank, world, port, out_path):
    """Sequence split as a real 2-rank job on one GPU: each
    rank decodes its token range of every sequence, then
    tp.seq_split_oproj_allreduce (LSE all-gather, rescale, fp32 o_proj GEMM,
    all-reduce)."""
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_21487_b200 import glad, tp
    Hs, hcs = 64, 2
    q, c, kr = synth.latent_kernel_inputs(B, Lq, Hs, hcs, d_c, d_R, int(SL.max()), seed=41)
    w_vo = synth.normal_bf16((Hs * d_c, D_MODEL), seed=42, std=1.0 / math.sqrt(Hs * d_c))
    rows = torch.cat([c.reshape(B, int(SL.max()), -1), kr], -1).contiguous()
    begin, end, causal = tp.seq_split_ranges(SL, 16, Lq, world, rank)
    n = end - begin
    loc = torch.zeros(B, max(int(n.max()), 1), rows.shape[-1], dtype=rows.dtype)
    for b in range(B):
        loc[b, :n[b]] = rows[b, begin[b]:end[b]]
    layout, pool, bt = build_paged(loc, n, 16, hcs, d_c, d_R, seed=rank)
    out, lse = glad.gla_decode(q.to(DEV), pool, layout, bt, torch.from_numpy(n.astype(np.int32)).to(DEV), SCALE,
                               causal=causal)
    y = tp.seq_split_oproj_allreduce(out.view(B * Lq, Hs, d_c), lse.view(B * Lq, Hs), w_vo.to(DEV))
    torch.cuda.synchronize()
    if rank == 0:
        np.save(out_path, y.float().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_seq_split_oproj_allreduce_two_processes(tmp_path):
    out = str(tmp_path / "y.npy")
    mp.start_processes(_worker_seq, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    Hs, hcs = 64, 2
    q, c, kr = synth.latent_kernel_inputs(B, Lq, Hs, hcs, d_c, d_R, int(SL.max()), seed=41)
    w_vo = synth.normal_bf16((Hs * d_c, D_MODEL), seed=42, std=1.0 / math.sqrt(Hs * d_c))
    o_ref, _ = OA.latent_decode(q.double().numpy(), c.double().numpy(), kr.double().numpy(), SL, SCALE)
    y_ref = OS.tp_oproj_allreduce(o_ref.reshape(B * Lq, Hs, d_c), w_vo.double().numpy().reshape(Hs, d_c, D_MODEL),
                                  1, hcs)
    _check(np.load(out), y_ref, "sequence split P=2 (two processes)")
