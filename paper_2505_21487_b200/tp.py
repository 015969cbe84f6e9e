"""Tensor-parallel GLA step: per-rank decode on the rank's latent
heads, row-parallel output projection, one all-reduce.

    O_r~ = O_r W_r^vo        (rank-local slice)
    O    = AllReduce(sum_r O_r~)

The decode runs in libglad; the o_proj is a plain library GEMM (cuBLAS via
torch.matmul) and the all-reduce is NCCL (gloo on CPU for the host-logic
tests).  Ownership comes from glad_tp_shard (C ABI).
"""

import torch
import torch.distributed as dist

from . import glad


def shard(h_q, n_kv_heads, world, rank):
    """(kv_begin, kv_end, q_begin, q_end) owned by `rank` (glad_tp_shard)."""
    return glad.tp_shard(h_q, n_kv_heads, world, rank)


def local_heads(h_q, n_kv_heads, world, rank):
    kb, ke, qb, qe = shard(h_q, n_kv_heads, world, rank)
    return ke - kb, qe - qb


def wvo_slice(w_vo_full, h_q, n_kv_heads, world, rank, d_c):
    """Rows of W^vo [h_q*d_c, d_model] that multiply this rank's heads."""
    _, _, qb, qe = shard(h_q, n_kv_heads, world, rank)
    return w_vo_full[qb * d_c:qe * d_c]


def oproj_allreduce(o_local, w_vo_local, out=None, group=None):
    """o_local [T, H_loc, d_c] (latent-space attention output of this rank),
    w_vo_local [H_loc*d_c, d_model] -> all-reduced [T, d_model]."""
    T = o_local.shape[0]
    y = torch.matmul(o_local.reshape(T, -1), w_vo_local, out=out)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(y, group=group)
    return y
