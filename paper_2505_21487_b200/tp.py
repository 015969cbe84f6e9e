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


# ------------------------------------------------------------ sequence split
# SURVEY §8(f)-1 (north_star: "optional sequence-split for long context
# merged with an LSE all-gather"): the P ranks of a head group each hold a
# contiguous page-aligned token range of every sequence (glad_seq_split_range)
# in their own pool, decode it (rank P-1 causal, the others not: it holds the
# last Lq - 1 keys), all-gather only the LSE [B, Lq, H_loc] fp32, rescale their
# partial output by exp(lse_r - lse) (glad_seq_split_rescale) and let the
# o_proj all-reduce (linear) do the sum.


def seq_split_ranges(seqlens, page_size, Lq, P, rank):
    """Per-sequence (begin, end) token ranges of `rank` -> int32 arrays, and
    the causal flag its decode call uses."""
    import numpy as np
    rng = [glad.seq_split_range(int(L), page_size, Lq, P, rank) for L in seqlens]
    begin = np.array([b for b, _ in rng], dtype=np.int32)
    end = np.array([e for _, e in rng], dtype=np.int32)
    return begin, end, rank == P - 1


def gather_lse(lse_local, group=None):
    """[P, *lse.shape]: every rank's lse of the same rows (all-gather over the
    sequence-split group; NCCL on GPUs, gloo in the CPU tests)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return lse_local.unsqueeze(0).contiguous()
    src = lse_local.contiguous()
    if src.is_cuda and dist.get_backend(group) == "gloo":  # gloo all-gathers host tensors only
        src = src.cpu()
    parts = [torch.empty_like(src) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, src, group=group)
    return torch.stack(parts).to(lse_local.device).contiguous()


def seq_split_oproj_allreduce(o_local, lse_local, w_vo_local, split_group=None, group=None, out=None):
    """o_local [T, H_loc, d_c] bf16 (this rank's normalised output over its
    token range), lse_local [T, H_loc] fp32 -> all-reduced [T, d_model]:
    sum over ranks of (o_r exp(lse_r - lse)) W_r^vo."""
    lse_all = gather_lse(lse_local, split_group)
    rank = dist.get_rank(split_group) if (dist.is_available() and dist.is_initialized()) else 0
    o_scaled, _ = glad.seq_split_rescale(lse_all, rank, o_local.contiguous())
    # the rescaled partial stays fp32 through the GEMM and the all-reduce:
    # o is rounded to bf16 once (by the decode), as in the unsplit path
    y = oproj_allreduce(o_scaled, w_vo_local.to(torch.float32), group=group)
    if out is not None:
        out.copy_(y)
        return out
    return y
