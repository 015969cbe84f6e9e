"""Seeded synthetic input generators shared by the tests, bench.py and smoke().

This module holds NO arithmetic of the method (no RoPE, no absorption, no
softmax, no paging arithmetic beyond drawing a random page permutation): it
only draws random numbers with the shapes, value distributions and length
mixes of the paper's workloads, and rounds them to
bf16.  Both the oracle side and the CUDA side read these same tensors.

Recipe:
  * activations / cache entries ~ N(0, 1), up-projections ~ N(0, 1/d_c),
    drawn in fp32 by torch.Generator(seed) and rounded RNE to bf16;
  * "peaked" regime multiplies queries by 4;
  * sequence lengths: fixed, uniform in [r*max, max] with r = 0.125
    ("random ratio"), or the skew profile [1024]*15 + [X];
  * block tables: a seeded random permutation of physical pages with ~3 %
    slack so that pages are never accidentally contiguous.
"""

import math

import numpy as np
import torch


def _gen(seed, device="cpu"):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def normal_bf16(shape, seed, std=1.0, device="cpu"):
    """N(0, std^2) drawn in fp32, rounded to bf16."""
    g = _gen(seed, device)
    x = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    return x.to(torch.bfloat16)


def seqlens(B, max_len, kind="fixed", r=0.125, seed=0, skew_long=None):
    """Per-sequence KV lengths as an int32 numpy array."""
    if kind == "fixed":
        return np.full(B, max_len, dtype=np.int32)
    if kind == "uniform":
        rng = np.random.default_rng(seed)
        lo = max(1, int(math.ceil(r * max_len)))
        return rng.integers(lo, max_len + 1, size=B).astype(np.int32)
    if kind == "skew":
        long = max_len if skew_long is None else skew_long
        base = [1024] * 15 + [long]
        return np.array([base[i % 16] for i in range(B)], dtype=np.int32)
    raise ValueError(kind)


def block_table(seqlens_arr, page_size, seed=0, slack=0.03, min_pages_per_seq=0):
    """Random page assignment.

    Returns (block_table [B, max_pages] int32 with unused entries = -1,
             num_pages).  Pages are a random permutation of the pool, so no two
    logically adjacent pages are physically adjacent by construction.
    """
    seqlens_arr = np.asarray(seqlens_arr)
    B = len(seqlens_arr)
    need = [max(min_pages_per_seq, -(-int(L) // page_size)) for L in seqlens_arr]
    max_pages = max(1, max(need) if need else 1)
    total = sum(need)
    num_pages = max(1, int(math.ceil(total * (1.0 + slack))) + 1)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(num_pages)
    bt = np.full((B, max_pages), -1, dtype=np.int32)
    k = 0
    for b in range(B):
        bt[b, : need[b]] = perm[k: k + need[b]]
        k += need[b]
    return bt, num_pages


def latent_kernel_inputs(B, Lq, H, h_c, d_c, d_R, Lmax, seed, q_scale=1.0):
    """GLA/MLA inputs in the kernel's (absorbed) form, bf16 on CPU.

    q [B, Lq, H, d_c + d_R], c [B, Lmax, h_c, d_c], k_rope [B, Lmax, d_R].
    """
    q = normal_bf16((B, Lq, H, d_c + d_R), seed * 7 + 1, std=q_scale)
    c = normal_bf16((B, Lmax, h_c, d_c), seed * 7 + 2)
    kr = normal_bf16((B, Lmax, d_R), seed * 7 + 3)
    return q, c, kr


def gla_method_inputs(B, Lq, H, h_c, d_c, d_R, d_h, Lmax, seed):
    """Raw (un-absorbed, un-rotated) GLA tensors, bf16 on CPU.

    q_nope [B,Lq,H,d_h], q_pe [B,Lq,H,d_R], c [B,Lmax,h_c,d_c],
    k_pe [B,Lmax,d_R], W_UK / W_UV [H, d_c, d_h] ~ N(0, 1/d_c).
    """
    return dict(
        q_nope=normal_bf16((B, Lq, H, d_h), seed * 11 + 1),
        q_pe=normal_bf16((B, Lq, H, d_R), seed * 11 + 2),
        c=normal_bf16((B, Lmax, h_c, d_c), seed * 11 + 3),
        k_pe=normal_bf16((B, Lmax, d_R), seed * 11 + 4),
        W_UK=normal_bf16((H, d_c, d_h), seed * 11 + 5, std=1.0 / math.sqrt(d_c)),
        W_UV=normal_bf16((H, d_c, d_h), seed * 11 + 6, std=1.0 / math.sqrt(d_c)),
    )


def gta_kernel_inputs(B, Lq, H, h_kv, d_h, Lmax, seed, q_scale=1.0):
    """GTA inputs: q [B,Lq,H,d_h] (nope || rope half), tied kv
    [B,Lmax,h_kv,d_h], single-head k_rope [B,Lmax,d_h/2]; bf16 on CPU."""
    q = normal_bf16((B, Lq, H, d_h), seed * 13 + 1, std=q_scale)
    kv = normal_bf16((B, Lmax, h_kv, d_h), seed * 13 + 2)
    kr = normal_bf16((B, Lmax, d_h // 2), seed * 13 + 3)
    return q, kv, kr


def device_pool(num_pages, page_size, row_stride, seed, device, chunk_bytes=1 << 30):
    """A whole pool of N(0,1) bf16 rows drawn directly on ``device`` (bench
    sizes; the oracle reads sampled rows back through the block table).
    Drawn in ~1 GB fp32 chunks from one seeded generator, so the peak memory
    is the bf16 pool plus one chunk (the C5 TP1 pool is 53 GB)."""
    pool = torch.empty((num_pages, page_size, row_stride), dtype=torch.bfloat16, device=device)
    flat = pool.view(num_pages, -1)
    per = max(1, chunk_bytes // max(1, 4 * flat.shape[1]))
    g = _gen(seed, device)
    for p0 in range(0, num_pages, per):
        p1 = min(num_pages, p0 + per)
        flat[p0:p1] = torch.randn(p1 - p0, flat.shape[1], generator=g, device=device, dtype=torch.float32)
    return pool


def device_queries(B, Lq, H, d_qk, seed, device, q_scale=1.0):
    return normal_bf16((B, Lq, H, d_qk), seed + 1000003, std=q_scale, device=device)
