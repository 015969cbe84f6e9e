"""Helpers on the CUDA side of the parity tests: build paged pools through the
library's own append kernel, form kernel inputs (absorbed query, rotated RoPE
parts) with torch, and error metrics.  Independent of oracle/ (no imports
from it, no shared arithmetic)."""

import math

import numpy as np
import torch

import synth
from paper_2505_21487_b200 import glad

DEV = "cuda"


def rel_l2(a, b):
    a = torch.as_tensor(a, dtype=torch.float64).flatten()
    b = torch.as_tensor(b, dtype=torch.float64).flatten()
    return float((a - b).norm() / b.norm().clamp_min(1e-300))


def max_abs(a, b):
    a = torch.as_tensor(a, dtype=torch.float64)
    b = torch.as_tensor(b, dtype=torch.float64)
    return float((a - b).abs().max()) if a.numel() else 0.0


def build_paged(rows, seqlens, page_size, n_heads_kv, d_head, d_rope, seed=0, row_stride=None,
                fill=float("nan"), min_pages_per_seq=0):
    """Scatter logical rows [B, Lmax, W] (bf16, CPU) into a NaN-filled pool on
    the GPU with glad_cache_append, one call per sequence (ragged lengths)."""
    B = rows.shape[0]
    bt, num_pages = synth.block_table(seqlens, page_size, seed=seed, min_pages_per_seq=min_pages_per_seq)
    layout = glad.make_layout(num_pages, page_size, n_heads_kv, d_head, d_rope, row_stride)
    pool = torch.full((num_pages, page_size, layout.row_stride), fill, dtype=torch.bfloat16, device=DEV)
    bt_d = torch.from_numpy(bt).to(DEV)
    zero = torch.zeros(1, dtype=torch.int32, device=DEV)
    for b in range(B):
        L = int(seqlens[b])
        if L > 0:
            glad.cache_append(layout, pool, bt_d[b:b + 1].contiguous(), zero,
                              rows[b:b + 1, :L].contiguous().to(DEV))
    torch.cuda.synchronize()
    return layout, pool, bt_d


def latent_rows(c, k_rope):
    """[B, L, h_c, d_c] + [B, L, d_R] -> cache rows [B, L, h_c*d_c + d_R]."""
    B, L = c.shape[:2]
    return torch.cat([c.reshape(B, L, -1), k_rope], dim=-1).contiguous()


def rope_torch(x, pos, base=10000.0):
    """RoPE (reading R5: interleaved pairs, base 10000) in fp64 torch; the
    GPU-side harness's own implementation (upstream of the kernel)."""
    x = x.to(torch.float64)
    d = x.shape[-1]
    i = torch.arange(d // 2, dtype=torch.float64)
    theta = base ** (-2.0 * i / d)
    ang = torch.as_tensor(pos, dtype=torch.float64)[..., None] * theta
    c, s = torch.cos(ang), torch.sin(ang)
    out = torch.empty_like(x)
    out[..., 0::2] = x[..., 0::2] * c - x[..., 1::2] * s
    out[..., 1::2] = x[..., 0::2] * s + x[..., 1::2] * c
    return out


def absorb_inputs(x, seqlens, Lq):
    """Kernel inputs from raw GLA tensors: q = [W_UK q_nope || RoPE(q_pe, p_t)],
    cache rows = [c || RoPE(k_pe, j)], rounded to bf16 (upstream step)."""
    q_abs = torch.einsum("hcd,bthd->bthc", x["W_UK"].double(), x["q_nope"].double())
    B = q_abs.shape[0]
    pos_q = torch.tensor([[int(seqlens[b]) - Lq + t for t in range(Lq)] for b in range(B)])[..., None]
    q_r = rope_torch(x["q_pe"], pos_q)
    L = x["k_pe"].shape[1]
    k_r = rope_torch(x["k_pe"], torch.arange(L)[None, :].expand(B, L))
    q = torch.cat([q_abs, q_r], dim=-1).to(torch.bfloat16)
    return q, x["c"], k_r.to(torch.bfloat16)


def check(o_gpu, lse_gpu, o_ref, lse_ref, tol_abs=1e-2, tol_rel=5e-3, tol_lse=1e-2, what="", abs_per_unit=False):
    """North-star tolerance.  abs_per_unit (R18, head-space outputs
    whose magnitude exceeds 1): the max-abs bound applies to
    |err| / max(1, |ref|), since the bf16 output format alone rounds a value
    in [2, 4) by up to 2^-8."""
    o_gpu = o_gpu.float().cpu().double()
    o_ref = torch.as_tensor(o_ref, dtype=torch.float64)
    lse_gpu = lse_gpu.float().cpu().double()
    lse_ref = torch.as_tensor(lse_ref, dtype=torch.float64)
    assert torch.isfinite(o_gpu).all(), f"{what}: non-finite output"
    fin = torch.isfinite(lse_ref)
    assert torch.equal(torch.isfinite(lse_gpu), fin), f"{what}: lse finiteness pattern differs"
    ma, rl = max_abs(o_gpu, o_ref), rel_l2(o_gpu, o_ref)
    if abs_per_unit and o_gpu.numel():
        ma = float(((o_gpu - o_ref).abs() / o_ref.abs().clamp_min(1.0)).max())
    ml = max_abs(lse_gpu[fin], lse_ref[fin]) if fin.any() else 0.0
    assert ma <= tol_abs and rl <= tol_rel and ml <= tol_lse, \
        f"{what}: max_abs={ma:.3e} rel_l2={rl:.3e} lse_max_abs={ml:.3e}"
    return ma, rl, ml
