"""BASELINE.json workloads (C1-C5) as concrete synthetic device inputs, the
algorithmic byte / FLOP accounting of SURVEY §8(d), and the call that runs one
decode step through the C ABI.  Product-side module: never imports oracle/.

Accounting (MAC-only convention; RoPE MACs counted because the tensor
cores execute them):
  bytes = sum_b L_b * W_unique * 2            (cache rows, RoPE counted once)
        + B*Lq*H*d_qk*2 + B*Lq*H*d_v*2 + B*Lq*H*4      (q, out, lse)
  flops = 2 * H * (d_qk + d_v) * sum_b sum_t vis(b, t)
with W_unique = h_c*d_c + d_R (GLA/MLA) or h_kv*d_h + d_h/2 (GTA),
d_qk = d_c + d_R (GLA/MLA) or d_h (GTA), d_v = d_c or d_h.
"""

import dataclasses
import math

import numpy as np
import torch

import synth

from . import glad


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    variant: str          # "gla" | "mla" | "gta"
    B: int
    Lq: int
    H: int
    h_c: int              # latent heads (GLA/MLA) or tied KV heads (GTA) on this rank
    d_c: int              # d_c or d_h
    d_R: int              # d_R or d_h/2
    L: int                # max / fixed KV length
    len_kind: str = "fixed"
    len_min_ratio: float = 0.125
    page: int = 64
    causal: bool = True
    scale: float = 1.0
    seed: int = 1
    description: str = ""
    kind: str = "decode"  # "decode" | "prefill_mat" (glad_gla_prefill, materialised K / V)
    d_h: int = 128        # per-head width of the materialised prefill

    @property
    def d_qk(self):
        return self.d_c if self.variant == "gta" else self.d_c + self.d_R

    @property
    def d_v(self):
        return self.d_c

    @property
    def width(self):
        return self.h_c * self.d_c + self.d_R

    def seqlens(self):
        return synth.seqlens(self.B, self.L, self.len_kind, r=self.len_min_ratio, seed=self.seed)


def _c5(N, kind="uniform"):
    return Workload(f"c5_gla8_tp{N}" + ("" if kind == "uniform" else "_skew"), "gla", 256, 1, 128 // N, 8 // N, 256,
                    64, 65536, len_kind=kind, len_min_ratio=0.5, page=64, scale=1 / math.sqrt(192), seed=5,
                    description=f"GLA-8 (h_c=8, d_c=256, d_R=64, h_q=128) TP={N} shard on one rank, B=256, "
                                f"ctx U[32K,64K]" if kind == "uniform" else "skew [1024]*15+[64K]")


WORKLOADS = {w.name: w for w in [
    Workload("c1_gla2", "gla", 2, 1, 16, 2, 128, 32, 256, page=16, scale=1 / math.sqrt(96), seed=0,
             description="GLA-2 oracle-scale: B=2, ctx 256, q_len 1, 16 q heads, 2x128 + 32, page 16"),
    Workload("c2_gla2", "gla", 128, 1, 128, 2, 256, 64, 8192, page=64, scale=1 / math.sqrt(192), seed=1,
             description="GLA-2 DeepSeek-V3 shape: B=128, ctx 8K, h_q=128, 2x256 + 64, page 64"),
    Workload("c2_mla", "mla", 128, 1, 128, 1, 512, 64, 8192, page=64, scale=1 / math.sqrt(192), seed=1,
             description="MLA DeepSeek-V3 shape: B=128, ctx 8K, h_q=128, 1x512 + 64, page 64"),
    Workload("c3_gla2_q2", "gla", 64, 2, 128, 2, 256, 64, 16384, len_kind="uniform", scale=1 / math.sqrt(192),
             seed=3, description="GLA-2 speculative q_len 2, B=64, ctx U[2K,16K]"),
    Workload("c3_gla2_q4", "gla", 64, 4, 128, 2, 256, 64, 16384, len_kind="uniform", scale=1 / math.sqrt(192),
             seed=3, description="GLA-2 speculative q_len 4, B=64, ctx U[2K,16K]"),
    Workload("c3_mla_q2", "mla", 64, 2, 128, 1, 512, 64, 16384, len_kind="uniform", scale=1 / math.sqrt(192),
             seed=3, description="MLA speculative q_len 2, B=64, ctx U[2K,16K]"),
    Workload("c4_gta", "gta", 256, 1, 64, 8, 128, 64, 4096, page=64, scale=1 / math.sqrt(128), seed=4,
             description="GTA Llama-style: h_q=64, 8 tied KV heads, d_h=128 half-RoPE, B=256, ctx 4K"),
    _c5(1), _c5(2), _c5(4), _c5(8), _c5(8, "skew"),
    # prefill in the absorbed form: every prompt token is a query (Lq = L)
    Workload("c6_prefill_gla2", "gla", 2, 4096, 128, 2, 256, 64, 4096, page=64, scale=1 / math.sqrt(192), seed=6,
             description="GLA-2 prefill as a full-length causal query: B=2, L=Lq=4096, h_q=128, 2x256 + 64"),
    # prefill in the materialised form: per-head K / V up-projected, then attention over them
    Workload("c6_prefill_gla2_mat", "gla", 2, 4096, 128, 2, 256, 64, 4096, page=64, scale=1 / math.sqrt(192), seed=6,
             kind="prefill_mat", d_h=128,
             description="GLA-2 prefill, materialised K/V (d_h 128 + RoPE 64): B=2, L=4096, h_q=128, d_c=256"),
    Workload("c7_prefill_gta", "gta", 2, 4096, 64, 8, 128, 64, 4096, page=64, scale=1 / math.sqrt(128), seed=7,
             description="GTA prefill as a full-length causal query: B=2, L=Lq=4096, h_q=64, 8 tied heads d_h=128"),
    # page-size ablation (page 1 vs 64 for GLA 2x256+64)
    Workload("c2_gla2_p1", "gla", 128, 1, 128, 2, 256, 64, 8192, page=1, scale=1 / math.sqrt(192), seed=1,
             description="C2 GLA-2 with page size 1 (prefix caching, P:316)"),
    Workload("c2_gla2_p16", "gla", 128, 1, 128, 2, 256, 64, 8192, page=16, scale=1 / math.sqrt(192), seed=1,
             description="C2 GLA-2 with page size 16"),
    Workload("c3_gla2_q2_p1", "gla", 64, 2, 128, 2, 256, 64, 16384, len_kind="uniform", page=1,
             scale=1 / math.sqrt(192), seed=3, description="C3 GLA-2 q_len 2 with page size 1 (P:1412 setting)"),
]}


def get(name):
    return WORKLOADS[name]


def visible_counts(seqlens, Lq, causal):
    out = []
    for L in seqlens:
        for t in range(Lq):
            out.append(max(0, min(int(L), int(L) - Lq + t + 1)) if causal else int(L))
    return np.array(out, dtype=np.int64)


def algorithmic_bytes(wl, seqlens):
    if wl.kind == "prefill_mat":  # raw inputs once + weights + output
        n = int(np.sum(seqlens))
        return int(2 * (n * wl.H * (wl.d_h + wl.d_R) + n * (wl.h_c * wl.d_c + wl.d_R) + 2 * wl.H * wl.d_c * wl.d_h
                        + n * wl.H * wl.d_h) + 4 * n * wl.H)
    rows = wl.B * wl.Lq * wl.H
    return int(np.sum(seqlens, dtype=np.int64) * wl.width * 2 + rows * wl.d_qk * 2 + rows * wl.d_v * 2 + rows * 4)


def algorithmic_flops(wl, seqlens):
    vis = visible_counts(seqlens, wl.Lq, wl.causal).sum()
    if wl.kind == "prefill_mat":  # attention over d_h + d_R keys, d_h values, plus the K / V up-projections
        return int(2 * wl.H * (2 * wl.d_h + wl.d_R) * vis + 2 * 2 * int(np.sum(seqlens)) * wl.H * wl.d_c * wl.d_h)
    return int(2 * wl.H * (wl.d_qk + wl.d_v) * vis)


def build_prefill_state(wl, seed=None, device="cuda", num_ctas=0):
    """Raw GLA tensors of a prompt batch, drawn on the device (materialised prefill)."""
    seed = wl.seed if seed is None else seed
    sl = wl.seqlens()
    B, L, H = wl.B, wl.L, wl.H
    g = lambda shape, k, std=1.0: synth.normal_bf16(shape, seed * 11 + k, std=std, device=device)
    st = dict(q_nope=g((B, L, H, wl.d_h), 1), q_pe=g((B, L, H, wl.d_R), 2), c=g((B, L, wl.h_c, wl.d_c), 3),
              k_pe=g((B, L, wl.d_R), 4), W_UK=g((H, wl.d_c, wl.d_h), 5, 1.0 / math.sqrt(wl.d_c)),
              W_UV=g((H, wl.d_c, wl.d_h), 6, 1.0 / math.sqrt(wl.d_c)),
              seqlens=torch.from_numpy(sl.astype(np.int32)).to(device), seqlens_host=sl, num_ctas=num_ctas,
              out=torch.empty(B, L, H, wl.d_h, dtype=torch.bfloat16, device=device),
              lse=torch.empty(B, L, H, dtype=torch.float32, device=device), workspace=glad.Workspace(device))
    st["workspace"].get(glad.gla_prefill_workspace_bytes(B, L, H, wl.d_h, wl.d_R, num_ctas))
    st["q"] = st["q_nope"]
    return st


def build_device_state(wl, seed=None, device="cuda", num_ctas=0):
    """Seeded synthetic device state: pool of N(0,1) bf16 rows (pages are a
    random permutation), block table, seqlens, queries, preallocated outputs
    and split workspace (so the step is CUDA-graph capturable)."""
    if wl.kind == "prefill_mat":
        return build_prefill_state(wl, seed, device, num_ctas)
    seed = wl.seed if seed is None else seed
    sl = wl.seqlens()
    bt, num_pages = synth.block_table(sl, wl.page, seed=seed)
    layout = glad.make_layout(num_pages, wl.page, wl.h_c, wl.d_c, wl.d_R)
    pool = synth.device_pool(num_pages, wl.page, layout.row_stride, seed, device)
    q = synth.device_queries(wl.B, wl.Lq, wl.H, wl.d_qk, seed, device)
    variant = {"gla": glad.GLA, "mla": glad.MLA, "gta": glad.GTA}[wl.variant]
    ws = glad.Workspace(device)
    ws.get(glad.workspace_bytes(layout, wl.B, wl.Lq, wl.H, variant, num_ctas))
    return dict(layout=layout, pool=pool, block_table=torch.from_numpy(bt).to(device),
                seqlens=torch.from_numpy(sl.astype(np.int32)).to(device), seqlens_host=sl, q=q,
                out=torch.empty(wl.B, wl.Lq, wl.H, wl.d_v, dtype=torch.bfloat16, device=device),
                lse=torch.empty(wl.B, wl.Lq, wl.H, dtype=torch.float32, device=device),
                num_ctas=num_ctas, workspace=ws)


def run(wl, st, stream=None, q=None):
    """One decode step through the C ABI (plan + decode + merge kernels)."""
    if wl.kind == "prefill_mat":
        return glad.gla_prefill(st["q_nope"] if q is None else q, st["q_pe"], st["c"], st["k_pe"], st["W_UK"],
                                st["W_UV"], st["seqlens"], wl.scale, out=st["out"], lse=st["lse"],
                                num_ctas=st["num_ctas"], workspace=st["workspace"], stream=stream)
    fn = {"gla": glad.gla_decode, "mla": glad.mla_decode, "gta": glad.gta_decode}[wl.variant]
    return fn(st["q"] if q is None else q, st["pool"], st["layout"], st["block_table"], st["seqlens"], wl.scale,
              causal=wl.causal, out=st["out"], lse=st["lse"], num_ctas=st["num_ctas"], workspace=st["workspace"],
              stream=stream)
