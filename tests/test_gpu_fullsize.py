"""Full-size parity for every workload bench.py times (BASELINE.json configs
at their benchmark sizes, in bench.py's launch configuration: the same
workloads.build_device_state + workloads.run call, default persistent grid).

The fp64 oracle cannot run a whole config (C2 is 17.7 TFLOP unabsorbed), so
each test recomputes sampled units one by one: a unit is one (sequence, KV
head) pair with all the query rows of its group, always including the
longest sequence of the batch.  The kernel output for those rows is compared
element by element at the north-star tolerance (max-abs 1e-2, rel-L2 5e-3,
LSE max-abs 1e-2).  Inputs are read back from the device pool through the
block table, so the paging is covered too (a wrong page lookup fails the
comparison)."""

import gc

import numpy as np
import pytest
import torch

from oracle import attention as OA
from paper_2505_21487_b200 import workloads

from gpu_side import DEV, check

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _free():
    gc.collect()
    torch.cuda.empty_cache()


def _logical_rows(st, b, L):
    """Cache rows [L, W] of sequence b, gathered through the block table."""
    layout, pool, bt = st["layout"], st["pool"], st["block_table"]
    pos = torch.arange(L, device=DEV)
    prow = bt[b, pos // layout.page_size].long() * layout.page_size + pos % layout.page_size
    return pool.reshape(-1, layout.row_stride)[prow]


def _samples(wl, st, n_extra=3, seed=0):
    """(b, head) units: the longest sequence (both ends of the head range),
    the shortest one and seeded random others."""
    sl = st["seqlens_host"]
    rng = np.random.default_rng(seed)
    b_long, b_short = int(np.argmax(sl)), int(np.argmin(sl))
    out = [(b_long, 0), (b_long, wl.h_c - 1), (b_short, wl.h_c // 2)]
    for _ in range(n_extra):
        out.append((int(rng.integers(0, wl.B)), int(rng.integers(0, wl.h_c))))
    return list(dict.fromkeys(out))


def latent_check(wl, st, out, lse, samples, t_rows=None):
    """GLA/MLA: q rows of head group i against latent head i + shared RoPE."""
    q = st["q"]
    g_q = wl.H // wl.h_c
    ts = list(range(wl.Lq)) if t_rows is None else list(t_rows)
    for b, i in samples:
        L = int(st["seqlens_host"][b])
        rows = _logical_rows(st, b, L)
        c_i = rows[:, i * wl.d_c:(i + 1) * wl.d_c].cpu()
        kr = rows[:, wl.h_c * wl.d_c: wl.h_c * wl.d_c + wl.d_R].cpu()
        qr = q[b, ts, i * g_q:(i + 1) * g_q].reshape(-1, q.shape[-1]).cpu()
        nvis = [OA.visible_count(L, wl.Lq, t, wl.causal) for t in ts for _ in range(g_q)]
        o_ref, lse_ref = OA.latent_decode_unit(qr, c_i, kr, nvis, wl.scale)
        o_g = out[b, ts, i * g_q:(i + 1) * g_q].reshape(-1, wl.d_c)
        l_g = lse[b, ts, i * g_q:(i + 1) * g_q].reshape(-1)
        check(o_g, l_g, o_ref, lse_ref, what=f"{wl.name} b={b} head={i} L={L}")


def gta_check(wl, st, out, lse, samples):
    """GTA: q rows of KV group g against the tied state g (+ shared K_RoPE)."""
    q = st["q"]
    g_q = wl.H // wl.h_c
    d_h = wl.d_c
    for b, g in samples:
        L = int(st["seqlens_host"][b])
        rows = _logical_rows(st, b, L)
        kv = rows[:, g * d_h:(g + 1) * d_h].cpu()[None, :, None, :]
        kr = rows[:, wl.h_c * d_h: wl.h_c * d_h + d_h // 2].cpu()[None]
        qg = q[b:b + 1, :, g * g_q:(g + 1) * g_q].cpu()
        o_ref, lse_ref = OA.tied_decode(qg, kv, kr, [L], wl.scale, causal=wl.causal)
        check(out[b:b + 1, :, g * g_q:(g + 1) * g_q], lse[b:b + 1, :, g * g_q:(g + 1) * g_q], o_ref, lse_ref,
              what=f"{wl.name} b={b} group={g} L={L}")


def _run(name, seed=None):
    wl = workloads.get(name)
    st = workloads.build_device_state(wl, seed=seed)
    out, lse = workloads.run(wl, st)
    torch.cuda.synchronize()
    return wl, st, out, lse


@pytest.mark.parametrize("name", ["c2_gla2", "c2_mla", "c2_gla2_p1", "c2_gla2_p16"])
def test_c2_full_size(name):
    """BASELINE configs[1]: GLA-2 and the MLA baseline, B=128, ctx 8K,
    DeepSeek-V3 shape; page 64 (and the page-1 / page-16 ablation)."""
    wl, st, out, lse = _run(name)
    latent_check(wl, st, out, lse, _samples(wl, st, seed=1))
    del st
    _free()


@pytest.mark.parametrize("name", ["c3_gla2_q2", "c3_gla2_q4", "c3_mla_q2", "c3_gla2_q2_p1"])
def test_c3_full_size(name):
    """BASELINE configs[2]: speculative q_len 2 / 4, B=64, ctx U[2K,16K]
    (variable lengths, causal among the new tokens)."""
    wl, st, out, lse = _run(name)
    latent_check(wl, st, out, lse, _samples(wl, st, seed=3))
    del st
    _free()


def test_c4_gta_full_size():
    """BASELINE configs[3]: GTA, 64 q heads / 8 tied KV heads, d_h 128 with
    half-RoPE, B=256, ctx 4K (the 144-CTA head-group grid)."""
    wl, st, out, lse = _run("c4_gta")
    gta_check(wl, st, out, lse, _samples(wl, st, n_extra=4, seed=4))
    del st
    _free()


@pytest.mark.parametrize("name", ["c5_gla8_tp1", "c5_gla8_tp8", "c5_gla8_tp8_skew"])
def test_c5_full_size(name):
    """BASELINE configs[4]: GLA-8 at ctx U[32K,64K], B=256: the TP1 problem
    on one GPU (53 GB pool) and one rank's TP8 shard (1 latent head + the
    replicated RoPE, 16 query heads), plus the skew length profile."""
    wl, st, out, lse = _run(name)
    latent_check(wl, st, out, lse, _samples(wl, st, seed=5))
    del st
    _free()


def test_c6_prefill_full_size():
    """Prefill workload (B=2, L = Lq = 4096, GLA-2, h_q 128): sampled query
    positions (first, tile and block edges, last) of both sequences, both
    latent heads."""
    wl, st, out, lse = _run("c6_prefill_gla2")
    ts = [0, 1, 63, 64, 127, 128, 1000, 2047, 4094, 4095]
    latent_check(wl, st, out, lse, [(0, 0), (0, 1), (1, 0), (1, 1)], t_rows=ts)
    del st
    _free()

