"""CPU tests of the C-ABI library (no kernel launches): it loads, exports every
symbol include/glad.h declares, validates arguments before touching the GPU,
and its host-only helpers (tp_shard, duplication factor, KV bytes) reproduce
the paper's numbers.  Plus the product-side byte/FLOP accounting."""

import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

from oracle import roofline as RF
from oracle import sharding as SH
from paper_2505_21487_b200 import glad, workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "glad.h")).read()
    return sorted(set(re.findall(r"GLAD_API\s+[\w\s\*]+?\b(glad_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = glad.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(glad.exported_symbols())
    assert "sm_100a" in glad.version()


def test_kv_bytes_reproduce_paper_tables(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "kv_bytes_per_token.json")))
    t = g["xl_tab_val_ppl_downstream_xl_kv"]  # P:1000-1004, h_q=16, d_h=128, d_R=64
    spec = {"MHA": (glad.MHA, 16, 128, 0), "GQA-4": (glad.GQA, 4, 128, 0), "GTA-4": (glad.GTA, 4, 128, 64),
            "GLA-2": (glad.GLA, 2, 256, 64), "MLA": (glad.MLA, 1, 512, 64)}
    for name, vals in t["rows"].items():
        v, n, dh, dr = spec[name]
        assert [glad.kv_bytes_per_token_per_device(v, n, dh, dr, N) for N in t["tp"]] == vals, name
    assert glad.kv_bytes_per_token_per_device(99, 1, 1, 1, 1) == -1


def test_tp_helpers_match_oracle():
    # P:153 duplication factor, S:363-365 spot values
    assert glad.tp_duplication(8, 128, 128) == 8
    assert glad.tp_duplication(8, 2, 16) == 1
    assert glad.tp_duplication(8, 4, 16) == 2
    for h_q in (16, 32, 64, 128):
        for n_kv in [d for d in (1, 2, 4, 8, 16) if h_q % d == 0]:
            for N in (1, 2, 4, 8):
                if h_q % N or (n_kv >= N and n_kv % N) or (n_kv < N and N % n_kv):
                    with pytest.raises(glad.GladError):
                        glad.tp_shard(h_q, n_kv, N, 0)
                    continue
                for r in range(N):
                    assert glad.tp_shard(h_q, n_kv, N, r) == SH.tp_shard(h_q, n_kv, N, r)
                assert glad.tp_duplication(N, h_q // n_kv, h_q) == SH.duplication_factor(N, h_q // n_kv, h_q)


FAKE = ctypes.c_void_p(1 << 20)  # never dereferenced: validation fails first


def _decode_status(layout, B=2, Lq=1, H=16, scale=0.1, ws_bytes=1 << 30, fn="glad_gla_decode", q=FAKE):
    return getattr(glad.lib(), fn)(q, FAKE, ctypes.byref(layout), FAKE, 4, FAKE, B, Lq, H, scale, 1, FAKE, FAKE,
                                   ctypes.c_void_p(1 << 20), ws_bytes, 0, None)


def test_argument_validation_before_launch():
    ok = glad.make_layout(10, 16, 2, 128, 32)
    assert _decode_status(ok, Lq=0) == glad.GLAD_ERR_INVALID_ARG
    assert "Lq" in glad.lib().glad_last_error().decode()
    assert _decode_status(ok, H=15) == glad.GLAD_ERR_INVALID_ARG
    assert _decode_status(ok, scale=0.0) == glad.GLAD_ERR_INVALID_ARG
    assert _decode_status(ok, scale=float("nan")) == glad.GLAD_ERR_INVALID_ARG
    assert _decode_status(ok, q=ctypes.c_void_p((1 << 20) + 2)) == glad.GLAD_ERR_INVALID_ARG  # misaligned
    assert _decode_status(ok, ws_bytes=16) == glad.GLAD_ERR_WORKSPACE
    assert _decode_status(glad.make_layout(10, 16, 2, 192, 32)) == glad.GLAD_ERR_UNSUPPORTED
    assert _decode_status(glad.make_layout(10, 12, 2, 128, 32)) == glad.GLAD_ERR_INVALID_ARG  # page not pow2
    assert _decode_status(glad.make_layout(10, 16, 2, 128, 32, row_stride=100)) == glad.GLAD_ERR_INVALID_ARG
    assert _decode_status(ok, fn="glad_mla_decode") == glad.GLAD_ERR_INVALID_ARG  # MLA needs 1 latent head
    assert _decode_status(glad.make_layout(10, 16, 8, 128, 32), fn="glad_gta_decode") == glad.GLAD_ERR_INVALID_ARG
    assert _decode_status(ok, B=0) == glad.GLAD_OK  # empty batch: nothing to do
    # append / gather / combine validate too
    lib = glad.lib()
    assert lib.glad_cache_append(ctypes.byref(ok), FAKE, FAKE, 4, FAKE, FAKE, -1, 1, None) == glad.GLAD_ERR_INVALID_ARG
    assert lib.glad_splitkv_combine(FAKE, FAKE, 0, 1, 1, 1, 256, FAKE, FAKE, None) == glad.GLAD_ERR_INVALID_ARG
    assert lib.glad_splitkv_combine(FAKE, FAKE, 2, 1, 1, 1, 12, FAKE, FAKE, None) == glad.GLAD_ERR_INVALID_ARG


def test_workspace_and_pool_bytes():
    L = glad.make_layout(16876, 64, 2, 256, 64)
    assert glad.pool_bytes(L) == 16876 * 64 * 576 * 2
    w1 = glad.workspace_bytes(L, 128, 1, 128, glad.GLA, 148)
    w2 = glad.workspace_bytes(L, 128, 1, 128, glad.GLA, 296)
    assert 0 < w1 < w2 < 64 << 20  # plan + (G + U) partial slots, tens of MB at most
    assert glad.workspace_bytes(L, 0, 1, 128, glad.GLA, 148) == 0


def test_accounting_matches_paper_and_baseline():
    wl = workloads.get("c2_gla2")
    sl = wl.seqlens()
    b, f = workloads.algorithmic_bytes(wl, sl), workloads.algorithmic_flops(wl, sl)
    # C2 GLA-2 1.227 GB, 0.155 TF
    assert abs(b / 1e9 - 1.227) < 0.005 and abs(f / 1e12 - 0.155) < 0.001
    # Table 1: GLA-2 arithmetic intensity -> h_q for L >> h_q
    # (with RoPE counted on both sides, d_qk + d_v equals the row width)
    big = workloads.Workload("x", "gla", 1, 1, 128, 2, 256, 64, 1 << 20)
    ai = workloads.algorithmic_flops(big, big.seqlens()) / workloads.algorithmic_bytes(big, big.seqlens())
    assert abs(ai / RF.ai_asymptote("GLA-2", 128) - 1) < 0.01
    # GTA at g_q = 8: Table 1 asymptote 2 g_q = 16, our RoPE-inclusive count 15.06
    gta = workloads.get("c4_gta")
    ai = workloads.algorithmic_flops(gta, gta.seqlens()) / workloads.algorithmic_bytes(gta, gta.seqlens())
    assert 14.5 < ai < RF.ai_asymptote("GTA", 64, g_q=8)


def test_header_documents_every_entry_point():
    txt = open(os.path.join(ROOT, "include", "glad.h")).read()
    for m in re.finditer(r"\nGLAD_API\s+[\w\s\*]+?\b(glad_\w+)\s*\(", txt):
        prefix = txt[:m.start()].rstrip()
        assert prefix.endswith("*/"), f"{m.group(1)} has no comment block right above it"
