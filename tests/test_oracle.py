"""Pins for the fp64 oracle (CPU only): each test ties the oracle to something
other than itself — a number printed in the paper, a hand-worked example, a
closed form, an algebraic identity of the method, or a library routine
(torch SDPA in fp64).  A dropped term, wrong sign/index or transposed operand
in the oracle fails at least one of these."""

import json
import math
import os

import numpy as np
import pytest
import torch

import synth
from oracle import attention as A
from oracle import paging as PG
from oracle import roofline as RF
from oracle import rope as R
from oracle import sharding as SH


def f64(t):
    return t.to(torch.float64).numpy()


# ---------------------------------------------------------------- golden ---
def test_hand_example(golden_dir):
    d = json.load(open(os.path.join(golden_dir, "hand_example.json")))
    for case, tol in ((d, 1e-13), (d["second_case"], d["second_case"]["tol"])):
        q = np.array(case["q"])[None, None, None, :]
        c = np.array(case["c"])[None, :, None, :]
        kr = np.zeros((1, c.shape[1], 0))
        o, lse = A.latent_decode(q, c, kr, [c.shape[1]], case["scale"], causal=False)
        np.testing.assert_allclose(o[0, 0, 0], case["o"], rtol=0, atol=tol)
        assert abs(lse[0, 0, 0] - case["lse"]) < tol


def test_kv_bytes_tables(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "kv_bytes_per_token.json")))
    name_map = {"GQA-4": ("GQA", 4), "GTA-4": ("GTA", 4), "GLA-2": ("GLA", 2)}

    def heads_and_dims(v, h_q, d_h, d_R, h_kv=None):
        if v == "MHA":
            return "MHA", h_q, d_h, 0
        if v == "MQA":
            return "MQA", 1, d_h, 0
        if v == "MLA":
            return "MLA", 1, 4 * d_h, d_R
        kind, n = name_map[v]
        if h_kv is not None and kind in ("GQA", "GTA"):
            n = h_kv
        if kind == "GLA":
            return "GLA", n, 2 * d_h, d_R
        return kind, n, d_h, (d_h // 2 if kind == "GTA" else 0)

    for key in ("xl_tab_main_combined_summary_xl", "xl_tab_val_ppl_downstream_xl_kv"):
        t = g[key]
        for v, vals in t["rows"].items():
            kind, n, dh, dr = heads_and_dims(v, t["dims"]["h_q"], t["dims"]["d_h"], t["dims"]["d_R"])
            got = [SH.kv_bytes_per_token_per_device(kind, n, dh, dr, N) for N in t["tp"]]
            assert got == vals, (key, v, got, vals)
    t = g["medium_tab_ablation_change_hq"]
    for v, vals in t["rows"].items():
        kind, n, dh, dr = heads_and_dims(v, t["h_q"][v], t["dims"]["d_h"], t["dims"]["d_R"])
        got = [SH.kv_bytes_per_token_per_device(kind, n, dh, dr, N) for N in t["tp"]]
        assert got == vals, (v, got, vals)
    t = g["llama3_8b_tab_kv_cache_sizes_dh_units"]
    d_h = 128  # any d_h: the table is in d_h units
    for v, vals in t["rows"].items():
        kind, n, dh, dr = heads_and_dims(v, t["dims"]["h_q"], d_h, d_h // 2, h_kv=t["dims"]["h_kv"])
        got = [SH.kv_elems_per_token_per_device(kind, n, dh, dr, N) / d_h for N in t["tp"]]
        assert got == vals, (v, got, vals)


def test_kv_bytes_formula_p123():
    # P:123-131 with MHA h_q=16,d_h=128 (g_q=1, m_kv=2) at one token -> 8192
    assert SH.kv_bytes(2, 1, 1, 16, 1, 128) == 8192
    assert SH.kv_bytes(2, 3, 5, 16, 1, 128) == 15 * 8192


def test_duplication_factor_spot_values():
    # S:363-365 and the zero-redundancy bound P:159-162
    assert SH.duplication_factor(8, 128, 128) == 8
    assert SH.duplication_factor(8, 2, 16) == 1
    assert SH.duplication_factor(8, 4, 16) == 2
    for h_q in range(1, 65):
        for N in (1, 2, 4, 8):
            for g_q in [g for g in range(1, h_q + 1) if h_q % g == 0]:
                D = SH.duplication_factor(N, g_q, h_q)
                assert 1 <= D <= N or (N * g_q > h_q * N)
                assert (D == 1) == SH.zero_redundancy(N, g_q, h_q)


def test_ai_closed_forms():
    # MLA h_q=128 at L=8192 -> 248.24 ; asymptotes of Table 1
    assert abs(RF.ai_closed_form("MLA", 8192, 128) - 248.24) < 0.01
    L = 10 ** 6
    for v, kw in [("GLA-2", dict(h_q=128)), ("GLA", dict(h_q=128, g_q=16)), ("MLA", dict(h_q=128)),
                  ("MQA", dict(h_q=32)), ("GQA", dict(h_q=32, g_q=4)), ("GTA", dict(h_q=32, g_q=4)),
                  ("MHA", dict(h_q=32)), ("General", dict(h_q=32, g_q=8, m_kv=1))]:
        a = RF.ai_closed_form(v, L, **kw)
        assert abs(a / RF.ai_asymptote(v, **kw) - 1) < 5e-3, v
    # GTA doubles GQA at equal g_q
    assert abs(RF.ai_closed_form("GTA", L, 32, 4) / RF.ai_closed_form("GQA", L, 32, 4) - 2) < 1e-4


# ------------------------------------------------------------------ rope ---
def test_rope_properties():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 64))
    np.testing.assert_array_equal(R.rope_rotate(x, 0), x)                       # pos 0 identity
    y = R.rope_rotate(x, 37)
    np.testing.assert_allclose(np.hypot(y[:, 0::2], y[:, 1::2]),
                               np.hypot(x[:, 0::2], x[:, 1::2]), rtol=1e-12)     # per-pair norm
    np.testing.assert_allclose(R.rope_unrotate(y, 37), x, atol=1e-12)           # inverse
    for _ in range(100):                                                          # relative position
        q, k = rng.standard_normal(32), rng.standard_normal(32)
        a, b, dl = rng.integers(0, 5000, 3)
        lhs = R.rope_rotate(q, a + dl) @ R.rope_rotate(k, b + dl)
        rhs = R.rope_rotate(q, a) @ R.rope_rotate(k, b)
        assert abs(lhs - rhs) < 1e-9 * max(1, abs(rhs))
    # angle convention: pair i rotates by pos * 10000^(-2i/d); pair 0 by pos rad
    e = np.zeros(8); e[0] = 1.0
    np.testing.assert_allclose(R.rope_rotate(e, 1.0)[:2], [math.cos(1), math.sin(1)], atol=1e-15)
    e = np.zeros(8); e[2] = 1.0
    th = 10000 ** (-2 / 8)
    np.testing.assert_allclose(R.rope_rotate(e, 3.0)[2:4], [math.cos(3 * th), math.sin(3 * th)], atol=1e-15)


# -------------------------------------------------------- closed forms ---
def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def test_latent_closed_forms():
    d_c, d_R = 8, 4
    c = _rand((1, 6, 1, d_c), 1)
    kr = _rand((1, 6, d_R), 2)
    # L = 1: o = V[0], lse = s_0
    q = _rand((1, 1, 1, d_c + d_R), 3)
    o, lse = A.latent_decode(q, c, kr, [1], 0.3, causal=True)
    np.testing.assert_allclose(o[0, 0, 0], c[0, 0, 0], atol=1e-15)
    s0 = 0.3 * (q[0, 0, 0, :d_c] @ c[0, 0, 0] + q[0, 0, 0, d_c:] @ kr[0, 0])
    assert abs(lse[0, 0, 0] - s0) < 1e-13
    # zero query: uniform weights, o = mean V, lse = ln L
    o, lse = A.latent_decode(np.zeros((1, 1, 1, d_c + d_R)), c, kr, [6], 0.3, causal=False)
    np.testing.assert_allclose(o[0, 0, 0], c[0, :6, 0].mean(0), atol=1e-14)
    assert abs(lse[0, 0, 0] - math.log(6)) < 1e-14
    # one dominant score -> that row
    cc = np.zeros((1, 3, 1, d_c)); cc[0, :, 0, :] = np.eye(3, d_c)
    q = np.zeros((1, 1, 1, d_c + d_R)); q[0, 0, 0, 1] = 2000.0
    o, lse = A.latent_decode(q, cc, np.zeros((1, 3, d_R)), [3], 1.0, causal=False)
    np.testing.assert_allclose(o[0, 0, 0], cc[0, 1, 0], atol=1e-12)
    assert abs(lse[0, 0, 0] - 2000.0) < 1e-9
    # identical keys -> uniform; empty -> 0 / -inf
    cc = np.repeat(_rand((1, 1, 1, d_c), 5), 4, axis=1)
    krr = np.repeat(_rand((1, 1, d_R), 6), 4, axis=1)
    q = _rand((1, 1, 1, d_c + d_R), 7)
    o, lse = A.latent_decode(q, cc, krr, [4], 0.5, causal=False)
    s = 0.5 * (q[0, 0, 0, :d_c] @ cc[0, 0, 0] + q[0, 0, 0, d_c:] @ krr[0, 0])
    np.testing.assert_allclose(o[0, 0, 0], cc[0, 0, 0], atol=1e-13)
    assert abs(lse[0, 0, 0] - (s + math.log(4))) < 1e-12
    o, lse = A.latent_decode(q, cc, krr, [0], 0.5, causal=False)
    assert np.all(o == 0) and lse[0, 0, 0] == -np.inf


def test_softmax_shift_invariance_and_stability():
    s = _rand(17, 8)
    p1, l1 = A.softmax_row(s)
    p2, l2 = A.softmax_row(s + 123.456)
    np.testing.assert_allclose(p1, p2, atol=1e-14)
    assert abs((l2 - l1) - 123.456) < 1e-11
    p, _ = A.softmax_row([1000.0, 0.0])
    np.testing.assert_allclose(p, [1.0, 0.0], atol=1e-300)
    assert abs(p.sum() - 1) < 1e-15


def test_brute_force_tiny():
    """L <= 3, d <= 4 evaluated term by term with scalar Python."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        L = int(rng.integers(1, 4))
        d_c, d_R = 3, 2
        q = rng.standard_normal(d_c + d_R)
        c = rng.standard_normal((L, d_c))
        kr = rng.standard_normal((L, d_R))
        sc = float(rng.uniform(0.1, 1.0))
        s = []
        for j in range(L):
            acc = 0.0
            for k in range(d_c):
                acc += q[k] * c[j, k]
            for k in range(d_R):
                acc += q[d_c + k] * kr[j, k]
            s.append(sc * acc)
        z = sum(math.exp(v) for v in s)
        want = [sum(math.exp(s[j]) / z * c[j, k] for j in range(L)) for k in range(d_c)]
        o, lse = A.latent_decode(q[None, None, None], c[None, :, None], kr[None], [L], sc, causal=False)
        np.testing.assert_allclose(o[0, 0, 0], want, atol=1e-13)
        assert abs(lse[0, 0, 0] - math.log(z)) < 1e-13


# ------------------------------------------------- library routine pins ---
def _sdpa(q, K, V, scale, mask):
    """torch SDPA in fp64 on CPU.  q [n, d], K [L, d], V [L, dv], mask [n, L] bool."""
    return torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q)[None, None], torch.from_numpy(K)[None, None],
        torch.from_numpy(V)[None, None], attn_mask=torch.from_numpy(mask)[None, None],
        scale=scale)[0, 0].numpy()


@pytest.mark.parametrize("Lq,causal", [(1, True), (2, True), (4, True), (3, False)])
def test_latent_decode_vs_sdpa(Lq, causal):
    B, H, h_c, d_c, d_R, L = 2, 8, 2, 16, 8, 21
    q, c, kr = (f64(t) for t in synth.latent_kernel_inputs(B, Lq, H, h_c, d_c, d_R, L, seed=3))
    sl = [L, 13]
    o, lse = A.latent_decode(q, c, kr, sl, 0.17, causal=causal)
    g_q = H // h_c
    for b in range(B):
        pos = np.arange(sl[b])
        for h in range(H):
            i = h // g_q
            K = np.concatenate([c[b, :sl[b], i], kr[b, :sl[b]]], 1)
            V = c[b, :sl[b], i]
            qt = np.arange(Lq)
            mask = (pos[None, :] <= (sl[b] - Lq + qt)[:, None]) if causal else np.ones((Lq, sl[b]), bool)
            ref = _sdpa(q[b, :, h], K, V, 0.17, mask)
            np.testing.assert_allclose(o[b, :, h], ref, atol=1e-12)


def test_gqa_and_degeneracies_vs_sdpa():
    B, Lq, H, d, L = 1, 2, 8, 16, 11
    rng = np.random.default_rng(4)
    q = rng.standard_normal((B, Lq, H, d))
    for h_kv in (8, 2, 1):                  # MHA, GQA, MQA
        k = rng.standard_normal((B, L, h_kv, d))
        v = rng.standard_normal((B, L, h_kv, d))
        o, _ = A.gqa_decode(q, k, v, [L], 0.25, causal=True)
        qt = np.arange(Lq)
        mask = np.arange(L)[None, :] <= (L - Lq + qt)[:, None]
        for h in range(H):
            g = h // (H // h_kv)
            ref = _sdpa(q[0, :, h], k[0, :, g], v[0, :, g], 0.25, mask)
            np.testing.assert_allclose(o[0, :, h], ref, atol=1e-12)


# ------------------------------------------------------ method identities ---
@pytest.mark.parametrize("h_c,d_h,Lq", [(2, 8, 1), (2, 8, 2), (1, 8, 2), (4, 4, 1)])
def test_absorbed_equals_unabsorbed(h_c, d_h, Lq):
    """W_UK absorbed into the query gives the same scores; the latent
    output up-projected by W_UV gives the head output (associativity)."""
    B, H, d_R, L = 2, 8, 4, 9
    d_c = 2 * d_h if h_c > 1 else 4 * d_h
    x = {k: f64(v) for k, v in synth.gla_method_inputs(B, Lq, H, h_c, d_c, d_R, d_h, L, seed=5).items()}
    sl = [L, 6]
    o_head, o_lat, lse_u = A.gla_unabsorbed(x["q_nope"], x["q_pe"], x["c"], x["k_pe"],
                                            x["W_UK"], x["W_UV"], sl, 0.2)
    # absorbed inputs: q_abs[h] = W_UK[h] q_nope[h]; RoPE on q_pe at p_t, on k_pe at j
    q_abs = np.einsum("hcd,bthd->bthc", x["W_UK"], x["q_nope"])
    q_r = np.zeros_like(x["q_pe"])
    k_r = np.zeros_like(x["k_pe"])
    for b in range(B):
        for t in range(Lq):
            q_r[b, t] = R.rope_rotate(x["q_pe"][b, t], sl[b] - Lq + t)
        k_r[b] = R.rope_rotate(x["k_pe"][b], np.arange(L)[:, None].repeat(1, 1)[:, 0])
    o_lat2, lse_a = A.latent_decode(np.concatenate([q_abs, q_r], -1), x["c"], k_r, sl, 0.2)
    np.testing.assert_allclose(o_lat2, o_lat, atol=1e-12)
    np.testing.assert_allclose(lse_a, lse_u, atol=1e-12)
    up = np.einsum("bthc,hcd->bthd", o_lat, x["W_UV"])
    np.testing.assert_allclose(up, o_head, atol=1e-12)


@pytest.mark.parametrize("Lq,causal", [(1, True), (2, True), (3, False)])
def test_mla_is_one_group_vs_sdpa(Lq, causal):
    """MLA = GLA with one latent head (h_c = 1, d_c = 4 d_h): every
    query head attends to the same latent + shared RoPE key.  Pinned against
    torch SDPA (fp64, a library routine) per head, so a wrong head-to-group
    map at h_c = 1 (e.g. h // g_q off by one) fails here."""
    B, H, d_h, d_R, L = 2, 6, 4, 4, 15
    d_c = 4 * d_h
    q, c, kr = (f64(t) for t in synth.latent_kernel_inputs(B, Lq, H, 1, d_c, d_R, L, seed=9))
    sl = [L, 9]
    o, lse = A.latent_decode(q, c, kr, sl, 0.3, causal=causal)
    for b in range(B):
        pos = np.arange(sl[b])
        K = np.concatenate([c[b, :sl[b], 0], kr[b, :sl[b]]], 1)
        V = c[b, :sl[b], 0]
        qt = np.arange(Lq)
        mask = (pos[None, :] <= (sl[b] - Lq + qt)[:, None]) if causal else np.ones((Lq, sl[b]), bool)
        for h in range(H):
            np.testing.assert_allclose(o[b, :, h], _sdpa(q[b, :, h], K, V, 0.3, mask), atol=1e-12)
            # lse against the log-sum-exp of the masked scores (numpy, fp64)
            s = 0.3 * (q[b, :, h] @ K.T)
            s = np.where(mask, s, -np.inf)
            np.testing.assert_allclose(lse[b, :, h], np.log(np.exp(s).sum(-1)), atol=1e-12)


def test_gta_structure_and_gqa_equivalence():
    """V == KV bit-exact; K[:d_h/2] == KV[:d_h/2] bit-exact; the
    tied half is never rotated; with K/V materialised, GTA == GQA."""
    B, Lq, H, h_kv, d_h, L = 2, 2, 8, 2, 16, 10
    q, kv, kr = (f64(t) for t in synth.gta_kernel_inputs(B, Lq, H, h_kv, d_h, L, seed=6))
    K, V = A.gta_keys_values(kv[0], kr[0])
    np.testing.assert_array_equal(V, kv[0])
    np.testing.assert_array_equal(K[:, :, : d_h // 2], kv[0][:, :, : d_h // 2])
    for g in range(h_kv):
        np.testing.assert_array_equal(K[:, g, d_h // 2:], kr[0])
    sl = [L, 7]
    o, lse = A.tied_decode(q, kv, kr, sl, 0.2)
    Kf = np.zeros_like(kv)
    for b in range(B):
        Kf[b] = A.gta_keys_values(kv[b], kr[b])[0]
    o2, lse2 = A.gqa_decode(q, Kf, kv, sl, 0.2)
    np.testing.assert_allclose(o, o2, atol=1e-13)
    np.testing.assert_allclose(lse, lse2, atol=1e-13)


def test_gta_rotation_only_on_rope_half():
    """gta_decode (unrotated inputs) == tied_decode on pre-rotated inputs;
    rotating the tied half instead changes the result."""
    B, Lq, H, h_kv, d_h, L = 1, 2, 4, 2, 8, 9
    q, kv, kr = (f64(t) for t in synth.gta_kernel_inputs(B, Lq, H, h_kv, d_h, L, seed=8))
    o, lse = A.gta_decode(q, kv, kr, [L], 0.3)
    qr = q.copy()
    for t in range(Lq):
        qr[0, t, :, d_h // 2:] = R.rope_rotate(q[0, t, :, d_h // 2:], L - Lq + t)
    krr = R.rope_rotate(kr[0], np.arange(L))[None]
    o2, lse2 = A.tied_decode(qr, kv, krr, [L], 0.3)
    np.testing.assert_allclose(o, o2, atol=1e-13)
    o3, _ = A.tied_decode(q, kv, kr, [L], 0.3)   # no rotation at all -> differs
    assert np.abs(o3 - o).max() > 1e-3


def test_gta_is_zero_padded_latent():
    """GTA == GLA with h_c = h_kv, d_c = d_h, d_R = d_h/2 and the latent query
    zero-padded q_c = [q_nope, 0] (SURVEY §8(c) bridge identity)."""
    B, Lq, H, h_kv, d_h, L = 2, 2, 8, 4, 16, 12
    q, kv, kr = (f64(t) for t in synth.gta_kernel_inputs(B, Lq, H, h_kv, d_h, L, seed=10))
    sl = [L, 5]
    o, lse = A.tied_decode(q, kv, kr, sl, 0.25)
    half = d_h // 2
    qpad = np.concatenate([q[..., :half], np.zeros_like(q[..., :half]), q[..., half:]], -1)
    o2, lse2 = A.latent_decode(qpad, kv, kr, sl, 0.25)
    np.testing.assert_allclose(o, o2, atol=1e-13)
    np.testing.assert_allclose(lse, lse2, atol=1e-13)


def test_causal_lq2_equals_two_steps():
    """a causal Lq=2 step equals two successive Lq=1 steps."""
    B, H, h_c, d_c, d_R, L = 2, 4, 2, 8, 4, 10
    q, c, kr = (f64(t) for t in synth.latent_kernel_inputs(B, 2, H, h_c, d_c, d_R, L, seed=12))
    sl = np.array([L, 6])
    o, lse = A.latent_decode(q, c, kr, sl, 0.3, causal=True)
    o0, l0 = A.latent_decode(q[:, :1], c, kr, sl - 1, 0.3, causal=True)
    o1, l1 = A.latent_decode(q[:, 1:], c, kr, sl, 0.3, causal=True)
    np.testing.assert_allclose(o[:, 0], o0[:, 0], atol=1e-14)
    np.testing.assert_allclose(o[:, 1], o1[:, 0], atol=1e-14)
    np.testing.assert_allclose(lse[:, 0], l0[:, 0], atol=1e-14)


@pytest.mark.parametrize("n_splits", [1, 2, 3, 7])
def test_split_merge_equals_unsplit(n_splits):
    L, d_c, d_R = 29, 8, 4
    rng = np.random.default_rng(n_splits)
    q = rng.standard_normal((3, d_c + d_R))
    c = rng.standard_normal((L, d_c))
    kr = rng.standard_normal((L, d_R))
    full, lse = A.latent_decode_unit(q, c, kr, [L] * 3, 0.4)
    parts_o, parts_l = [], []
    for (a, b) in A.split_ranges(L, n_splits):
        o_s, l_s = A.latent_decode_unit(q, c[a:b], kr[a:b], [b - a] * 3, 0.4)
        parts_o.append(o_s)
        parts_l.append(l_s)
    o, l = A.merge_partials(np.stack(parts_o), np.stack(parts_l))
    np.testing.assert_allclose(o, full, atol=1e-13)
    np.testing.assert_allclose(l, lse, atol=1e-13)
    # an empty split (lse = -inf, o = 0) is neutral
    o2, l2 = A.merge_partials(np.stack(parts_o + [np.zeros_like(full)]),
                              np.stack(parts_l + [np.full(3, -np.inf)]))
    np.testing.assert_allclose(o2, full, atol=1e-13)


# ---------------------------------------------------------------- paging ---
@pytest.mark.parametrize("page_size", [1, 2, 8, 16, 64])
def test_paging_round_trip_and_invariance(page_size):
    rows = np.arange(3 * 70 * 5, dtype=np.float64).reshape(3, 70, 5)
    sl = synth.seqlens(3, 70, "uniform", seed=page_size)
    bt, npg = synth.block_table(sl, page_size, seed=page_size)
    pool = PG.build_pool(rows, sl, bt, page_size, npg, row_stride=8, fill=-1)
    dense = PG.gather_naive(pool, bt, sl, page_size, 70, 5)
    for b in range(3):
        np.testing.assert_array_equal(dense[b, : sl[b]], rows[b, : sl[b]])
        assert np.all(dense[b, sl[b]:] == 0)


def test_physical_row_hand_values():
    """token j of sequence b lives in page block_table[b][j // page] at
    offset j % page.  Hand-computed values (not a round trip): pool rows of
    a 4-token-page table [[3, 0, 2], [1, 4, 5]]."""
    bt = [[3, 0, 2], [1, 4, 5]]
    want = {(0, 0): 12, (0, 3): 15, (0, 4): 0, (0, 5): 1, (0, 9): 9, (0, 11): 11,
            (1, 0): 4, (1, 6): 18, (1, 8): 20, (1, 10): 22}
    for (b, j), r in want.items():
        assert PG.physical_row(bt, 4, b, j) == r, (b, j)
    # page size 1: the block table is the row map itself
    assert [PG.physical_row([[7, 2, 9]], 1, 0, j) for j in range(3)] == [7, 2, 9]


def test_cooperative_offsets_match_naive():
    rng = np.random.default_rng(0)
    for trial in range(200):
        page_size = int(rng.choice([1, 2, 8, 64]))
        n_tok = 128 * 3
        bt_row = rng.permutation(4096)[: -(-n_tok // page_size)]
        start = 128 * int(rng.integers(0, 3))
        addr, trace = PG.cooperative_offsets(bt_row, page_size, start)
        naive = [PG.physical_row([bt_row], page_size, 0, start + r) for r in range(128)]
        np.testing.assert_array_equal(addr, naive)
        assert sorted(r for r, _, _ in trace) == list(range(128))
    # P:311-312 spot case: lane 17 computes row 9; row 9 is read from lane 17
    _, trace = PG.cooperative_offsets(np.arange(10), 64, 0)
    src_of_row = {r: s for r, s, _ in trace}
    assert src_of_row[9] == 17
    assert 1 + (17 % 16) * 8 == 9


# -------------------------------------------------------------- sharding ---
@pytest.mark.parametrize("h_c,N", [(2, 2), (4, 4), (8, 8), (4, 2), (2, 4), (1, 1)])
def test_shard_sum_equals_unsharded(h_c, N):
    T, H, d_c, D = 3, 16, 8, 12
    rng = np.random.default_rng(h_c * 10 + N)
    o = rng.standard_normal((T, H, d_c))
    W = rng.standard_normal((H, d_c, D))
    full = o.reshape(T, -1) @ W.reshape(-1, D)
    np.testing.assert_allclose(SH.tp_oproj_allreduce(o, W, N, h_c), full, atol=1e-12)
    # each rank's query heads belong to its own latent heads
    for r in range(N):
        k0, k1, q0, q1 = SH.tp_shard(H, h_c, N, r)
        g_q = H // h_c
        assert q0 // g_q >= k0 and (q1 - 1) // g_q < k1


def test_absorb_query_identity_with_unabsorbed_definition():
    """Pin of oracle.attention.absorb_query / rope_cache_rows (the upstream
    step): decoding the absorbed query against the rotated
    cache rows equals the unabsorbed definition (per-head K/V up-projection,
    RoPE, softmax) in fp64."""
    import synth
    from oracle import attention as OA
    B, Lq, H, h_c, d_c, d_R, d_h = 2, 3, 8, 2, 32, 16, 24
    sl = np.array([40, 17])
    x = synth.gla_method_inputs(B, Lq, H, h_c, d_c, d_R, d_h, 40, seed=5)
    q = OA.absorb_query(x["q_nope"], x["q_pe"], x["W_UK"], sl, Lq)
    rows = OA.rope_cache_rows(x["c"], x["k_pe"], np.zeros(B))
    c = rows[..., :h_c * d_c].reshape(B, 40, h_c, d_c)
    kr = rows[..., h_c * d_c:]
    o, lse = OA.latent_decode(q, c, kr, sl, 0.3)
    _, o_lat, lse_u = OA.gla_unabsorbed(x["q_nope"], x["q_pe"], x["c"], x["k_pe"], x["W_UK"], x["W_UV"], sl, 0.3)
    np.testing.assert_allclose(o, o_lat, atol=1e-12)
    np.testing.assert_allclose(lse, lse_u, atol=1e-12)


def test_rope_cache_rows_start_offset():
    """oracle.attention.rope_cache_rows at start > 0 (the append position of
    a decode step): (a) appending in chunks at their start offsets equals one
    bulk append from 0; (b) one row at start s equals the rotation of each
    pair (x0, x1) as the complex number x0 + i x1 times e^{i s theta_k}
    (independent complex arithmetic, R5: theta_k = 10000^(-2k/d)); (c) the
    latent part is copied unchanged."""
    from oracle import attention as OA
    rng = np.random.default_rng(11)
    B, n, h_c, d_c, d_R = 2, 9, 2, 4, 6
    c = rng.standard_normal((B, n, h_c, d_c))
    kp = rng.standard_normal((B, n, d_R))
    bulk = OA.rope_cache_rows(c, kp, np.zeros(B))
    parts = [OA.rope_cache_rows(c[:, a:e], kp[:, a:e], np.full(B, a)) for a, e in ((0, 2), (2, 3), (3, 9))]
    np.testing.assert_allclose(np.concatenate(parts, axis=1), bulk, atol=1e-12)
    start = np.array([5, 1234])
    rows = OA.rope_cache_rows(c[:, :1], kp[:, :1], start)
    for b in range(B):
        z = kp[b, 0, 0::2] + 1j * kp[b, 0, 1::2]
        th = 10000.0 ** (-2.0 * np.arange(d_R // 2) / d_R)
        w = z * np.exp(1j * start[b] * th)
        np.testing.assert_allclose(rows[b, 0, h_c * d_c::2], w.real, atol=1e-12)
        np.testing.assert_allclose(rows[b, 0, h_c * d_c + 1::2], w.imag, atol=1e-12)
        np.testing.assert_array_equal(rows[b, 0, :h_c * d_c], c[b, 0].reshape(-1))
