"""Decode attention for GLA / MLA / GTA, fp64, unabsorbed and latent forms
(oracle; test infrastructure only — never imported by the product path).

Every function evaluates the *plain definition*: scores, a max-subtracted
softmax over the visible keys, a weighted sum.  No tiling, no online softmax,
no split-KV: the kernel's rearrangements (online softmax, split + LSE merge,
weight absorption) are exact up to rounding, so the oracle is the definition
they must reproduce.

Conventions:
  R1 softmax_scale is an explicit argument (the paper never writes a scale).
  R2 causal (bottom-right aligned): query t of a step with Lq queries sits at
     absolute position p_t = L_b - Lq + t and sees keys j <= p_t; non-causal
     sees all j < L_b.  ``seqlens`` count the Lq new tokens (already appended).
  R3 lse is the natural log of sum_j exp(s_j), fp64 here; a query with no
     visible key gets o = 0 and lse = -inf.
  R4 GTA rotates the query's second half (the half matching K_RoPE) at p_t.
  Head grouping is contiguous: head h belongs to latent/KV group h // g_q
  ("partitions the query heads into two groups").
"""

import numpy as np

from .rope import rope_rotate


def _f64(x):
    """Upcast (exactly) anything array-like, incl. torch bf16, to numpy fp64."""
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


def visible_count(L_b, Lq, t, causal):
    """Number of keys query t (0-based within the step) may attend to (R2)."""
    if causal:
        return max(0, min(L_b, L_b - Lq + t + 1))
    return L_b


def softmax_row(s):
    """Max-subtracted softmax of a 1-D score vector; returns (p, lse).

    Empty input -> (empty, -inf).  (stable under large scores.)
    """
    s = np.asarray(s, dtype=np.float64)
    if s.size == 0:
        return s.copy(), -np.inf
    m = s.max()
    e = np.exp(s - m)
    z = e.sum()
    return e / z, m + np.log(z)


def attend(q, K, V, scale):
    """One query row against keys K [n, dk] and values V [n, dv].

    Returns (o [dv], lse).  The textbook definition softmax(scale*K q) V.
    """
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    if K.shape[0] == 0:
        return np.zeros(V.shape[1], dtype=np.float64), -np.inf
    s = scale * (K @ np.asarray(q, dtype=np.float64))
    p, lse = softmax_row(s)
    return p @ V, lse


# --------------------------------------------------------------------------
# GLA / MLA, latent ("absorbed") form on the kernel's own inputs.
# P:246-252:  O_i = softmax(Q_i (c_i^KV)^T) c_i^KV ; with the decoupled RoPE
# score term added as in P:48 (sigma(QK^T + Q_rope K_rope^T) V).
# --------------------------------------------------------------------------
def latent_decode(q, c, k_rope, seqlens, scale, causal=True):
    """GLA (h_c latent heads) / MLA (h_c = 1) decode on absorbed inputs.

    q       [B, Lq, H, d_c + d_R]  absorbed q_nope (d_c) || rotated q_rope (d_R)
    c       [B, Lmax, h_c, d_c]    latent cache (logical, unpaged)
    k_rope  [B, Lmax, d_R]         rotated decoupled RoPE key, ONE per token
    Returns o [B, Lq, H, d_c], lse [B, Lq, H]  (fp64).
    """
    q, c, kr = _f64(q), _f64(c), _f64(k_rope)
    B, Lq, H, dqk = q.shape
    h_c, d_c = c.shape[2], c.shape[3]
    d_R = kr.shape[2]
    assert dqk == d_c + d_R and H % h_c == 0
    g_q = H // h_c
    o = np.zeros((B, Lq, H, d_c))
    lse = np.full((B, Lq, H), -np.inf)
    for b in range(B):
        L_b = int(seqlens[b])
        for t in range(Lq):
            n = visible_count(L_b, Lq, t, causal)
            for h in range(H):
                i = h // g_q
                K = np.concatenate([c[b, :n, i, :], kr[b, :n, :]], axis=1)
                V = c[b, :n, i, :]
                o[b, t, h], lse[b, t, h] = attend(q[b, t, h], K, V, scale)
    return o, lse


def latent_decode_unit(q_rows, c_i, k_rope, n_visible, scale):
    """One (b, latent head) unit: q_rows [n_q, d_c+d_R] against c_i [L, d_c],
    k_rope [L, d_R] with per-row visible counts.  Used for sampled parity at
    full benchmark sizes.  Returns (o [n_q, d_c], lse [n_q])."""
    q_rows, c_i, kr = _f64(q_rows), _f64(c_i), _f64(k_rope)
    o = np.zeros((q_rows.shape[0], c_i.shape[1]))
    lse = np.full(q_rows.shape[0], -np.inf)
    for r in range(q_rows.shape[0]):
        n = int(n_visible[r])
        K = np.concatenate([c_i[:n], kr[:n]], axis=1)
        o[r], lse[r] = attend(q_rows[r], K, c_i[:n], scale)
    return o, lse


# --------------------------------------------------------------------------
# GLA / MLA, UNabsorbed definition (what the method computes before the
# absorption trick).  K_h = c_i W_UK[h], V_h = c_i W_UV[h].
# --------------------------------------------------------------------------
def gla_unabsorbed(q_nope, q_pe, c, k_pe, W_UK, W_UV, seqlens, scale,
                   causal=True, rope_base=10000.0):
    """Materialise per-head keys/values from the latent, rotate the decoupled
    RoPE parts, run standard softmax attention.

    q_nope [B, Lq, H, d_h], q_pe [B, Lq, H, d_R] (unrotated)
    c      [B, Lmax, h_c, d_c], k_pe [B, Lmax, d_R] (unrotated, one per token)
    W_UK, W_UV [H, d_c, d_h]  (latent -> per-head key / value up-projection)
    Returns o_head [B,Lq,H,d_h], o_lat [B,Lq,H,d_c], lse [B,Lq,H].
    o_lat = sum_j P_j c_j (the latent-space output the kernel writes; the
    head-space output equals o_lat @ W_UV[h] by linearity).
    """
    q_nope, q_pe, c, k_pe = _f64(q_nope), _f64(q_pe), _f64(c), _f64(k_pe)
    W_UK, W_UV = _f64(W_UK), _f64(W_UV)
    B, Lq, H, d_h = q_nope.shape
    h_c, d_c = c.shape[2], c.shape[3]
    g_q = H // h_c
    o_head = np.zeros((B, Lq, H, d_h))
    o_lat = np.zeros((B, Lq, H, d_c))
    lse = np.full((B, Lq, H), -np.inf)
    for b in range(B):
        L_b = int(seqlens[b])
        kR = rope_rotate(k_pe[b, :L_b], np.arange(L_b), rope_base)      # [L, d_R]
        for h in range(H):
            i = h // g_q
            K_h = c[b, :L_b, i, :] @ W_UK[h]                              # [L, d_h]
            V_h = c[b, :L_b, i, :] @ W_UV[h]
            for t in range(Lq):
                n = visible_count(L_b, Lq, t, causal)
                p_t = L_b - Lq + t
                qR = rope_rotate(q_pe[b, t, h], p_t, rope_base)
                if n == 0:
                    continue
                s = scale * (K_h[:n] @ q_nope[b, t, h] + kR[:n] @ qR)
                p, lse[b, t, h] = softmax_row(s)
                o_head[b, t, h] = p @ V_h[:n]
                o_lat[b, t, h] = p @ c[b, :n, i, :]
    return o_head, o_lat, lse


# --------------------------------------------------------------------------
# GTA:  K_NoPE = KV[..., :d_h/2], V = KV,
#   K = concat(K_NoPE, broadcast(K_RoPE, h_kv))  -- tied half never rotated.
# --------------------------------------------------------------------------
def gta_keys_values(kv, k_rope_rot):
    """Build per-group K and V from the tied state.

    kv [L, h_kv, d_h], k_rope_rot [L, d_h/2] (already rotated).
    Returns K, V each [L, h_kv, d_h]."""
    kv, kr = _f64(kv), _f64(k_rope_rot)
    L, h_kv, d_h = kv.shape
    V = kv.copy()
    K = np.concatenate([kv[:, :, : d_h // 2],
                        np.broadcast_to(kr[:, None, :], (L, h_kv, d_h // 2))], axis=2)
    return K, V


def gta_decode(q, kv, k_rope, seqlens, scale, causal=True, rope_base=10000.0):
    """GTA decode from *unrotated* inputs.

    q      [B, Lq, H, d_h]    = [q_nope (d_h/2) || q_rope (d_h/2, unrotated)]
    kv     [B, Lmax, h_kv, d_h] tied KV state
    k_rope [B, Lmax, d_h/2]   single-head RoPE key, unrotated
    Returns o [B,Lq,H,d_h], lse [B,Lq,H].
    """
    q, kv, k_rope = _f64(q), _f64(kv), _f64(k_rope)
    B, Lq, H, d_h = q.shape
    h_kv = kv.shape[2]
    g_q = H // h_kv
    half = d_h // 2
    o = np.zeros((B, Lq, H, d_h))
    lse = np.full((B, Lq, H), -np.inf)
    for b in range(B):
        L_b = int(seqlens[b])
        kR = rope_rotate(k_rope[b, :L_b], np.arange(L_b), rope_base)
        K, V = gta_keys_values(kv[b, :L_b], kR)
        for t in range(Lq):
            n = visible_count(L_b, Lq, t, causal)
            p_t = L_b - Lq + t
            for h in range(H):
                g = h // g_q
                q_eff = np.concatenate([q[b, t, h, :half],
                                        rope_rotate(q[b, t, h, half:], p_t, rope_base)])
                o[b, t, h], lse[b, t, h] = attend(q_eff, K[:n, g], V[:n, g], scale)
    return o, lse


def tied_decode(q, kv, k_rope_rot, seqlens, scale, causal=True):
    """GTA on the kernel's own (pre-rotated) inputs.

    q [B,Lq,H,d_h] = [q_nope || rotated q_rope]; kv [B,Lmax,h_kv,d_h];
    k_rope_rot [B,Lmax,d_h/2].  Score s = scale*(q_nope.KV[:d_h/2] + q_rope.k_rope),
    value = full tied state.  Returns o [B,Lq,H,d_h], lse.
    """
    q, kv, kr = _f64(q), _f64(kv), _f64(k_rope_rot)
    B, Lq, H, d_h = q.shape
    h_kv = kv.shape[2]
    g_q = H // h_kv
    o = np.zeros((B, Lq, H, d_h))
    lse = np.full((B, Lq, H), -np.inf)
    for b in range(B):
        L_b = int(seqlens[b])
        K, V = gta_keys_values(kv[b, :L_b], kr[b, :L_b])
        for t in range(Lq):
            n = visible_count(L_b, Lq, t, causal)
            for h in range(H):
                g = h // g_q
                o[b, t, h], lse[b, t, h] = attend(q[b, t, h], K[:n, g], V[:n, g], scale)
    return o, lse


# --------------------------------------------------------------------------
# Textbook GQA (separate K and V heads) — degeneracy target for GTA.
# --------------------------------------------------------------------------
def gqa_decode(q, k, v, seqlens, scale, causal=True):
    """q [B,Lq,H,d], k/v [B,Lmax,h_kv,d]; head h uses KV head h // (H/h_kv)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, Lq, H, _ = q.shape
    h_kv = k.shape[2]
    g_q = H // h_kv
    o = np.zeros((B, Lq, H, v.shape[3]))
    lse = np.full((B, Lq, H), -np.inf)
    for b in range(B):
        L_b = int(seqlens[b])
        for t in range(Lq):
            n = visible_count(L_b, Lq, t, causal)
            for h in range(H):
                g = h // g_q
                o[b, t, h], lse[b, t, h] = attend(q[b, t, h], k[b, :n, g], v[b, :n, g], scale)
    return o, lse


# --------------------------------------------------------------------------
# Split-KV merge.  Not in the paper (BASELINE.json north_star: "a split-KV
# softmax and a log-sum-exp merge").  Definition:
#   lse = ln sum_s exp(lse_s),  O = sum_s exp(lse_s - lse) O_s
# where O_s is the *normalised* partial output over split s.
# --------------------------------------------------------------------------
def absorb_query(q_nope, q_pe, W_UK, seqlens, Lq, rope_base=10000.0):
    """Kernel query from raw tensors (P:48 weight absorption, R2 positions,
    R5 RoPE): q[b,t,h] = [ W_UK[h] q_nope[b,t,h] || RoPE(q_pe[b,t,h], L_b - Lq + t) ].

    q_nope [B,Lq,H,d_h], q_pe [B,Lq,H,d_R], W_UK [H,d_c,d_h] -> [B,Lq,H,d_c+d_R] fp64.
    """
    q_nope, q_pe, W_UK = _f64(q_nope), _f64(q_pe), _f64(W_UK)
    B, _, H, _ = q_nope.shape
    q_abs = np.einsum("hcd,bthd->bthc", W_UK, q_nope)
    pos = np.array([[int(seqlens[b]) - Lq + t for t in range(Lq)] for b in range(B)], dtype=np.float64)
    q_r = rope_rotate(q_pe, pos[:, :, None], rope_base)
    return np.concatenate([q_abs, q_r], axis=-1)


def rope_cache_rows(c, k_pe, start, rope_base=10000.0):
    """Cache rows [c || RoPE(k_pe, start_b + i)] (P:304 append with the RoPE
    key rotated at its position).  c [B,n,h_c,d_c], k_pe [B,n,d_R] -> [B,n,W]."""
    c, k_pe = _f64(c), _f64(k_pe)
    B, n = c.shape[:2]
    pos = np.asarray(start, dtype=np.float64)[:, None] + np.arange(n)[None, :]
    return np.concatenate([c.reshape(B, n, -1), rope_rotate(k_pe, pos, rope_base)], axis=-1)


def merge_partials(o_parts, lse_parts):
    """o_parts [S, ..., d], lse_parts [S, ...] -> (o [..., d], lse [...])."""
    o_parts, lse_parts = _f64(o_parts), _f64(lse_parts)
    m = np.max(lse_parts, axis=0)
    m_safe = np.where(np.isfinite(m), m, 0.0)
    w = np.exp(lse_parts - m_safe)                          # exp(-inf) = 0
    z = w.sum(axis=0)
    with np.errstate(divide="ignore", invalid="ignore"):
        lse = np.where(z > 0, m_safe + np.log(z), -np.inf)
        wn = np.where(z > 0, w / np.where(z > 0, z, 1.0), 0.0)
    o = (wn[..., None] * o_parts).sum(axis=0)
    return o, lse


def split_ranges(L, n_splits):
    """Contiguous token ranges covering [0, L) (helper for split tests)."""
    edges = np.linspace(0, L, n_splits + 1).round().astype(int)
    return [(int(edges[s]), int(edges[s + 1])) for s in range(n_splits)]
