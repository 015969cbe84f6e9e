"""Tensor-parallel sharding arithmetic (oracle; test infrastructure only).

P:147-162: duplication factor D = ceil(N g_q / h_q), 1 <= D <= N; zero
redundancy D = 1 <=> g_q <= floor(h_q / N).  P:123-131: KV_Bytes =
m_kv * B * L * (h_q / g_q) * d_h * sizeof(dtype).  The decoupled / GTA RoPE
head is single and replicated on every rank ("broadcast across all
groups"; pinned by the byte tables P:624-628, P:1000-1004, P:1299-1305,
P:1381-1386).
"""

import math

import numpy as np

# Variant -> (m_kv, has_rope)
VARIANTS = {
    "MHA": (2, False), "MQA": (2, False), "GQA": (2, False),
    "GTA": (1, True), "GLA": (1, True), "MLA": (1, True),
}


def duplication_factor(N, g_q, h_q):
    """D = ceil(N * g_q / h_q)."""
    return math.ceil(N * g_q / h_q)


def zero_redundancy(N, g_q, h_q):
    """D == 1 iff g_q <= floor(h_q / N)."""
    return g_q <= h_q // N


def kv_elems_per_token_per_device(variant, n_kv_heads, d_head, d_rope, N):
    """Cached elements per token on one of N ranks.

    n_kv_heads: distinct cached heads (h_q for MHA, 1 for MQA/MLA, h_kv for
    GQA/GTA, h_c for GLA); d_head: d_h (MHA/MQA/GQA/GTA) or d_c (GLA/MLA);
    d_rope: d_h/2 (GTA) or d_R (GLA/MLA), ignored otherwise.
    A rank holds ceil(n_kv_heads / N) heads (at least one: duplication
    when n_kv_heads < N), plus the replicated single RoPE head.
    """
    m_kv, has_rope = VARIANTS[variant]
    heads = max(1, math.ceil(n_kv_heads / N))
    return m_kv * heads * d_head + (d_rope if has_rope else 0)


def kv_bytes_per_token_per_device(variant, n_kv_heads, d_head, d_rope, N, dtype_bytes=2):
    return kv_elems_per_token_per_device(variant, n_kv_heads, d_head, d_rope, N) * dtype_bytes


def kv_bytes(m_kv, B, L, h_q, g_q, d_h, dtype_bytes=2):
    """P:123-131 verbatim (no RoPE term)."""
    return m_kv * B * L * (h_q // g_q) * d_h * dtype_bytes


def tp_shard(h_q, n_kv_heads, N, rank):
    """Contiguous head ranges for rank r (each rank owns its latent
    head(s) and the query group that attends to them).

    Returns (kv_begin, kv_end, q_begin, q_end).  When n_kv_heads < N each
    KV/latent head is duplicated on D = N / n_kv_heads ranks and its g_q
    query heads are split across those replicas.
    """
    assert h_q % N == 0, "h_q must divide by N"
    if n_kv_heads >= N:
        assert n_kv_heads % N == 0
        per = n_kv_heads // N
        kv = (rank * per, (rank + 1) * per)
    else:
        assert N % n_kv_heads == 0
        D = N // n_kv_heads
        kv = (rank // D, rank // D + 1)
    qp = h_q // N
    return kv[0], kv[1], rank * qp, (rank + 1) * qp


def tp_oproj_allreduce(o_lat, W_vo, N, n_kv_heads):
    """O = AllReduce(sum_r O_r W_r^vo).

    o_lat [T, H, d_c] latent-space attention output, W_vo [H, d_c, D_model].
    Evaluates the per-rank partial products over the rank's query heads and
    sums them (the all-reduce).  Returns [T, D_model].
    """
    o_lat, W_vo = np.asarray(o_lat, np.float64), np.asarray(W_vo, np.float64)
    T, H, d_c = o_lat.shape
    total = np.zeros((T, W_vo.shape[2]))
    for r in range(N):
        _, _, q0, q1 = tp_shard(H, n_kv_heads, N, r)
        part = o_lat[:, q0:q1, :].reshape(T, -1) @ W_vo[q0:q1].reshape(-1, W_vo.shape[2])
        total += part
    return total


def seq_split_ranges(L, page_size, Lq, P):
    """Sequence split of one head group (reading R17 in
    DESIGN.md): the P ranks own contiguous page-aligned token ranges,
    later ranks first in line for the extra pages, and the last rank holds
    the last min(L, Lq - 1) keys so that it alone needs the causal mask.

    Written page by page: pages are dealt out in rank order with counts
    floor(n/P) (+1 for the last n mod P ranks); then whole pages move from
    the earlier ranks to the last one until it holds every key index
    >= L - (Lq - 1).  Returns [(begin, end)] per rank.
    """
    n = -(-L // page_size)
    counts = [n // P + (1 if r >= P - n % P else 0) for r in range(P)]
    owner = []
    for r in range(P):
        owner += [r] * counts[r]
    must = max(0, L - (Lq - 1))          # keys with index >= must belong to the last rank
    for pg in range(n):
        if (pg + 1) * page_size > must:  # page holds a key >= must
            owner[pg] = P - 1
    ranges = []
    for r in range(P):
        toks = [j for j in range(L) if owner[j // page_size] == r]
        ranges.append((toks[0], toks[-1] + 1) if toks else None)
    # empty ranges sit where the rank's pages would have started
    out = []
    for r in range(P):
        if ranges[r] is not None:
            out.append(ranges[r])
        else:
            nxt = [ranges[q][0] for q in range(r + 1, P) if ranges[q] is not None]
            prv = [ranges[q][1] for q in range(r) if ranges[q] is not None]
            pos = prv[-1] if prv else (nxt[0] if nxt else 0)
            out.append((pos, pos))
    return out
