"""Paged KV cache addressing (oracle; test infrastructure only).

Paged KV ("Paged KV ... has become a standard way of storing the KV
cache"): token position j of sequence b lives in physical page
block_table[b][j // page_size] at in-page offset j % page_size.  Page size 1
must work.  Row layout (reading R6): [head_0 | ... | head_{n-1} |
rope], RoPE stored once per token (pinned by P:627, P:1003 byte counts).
"""

import numpy as np


def physical_row(block_table, page_size, b, j):
    """Naive 64-bit address of logical token j of sequence b, in pool rows."""
    return int(block_table[b][j // page_size]) * page_size + (j % page_size)


def build_pool(rows, seqlens, block_table, page_size, num_pages, row_stride=None,
               fill=0.0):
    """Scatter logical rows [B, Lmax, W] into a pool [num_pages, page_size, stride]."""
    rows = np.asarray(rows)
    B, _, W = rows.shape
    stride = W if row_stride is None else row_stride
    pool = np.full((num_pages * page_size, stride), fill, dtype=rows.dtype)
    for b in range(B):
        for j in range(int(seqlens[b])):
            pool[physical_row(block_table, page_size, b, j), :W] = rows[b, j]
    return pool.reshape(num_pages, page_size, stride)


def gather_naive(pool, block_table, seqlens, page_size, max_len, width):
    """Dense [B, max_len, width] view; positions >= L_b are zero."""
    pool2 = np.asarray(pool).reshape(-1, np.asarray(pool).shape[-1])
    B = len(seqlens)
    out = np.zeros((B, max_len, width), dtype=pool2.dtype)
    for b in range(B):
        for j in range(min(int(seqlens[b]), max_len)):
            out[b, j] = pool2[physical_row(block_table, page_size, b, j), :width]
    return out


def cooperative_offsets(block_table_row, page_size, block_start, n_threads=128,
                        group_size=16):
    """Emulate the paper's distributed offset calculation.

    128 threads in 8 groups of 16; group g loads rows g, g+8, ..., g+120.
    Step 2: thread t (group g = t // 16) computes the address of row
            g + (t mod 16) * 8 (one register per thread).
    Step 3: for row r of group g, the address is read (warp shuffle) from
            thread g*16 + (r - g)/8.
    Returns (addr_of_row [128], trace) where trace lists
    (row, computing_thread, reading_group) and each thread stores 1 offset.
    """
    n_groups = n_threads // group_size
    reg = {}
    for t in range(n_threads):
        g = t // group_size
        r = g + (t % group_size) * n_groups
        j = block_start + r
        reg[t] = int(block_table_row[j // page_size]) * page_size + (j % page_size)
    addr = np.zeros(n_threads, dtype=np.int64)
    trace = []
    for g in range(n_groups):
        for r in range(g, n_threads, n_groups):
            src = g * group_size + (r - g) // n_groups
            addr[r] = reg[src]
            trace.append((r, src, g))
    return addr, trace
