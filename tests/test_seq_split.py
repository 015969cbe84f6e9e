"""Sequence split (context-parallel decode): the token ranges
(oracle pinned by properties; C ABI == oracle) and the merge identity that
makes the split exact (oracle only, fp64).  CPU tests."""

import numpy as np
import pytest

import synth
from oracle import attention as OA
from oracle import sharding as SH
from paper_2505_21487_b200 import glad

CASES = [(L, page, Lq, P) for L in [0, 1, 2, 3, 63, 64, 65, 127, 129, 300, 1000, 8191]
         for page in [1, 16, 64] for Lq in [1, 2, 4, 8] for P in [1, 2, 3, 4, 8]]


@pytest.mark.parametrize("L,page,Lq,P", CASES[::7] + [(65, 64, 4, 8), (2, 64, 8, 4), (8191, 64, 2, 8)])
def test_oracle_ranges_properties(L, page, Lq, P):
    """Pins of oracle.sharding.seq_split_ranges: the ranges partition [0, L)
    in rank order, interior boundaries are page-aligned, the last rank holds
    every key >= L - (Lq - 1), and ranks differ by at most one page unless
    pages moved to the last rank for the causal rule."""
    r = SH.seq_split_ranges(L, page, Lq, P)
    assert len(r) == P
    covered = []
    for b, e in r:
        assert 0 <= b <= e <= L
        covered += list(range(b, e))
    assert covered == list(range(L))
    for b, e in r[:-1]:
        if e > b:
            assert b % page == 0 and e % page == 0
    assert r[-1][1] == L or L == 0
    assert r[-1][0] <= max(0, L - (Lq - 1))
    pages = [-(-(e - b) // page) if e > b else 0 for b, e in r]
    if r[-1][0] == (-(-L // page) - pages[-1]) * page and max(0, L - (Lq - 1)) >= r[-1][0]:
        assert max(pages[:-1] or [0]) - min(pages[:-1] or [0]) <= 1


def test_c_abi_ranges_match_oracle():
    """glad_seq_split_range == oracle on every case (non-empty ranges exact,
    empty ranges begin == end)."""
    for L, page, Lq, P in CASES:
        o = SH.seq_split_ranges(L, page, Lq, P)
        c = [glad.seq_split_range(L, page, Lq, P, r) for r in range(P)]
        assert [x for x in o if x[1] > x[0]] == [x for x in c if x[1] > x[0]], (L, page, Lq, P, o, c)
        assert all(e >= b for b, e in c)


def test_c_abi_range_errors():
    with pytest.raises(RuntimeError):
        glad.seq_split_range(10, 0, 1, 2, 0)
    with pytest.raises(RuntimeError):
        glad.seq_split_range(10, 16, 1, 2, 2)


@pytest.mark.parametrize("L,Lq,P,page", [(300, 1, 2, 16), (300, 4, 3, 16), (129, 8, 4, 64), (70, 2, 8, 1),
                                         (5, 4, 2, 64)])
def test_split_merge_equals_unsplit(L, Lq, P, page):
    """The identity the sequence split relies on (fp64 oracle): attention of
    rank r over its range (causal only on the last rank, bottom-right aligned
    on its local length, R2), merged by LSE (the all-gather + rescale + sum),
    equals causal attention over the whole sequence."""
    q, c, kr = synth.latent_kernel_inputs(1, Lq, 8, 2, 32, 16, L, seed=L + P)
    q, c, kr = q.double().numpy(), c.double().numpy(), kr.double().numpy()
    scale = 0.2
    o_ref, lse_ref = OA.latent_decode(q, c, kr, np.array([L]), scale, causal=True)
    o_parts, lse_parts = [], []
    for r, (b, e) in enumerate(SH.seq_split_ranges(L, page, Lq, P)):
        o_r, lse_r = OA.latent_decode(q, c[:, b:e], kr[:, b:e], np.array([e - b]), scale, causal=(r == P - 1))
        o_parts.append(o_r)
        lse_parts.append(lse_r)
    o, lse = OA.merge_partials(np.stack(o_parts), np.stack(lse_parts))
    np.testing.assert_allclose(o, o_ref, atol=1e-12)
    np.testing.assert_allclose(lse, lse_ref, atol=1e-12)
