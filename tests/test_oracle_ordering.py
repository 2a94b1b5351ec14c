"""Pins for the parallel ordering (reading R1).

b = 1 must reproduce the merry-go-round prefix the paper prints:
"(1,2),(3,4),...,(n-1,n),(1,4),...,(n-3,n-1),(1,6),...,(n,n-2)".
Every b must give n_p - 1 perfect matchings covering each pair exactly once."""
import itertools

import pytest


@pytest.mark.parametrize("n", [8, 10, 16, 64])
def test_b1_is_papers_merry_go_round(orc, n):
    P, Q = orc.schedule(n, 1)
    one = lambda r: [(int(p) + 1, int(q) + 1) for p, q in zip(P[r], Q[r])]  # 1-based
    # round 1: (1,2),(3,4),...,(n-1,n)
    assert one(0) == [(2 * k + 1, 2 * k + 2) for k in range(n // 2)]
    # round 2 starts (1,4) and ends (n-3,n-1)
    assert one(1)[0] == (1, 4) and one(1)[-1] == (n - 3, n - 1)
    # round 3 starts (1,6)
    assert one(2)[0] == (1, 6)
    # the sweep ends with the pair printed as (n, n-2)
    assert one(n - 2)[-1] == (n - 2, n)


@pytest.mark.parametrize("n,b", [(8, 1), (9, 1), (2, 1), (3, 1), (32, 2), (64, 8), (64, 32),
                                 (100, 8), (130, 16), (33, 4), (256, 32)])
def test_perfect_matchings_cover_all_pairs(orc, n, b):
    P, Q = orc.schedule(n, b)
    np_ = orc.padded_n(n, b)
    assert np_ % (2 * b) == 0 and np_ >= n and np_ - n < 2 * b
    assert P.shape == (np_ - 1, np_ // 2)
    seen = set()
    for r in range(P.shape[0]):
        idx = list(P[r]) + list(Q[r])
        assert sorted(idx) == list(range(np_))          # perfect matching
        for p, q in zip(P[r], Q[r]):
            assert p < q                                 # p = min (R1, Lemma 3.1 i<j)
            assert (p, q) not in seen
            seen.add((int(p), int(q)))
    assert seen == set(itertools.combinations(range(np_), 2))


def test_block_structure(orc):
    """Reading R1: with b > 1 the rounds group into block rounds; during a
    cross round of block pair (I,J), I*b+i meets J*b+((i+s) mod b)."""
    n, b = 64, 8
    P, Q = orc.schedule(n, b)
    # the first b-1 rounds are intra-block
    for r in range(b - 1):
        for p, q in zip(P[r], Q[r]):
            assert p // b == q // b
    # every later round pairs whole blocks, as a cyclic shift inside the pair
    for r in range(b - 1, n - 1):
        blocks = {}
        for p, q in zip(P[r], Q[r]):
            assert p // b != q // b
            blocks.setdefault((p // b, q // b), []).append((p % b, q % b))
        for (I, J), prs in blocks.items():
            assert len(prs) == b
            shifts = {(qq - pp) % b for pp, qq in prs}
            assert len(shifts) == 1
