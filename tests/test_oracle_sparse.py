"""Pins for O-17, the l1 Pair-(2:4) pruning of SURVEY 8(f) NEXT-4:
hand-evaluated groups (ties, zeros, signs), brute force over every ordering of four distinct
magnitudes, and the structural invariants (two zeros per group of four, kept values untouched,
the kept pair maximises the retained l1 mass).  The sparse linear itself is O-4 / O-5 on the
pruned weights, pinned in test_oracle_gemm.py."""
import itertools

import numpy as np

from paper_2301_12017_b200 import synth

GOLD = [  # (group of four, pruned) by hand: keep the two largest |w|, ties -> lower index
    ([1.0, -3.0, 2.0, 0.5], [0.0, -3.0, 2.0, 0.0]),
    ([1.0, 1.0, 1.0, 1.0], [1.0, 1.0, 0.0, 0.0]),
    ([0.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0]),
    ([0.0, 0.0, -2.0, 0.0], [0.0, 0.0, -2.0, 0.0]),     # fewer than two nonzeros: stays as is
    ([-0.25, 0.25, 0.125, -0.5], [-0.25, 0.0, 0.0, -0.5]),  # |.| tie between 0 and 1 -> index 0
]


def test_prune24_golden(orc):
    w = np.array([np.concatenate([g for g, _ in GOLD])], np.float16)
    got = orc.prune_24(w)[0].reshape(-1, 4)
    for (g, want), row in zip(GOLD, got):
        assert row.tolist() == want, g


def test_prune24_brute_force_orderings(orc):
    """Every arrangement of four distinct magnitudes with random signs: the two largest |w| survive."""
    rng = np.random.default_rng(31)
    rows = []
    for perm in itertools.permutations([0.5, 1.0, 2.0, 4.0]):
        rows.append(np.array(perm) * rng.choice([-1.0, 1.0], 4))
    w = np.array([np.concatenate(rows)], np.float16)
    got = orc.prune_24(w)[0].reshape(-1, 4)
    for g, row in zip(np.array(rows), got):
        keep = np.argsort(-np.abs(g), kind="stable")[:2]
        want = np.where(np.isin(np.arange(4), keep), g, 0.0)
        assert np.array_equal(row, want.astype(np.float16))


def test_prune24_invariants(orc):
    w = synth.weight(96, 256, "p24")
    p = orc.prune_24(w)
    g, pg = w.reshape(96, -1, 4).astype(np.float64), p.reshape(96, -1, 4).astype(np.float64)
    assert ((pg == 0).sum(-1) >= 2).all()                   # at least two zeros per group
    assert np.array_equal(pg[pg != 0], g[pg != 0])          # kept values untouched
    # the kept pair has the largest l1 mass of all six pairs
    best = np.max([np.abs(g[..., i]) + np.abs(g[..., j]) for i, j in itertools.combinations(range(4), 2)], 0)
    assert np.allclose(np.abs(pg).sum(-1), best)
