"""Pins of the embedding-similarity oracle (NEXT-3): closed forms and a library routine."""
import numpy as np
from sklearn.metrics.pairwise import cosine_similarity

import oracle
from tests.helpers import bf16_bits, grid_values


def test_matches_sklearn_cosine():
    rng = np.random.default_rng(0)
    e = grid_values(rng, (50, 64)); q = grid_values(rng, (3, 64))
    got = oracle.embed_scores(bf16_bits(e), bf16_bits(q))
    ref = cosine_similarity(q.astype(np.float64), e.astype(np.float64))
    assert np.allclose(got, ref, atol=1e-14)


def test_closed_forms():
    q = np.zeros((1, 16), np.float32); q[0, 0] = 1.0
    e = np.zeros((4, 16), np.float32)
    e[0] = q[0] * 2.0          # same direction → 1
    e[1] = -q[0]               # opposite → −1
    e[2, 1] = 1.0              # orthogonal → 0
    # e[3] = 0                 # zero vector → 0 by convention
    got = oracle.embed_scores(bf16_bits(e), bf16_bits(q))[0]
    assert got.tolist() == [1.0, -1.0, 0.0, 0.0]
