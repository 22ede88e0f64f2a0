"""Pins of the oracle priority select (Alg.1 l.12-14, A-1/A-2)."""
import itertools
import random

import numpy as np
import pytest

from conftest import golden
from oracle import ztp_oracle as O


def test_worked_example_S384():
    g = golden("select_worked.json")
    S, P = O.select(np.array(g["scores"], dtype=np.float32), g["n_prune"])
    assert list(P) == g["pruned"] and list(S) == g["kept"]


@pytest.mark.parametrize("seed", range(60))
def test_bruteforce_unique_threshold_subset(seed):
    """For L <= 10: exactly one of the C(L,k) subsets P satisfies
    min key(S) > max key(P) with key = (score, index); it must be the output."""
    rng = random.Random(seed)
    L = rng.randint(1, 10)
    k = rng.randint(0, L)
    levels = rng.choice([0, 2, 3])                 # tie-stress
    if levels:
        sc = np.array([rng.randrange(levels) * 0.25 for _ in range(L)], dtype=np.float32)
    else:
        sc = np.array([rng.uniform(-1, 1) for _ in range(L)], dtype=np.float32)
    key = [(float(sc[i]), i) for i in range(L)]
    valid = []
    for Pset in itertools.combinations(range(L), k):
        Sset = [i for i in range(L) if i not in Pset]
        if not Pset or not Sset or min(key[i] for i in Sset) > max(key[i] for i in Pset):
            valid.append(Pset)
    assert len(valid) == 1
    S, P = O.select(sc, k)
    assert tuple(P) == valid[0]
    assert list(S) == sorted(set(range(L)) - set(valid[0]))


def test_all_equal_prunes_lowest_indices():
    S, P = O.select(np.full(9, 0.5, dtype=np.float32), 4)
    assert list(P) == [0, 1, 2, 3] and list(S) == [4, 5, 6, 7, 8]


def test_zero_prune_keeps_all_and_signed_zero():
    S, P = O.select(np.array([3.0, 1.0, 2.0], dtype=np.float32), 0)
    assert list(S) == [0, 1, 2] and len(P) == 0
    # -0 == +0: ties broken by index
    S, P = O.select(np.array([0.0, -0.0, 1.0, -0.0], dtype=np.float32), 2)
    assert list(P) == [0, 1]


def test_nan_rejected():
    with pytest.raises(O.OracleError) as ei:
        O.select(np.array([1.0, np.nan], dtype=np.float32), 1)
    assert ei.value.code == "ZTP_EINVAL"
