"""Pins of the oracle priority select (Alg.1 l.12-14, A-1/A-2)."""
import itertools
import math
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


# ------------------------------------------------ NEXT-1 priority maintenance

def test_column_delta_worked_example():
    """S:87 / Alg.1 l.4: paper-view weights [R, L]; our Wt is the transpose."""
    g = golden("column_delta.json")
    Wo = np.array(g["w_old"], dtype=np.float64).T
    Wn = np.array(g["w_new"], dtype=np.float64).T
    assert O.column_delta(Wn, Wo).tolist() == g["delta"]


def test_column_delta_constant_shift_closed_form():
    rng = np.random.default_rng(3)
    W = rng.standard_normal((37, 19))
    for c in (0.25, -3.0, 0.0):
        d = O.column_delta(W + c, W)
        assert np.allclose(d, abs(c), rtol=0, atol=1e-15)
    # rows changed in a single element j: delta = |dw| / R exactly
    W2 = W.copy()
    W2[5, 7] += 0.5
    d = O.column_delta(W2, W)
    assert d[5] == pytest.approx(0.5 / 19, abs=1e-15) and np.count_nonzero(d) == 1


def test_priority_update_carries_pruned_columns():
    """pruned columns keep their old variation (no endless loop);
    every other column is recomputed."""
    rng = np.random.default_rng(4)
    K, n = 50, 23
    W0 = rng.standard_normal((K, n))
    d0 = rng.random(K)
    S, P = O.select(d0.astype(np.float32), 20)
    W1 = W0 + 0.01 * rng.standard_normal((K, n))
    W1[P] = W0[P]                       # pruned rows: zero-imputed grads -> unchanged
    d1 = O.priority_update(d0, W1, W0, P)
    assert np.array_equal(d1[P], d0[P])                           # carried over, bit-exact
    assert np.allclose(d1[S], O.column_delta(W1, W0)[S], rtol=0, atol=0)
    # without carry-over the pruned columns would collapse to 0 (the loop)
    assert np.all(O.priority_update(d0, W1, W0, None)[P] == 0.0)
    # first epoch: everything recomputed
    assert np.array_equal(O.priority_update(d0, W1, W0, None), O.column_delta(W1, W0))


def test_pridiff_gamma_rules():
    """Alg.1 l.9-11: gamma_k = 1 - #{delta > theta}/L, floored at alpha*gamma."""
    d = np.array([0.5, 0.001, 0.002, 0.3, 0.0, 0.001])
    theta = 0.001                        # strict '>' : 0.001 is not above
    assert O.pridiff_gamma(d, theta, 0.0) == pytest.approx(1 - 3 / 6)
    assert O.pridiff_gamma(d, theta, 0.9) == pytest.approx(0.8 * 0.9)   # alpha floor wins
    assert O.pridiff_gamma(np.full(8, 1.0), theta, 0.5) == pytest.approx(0.4)
    assert O.pridiff_gamma(np.zeros(8), theta, 0.5) == 1.0
    with pytest.raises(O.OracleError):
        O.pridiff_gamma(np.zeros(0), theta, 0.5)


def anti_endless_loop_run(incremental: bool, epochs: int = 10, K: int = 64, n: int = 32, gamma: float = 0.25,
                          seed: int = 410):
    """Seeded scenario of S:410 / P:190: each epoch "trains" the weight W^T
    [K, n] by an update of per-row scale drawn fresh every epoch (the rows'
    real variation), except that rows pruned this epoch receive none (their
    Zero-imputed gradient rows, leave them unchanged under SGD).  At
    the epoch end delta is updated (incrementally, or naively: every
    row recomputed) and the next pruned set is selected (Alg.1 l.12-14).
    Returns the pruned sets of every epoch."""
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((K, n))
    npr = int(math.floor(K * gamma + 0.5))
    delta = rng.random(K).astype(np.float32)          # epoch-0 scores
    _, P = O.select(delta, npr)
    sets = [tuple(P)]
    for _ in range(epochs - 1):
        W_old = W.copy()
        scale = rng.lognormal(-3.0, 1.0, size=K)
        upd = rng.standard_normal((K, n)) * scale[:, None]
        upd[np.asarray(P)] = 0.0
        W = W + upd
        delta = O.priority_update(delta, W, W_old, P if incremental else None).astype(np.float32)
        _, P = O.select(delta, npr)
        sets.append(tuple(P))
    return sets


def test_anti_endless_loop_S410():
    """S:410 invariant: with the incremental rule the pruned set rotates (>= 3
    distinct sets in 10 epochs); the naive full update freezes on a fixed set
    by epoch 3 (pruned rows show zero variation and are pruned again)."""
    inc = anti_endless_loop_run(True)
    naive = anti_endless_loop_run(False)
    assert len(set(inc)) >= 3
    assert all(sset == naive[2] for sset in naive[2:])
    assert naive[1] == naive[2]
