"""Pins of the stochastic-acceptance oracle (oracle/sampling.py, SURVEY §8(f) f2,
reading R24) against what the mathematics fixes, independent of the oracle:

* losslessness: for children drawn from the draft q without
  replacement, the committed token's law equals the base distribution p --
  exactly on a uniform grid for one child, within total variation 0.01 over
  60k seeded trials for several children;
* sensitivity: a mutant that forgets the draft update (with-replacement rule on
  distinct children) fails the same test;
* the temperature -> 0 limit (one-hot p) reproduces the greedy walk
  (oracle/tree.py accept_walk) on random trees.
"""
import numpy as np
import pytest

from oracle import sampling as S
from oracle import tree as T


def _law_one_child(p, q, c, n=20000):
    """Law of the committed token with a single child carrying token c, with
    the accept uniform and the residual uniform each on an n-point midpoint grid
    (they are independent: the accept decision sees only attempt 0)."""
    grid = (np.arange(n) + 0.5) / n
    acc = 0
    for u in grid:
        i, _, _ = S.branch_step(p, q, [c], lambda a, u=u: u)
        acc += i == 0
    a = acc / n
    law = np.zeros(len(p))
    law[c] += a
    if a < 1.0:
        rej = np.zeros(len(p))
        for u in grid:   # attempt 0 rejected (u0 = 1 - 1e-12 > ratio), attempt 1 on the grid
            i, t, _ = S.branch_step(p, q, [c], lambda k, u=u: (1 - 1e-12) if k == 0 else u)
            assert i == -1
            rej[t] += 1
        law += (1 - a) * rej / n
    return law


def test_single_child_law_equals_base_distribution():
    p = np.array([0.1, 0.5, 0.3, 0.1])
    q = np.array([0.4, 0.2, 0.3, 0.1])
    law = sum(q[c] * _law_one_child(p, q, c, n=4000) for c in range(4))
    assert np.abs(law - p).max() < 1e-3, law


def _trials(p, q, k, n_trials, step, seed=7):
    rng = np.random.default_rng(seed)
    counts = np.zeros(len(p))
    for trial in range(n_trials):
        kids, qq = [], q.copy()
        for _ in range(k):   # k distinct children drawn from q without replacement
            t = int(rng.choice(len(q), p=qq / qq.sum()))
            kids.append(t)
            qq[t] = 0.0
        i, t, _ = step(p, q, kids, lambda a, trial=trial: S.uniform(1234, trial, a))
        counts[kids[i] if i >= 0 else t] += 1
    return counts / n_trials


P5 = np.array([0.05, 0.40, 0.25, 0.20, 0.10])
Q5 = np.array([0.45, 0.05, 0.30, 0.10, 0.10])


@pytest.mark.parametrize("k", [1, 2, 3])
def test_multi_branch_law_equals_base_distribution(k):
    law = _trials(P5, Q5, k, 60_000, S.branch_step)
    tv = 0.5 * np.abs(law - P5).sum()
    assert tv < 0.01, (k, tv, law)


def _mutant_no_draft_update(p, q, child_tokens, u_of):
    """The rule with the draft left unchanged after a rejection (the
    with-replacement form): not lossless for distinct children."""
    r = np.array(p, np.float64)
    for i, t in enumerate(child_tokens):
        if u_of(i) < (r[t] / q[t] if q[t] > 0 else np.inf):
            return i, -1, 1.0
        r = np.maximum(r - q, 0.0)
        r = r / r.sum()
    t, m = S.inverse_cdf(r, u_of(len(child_tokens)))
    return -1, t, m


def test_pin_detects_missing_draft_update():
    law = _trials(P5, Q5, 3, 60_000, _mutant_no_draft_update)
    assert 0.5 * np.abs(law - P5).sum() > 0.02


def test_uniform_generator_range_and_determinism():
    us = [S.uniform(99, i, a) for i in range(200) for a in range(4)]
    assert all(0.0 <= u < 1.0 for u in us)
    assert all(u * (1 << 24) == int(u * (1 << 24)) for u in us)   # exact 24-bit grid (fp32-exact)
    assert S.uniform(99, 5, 1) == S.uniform(99, 5, 1) and S.uniform(99, 5, 1) != S.uniform(99, 5, 2)
    assert abs(np.mean(us) - 0.5) < 0.03


@pytest.mark.parametrize("seed", range(20))
def test_one_hot_base_reduces_to_greedy_walk(seed):
    rng = np.random.default_rng(seed)
    n, V = 30, 6
    parent = [-1] + [int(rng.integers(0, i)) for i in range(1, n)]
    token = [0] * n
    for i in range(1, n):   # distinct sibling tokens
        used = {token[j] for j in range(1, i) if parent[j] == parent[i]}
        free = [t for t in range(V) if t not in used]
        token[i] = int(rng.choice(free)) if free else -1
    verified = rng.random(n) < 0.7
    verified[0] = True
    am = rng.integers(0, V, n)
    g = T.accept_walk(parent, token, am, verified)
    q_rng = np.random.default_rng(seed + 100)
    qs = {v: (lambda x: x / x.sum())(q_rng.random(V) + 0.05) for v in range(n)}
    s = S.accept_walk_stochastic(
        0, lambda v: [c for c in range(n) if parent[c] == v and token[c] >= 0], lambda c: token[c],
        lambda v: bool(verified[v]), lambda v: v, lambda v: np.eye(V)[am[v]], lambda v: qs[v], seed)
    assert s["progress"] == g["progress"] == 1
    assert (s["acc"], s["x_new"], s["n_new"], s["cont"]) == (g["acc"], g["x_new"], g["n_new"], g["cont"])
