"""Stochastic acceptance (temperature 1) of a draft tree, written out plainly.
TEST INFRASTRUCTURE ONLY (first step: the oracle and its
pins; the CUDA path is the next step and shares nothing with this file).

The paper evaluates at temperature 0 and 1 (Table 1) and
accepts "tokens that lead to an aligned distribution" (§3.3) without
giving the rule.  Reading R24: standard multi-branch
speculative rejection sampling (accept_walk stochastic mode),
in the lossless form for children drawn from the draft distribution WITHOUT
replacement (siblings never repeat a token):

  at the current node v (verified), with base distribution p_v and draft
  distribution q_v, residual r = p_v, draft q = q_v; for the children c_1..c_k
  of v in the given order (the order they were drawn):
      accept c_i with probability min(1, r(t_i) / q(t_i))          (u_i < ratio)
      on rejection:  r <- norm(max(r - q, 0)),  q <- norm(q with q(t_i) = 0)
  if every child is rejected, x_new ~ r (inverse CDF with u_k) and the round
  exits (Eq. 2 false); if child c is accepted and verified the walk descends
  (v = c); if c is accepted but not yet verified the walk stops with
  x_new = token(c), n_new = c (Eq. 2 true, the round continues).

Uniforms: u(seed, node id, attempt) from a counter-based generator that the
CUDA side will implement independently (splitmix64 finalizer; 24-bit uniform,
exact in fp32).  Decisions whose margin |u - ratio| (or the inverse-CDF
boundary distance) is below FLAG are flagged, as the greedy near-ties are.
"""
import numpy as np

FLAG = 1e-6
_M64 = (1 << 64) - 1


def _mix(z):
    """splitmix64 finalizer (SURVEY §8(d) hash)."""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def uniform(seed, node_id, attempt):
    """u in [0, 1) on a 2^-24 grid: mix(mix(seed ^ 0x5EED5A3C) ^ (node_id * 2^16 + attempt)) >> 40."""
    h = _mix(_mix((seed ^ 0x5EED5A3C) & _M64) ^ ((node_id << 16) + attempt))
    return (h >> 40) / float(1 << 24)


def softmax(logits, temperature=1.0):
    """Base distribution at temperature T > 0 (fp64)."""
    z = np.asarray(logits, np.float64) / temperature
    z = z - z.max()
    e = np.exp(z)
    return e / e.sum()


def inverse_cdf(r, u):
    """Smallest token t with sum_{s <= t} r(s) > u * sum(r); boundary distance for flagging."""
    c = np.cumsum(r)
    target = u * c[-1]
    t = int(np.searchsorted(c, target, side="right"))
    t = min(t, len(r) - 1)
    lo = c[t - 1] if t > 0 else 0.0
    return t, min(target - lo, c[t] - target) / c[-1]


def branch_step(p, q, child_tokens, u_of):
    """One node of the walk: returns (index of the accepted child or -1,
    sampled token or -1, smallest decision margin).  u_of(i) gives the
    uniform of attempt i (attempt k = the residual draw)."""
    r = np.array(p, np.float64)
    qq = np.array(q, np.float64)
    margin = np.inf
    for i, t in enumerate(child_tokens):
        ratio = r[t] / qq[t] if qq[t] > 0 else np.inf
        u = u_of(i)
        margin = min(margin, abs(u - ratio))
        if u < ratio:
            return i, -1, margin
        r = np.maximum(r - qq, 0.0)
        r = r / r.sum()
        qq[t] = 0.0
        qq = qq / qq.sum() if qq.sum() > 0 else qq
    t, m = inverse_cdf(r, u_of(len(child_tokens)))
    return -1, t, min(margin, m)


def accept_walk_stochastic(root, children, token, verified, node_id, p_of, q_of, seed, flag=FLAG):
    """The walk from the current root (R23: no progress until the root is
    verified).  children(v) -> child nodes of v in draw order; p_of / q_of(v)
    -> base / draft distribution at v.  Returns a dict like the greedy walk's:
    progress, acc (nodes of S_acc), x_new, n_new, cont, flagged (node ids)."""
    if not verified(root):
        return dict(progress=0)
    v, acc, flagged = root, [root], []
    while True:
        kids = children(v)
        i, t, margin = branch_step(p_of(v), q_of(v), [token(c) for c in kids],
                                   lambda a: uniform(seed, node_id(v), a))
        if margin < flag:
            flagged.append(node_id(v))
        if i < 0:
            return dict(progress=1, acc=acc, x_new=t, n_new=-1, cont=0, flagged=flagged)
        c = kids[i]
        if not verified(c):
            return dict(progress=1, acc=acc, x_new=token(c), n_new=c, cont=1, flagged=flagged)
        acc.append(c)
        v = c
