"""Counter-based generators for host-side inputs (SURVEY.md §8(d) "Generators").

* ``mix64``           splitmix64 finalizer (the same counter hash both sides
                      implement independently for weights; here it only drives
                      host inputs).
* ``prefix_tokens``   prompt tokens ``mix(seed_p ^ i) mod V``.
* ``planted_tree``    a draft tree (parent ids, tokens, own scores) that carries
                      a planted path g_1..g_a under the root, with target score
                      ranks (SURVEY §8(d) "Trees (planted path)").

Nothing here computes the method: the consumer re-derives the score order
from (parent, own) and the tests check it against ``order`` (target scores
are 1 - 0.9 r/(n+1), gaps of ~1e-2 that fp32 rounding of the own-score
quotients, ~1e-7, cannot reorder).
"""
import numpy as np

M64 = (1 << 64) - 1


def mix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class Rng:
    """Tiny counter-based RNG (host inputs only)."""

    def __init__(self, seed: int):
        self.key = mix64(seed & M64)
        self.ctr = 0

    def next(self) -> int:
        self.ctr += 1
        return mix64(self.key ^ self.ctr)

    def below(self, n: int) -> int:
        return self.next() % n

    def uniform(self) -> float:
        return (self.next() >> 11) / float(1 << 53)


def prefix_tokens(seed: int, n: int, vocab: int):
    return [mix64((seed ^ i) & M64) % vocab for i in range(n)]


def planted_tree(seed: int, n_nodes: int, max_depth: int, stream, planted_ranks,
                 vocab: int, max_tries: int = 200):
    """Draft tree with a planted greedy path.

    stream        greedy tokens [g_0 = root token, g_1, g_2, ...] (len >= a+2)
    planted_ranks target S ranks of [root, g_1, ..., g_a] (rank of root = 0)

    Returns dict(parent, token, own, order, planted_ids) with node ids in
    creation order (parent id < id) and ``order`` the target S order (node ids).
    No child of planted node g_j carries g_{j+1} except g_{j+1} itself, and no
    child of g_a carries g_{a+1}: a round commits exactly a+1 tokens (scenario R).
    """
    a = len(planted_ranks) - 1
    assert planted_ranks[0] == 0 and list(planted_ranks) == sorted(planted_ranks)
    assert a <= max_depth and len(stream) >= a + 2 and n_nodes >= a + 1
    for attempt in range(max_tries):
        rng = Rng(seed * 1000003 + attempt)
        parent = [-1]
        token = [stream[0]]
        depth = [0]
        planted_ids = [0]
        for j in range(1, a + 1):      # planted chain root -> g1 -> ... -> ga
            parent.append(planted_ids[-1])
            token.append(stream[j])
            depth.append(j)
            planted_ids.append(len(parent) - 1)
        children = {i: {token[c] for c in range(len(parent)) if parent[c] == i}
                    for i in range(len(parent))}
        forbidden = {planted_ids[j]: stream[j + 1] for j in range(a + 1)}
        ok = True
        while len(parent) < n_nodes:
            cand = [i for i in range(len(parent)) if depth[i] < max_depth]
            p = cand[rng.below(len(cand))]
            for _ in range(64):
                t = rng.below(vocab)
                if t not in children.setdefault(p, set()) and forbidden.get(p) != t:
                    break
            else:
                ok = False
                break
            parent.append(p)
            token.append(t)
            depth.append(depth[p] + 1)
            children[p].add(t)
            children[len(parent) - 1] = set()
        if not ok:
            continue
        n = n_nodes
        # random topological order with planted nodes pinned at their ranks
        pinned = {planted_ranks[j]: planted_ids[j] for j in range(a + 1)}
        pinned_ids = set(pinned.values())
        placed = [False] * n
        order = []
        for r in range(n):
            if r in pinned:
                nid = pinned[r]
                if parent[nid] >= 0 and not placed[parent[nid]]:
                    ok = False
                    break
            else:
                avail = [i for i in range(n) if not placed[i] and i not in pinned_ids
                         and (parent[i] < 0 or placed[parent[i]])]
                if not avail:
                    ok = False
                    break
                nid = avail[rng.below(len(avail))]
            placed[nid] = True
            order.append(nid)
        if not ok:
            continue
        rank = {nid: r for r, nid in enumerate(order)}
        cu_t = [np.float32(1.0 - 0.9 * rank[i] / (n + 1)) for i in range(n)]
        own = [np.float32(1.0)] + [np.float32(cu_t[i] / cu_t[parent[i]]) for i in range(1, n)]
        if not all(0.0 < float(o) <= 1.0 for o in own):
            continue
        return dict(parent=np.array(parent, np.int32), token=np.array(token, np.int32),
                    own=np.array(own, np.float32), order=np.array(order, np.int32),
                    planted_ids=planted_ids)
    raise RuntimeError("planted_tree: could not meet the target ranks")


def random_tree(seed: int, n_nodes: int, max_depth: int, vocab: int, root_token: int,
                own_lo: float = 1.0 / 64):
    """Unplanted random tree (parent id < id, unique sibling tokens, own in [own_lo,1])."""
    rng = Rng(seed)
    parent, token, depth, own = [-1], [root_token], [0], [np.float32(1.0)]
    kids = {0: set()}
    while len(parent) < n_nodes:
        cand = [i for i in range(len(parent)) if depth[i] < max_depth and len(kids[i]) < vocab]
        p = cand[rng.below(len(cand))]
        while True:
            t = rng.below(vocab)
            if t not in kids[p]:
                break
        kids[p].add(t)
        parent.append(p)
        token.append(t)
        depth.append(depth[p] + 1)
        kids[len(parent) - 1] = set()
        # quantised scores make exact ties (exercise the id tie-break)
        q = rng.below(8)
        own.append(np.float32(own_lo + (1.0 - own_lo) * q / 7.0))
    return dict(parent=np.array(parent, np.int32), token=np.array(token, np.int32),
                own=np.array(own, np.float32))


class SteadyExpansion:
    """Scenario S input (SURVEY §8(d) "Trees", configs[3]): the planted greedy
    chain continues in appended batches (S_mer = S_pr || S_app) so the
    pipeline never runs dry.  Every batch holds q chain nodes
    g_{k+1..k+q} hanging off the current chain tip, plus distractors under the
    tip, the new chain nodes and earlier batch nodes; sibling tokens stay unique
    across batches and no distractor under a chain node carries the next chain
    token, so each verified batch commits exactly q tokens.

    tree      the initial NEW_ROUND tree from planted_tree (its planted chain
              ends at the tip g_a); stream[j] = g_j for j >= 0."""

    def __init__(self, seed, tree, stream, q=2, batch=16, vocab=32000):
        self.rng = Rng(seed)
        self.stream = stream
        self.q, self.batch, self.vocab = q, batch, vocab
        par = [int(p) for p in tree["parent"]]
        tok = [int(t) for t in tree["token"]]
        self.kids = {}
        for i, p in enumerate(par):
            if p >= 0:
                self.kids.setdefault(p, set()).add(tok[i])
        self.tip = int(tree["planted_ids"][-1])
        self.k = len(tree["planted_ids"]) - 1        # tip carries g_k
        self.next_id = len(par)

    def next_batch(self):
        """(parent ids, tokens, own) of the next APPEND batch (ids continue at
        next_id; parents precede children)."""
        q, base = self.q, self.next_id
        if self.k + q + 1 >= len(self.stream):
            raise IndexError("stream exhausted")
        parent, token, own = [], [], []
        chain = []
        p = self.tip
        for j in range(q):                      # chain g_{k+1} .. g_{k+q}
            t = self.stream[self.k + 1 + j]
            self.kids.setdefault(p, set()).add(t)
            parent.append(p)
            token.append(t)
            own.append(np.float32(0.95))
            chain.append(base + j)
            p = base + j
        forbid = {self.tip: self.stream[self.k + 1]}
        for j in range(q):
            forbid[chain[j]] = self.stream[self.k + 2 + j]
        anchors = [self.tip] + chain
        for i in range(q, self.batch):
            cand = anchors + [base + j for j in range(q, i)]
            pid = cand[self.rng.below(len(cand))]
            kids = self.kids.setdefault(pid, set())
            while True:
                t = self.rng.below(self.vocab)
                if t not in kids and forbid.get(pid) != t:
                    break
            kids.add(t)
            parent.append(pid)
            token.append(t)
            own.append(np.float32(0.05 + 0.75 * self.rng.uniform()))
        self.tip = chain[-1]
        self.k += q
        self.next_id = base + self.batch
        return (np.array(parent, np.int32), np.array(token, np.int32), np.array(own, np.float32))
