"""Pins of the oracle's tree algorithms (oracle/tree.py) against what the paper
and plain mathematics fix: closed forms, the Fig. 3 caption, App. A.1 sizes,
brute force on small inputs.  CPU only."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import tree as T
from synth import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ Eq. 1
def test_eq1_closed_forms():
    # root = empty product = 1; one step 0.5 * 0.4 = 0.2
    cu = T.cumulative_scores([-1, 0, 1], [1.0, 0.5, 0.4])
    assert cu[0] == np.float32(1.0)
    assert cu[1] == np.float32(0.5)
    assert cu[2] == np.float32(np.float32(0.5) * np.float32(0.4))
    assert abs(float(cu[2]) - 0.2) < 1e-7


@pytest.mark.parametrize("seed", range(20))
def test_eq1_equals_path_product_walk(seed):
    t = gen.random_tree(seed, 40, 8, 50, 3)
    cu = T.cumulative_scores(t["parent"], t["own"])
    for i in range(40):
        # brute force: walk to the root collecting own scores, multiply root->node
        path, p = [], i
        while p >= 0:
            path.append(p)
            p = t["parent"][p]
        prod = np.float32(1.0)
        for j in reversed(path[:-1]):
            prod = np.float32(prod * np.float32(t["own"][j]))
        assert prod == cu[i]
        assert abs(float(cu[i]) - float(np.prod(np.float64(t["own"][path[:-1]])))) < 1e-5
        if t["parent"][i] >= 0:  # scores never increase down the tree
            assert cu[i] <= cu[t["parent"][i]]


# ------------------------------------------------------------------ order
@pytest.mark.parametrize("seed", range(20))
def test_order_is_bruteforce_sort_and_topological(seed):
    t = gen.random_tree(100 + seed, 60, 6, 40, 1)
    cu = T.cumulative_scores(t["parent"], t["own"])
    ids = np.arange(60)
    order = T.score_order(cu, ids)
    # brute force: repeatedly extract the max (cu, then smallest id)
    rest, bf = set(range(60)), []
    while rest:
        best = None
        for i in rest:
            if best is None or cu[i] > cu[best] or (cu[i] == cu[best] and i < best):
                best = i
        bf.append(best)
        rest.remove(best)
    assert order == bf
    pos = {v: k for k, v in enumerate(order)}
    for i in range(1, 60):  # parent before child
        assert pos[t["parent"][i]] < pos[i]
    # every prefix is ancestor-closed, so every top-L is a connected tree
    for L in range(1, 61):
        keep = set(T.top_L(order, L))
        assert all(t["parent"][i] in keep for i in keep if i != 0)


def test_planted_tree_meets_target_order():
    for seed in range(10):
        stream = list(range(10, 20))
        t = gen.planted_tree(seed, 64, 6, stream, (0, 2, 5, 17, 21), 1000)
        cu = T.cumulative_scores(t["parent"], t["own"])
        assert [int(i) for i in T.score_order(cu, np.arange(64))] == list(t["order"])


def test_segments_appendix_a1():
    g = _gold("appendix_a1_segments.json")
    for c in g["cases"]:
        b = T.segment_bounds(c["n"], c["l_max"])
        assert [e - s for s, e in b] == c["lengths"]
        assert b[0][0] == 0 and b[-1][1] == c["n"]
        assert all(b[k][1] == b[k + 1][0] for k in range(len(b) - 1))


# ------------------------------------------------------------------ masks
def test_mask_special_cases():
    # chain -> lower-triangular; root with two children -> siblings invisible
    assert T.ancestors_or_self([-1, 0, 1]) == [{0}, {0, 1}, {0, 1, 2}]
    assert T.ancestors_or_self([-1, 0, 0]) == [{0}, {0, 1}, {0, 2}]


@pytest.mark.parametrize("seed", range(10))
def test_mask_equals_transitive_closure(seed):
    t = gen.random_tree(500 + seed, 30, 7, 30, 0)
    n = 30
    A = np.zeros((n, n), bool)  # A[i, j]: j is the parent of i
    for i in range(1, n):
        A[i, t["parent"][i]] = True
    R = np.eye(n, dtype=bool)
    for _ in range(n):  # reflexive-transitive closure by repeated squaring-ish
        R = R | (R.astype(np.int32) @ A.astype(np.int32) > 0)
    anc = T.ancestors_or_self(list(t["parent"]))
    for i in range(n):
        assert anc[i] == set(np.nonzero(R[i])[0].tolist())
    d = T.depth_of(list(t["parent"]))
    assert all(len(anc[i]) == d[i] + 1 for i in range(n))


# ------------------------------------------------------------------ accept
def test_accept_zero_acceptance_and_perfect_alignment():
    par = [-1, 0, 1, 2]
    tok = [5, 6, 7, 8]
    # argmax at root not among its children: S_acc = [root] (R2), exit
    r = T.accept_walk(par, tok, [9, 0, 0, 0], [True] * 4)
    assert r == dict(progress=1, acc=[0], x_new=9, n_new=-1, cont=0)
    # perfectly aligned chain: accept everything, bonus token after the leaf
    r = T.accept_walk(par, tok, [6, 7, 8, 3], [True] * 4)
    assert r["acc"] == [0, 1, 2, 3] and r["x_new"] == 3 and not r["cont"]
    # unverified child matching the argmax: stop before it, continue (R3, Eq. 2)
    r = T.accept_walk(par, tok, [6, 7, 0, 0], [True, True, False, False])
    assert r["acc"] == [0, 1] and r["n_new"] == 2 and r["cont"] == 1
    # root unverified: no progress (R23)
    assert T.accept_walk(par, tok, [6, 7, 8, 3], [False] * 4) == dict(progress=0)


@pytest.mark.parametrize("seed", range(30))
def test_accept_matches_bruteforce_path_search(seed):
    rng = gen.Rng(seed)
    t = gen.random_tree(900 + seed, 25, 5, 6, 0)
    par, tok = list(t["parent"]), list(t["token"])
    am = [rng.below(6) for _ in range(25)]
    ver = [True] * 25
    r = T.accept_walk(par, tok, am, ver)
    # brute force: the longest root path whose every step follows the argmax;
    # Eq. 2 by a linear scan over all node paths
    paths = {}
    for i in range(25):
        p, pth = i, []
        while p >= 0:
            pth.append(tok[p])
            p = par[p]
        paths[i] = tuple(reversed(pth))
    best = [0]
    for i in range(25):
        pth = [i]
        p = par[i]
        while p >= 0:
            pth.append(p)
            p = par[p]
        pth.reverse()
        if all(tok[pth[k + 1]] == am[pth[k]] for k in range(len(pth) - 1)) and len(pth) > len(best):
            best = pth
    assert r["acc"] == best
    want = paths[best[-1]] + (am[best[-1]],)
    found = [i for i in range(25) if paths[i] == want]
    assert r["cont"] == int(bool(found)) and (r["n_new"] == (found[0] if found else -1))


# ------------------------------------------------------------------ prune
def test_fig3_prune_vector():
    g = _gold("fig3_pruning.json")
    par = g["parent_s"]
    anc = T.ancestors_or_self(par)
    i_acc, i_pr, i_ret = T.prune_sets(g["acc"], g["n_new"], anc, len(par))
    assert i_acc == g["I_acc"] and i_pr == g["I_pr"] and i_ret == g["I_retain"]
    assert T.rank_map(i_ret) == {int(k): v for k, v in g["rank_map"].items()}
    assert T.segment_bounds(len(par), g["l_max"]) == [tuple(s) for s in g["segments"]]


@pytest.mark.parametrize("seed", range(30))
def test_prune_equals_path_prefix_bruteforce(seed):
    rng = gen.Rng(7 * seed + 1)
    t = gen.random_tree(300 + seed, 40, 6, 5, 2)
    par, tok = list(t["parent"]), list(t["token"])
    am = [rng.below(5) for _ in range(40)]
    r = T.accept_walk(par, tok, am, [True] * 40)
    anc = T.ancestors_or_self(par)
    i_acc, i_pr, i_ret = T.prune_sets(r["acc"], r["n_new"], anc, 40)
    # brute force: keep nodes whose token path has S_acc||x_new as prefix
    def path(i):
        out = []
        while i >= 0:
            out.append(tok[i])
            i = par[i]
        return out[::-1]
    pre = [tok[i] for i in r["acc"]] + [r["x_new"]]
    bf = [i for i in range(40) if path(i)[:len(pre)] == pre]
    assert i_pr == (bf if r["cont"] else [])
    # causality: retained entries keep their retained ancestors before them
    for i in i_pr:
        assert all(a in i_pr for a in anc[i] if a >= r["n_new"] and a in anc[i] and r["n_new"] in anc[a])
    # accepted indices all precede retained draft indices (so accepted rows land
    # at l_glo..l_glo'-1 after compaction, SURVEY §8(c) "Compaction")
    if i_pr:
        assert max(i_acc) < min(i_pr)


# ------------------------------------------------------------------ BFS ablation order (f1)
def _levels_by_children(parent):
    """Independent construction: level sets by walking parent -> children from
    the roots, each level emitted in id order."""
    kids = {}
    for i, p in enumerate(parent):
        kids.setdefault(p, []).append(i)
    out, level = [], sorted(kids.get(-1, []))
    while level:
        out += level
        level = sorted(c for v in level for c in kids.get(v, []))
    return out


@pytest.mark.parametrize("seed", range(20))
def test_bfs_order_is_layer_order(seed):
    t = gen.random_tree(seed, 48, 7, 50, 3)
    par = t["parent"]
    order = T.bfs_order(T.depth_of(par), list(range(len(par))))
    assert order == _levels_by_children(par)
    pos = {v: k for k, v in enumerate(order)}
    for i, p in enumerate(par):   # topological: every prefix is ancestor-closed
        if p >= 0:
            assert pos[p] < pos[i]


def test_bfs_equals_score_order_on_a_chain():
    par = [-1, 0, 1, 2, 3]
    cu = T.cumulative_scores(par, [1.0, 0.9, 0.8, 0.7, 0.6])
    ids = list(range(5))
    assert T.bfs_order(T.depth_of(par), ids) == T.score_order(cu, ids) == ids


# ------------------------------------------------------------------ f4 merge
def _tree_paths(parent, token):
    """Brute force: every node's root path, walked independently of oracle/tree.py."""
    out = []
    for i in range(len(parent)):
        p, j = [], i
        while j >= 0:
            p.insert(0, int(token[j]))
            j = int(parent[j])
        out.append(tuple(p))
    return out


def _overlapping_trees(seed, vocab=6):
    """T_pr and T_new rooted at the same token with a small vocabulary, so many
    paths coincide."""
    a = gen.random_tree(seed, 25, 4, vocab, 3)
    b = gen.random_tree(seed + 1000, 25, 4, vocab, 3)
    return a, b


@pytest.mark.parametrize("seed", range(12))
def test_merge_path_set_is_union(seed):
    """Tree merging: after merging, the tree holds every path of
    T_pr and T_new exactly once; S_pr stays at the front in its order; every
    T_new node maps to the node with its path."""
    from oracle.pipeline import OraclePipeline
    from synth.configs import SHAPES
    a, b = _overlapping_trees(seed)
    op = OraclePipeline(SHAPES["tiny"], 1, n_stages=1, max_slots=256)
    op.x_new, op.l_glo = 3, 10
    op.submit(True, a["parent"], a["token"], a["own"], l_max=8)
    before_nodes = list(op.node)
    out = op.merge(b["parent"], b["token"], b["own"], l_max=8)
    P_a = set(_tree_paths(a["parent"], a["token"]))
    P_b = set(_tree_paths(b["parent"], b["token"]))
    paths = _tree_paths(op.par, op.tok)
    assert len(paths) == len(set(paths)) and set(paths) == P_a | P_b
    assert op.node[:len(before_nodes)] == before_nodes            # S_mer = S_pr || S_app
    assert len(op.node) == len(before_nodes) + len(P_b - P_a)
    bp = _tree_paths(b["parent"], b["token"])
    for i, nid in enumerate(out["merged"]):
        assert paths[op.id2s[nid]] == bp[i]
    # appended nodes come after their parents (ancestor-closed prefixes)
    for s in range(len(op.node)):
        assert op.par[s] < s


def test_merge_special_cases():
    from oracle.pipeline import OraclePipeline
    from synth.configs import SHAPES
    a = gen.random_tree(5, 20, 4, 50, 7)
    op = OraclePipeline(SHAPES["tiny"], 1, n_stages=1, max_slots=256)
    op.x_new, op.l_glo = 7, 10
    op.submit(True, a["parent"], a["token"], a["own"], l_max=8)
    n0 = len(op.node)
    # T_new == T_pr: nothing new
    out = op.merge(a["parent"], a["token"], a["own"], l_max=8)
    assert out["order"] == [] and len(op.node) == n0 and out["merged"] == list(range(20))
    # a chain whose first token is new below the root: all of it is appended
    toks = [7] + [t for t in range(60, 64)]
    out = op.merge([-1, 0, 1, 2, 3], toks, [1.0, 0.9, 0.9, 0.9, 0.9], l_max=8)
    assert len(out["order"]) == 4 and len(op.node) == n0 + 4


@pytest.mark.parametrize("seed", range(6))
def test_score_aware_top_l_is_score_prefix_of_new_nodes(seed):
    """Score-aware expansion: of the nodes not yet in T, the top-L_se
    by cumulative score are appended; the kept set is closed under parents."""
    from oracle.pipeline import OraclePipeline
    from synth.configs import SHAPES
    a, b = _overlapping_trees(seed + 50, vocab=8)
    op = OraclePipeline(SHAPES["tiny"], 1, n_stages=1, max_slots=256)
    op.x_new, op.l_glo = 3, 10
    op.submit(True, a["parent"], a["token"], a["own"], l_max=8)
    n0 = len(op.node)
    cu_pr = {op.node[s]: float(c) for s, c in enumerate(op.cu())}
    new, _ = T.merge_new_nodes(op.par, op.tok, b["parent"], b["token"])
    out = op.merge(b["parent"], b["token"], b["own"], l_max=8, l_top=5)
    kept = len(out["order"])
    assert kept == min(5, len(new)) and len(op.node) == n0 + kept
    # brute force: Eq. 1 of every new node in the merged tree (fp32 products
    # along T_new, starting from the matched T_pr ancestor's score)
    P_a = {p: i for i, p in enumerate(_tree_paths(a["parent"], a["token"]))}
    bp = _tree_paths(b["parent"], b["token"])
    cu_a = T.cumulative_scores(a["parent"], a["own"])
    cu_b = {}
    for i in range(len(bp)):
        if bp[i] in P_a:
            cu_b[i] = np.float32(cu_a[P_a[bp[i]]])
        else:
            cu_b[i] = np.float32(cu_b[int(b["parent"][i])] * np.float32(b["own"][i]))
    cand = sorted((i for i in range(len(bp)) if bp[i] not in P_a), key=lambda i: (-float(cu_b[i]), i))
    want = {bp[i] for i in cand[:5]}
    got = set(_tree_paths(op.par, op.tok)[n0:])
    assert got == want
    assert all(op.par[s] < s for s in range(len(op.node)))
