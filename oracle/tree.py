"""Tree algorithms of FlowSpec, written out plainly.  TEST INFRASTRUCTURE ONLY.

Each function follows one passage of /root/reference/PAPER.md (cited as P:line,
section, equation) in the paper's order and notation; where the paper is silent
the DESIGN.md reading (R1..R23) is named.  Sets are
Python sets, loops are plain loops: sizes here are <= a few hundred nodes.
"""
import numpy as np

MARGIN_FLAG = 1e-2  # north_star: nodes whose oracle top-2 margin < 1e-2 are flagged


def cumulative_scores(parent, own):
    """Eq. 1 (§3.2): c_cu(n_i) = c(n_i) * c_cu(parent(n_i)); root = 1.

    parent[i] < i (R10) so one pass in index order folds root -> node.
    fp32 products, round-to-nearest (R11)."""
    n = len(parent)
    cu = np.zeros(n, np.float32)
    for i in range(n):
        if parent[i] < 0:
            cu[i] = np.float32(1.0)
        else:
            cu[i] = np.float32(np.float32(cu[parent[i]]) * np.float32(own[i]))
    return cu


def score_order(cu, ids):
    """Score-based ordering (§3.2): descending cumulative score; ties by
    node id ascending (R10).  Returns positions into cu/ids."""
    return sorted(range(len(cu)), key=lambda i: (-float(cu[i]), int(ids[i])))


def bfs_order(depth, ids):
    """Breadth-first (layer) order: the "FlowSpec w/o Score-Based Draft"
    ablation (Table 2).  The paper does
    not name the replacement order; BFS is the reading SPEC S:506 takes.  Depth
    ascending, ties by node id ascending; topological because a parent is one
    layer shallower.  Returns positions into depth/ids."""
    return sorted(range(len(depth)), key=lambda i: (int(depth[i]), int(ids[i])))


def top_L(order, L):
    """Top-L refinement: keep the L highest-scoring nodes."""
    return list(order[:L])


def segment_bounds(n, l_max, base=0):
    """Segmentation (R12): consecutive slices of at most L_max."""
    return [(base + b, base + min(b + l_max, n)) for b in range(0, n, l_max)]


def depth_of(parent_s):
    """Depth by walking parents (root depth 0)."""
    d = []
    for i in range(len(parent_s)):
        k, p = 0, parent_s[i]
        while p >= 0:
            k += 1
            p = parent_s[p]
        d.append(k)
    return d


def ancestors_or_self(parent_s):
    """Tree attention mask (§3.1) in set form: entry i attends to its
    ancestors and itself (plus the committed context)."""
    out = []
    for i in range(len(parent_s)):
        s, p = {i}, parent_s[i]
        while p >= 0:
            s.add(p)
            p = parent_s[p]
        out.append(s)
    return out


def argmax_margin(logits):
    """Greedy target token (lowest id on ties) and top-1 minus top-2."""
    am = int(np.argmax(logits))
    srt = np.sort(logits.astype(np.float32))
    margin = float(np.float32(srt[-1]) - np.float32(srt[-2])) if logits.size > 1 else float("inf")
    return am, margin


def accept_walk(parent_s, token, am, verified):
    """Acceptance + continuous condition (§3.3, Eq. 2), greedy (R1).

    From the root (S index 0): while the child of v whose token equals the base
    argmax at v exists and is verified (R3), descend.  S_acc = root..v (R2),
    x_new = am[v], n_new = the child of v carrying x_new (unverified) or -1;
    continue iff n_new exists (Eq. 2).  Root not verified -> progress 0 (R23).
    """
    n = len(parent_s)
    if n == 0 or not verified[0]:
        return dict(progress=0)
    kids = {}
    for j in range(n):
        if parent_s[j] >= 0:
            kids.setdefault(parent_s[j], {})[int(token[j])] = j
    v, path = 0, [0]
    while True:
        c = kids.get(v, {}).get(int(am[v]), -1)
        if c >= 0 and verified[c]:
            v = c
            path.append(c)
        else:
            break
    x_new = int(am[v])
    n_new = kids.get(v, {}).get(x_new, -1)
    return dict(progress=1, acc=path, x_new=x_new, n_new=n_new, cont=int(n_new >= 0))


def prune_sets(acc, n_new, anc, n_live):
    """Tree pruning (§3.3, Fig. 3): I_acc = indices of S_acc;
    I_pr = n_new and its descendants (entries whose ancestor set holds n_new);
    I_retain = I_acc ∪ I_pr.  On exit (n_new = -1) I_retain = I_acc (R16)."""
    i_acc = sorted(acc)
    i_pr = [j for j in range(n_live) if n_new >= 0 and n_new in anc[j]]
    return i_acc, i_pr, sorted(set(i_acc) | set(i_pr))


def rank_map(i_retain):
    """Position of each retained index in I_retain (order preserved)."""
    return {i: k for k, i in enumerate(i_retain)}


def path_of(parent, token, i):
    """path_T(n): the token sequence from the root to node i."""
    p = []
    while i >= 0:
        p.append(int(token[i]))
        i = parent[i]
    return tuple(reversed(p))


def merge_new_nodes(pr_parent, pr_token, new_parent, new_token):
    """Context-aware expansion, tree merging (§3.4).

    P_pr = {path_Tpr(n) | n in T_pr};  N_new = {n in T_new | path_Tnew(n) not
    in P_pr}.  Both trees are rooted at the current root x_new (T_pr: S index 0;
    T_new: index 0).  Returns (N_new as T_new indices in T_new order, match)
    where match[i] = the T_pr node with the same path, or -1 for new nodes."""
    P_pr = {}
    for n in range(len(pr_parent)):
        P_pr[path_of(pr_parent, pr_token, n)] = n
    new, match = [], []
    for i in range(len(new_parent)):
        m = P_pr.get(path_of(new_parent, new_token, i), -1)
        match.append(m)
        if m < 0:
            new.append(i)
    return new, match
