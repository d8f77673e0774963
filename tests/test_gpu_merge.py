"""f4 draft-side expansion on the GPU (PAPER.md:383-392
context-aware tree merging, P:399-402 score-aware top-L_se selection):
merge_kernel (path-hash table + exact path check) + submit_kernel in lockstep
with OraclePipeline.merge (the plain path-set definition, pinned in
tests/test_oracle_tree.py): appended order, segment bounds and the node id of
every T_new node bit-exact, then the usual tree / schedule / logits lockstep."""
import numpy as np
import pytest

from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES
from tests.lockstep import compare_tree, planted_trees, run_lockstep

pytestmark = pytest.mark.gpu
SEED = 0x5EED01


def overlap_tree(op, rng, n_extra, vocab):
    """T_new rooted at the current root: a random ancestor-closed subset of the
    live tree (paths that already exist) plus n_extra random nodes (some of
    which hit existing paths by token)."""
    keep = {0: 0}
    par, tok = [-1], [op.tok[0]]
    for s in range(1, len(op.node)):
        if op.par[s] in keep and rng.below(2):
            keep[s] = len(par)
            par.append(keep[op.par[s]])
            tok.append(op.tok[s])
    kids = {}
    for i in range(1, len(par)):
        kids.setdefault(par[i], set()).add(tok[i])
    for _ in range(n_extra):
        p = rng.below(len(par))
        while True:
            t = rng.below(min(vocab, 12))       # small alphabet: frequent path hits
            if t not in kids.setdefault(p, set()):
                break
        kids[p].add(t)
        par.append(p)
        tok.append(t)
    own = [1.0] + [0.05 + 0.9 * rng.uniform() for _ in range(len(par) - 1)]
    return np.array(par, np.int32), np.array(tok, np.int32), np.array(own, np.float32)


@pytest.mark.parametrize("name,P,l_top", [("tiny", 1, 0), ("tiny", 2, 0), ("tiny", 1, 5), ("small", 1, 6)])
def test_merge_lockstep(name, P, l_top):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    shape = SHAPES[name]
    if P == 1:
        gp = F.Pipeline(shape, max_ctx=1024, max_seg=16)
        stages = [gp]
    else:
        gp = F.LocalPipeline(shape, P, max_ctx=1024, max_seg=16)
        stages = gp.stages
    gp.fs_load_random_weights(SEED)
    gp.enable_logits()
    lps = [st.state()["layer_end"] - st.state()["layer_begin"] for st in stages]
    op = OraclePipeline(shape, SEED, n_stages=P, layers_per_stage=lps, max_slots=1024)
    prefix = gen.prefix_tokens(SEED, 32, shape.vocab)
    assert gp.fs_set_prefix(prefix) == op.set_prefix(prefix)
    rng = gen.Rng(77)
    merges = [0, 0]

    def merge(r, ticks, gp_, op_):
        if not op_.live or not op_.node or len(op_.node) > 300:
            return
        par, tok, own = overlap_tree(op_, rng, 6, shape.vocab)
        so = op_.merge(par, tok, own, l_max=8, l_top=l_top)
        sg = gp_.fs_submit_segment(F.FS_MERGE, par, tok, own, 8, l_top)
        assert sg["order"] == so["order"] and sg["bounds"] == [tuple(b) for b in so["bounds"]]
        assert sg["merged"] == so["merged"]
        merges[0] += 1
        merges[1] += len(so["order"])
        for st in stages:
            compare_tree(st, op_, st.cfg.max_live // 32, "merge")

    n_nodes, planted = (15, (0, 1, 2, 9)) if name == "tiny" else (30, (0, 2, 5, 17, 21))
    st = run_lockstep(gp, op, planted_trees(shape, n_nodes, 5, planted, SEED), n_rounds=4, l_max=8,
                      tol=1e-4 if name == "tiny" else 2e-2, append_fn=merge)
    print(f"{name} P={P} L_se={l_top}: merges {merges[0]} appended {merges[1]} decisions {st.decisions}")
    assert merges[0] > 0 and merges[1] > 0
    gp.close()
