"""Lockstep parity harness: drive the CUDA path (C-ABI) and the oracle with the
same seeded inputs, compare every intermediate (SURVEY.md §8(c) parity rules):

  bit-exact  S order, segment bounds, positions, ancestor bitsets, cumulative
             scores, per-stage n_cached / segment schedule, l_glo, retain sets
  toleranced logits (max-abs <= tol), KV rows
  identical  accepted tokens, except where the oracle top-2 margin < 1e-2
             (flagged); then the oracle's decision is applied to both.
"""
import numpy as np

from oracle import tree as T
from oracle.pipeline import OraclePipeline
from synth import gen

FLAG = T.MARGIN_FLAG


def anc_bits_to_sets(words, n, ancw):
    w = np.asarray(words, np.uint32).reshape(n, ancw) if n else np.zeros((0, ancw), np.uint32)
    out = []
    for i in range(n):
        s = []
        for k in range(ancw):
            v = int(w[i, k])
            for b in range(32):
                if (v >> b) & 1:
                    s.append(32 * k + b)
        out.append(s)
    return out


class Stats:
    def __init__(self):
        self.max_abs = 0.0
        self.rows = 0
        self.flagged = 0
        self.decisions = 0
        self.overrides = 0
        self.committed = []
        self.kv_rows_checked = 0


def compare_tree(gp, op, ancw, where=""):
    from paper_2507_02620_b200 import flowspec as F
    snap = op.snapshot()
    st = gp.state()
    n = len(snap["node"])
    assert st["n_live"] == n, (where, st["n_live"], n)
    assert st["l_glo"] == snap["l_glo"], where
    assert st["n_cached"] == snap["n_cached"], (where, st["n_cached"], snap["n_cached"])
    assert [tuple(q) for q in st["queue"]] == [tuple(q) for q in snap["queue"]], where
    inf_o = [(-1, 0, 0) if s is None else tuple(s) for s in snap["inflight"]]
    inf_g = [tuple(s) if s[0] >= 0 else (-1, 0, 0) for s in st["inflight"]]
    assert inf_g == inf_o, (where, inf_g, inf_o)
    if n == 0:
        return
    assert list(gp.query(F.FS_Q_NODE)) == snap["node"], where
    assert list(gp.query(F.FS_Q_TOKEN)) == snap["token"], where
    assert list(gp.query(F.FS_Q_PARENT)) == snap["parent"], where
    assert list(gp.query(F.FS_Q_POS)) == snap["pos"], where
    assert anc_bits_to_sets(gp.query(F.FS_Q_ANC), n, ancw) == snap["anc"], where
    cu_g = gp.query(F.FS_Q_CU)
    cu_o = op.cu()
    assert np.array_equal(cu_g.view(np.uint32), np.asarray(cu_o, np.float32).view(np.uint32)), where


def kv_snapshot(stages):
    """Device KV rows of every cached draft slot, per stage (its own layers),
    K and V, first and last kv head: {(layer, which, kvh, S index): row}."""
    snap = {}
    for st in stages:
        s = st.state()
        nc = s["n_cached"][s["rank"]]
        hk = {0, st.shape.n_kv_heads - 1}
        for l in range(s["layer_begin"], s["layer_end"]):
            for w in (0, 1):
                for h in hk:
                    for i in range(nc):
                        snap[(l, w, h, i)] = (st, s["l_glo"], st.read_kv(l, w, h, s["l_glo"] + i))
    return snap


def check_kv_identity(snap, op):
    """SURVEY §8(c) "Compaction": after fs_prune_and_compact every retained
    cached draft row is byte-identical to its pre-compaction row, at slot
    l_glo_old + r(i) (accepted rows at l_glo_old .. l_glo_new - 1)."""
    lp = op.last_prune
    ret = set(lp["i_retain"])
    n = 0
    for (l, w, h, i), (st, l_old, row) in snap.items():
        if i not in ret:
            continue
        got = st.read_kv(l, w, h, l_old + lp["rank"][i])
        assert np.array_equal(got.view(np.uint32), row.view(np.uint32)), ("kv identity", l, w, h, i)
        n += 1
    return n


def run_lockstep(gp, op, trees_fn, n_rounds, l_max, tol, check_tree=True, check_kv=None,
                 append_fn=None, max_ticks=10000, bfs=False, kv_identity=None, l_top=0):
    """trees_fn(round, op) -> tree dict (parent, token, own); both sides get it.
    bfs: breadth-first submit order (the w/o-SBD ablation, FS_ORDER_BFS).
    kv_identity: stage contexts whose KV rows are checked byte-identical across
    every fs_prune_and_compact.  l_top: keep the top-L_top nodes."""
    stats = Stats()
    ancw = gp.cfg.max_live // 32
    for r in range(n_rounds):
        t = trees_fn(r, op)
        so = op.submit(True, t["parent"], t["token"], t["own"], l_max=l_max,
                       order_mode="bfs" if bfs else "score", l_top=l_top)
        sg = gp.fs_submit_segment(1 | (4 if bfs else 0), t["parent"], t["token"], t["own"], l_max,
                                  l_top)
        assert sg["order"] == so["order"], ("order", r)
        assert sg["bounds"] == [tuple(b) for b in so["bounds"]], ("bounds", r)
        if "order" in t and not bfs and not l_top:
            assert so["order"] == list(t["order"]), "generator target order not met"
        if check_tree:
            compare_tree(gp, op, ancw, f"submit r{r}")
        ticks = 0
        while True:
            ticks += 1
            assert ticks < max_ticks
            og = gp.fs_verify_step()
            oo = op.verify_step()
            assert og["seg_id"] == oo["seg_id"] and og["n_rows"] == oo["n_rows"], (og, oo)
            if oo["n_rows"]:
                assert og["node"] == oo["node"]
                for k in range(oo["n_rows"]):
                    stats.rows += 1
                    if oo["margin"][k] < FLAG:
                        stats.flagged += 1
                    else:
                        assert og["am"][k] == oo["am"][k], ("am", r, k, og["am"][k], oo["am"][k],
                                                            oo["margin"][k])
                if "logits" in og and oo["logits"] is not None:
                    err = float(np.max(np.abs(og["logits"] - oo["logits"])))
                    stats.max_abs = max(stats.max_abs, err)
                    assert err <= tol, ("logits", r, err)
            dg = gp.decision_dict(gp.fs_accept())
            do = op.accept()
            if not do["progress"]:
                assert not dg["progress"]
                if append_fn:
                    append_fn(r, ticks, gp, op)
                continue
            stats.decisions += 1
            want = dict(acc_ids=do["acc_ids"], acc_tokens=do["acc_tokens"], x_new=do["x_new"],
                        n_new_id=do["n_new_id"], cont=do["cont"])
            got = {k: dg[k] for k in want}
            if got != want:
                # allowed only through an oracle near-tie on a walked node
                walked = set(do["acc_ids"]) | set(dg.get("acc_ids", []))
                flagged = {op.node[i] for i in range(len(op.node)) if op.margin[i] < FLAG}
                assert walked & (flagged | set(do.get("flagged", []))), ("decision", r, got, want)
                stats.overrides += 1
            stats.committed += do["acc_tokens"]
            snap = kv_snapshot(kv_identity) if kv_identity else None
            gp.fs_prune_and_compact(want)
            op.prune(want)
            if snap:
                stats.kv_rows_checked += check_kv_identity(snap, op)
            if check_tree:
                compare_tree(gp, op, ancw, f"prune r{r} t{ticks}")
            if check_kv:
                check_kv(gp, op)
            if not do["cont"]:
                break
            if append_fn:
                append_fn(r, ticks, gp, op)
    return stats


def planted_trees(shape, n_nodes, depth, ranks, seed):
    def fn(r, op):
        stream = op.greedy_stream(len(ranks) + 1)
        return gen.planted_tree(seed + r, n_nodes, depth, stream, ranks, shape.vocab)
    return fn
