"""Oracle of the whole pipelined verification path.  TEST INFRASTRUCTURE ONLY.

``OraclePipeline`` mirrors the C-ABI calls of include/flowspec.h
(set_prefix / submit / verify_step / accept / prune_and_compact) and follows
the paper step by step:

  * segments are consecutive slices of the score-ordered sequence S and are
    fed to stage 0 one after the other; at tick t stage p holds the segment
    that entered stage 0 at tick t-p (§3.1);
  * after the last stage a segment is verified; acceptance and Eq. 2 run
    over every verified node;
  * pruning keeps I_retain = I_acc ∪ I_pr, prunes each stage's in-flight
    segment (I_local) and KV cache (I_incache), then l_glo += |S_acc|
    (§3.3);
  * when Eq. 2 fails all remaining drafts are dropped and the round ends
    (P:315);
  * appended batches go after S (S_mer = S_pr || S_app).

The decoder math runs in the C oracle (oracle/fso.c, fp64 + contract
rounding).  Every intermediate the GPU must match bit-exactly (S order,
segment bounds, positions, ancestor sets, retain sets, rank maps, per-stage
KV slot maps, l_glo) is exposed by ``snapshot()``.
"""
import numpy as np

from . import fso
from . import tree as T


class Seg:
    __slots__ = ("seg_id", "b", "e", "h")

    def __init__(self, seg_id, b, e, h=None):
        self.seg_id, self.b, self.e, self.h = seg_id, b, e, h


class OraclePipeline:
    def __init__(self, shape, seed, n_stages=1, layers_per_stage=None, max_slots=4096,
                 max_live=512, cache_weights=False, keep_logits=True, rank=None):
        self.shape = shape
        self.P = n_stages
        # SPMD mode (rank given): this process computes only stage `rank`; hidden
        # rows move p -> p+1 by torch.distributed send/recv and the last stage's
        # per-row (argmax, margin) is broadcast — the protocol of fs_verify_step.
        self.rank = rank
        if layers_per_stage is None:
            base, rem = divmod(shape.n_layers, n_stages)
            layers_per_stage = [base + (1 if p < rem else 0) for p in range(n_stages)]
        assert sum(layers_per_stage) == shape.n_layers and len(layers_per_stage) == n_stages
        self.lb = list(np.cumsum([0] + list(layers_per_stage[:-1])))
        self.le = list(np.cumsum(layers_per_stage))
        self.model = fso.Model(shape, seed, cache_weights=cache_weights)
        self.kv = fso.KV(self.model, max_slots)
        self.max_live = max_live
        self.keep_logits = keep_logits
        self.l_glo = 0
        self.x_new = -1
        self.live = False
        self._reset_round()

    # ------------------------------------------------------------ state
    def _reset_round(self):
        self.node = []      # node id per S index
        self.tok = []
        self.par = []       # parent S index (-1 root)
        self.own = []
        self.verified = []
        self.am = []
        self.margin = []
        self.logits = {}    # node id -> logits (verified nodes)
        self.id2s = {}
        self.next_id = 0
        self.queue = []
        self.slot = [None] * self.P
        self.n_cached = [0] * self.P
        self.seg_counter = getattr(self, "seg_counter", 0)

    def _derived(self):
        depth = T.depth_of(self.par)
        anc = T.ancestors_or_self(self.par)
        return depth, anc

    def cu(self):
        """Eq. 1 relative to the current root (R11), in S order."""
        # parent S index < S index, so the fold of Eq. 1 runs in S order
        return T.cumulative_scores(self.par, self.own)

    def snapshot(self):
        depth, anc = self._derived()
        return dict(l_glo=self.l_glo, x_new=self.x_new, live=self.live,
                    node=list(self.node), token=list(self.tok), parent=list(self.par),
                    pos=[self.l_glo + d for d in depth], anc=[sorted(a) for a in anc],
                    n_cached=list(self.n_cached),
                    queue=[(s.seg_id, s.b, s.e) for s in self.queue],
                    inflight=[None if s is None else (s.seg_id, s.b, s.e) for s in self.slot])

    # ------------------------------------------------------------ prefix
    def set_prefix(self, tokens, mode="prefill", kv_seed=0):
        """Prefilling: the prompt runs through the decoder to build the
        KV cache and the first sampled token x_new.  mode 'synth': slots
        [0,n-1) get synthetic K/V, the last prompt token runs for real
        (SURVEY §8(d) "Prefix")."""
        n = len(tokens)
        if n < 1:
            raise ValueError("empty prefix")
        if self.live:
            raise RuntimeError("round live")
        if mode == "prefill":
            vis = [list(range(i + 1)) for i in range(n)]
            _, lg = fso.forward(self.model, self.kv, 0, self.shape.n_layers, tokens,
                                list(range(n)), list(range(n)), vis)
        else:
            self.kv.synth(n - 1, kv_seed)
            _, lg = fso.forward(self.model, self.kv, 0, self.shape.n_layers, [tokens[-1]],
                                [n - 1], [n - 1], [list(range(n))])
        self.prefix_logits = lg[-1].copy()
        self.x_new, _ = T.argmax_margin(lg[-1])
        self.l_glo = n
        self._reset_round()
        return self.x_new

    def greedy_stream(self, count):
        """Greedy autoregressive continuation [x_new, g1, ..., g_count] from the
        committed context (R-def-2).  Uses draft slots >= l_glo as scratch; they
        are always rewritten before being read by verification."""
        if self.live:
            raise RuntimeError("greedy_stream needs an idle round")
        toks = [self.x_new]
        for j in range(count):
            p = self.l_glo + j
            _, lg = fso.forward(self.model, self.kv, 0, self.shape.n_layers, [toks[-1]], [p],
                                [p], [list(range(p + 1))])
            toks.append(T.argmax_margin(lg[0])[0])
        return toks

    # ------------------------------------------------------------ submit
    def submit(self, new_round, parent_ids, tokens, own, l_max, l_top=0, order_mode="score"):
        """Draft initialization or expansion append.

        NEW_ROUND: node 0 is the root (parent -1, token = x_new); ids 0..n-1.
        APPEND: new ids continue; parents are live ids or earlier batch ids.
        Returns the batch's S order (node ids) and its segment bounds."""
        parent_ids = [int(p) for p in parent_ids]
        tokens = [int(t) for t in tokens]
        own = [np.float32(o) for o in own]
        n = len(parent_ids)
        if n < 1 or l_max < 1 or l_top < 0 or len(tokens) != n or len(own) != n:
            raise ValueError("bad sizes")
        if new_round:
            if self.live:
                raise RuntimeError("round live")
            if parent_ids[0] != -1 or tokens[0] != self.x_new:
                raise ValueError("root must be x_new with parent -1")
            base_id = 0
        else:
            if not self.live:
                raise RuntimeError("no live round")
            base_id = self.next_id
        ids = [base_id + i for i in range(n)]
        # validate: topological ids, known parents, own in (0,1], unique sibling tokens
        bpar_cu = []
        kids = {}
        for s in range(len(self.node)):
            if self.par[s] >= 0:
                kids.setdefault(self.node[self.par[s]], set()).add(self.tok[s])
        cur_cu = self.cu() if self.node else np.zeros(0, np.float32)
        for i in range(n):
            p = parent_ids[i]
            if new_round and i == 0:
                continue
            if not (0.0 < float(own[i]) <= 1.0):
                raise ValueError("own score outside (0,1]")
            if p >= ids[i] or p < 0:
                raise ValueError("parent must precede child")
            if p < base_id and p not in self.id2s:
                raise ValueError("unknown or pruned parent")
            if tokens[i] in kids.setdefault(p, set()):
                raise ValueError("duplicate sibling token")
            kids[p].add(tokens[i])
        # Eq. 1 over the batch (parents in S use their current cu)
        cu = np.zeros(n, np.float32)
        for i in range(n):
            p = parent_ids[i]
            if new_round and i == 0:
                cu[i] = np.float32(1.0)
            elif p >= base_id:
                cu[i] = np.float32(cu[p - base_id] * own[i])
            else:
                cu[i] = np.float32(cur_cu[self.id2s[p]] * own[i])
        if order_mode == "bfs":   # ablation: breadth-first instead of score order
            cur_depth = T.depth_of(self.par) if self.node else []
            dep = [0] * n
            for i in range(n):
                p = parent_ids[i]
                if new_round and i == 0:
                    dep[i] = 0
                elif p >= base_id:
                    dep[i] = dep[p - base_id] + 1
                else:
                    dep[i] = cur_depth[self.id2s[p]] + 1
            order = T.bfs_order(dep, ids)
        else:
            order = T.score_order(cu, ids)
        if l_top:
            order = T.top_L(order, l_top)
            keep = set(order)
            for i in order:  # connectivity: parents of kept batch nodes are kept
                p = parent_ids[i]
                assert p < base_id or (p - base_id) in keep
        if len(self.node) + len(order) > self.max_live:
            raise OverflowError("max_live exceeded")
        b0 = len(self.node)
        for i in order:
            self.id2s[ids[i]] = len(self.node)
            self.node.append(ids[i])
            self.tok.append(tokens[i])
            p = parent_ids[i]
            self.par.append(-1 if p < 0 else self.id2s[p])
            self.own.append(np.float32(1.0) if p < 0 else own[i])
            self.verified.append(False)
            self.am.append(-1)
            self.margin.append(np.inf)
        bounds = T.segment_bounds(len(order), l_max, base=b0)
        for (b, e) in bounds:
            self.queue.append(Seg(self.seg_counter, b, e))
            self.seg_counter += 1
        self.next_id = base_id + n
        self.live = True
        return dict(order=[ids[i] for i in order], bounds=bounds)

    def merge(self, parent_rel, tokens, own, l_max, l_top=0, order_mode="score"):
        """Tree merging (§3.4 context-aware expansion; with l_top =
        L_se the score-aware expansion of P:399-402): T_new (parent_rel =
        parent indices within T_new, node 0 = the current root x_new) is
        merged into T_pr; the nodes whose path is new are appended as S_app
        (S_mer = S_pr || S_app), ordered by cumulative score in the merged
        tree, optionally only the top-l_top of them.  Returns submit()'s dict
        plus merged = the node id of every T_new node (existing or new)."""
        if not self.live:
            raise RuntimeError("no live round")
        parent_rel = [int(p) for p in parent_rel]
        tokens = [int(t) for t in tokens]
        if not parent_rel or parent_rel[0] != -1 or tokens[0] != self.tok[0]:
            raise ValueError("T_new must be rooted at the current root")
        for i in range(1, len(parent_rel)):
            if not (0 <= parent_rel[i] < i):
                raise ValueError("parent must precede child")
        new, match = T.merge_new_nodes(self.par, self.tok, parent_rel, tokens)
        base = self.next_id
        new_id = {i: base + k for k, i in enumerate(new)}
        merged = [self.node[match[i]] if match[i] >= 0 else new_id[i] for i in range(len(tokens))]
        if not new:
            return dict(order=[], bounds=[], merged=merged)
        par_ids = [merged[parent_rel[i]] for i in new]
        out = self.submit(False, par_ids, [tokens[i] for i in new], [own[i] for i in new], l_max,
                          l_top=l_top, order_mode=order_mode)
        out["merged"] = merged
        return out

    # ------------------------------------------------------------ verify
    def _rows(self, seg, depth, anc):
        rows = list(range(seg.b, seg.e))
        ctx = list(range(self.l_glo))
        toks = [self.tok[i] for i in rows]
        pos = [self.l_glo + depth[i] for i in rows]
        slot = [self.l_glo + i for i in rows]
        vis = [ctx + [self.l_glo + a for a in sorted(anc[i])] for i in rows]
        return rows, toks, pos, slot, vis

    def verify_step(self):
        """One pipeline tick: stage 0 takes the next queued segment,
        every stage forwards its segment through its layer block, the last
        stage's output is verified, segments shift one stage."""
        if self.queue and self.slot[0] is None:
            self.slot[0] = self.queue.pop(0)
        if self.rank is not None:
            return self._verify_step_spmd()
        depth, anc = self._derived()
        out = dict(seg_id=-1, s_begin=0, n_rows=0, node=[], am=[], margin=[], logits=None)
        for p in range(self.P):
            seg = self.slot[p]
            if seg is None:
                continue
            if seg.e > seg.b:
                rows, toks, pos, slot, vis = self._rows(seg, depth, anc)
                last = p == self.P - 1
                h, lg = fso.forward(self.model, self.kv, self.lb[p], self.le[p], toks, pos, slot,
                                    vis, h_in=seg.h, want_hidden=not last, want_logits=last)
                seg.h = h
                if last:
                    ams, mgs = [], []
                    for k, i in enumerate(rows):
                        a, mg = T.argmax_margin(lg[k])
                        self.verified[i] = True
                        self.am[i] = a
                        self.margin[i] = mg
                        ams.append(a)
                        mgs.append(mg)
                        if self.keep_logits:
                            self.logits[self.node[i]] = lg[k].copy()
                    out.update(node=[self.node[i] for i in rows], am=ams, margin=mgs,
                               logits=lg if self.keep_logits else None)
            self.n_cached[p] = max(self.n_cached[p], seg.e)
            if p == self.P - 1:
                out.update(seg_id=seg.seg_id, s_begin=seg.b, n_rows=seg.e - seg.b)
        for p in range(self.P - 1, 0, -1):
            self.slot[p] = self.slot[p - 1]
        self.slot[0] = None
        return out

    def _verify_step_spmd(self):
        import torch
        import torch.distributed as dist
        depth, anc = self._derived()
        p, P, d = self.rank, self.P, self.shape.d_model
        out = dict(seg_id=-1, s_begin=0, n_rows=0, node=[], am=[], margin=[], logits=None)
        seg = self.slot[p]
        last = p == P - 1
        if seg is not None and seg.e > seg.b:
            rows, toks, pos, slot, vis = self._rows(seg, depth, anc)
            h, lg = fso.forward(self.model, self.kv, self.lb[p], self.le[p], toks, pos, slot, vis,
                                h_in=seg.h, want_hidden=not last, want_logits=last)
            seg.h = h
            if last:
                res = torch.tensor([T.argmax_margin(lg[k]) for k in range(len(rows))],
                                   dtype=torch.float64)
                out["logits"] = lg
        # stage handoff: p sends its rows to p+1, receives p-1's rows
        prev = self.slot[p - 1] if p > 0 else None
        recv_h = None
        if p < P - 1 and seg is not None and seg.e > seg.b:
            dist.send(torch.from_numpy(np.ascontiguousarray(seg.h)), dst=p + 1)
        if prev is not None and prev.e > prev.b:
            recv_h = torch.empty((prev.e - prev.b, d), dtype=torch.float32)
            dist.recv(recv_h, src=p - 1)
        # the last stage's (argmax, margin) rows reach every replica
        oseg = self.slot[P - 1]
        if oseg is not None and oseg.e > oseg.b:
            n = oseg.e - oseg.b
            if not last:
                res = torch.empty((n, 2), dtype=torch.float64)
            dist.broadcast(res, src=P - 1)
            for k in range(n):
                i = oseg.b + k
                self.verified[i] = True
                self.am[i] = int(res[k, 0])
                self.margin[i] = float(res[k, 1])
            out.update(seg_id=oseg.seg_id, s_begin=oseg.b, n_rows=n,
                       node=[self.node[oseg.b + k] for k in range(n)],
                       am=[int(res[k, 0]) for k in range(n)], margin=[float(res[k, 1]) for k in range(n)])
        elif oseg is not None:
            out.update(seg_id=oseg.seg_id, s_begin=oseg.b, n_rows=0)
        for q in range(P):
            if self.slot[q] is not None:
                self.n_cached[q] = max(self.n_cached[q], self.slot[q].e)
        for q in range(P - 1, 0, -1):
            self.slot[q] = self.slot[q - 1]
        self.slot[0] = None
        if p > 0 and self.slot[p] is not None:
            self.slot[p].h = recv_h.numpy() if recv_h is not None else None
        return out

    # ------------------------------------------------------------ accept
    def accept(self):
        """Acceptance and Eq. 2 over all verified nodes."""
        if not self.live:
            return dict(progress=0)
        r = T.accept_walk(self.par, self.tok, self.am, self.verified)
        if not r["progress"]:
            return r
        r["acc_ids"] = [self.node[i] for i in r["acc"]]
        r["acc_tokens"] = [self.tok[i] for i in r["acc"]]
        r["n_new_id"] = self.node[r["n_new"]] if r["n_new"] >= 0 else -1
        r["flagged"] = [self.node[i] for i in r["acc"] if self.margin[i] < T.MARGIN_FLAG]
        return r

    def accept_stochastic(self, q_of, temperature, seed, flag=None):
        """Stochastic acceptance (R24, oracle/sampling.py) over the verified
        nodes: p = softmax(logits / T) of this oracle's own logits, q_of(node
        id) the draft distribution, children in draw order (node id
        ascending).  flag: decision-margin threshold for near-threshold flags."""
        from oracle import sampling as SM
        if not self.live:
            return dict(progress=0)
        kids = {}
        for s in range(len(self.node)):
            if self.par[s] >= 0:
                kids.setdefault(self.par[s], []).append(s)
        r = SM.accept_walk_stochastic(
            0, lambda v: sorted(kids.get(v, []), key=lambda c: self.node[c]),
            lambda s: self.tok[s], lambda s: bool(self.verified[s]), lambda s: self.node[s],
            lambda s: SM.softmax(self.logits[self.node[s]], temperature),
            lambda s: q_of(self.node[s]), seed, SM.FLAG if flag is None else flag)
        if not r["progress"]:
            return r
        r["acc_ids"] = [self.node[i] for i in r["acc"]]
        r["acc_tokens"] = [self.tok[i] for i in r["acc"]]
        r["n_new_id"] = self.node[r["n_new"]] if r["n_new"] >= 0 else -1
        return r

    # ------------------------------------------------------------ prune
    def prune(self, decision):
        """Collaborative pruning or round exit.

        decision: dict(acc_ids, x_new, n_new_id, cont) — node ids, so that a
        decision taken elsewhere (lockstep harness) can be applied."""
        if not self.live:
            raise RuntimeError("no live round")
        acc = [self.id2s[i] for i in decision["acc_ids"]]
        # consistency: acc is the root path, n_new (if any) a child of its end
        if not acc or acc[0] != 0:
            raise ValueError("S_acc must start at the root")
        for k in range(1, len(acc)):
            if self.par[acc[k]] != acc[k - 1]:
                raise ValueError("S_acc is not a path")
        cont = int(decision["cont"])
        n_new = self.id2s[decision["n_new_id"]] if cont else -1
        if cont and self.par[n_new] != acc[-1]:
            raise ValueError("n_new is not a child of the last accepted node")
        depth, anc = self._derived()
        i_acc, i_pr, i_ret = T.prune_sets(acc, n_new, anc, len(self.node))
        r = T.rank_map(i_ret)
        a = len(i_acc)
        self.last_prune = dict(i_acc=i_acc, i_pr=i_pr, i_retain=i_ret, rank=r)
        # KV cache pruning per stage (I_incache): retained draft
        # slot l_glo+i moves to l_glo+r(i); context slots untouched.
        for p in range(self.P):
            keep = [i for i in i_ret if i < self.n_cached[p]]
            self.kv.move(self.lb[p], self.le[p], [self.l_glo + i for i in keep],
                         [self.l_glo + r[i] for i in keep])
            self.n_cached[p] = len(keep) - a if cont else 0
        self.l_glo += a
        if not cont:
            self.x_new = int(decision["x_new"])
            self.live = False
            self._reset_round()
            return self.last_prune
        # segment pruning (I_local): keep rows in I_pr, order kept
        pr_set = set(i_pr)
        newidx = {i: k for k, i in enumerate(i_pr)}

        def remap(x):
            return sum(1 for j in i_pr if j < x)

        for p in range(self.P):
            s = self.slot[p]
            if s is None:
                continue
            keep_rows = [k for k, i in enumerate(range(s.b, s.e)) if i in pr_set]
            if s.h is not None:
                s.h = s.h[keep_rows]
            s.b, s.e = remap(s.b), remap(s.e)   # empty in-flight segment = bubble (R9)
        q = []
        for s in self.queue:
            s.b, s.e = remap(s.b), remap(s.e)
            if s.e > s.b:
                q.append(s)
        self.queue = q
        # S_pr preserves the original order; re-root at n_new (R4, R11)
        self.node = [self.node[i] for i in i_pr]
        self.tok = [self.tok[i] for i in i_pr]
        self.par = [-1 if i == n_new else newidx[self.par[i]] for i in i_pr]
        self.own = [np.float32(1.0) if i == n_new else self.own[i] for i in i_pr]
        self.verified = [self.verified[i] for i in i_pr]
        self.am = [self.am[i] for i in i_pr]
        self.margin = [self.margin[i] for i in i_pr]
        self.id2s = {nid: k for k, nid in enumerate(self.node)}
        self.x_new = int(decision["x_new"])
        return self.last_prune
