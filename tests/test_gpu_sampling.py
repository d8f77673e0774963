"""Stochastic acceptance on the GPU (Table 1 T=1
P:461; reading R24): sample_walk_kernel against the oracle walk
(oracle/sampling.py via OraclePipeline.accept_stochastic) in lockstep, and the
losslessness law on the GPU (the committed token's law equals the base
distribution p when the children are drawn from q without replacement).

Decisions may differ only where the oracle's own decision margin is below the
logit tolerance's effect on the ratio p/q or on the inverse-CDF boundary
(fp32: 1e-3, bf16: 5e-2); the oracle's decision is then applied to both."""
import numpy as np
import pytest

from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES, reduced
from tests.lockstep import compare_tree

pytestmark = pytest.mark.gpu
SEED = 0x5EED01


def _draft_q(tree, vocab, n_rows, seed):
    """Draft distributions by node id: half the mass on the node's first child
    token (so that child's ratio p/q straddles 1), half a peaked random
    distribution (counter-based)."""
    q = np.zeros((n_rows, vocab), np.float32)
    first = {}
    for i, p in enumerate(tree["parent"]):
        if p >= 0 and p not in first:
            first[int(p)] = int(tree["token"][i])
    for nid in range(len(tree["parent"])):
        rng = gen.Rng(seed * 7919 + nid)
        z = np.array([rng.uniform() for _ in range(vocab)])
        w = np.exp(4.0 * z)
        row = 0.5 * w / w.sum()
        if nid in first:
            row[first[nid]] += 0.5
        else:
            row *= 2.0
        q[nid] = row / row.sum()
    return q


def _setup(name, P, sampling=1, max_ctx=1024):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    shape = SHAPES[name] if ":" not in name else reduced(name.split(":")[0], int(name.split(":")[1]))
    if P == 1:
        gp = F.Pipeline(shape, max_ctx=max_ctx, max_seg=16, sampling=sampling)
        stages = [gp]
    else:
        gp = F.LocalPipeline(shape, P, max_ctx=max_ctx, max_seg=16, sampling=sampling)
        stages = gp.stages
    gp.fs_load_random_weights(SEED)
    gp.enable_logits()
    lps = [st.state()["layer_end"] - st.state()["layer_begin"] for st in stages]
    op = OraclePipeline(shape, SEED, n_stages=P, layers_per_stage=lps, max_slots=max_ctx)
    return F, torch, shape, gp, stages, op


@pytest.mark.parametrize("name,P,tol,flag", [("tiny", 1, 1e-4, 1e-3), ("tiny", 2, 1e-4, 1e-3),
                                             ("small", 1, 2e-2, 5e-2), ("smallq:4", 2, 2e-2, 5e-2)])
def test_stochastic_lockstep(name, P, tol, flag):
    F, torch, shape, gp, stages, op = _setup(name, P)
    prefix = gen.prefix_tokens(SEED, 32, shape.vocab)
    op.set_prefix(prefix)
    xg = gp.fs_set_prefix(prefix)
    assert xg == op.x_new
    n_nodes = 15 if name == "tiny" else 40
    decisions = flagged = overrides = rejects_at_root = 0
    for r in range(8):
        stream = op.greedy_stream(5)
        t = gen.planted_tree(SEED + r, n_nodes, 5, stream, (0, 1, 2, 9) if name == "tiny"
                             else (0, 2, 5, 17, 21), shape.vocab)
        q = _draft_q(t, shape.vocab, 64, SEED + r)
        qd = torch.from_numpy(q).cuda()
        seed = 1000 + r
        gp.fs_set_acceptance(F.FS_ACCEPT_STOCHASTIC, 1.0, seed, qd)
        op.submit(True, t["parent"], t["token"], t["own"], l_max=8)
        gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 8)
        while True:
            og = gp.fs_verify_step()
            oo = op.verify_step()
            assert og["seg_id"] == oo["seg_id"] and og["n_rows"] == oo["n_rows"]
            if oo["n_rows"]:
                err = float(np.max(np.abs(og["logits"] - oo["logits"])))
                assert err <= tol, err
            dg = gp.decision_dict(gp.fs_accept())
            do = op.accept_stochastic(lambda nid: q[nid], 1.0, seed, flag=flag)
            if not do["progress"]:
                assert not dg["progress"]
                continue
            decisions += 1
            want = dict(acc_ids=do["acc_ids"], acc_tokens=do["acc_tokens"], x_new=do["x_new"],
                        n_new_id=do["n_new_id"], cont=do["cont"])
            got = {k: dg[k] for k in want}
            flagged += len(do["flagged"])
            if got != want:
                walked = set(do["acc_ids"]) | set(dg["acc_ids"])
                assert walked & set(do["flagged"]), ("decision", r, got, want, do["flagged"])
                overrides += 1
            if len(want["acc_ids"]) == 1 and not want["cont"]:
                rejects_at_root += 1
            gp.fs_prune_and_compact(want)
            op.prune(want)
            for st in stages:
                compare_tree(st, op, st.cfg.max_live // 32, f"r{r}")
            if not want["cont"]:
                break
        gp.fs_set_acceptance(F.FS_ACCEPT_GREEDY)
    print(f"{name} P={P}: decisions {decisions} flagged {flagged} overrides {overrides} "
          f"root rejections {rejects_at_root}")
    assert decisions >= 8
    gp.close()


def test_stochastic_law_equals_base_distribution():
    """Losslessness on the GPU: root + 3 children drawn from
    q without replacement; over 3000 seeds the first committed token after the
    root (accepted child or residual sample) follows p_root = softmax of the
    oracle's root logits, not q."""
    F, torch, shape, gp, stages, op = _setup("tiny", 1)
    prefix = gen.prefix_tokens(SEED, 32, shape.vocab)
    x0 = op.set_prefix(prefix)
    assert gp.fs_set_prefix(prefix) == x0
    V = shape.vocab
    rng = gen.Rng(99)
    z = np.array([rng.uniform() for _ in range(V)])
    qrow = np.exp(3.0 * z)
    qrow /= qrow.sum()
    # p_root from the oracle: verify a root-only tree
    op.submit(True, [-1], [x0], [1.0], l_max=1)
    p_root = None
    oo = op.verify_step()
    from oracle import sampling as SM
    p_root = SM.softmax(oo["logits"][0], 1.0)
    counts = np.zeros(V)
    n_trials = 3000
    qd = torch.from_numpy(np.tile(qrow.astype(np.float32), (8, 1))).cuda()
    for trial in range(n_trials):
        kids, qq = [], qrow.copy()
        r2 = np.random.default_rng(trial)
        for _ in range(3):
            t = int(r2.choice(V, p=qq / qq.sum()))
            kids.append(t)
            qq[t] = 0.0
        gp.fs_set_prefix(prefix)
        gp.fs_set_acceptance(F.FS_ACCEPT_STOCHASTIC, 1.0, 5000 + trial, qd)
        gp.fs_submit_segment(F.FS_NEW_ROUND, [-1, 0, 0, 0], [x0] + kids, [1.0, 0.9, 0.8, 0.7], 4)
        while True:
            gp.fs_verify_step()
            d = gp.decision_dict(gp.fs_accept())
            if d["progress"]:
                break
        tok = d["acc_tokens"][1] if len(d["acc_tokens"]) > 1 else d["x_new"]
        counts[tok] += 1
        gp.fs_prune_and_compact(d)
        if d["cont"]:   # an accepted child is verified here, so the walk exits below it
            raise AssertionError("unexpected continue")
        gp.fs_set_acceptance(F.FS_ACCEPT_GREEDY)
    law = counts / n_trials
    tv_p = 0.5 * np.abs(law - p_root).sum()
    tv_q = 0.5 * np.abs(law - qrow).sum()
    # null distribution of the TV of n_trials exact draws from p_root
    nr = np.random.default_rng(1)
    null = np.sort([0.5 * np.abs(nr.multinomial(n_trials, p_root) / n_trials - p_root).sum()
                    for _ in range(400)])
    q995 = null[int(0.995 * len(null))]
    print(f"TV(law, p) {tv_p:.4f} (null median {null[200]:.4f}, 99.5% {q995:.4f})  TV(law, q) {tv_q:.4f}")
    assert tv_p <= q995 and tv_q > 5 * q995
    gp.close()
