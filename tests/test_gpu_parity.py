"""CUDA path vs oracle, element by element, through the C-ABI (B200 only).

Sizes span several GEMM tiles / attention chunks and ragged tails; full-size
7B checks sample outputs the oracle computes one by one."""
import numpy as np
import pytest

from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES
from tests.lockstep import compare_tree, planted_trees, run_lockstep

pytestmark = pytest.mark.gpu

SEED = 0x5EED01


def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    return F


def _pair(name, P=1, max_ctx=1024, max_seg=16, max_live=512, prefix_len=32, mode="prefill"):
    F = _gpu()
    shape = SHAPES[name]
    gp = F.Pipeline(shape, n_stages=P, max_ctx=max_ctx, max_live=max_live, max_seg=max_seg)
    gp.fs_load_random_weights(SEED)
    gp.enable_logits()
    op = OraclePipeline(shape, SEED, n_stages=P, max_slots=max_ctx)
    prefix = gen.prefix_tokens(SEED, prefix_len, shape.vocab)
    xo = op.set_prefix(prefix, mode="synth" if mode == "synth" else "prefill", kv_seed=7)
    xg = gp.fs_set_prefix(prefix, F.FS_SYNTH_KV if mode == "synth" else F.FS_PREFILL, kv_seed=7)
    return F, shape, gp, op, xo, xg


def test_tiny_fp32_lockstep_rounds():
    """configs[0]: tiny fp32, planted 3-token path, 15-node depth-4 trees, L_max 8."""
    F, shape, gp, op, xo, xg = _pair("tiny")
    assert xg == xo
    st = run_lockstep(gp, op, planted_trees(shape, 15, 4, (0, 1, 2, 9), SEED), n_rounds=8,
                      l_max=8, tol=1e-4)
    assert st.max_abs <= 1e-4
    assert len(st.committed) == 4 * 8  # a+1 tokens per round (scenario R)
    # greedy losslessness (R-def-2)
    ar = OraclePipeline(shape, SEED, max_slots=1024)
    ar.set_prefix(gen.prefix_tokens(SEED, 32, shape.vocab))
    assert st.committed == ar.greedy_stream(len(st.committed))[:len(st.committed)]


@pytest.mark.parametrize("l_max", [1, 3, 5, 16])
def test_tiny_fp32_segmentation_invariance(l_max):
    F, shape, gp, op, xo, xg = _pair("tiny", max_seg=16)
    st = run_lockstep(gp, op, planted_trees(shape, 15, 4, (0, 1, 2, 9), SEED), n_rounds=3,
                      l_max=l_max, tol=1e-4)
    assert len(st.committed) == 12


def test_tiny_random_trees_exercise_ties_and_prunes():
    F, shape, gp, op, xo, xg = _pair("tiny")

    def trees(r, op_):
        return gen.random_tree(100 + r, 40, 6, shape.vocab, op_.x_new)

    st = run_lockstep(gp, op, trees, n_rounds=6, l_max=7, tol=1e-4)
    assert st.decisions >= 6


@pytest.mark.parametrize("name", ["small", "smallq"])
def test_bf16_small_lockstep(name):
    """bf16 path (tcgen05 GEMMs, tensor-core attention), head_dim 128, MHA and
    GQA+bias, several tiles and a ragged tail."""
    F, shape, gp, op, xo, xg = _pair(name, max_ctx=1024, prefix_len=40)
    st = run_lockstep(gp, op, planted_trees(shape, 30, 5, (0, 2, 5, 17, 21), SEED), n_rounds=3,
                      l_max=16, tol=2e-2)
    assert st.max_abs <= 2e-2
    print(f"{name}: max|dlogit| {st.max_abs:.3e} rows {st.rows} flagged {st.flagged} "
          f"overrides {st.overrides}")


def test_bf16_synth_prefix_and_kv_rows():
    F, shape, gp, op, xo, xg = _pair("small", max_ctx=1024, prefix_len=300, mode="synth")
    assert op.prefix_logits is not None
    # synthetic KV rows are bit-identical (same counter generator, bf16 RNE)
    for (l, w, h, s) in [(0, 0, 0, 0), (1, 1, 3, 298), (0, 1, 2, 17)]:
        assert np.array_equal(gp.read_kv(l, w, h, s), op.kv.get(l, w, h, s))
    # the real last-token pass: K/V of slot n-1 within bf16 rounding
    for l in range(2):
        a, b = gp.read_kv(l, 0, 1, 299), op.kv.get(l, 0, 1, 299)
        assert np.max(np.abs(a - b)) <= 2 ** -7 * max(1.0, np.max(np.abs(b)))
    st = run_lockstep(gp, op, planted_trees(shape, 40, 6, (0, 2, 5, 17, 21), SEED), n_rounds=2,
                      l_max=16, tol=2e-2)
    assert st.max_abs <= 2e-2


def _append_batch(op, rng, n_new, vocab):
    """Random APPEND batch (a16): parents are live nodes or earlier
    batch nodes; sibling tokens unique; own scores in (0, 1]."""
    live = list(op.node)
    kids = {}
    for s in range(len(op.node)):
        if op.par[s] >= 0:
            kids.setdefault(op.node[op.par[s]], set()).add(op.tok[s])
    base = op.next_id
    parent, token, own = [], [], []
    for i in range(n_new):
        cand = live + [base + j for j in range(i)]
        p = cand[rng.below(len(cand))]
        while True:
            t = rng.below(vocab)
            if t not in kids.setdefault(p, set()):
                break
        kids[p].add(t)
        parent.append(p)
        token.append(t)
        own.append(np.float32(0.05 + 0.95 * rng.uniform()))
    return parent, token, own


def test_tiny_bfs_order_lockstep_and_strategy_independence():
    """f1 ablation: breadth-first submit order (FS_ORDER_BFS) is bit-exact with the
    oracle, and commits the same greedy stream as score order (SPEC strategy
    independence; R-def-2)."""
    F, shape, gp, op, xo, xg = _pair("tiny")
    st_b = run_lockstep(gp, op, planted_trees(shape, 15, 4, (0, 1, 2, 9), SEED), n_rounds=4,
                        l_max=5, tol=1e-4, bfs=True)
    F, shape, gp, op, xo, xg = _pair("tiny")
    st_s = run_lockstep(gp, op, planted_trees(shape, 15, 4, (0, 1, 2, 9), SEED), n_rounds=4,
                        l_max=5, tol=1e-4)
    assert st_b.committed == st_s.committed and len(st_s.committed) == 16


@pytest.mark.parametrize("name,P_l", [("tiny", 4), ("small", 8)])
def test_lockstep_with_appended_batches(name, P_l):
    """Expansion input (a16): after every progress-free tick or mid-round prune
    a batch is appended (S_mer = S_pr || S_app, own segments)."""
    F, shape, gp, op, xo, xg = _pair(name, max_ctx=1024, prefix_len=24)
    rng = gen.Rng(77)
    appended = [0]

    def append(r, ticks, gp_, op_):
        if not op_.live or len(op_.node) + 6 > 200 or appended[0] >= 12:
            return
        parent, token, own = _append_batch(op_, rng, 6, shape.vocab)
        so = op_.submit(False, parent, token, own, l_max=P_l)
        sg = gp_.fs_submit_segment(F.FS_APPEND, parent, token, own, P_l)
        assert sg["order"] == so["order"] and sg["bounds"] == [tuple(b) for b in so["bounds"]]
        appended[0] += 1

    st = run_lockstep(gp, op, planted_trees(shape, 20, 5, (0, 1, 3, 9), SEED), n_rounds=4,
                      l_max=P_l, tol=1e-4 if not shape.bf16 else 2e-2, append_fn=append)
    assert appended[0] > 0


def test_error_codes_leave_state_unchanged():
    F, shape, gp, op, xo, xg = _pair("tiny")

    def state():
        s = gp.state()
        s.pop("launches")
        return s

    before = state()

    def rc(f, *a):
        try:
            f(*a)
        except F.FlowSpecError as e:
            return e.code
        return 0

    x = before["x_new"]
    # root token != x_new, non-topological parent, duplicate siblings, own outside (0,1]
    assert rc(gp.fs_submit_segment, F.FS_NEW_ROUND, [-1, 0], [x + 1, 3], [1.0, 0.5], 4) == F.FS_EINVAL
    assert rc(gp.fs_submit_segment, F.FS_NEW_ROUND, [-1, 2, 0], [x, 3, 4], [1.0, 0.5, 0.5], 4) == F.FS_EINVAL
    assert rc(gp.fs_submit_segment, F.FS_NEW_ROUND, [-1, 0, 0], [x, 3, 3], [1.0, 0.5, 0.5], 4) == F.FS_EINVAL
    assert rc(gp.fs_submit_segment, F.FS_NEW_ROUND, [-1, 0], [x, 3], [1.0, 1.5], 4) == F.FS_EINVAL
    assert rc(gp.fs_submit_segment, F.FS_NEW_ROUND, [-1, 0], [x, 3], [1.0, 0.5], 0) == F.FS_EINVAL
    assert rc(gp.fs_submit_segment, F.FS_APPEND, [0], [3], [0.5], 4) == F.FS_ESTATE
    assert state() == before
    # a valid round; then NEW_ROUND while live, APPEND with a pruned/unknown parent
    gp.fs_submit_segment(F.FS_NEW_ROUND, [-1, 0, 0], [x, 3, 4], [1.0, 0.5, 0.4], 4)
    assert rc(gp.fs_submit_segment, F.FS_NEW_ROUND, [-1], [x], [1.0], 4) == F.FS_ESTATE
    assert rc(gp.fs_submit_segment, F.FS_APPEND, [99], [5], [0.5], 4) == F.FS_EINVAL
    # inconsistent decisions are rejected without touching the state
    s1 = state()
    assert rc(gp.fs_prune_and_compact, dict(acc_ids=[1], x_new=0, n_new_id=-1, cont=0)) == F.FS_ESTATE
    assert rc(gp.fs_prune_and_compact, dict(acc_ids=[0], x_new=0, n_new_id=7, cont=1)) == F.FS_ESTATE
    assert state() == s1
    o = gp.fs_verify_step()
    assert o["n_rows"] == 3


@pytest.mark.parametrize("name", ["small", "smallq"])
def test_bf16_wide_segments_lockstep(name):
    """max_seg = FS_MAX_SEG (64): the N = 64 GEMM configuration (one CTA per SM,
    its own split planning), 64-row prefill chunks, and a 60-node tree verified
    as one segment (ragged against the 64-row tile) next to 64-row segments."""
    F, shape, gp, op, xo, xg = _pair(name, max_ctx=1024, max_seg=64, prefix_len=150)
    st = run_lockstep(gp, op, planted_trees(shape, 60, 5, (0, 2, 5, 17, 21), SEED), n_rounds=2,
                      l_max=64, tol=2e-2)
    assert st.max_abs <= 2e-2
    print(f"{name} wide: max|dlogit| {st.max_abs:.3e} rows {st.rows} flagged {st.flagged} "
          f"overrides {st.overrides}")


def test_tiny_capacity_tree_max_live():
    """A 500-node tree against max_live = 512: submit (score order, 16-word
    ancestor bitsets), segment scheduling and prune at capacity, in lockstep."""
    F, shape, gp, op, xo, xg = _pair("tiny", max_ctx=1024, max_live=512)
    st = run_lockstep(gp, op, planted_trees(shape, 500, 9, (0, 3, 40, 170, 333, 401), SEED), n_rounds=1,
                      l_max=16, tol=1e-4)
    assert st.max_abs <= 1e-4
    print(f"tiny capacity: max|dlogit| {st.max_abs:.3e} rows {st.rows} decisions {st.decisions}")


@pytest.mark.parametrize("name", ["small", "smallq"])
def test_mha_tma_kernel_short_context(name, monkeypatch):
    """The TMA-ring MHA kernel (k_attn_mha.cuh) normally runs only above 2048
    keys; forced here on short contexts (ragged last sub-chunk, empty splits)."""
    monkeypatch.setenv("FS_MHA_TMA", "1")
    F, shape, gp, op, xo, xg = _pair(name, max_ctx=1024, prefix_len=40)
    st = run_lockstep(gp, op, planted_trees(shape, 30, 5, (0, 2, 5, 17, 21), SEED), n_rounds=2,
                      l_max=16, tol=2e-2)
    assert st.max_abs <= 2e-2


def test_async_submit_lockstep_and_deferred_error():
    """FS_SUBMIT_ASYNC: the same rounds without waiting for the device at
    submit (bench.py's timed path); a batch the device rejects poisons the
    context at the next verify step instead of corrupting it."""
    F, shape, gp, op, xo, xg = _pair("small", max_ctx=1024, prefix_len=40)
    trees = planted_trees(shape, 30, 5, (0, 2, 5, 17, 21), SEED)
    for r in range(2):
        t = trees(r, op)
        so = op.submit(True, t["parent"], t["token"], t["own"], l_max=16)
        sg = gp.fs_submit_segment(F.FS_NEW_ROUND | F.FS_SUBMIT_ASYNC, t["parent"], t["token"], t["own"], 16)
        assert sg["bounds"] == [tuple(b) for b in so["bounds"]]
        compare_tree(gp, op, gp.cfg.max_live // 32, f"async submit r{r}")
        while True:
            og, oo = gp.fs_verify_step(), op.verify_step()
            assert og["node"] == oo["node"]
            dg, do = gp.decision_dict(gp.fs_accept()), op.accept()
            if not do["progress"]:
                continue
            want = dict(acc_ids=do["acc_ids"], x_new=do["x_new"], n_new_id=do["n_new_id"], cont=do["cont"])
            gp.fs_prune_and_compact(want)
            op.prune(want)
            if not do["cont"]:
                break
    # duplicate sibling token: rejected on the device, surfaces at the next verify
    x = gp.state()["x_new"]
    gp.fs_submit_segment(F.FS_NEW_ROUND | F.FS_SUBMIT_ASYNC, [-1, 0, 0], [x, 5, 5], [1.0, 0.5, 0.4], 16)
    with pytest.raises(F.FlowSpecError):
        gp.fs_verify_step()
    with pytest.raises(F.FlowSpecError) as e:
        gp.fs_accept()
    assert e.value.code == F.FS_EPOISONED
