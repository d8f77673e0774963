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
