"""Multi-stage pipelines on ONE GPU (SURVEY §4 tier T3, §8(e)): P stage contexts
in one process joined by an fs_local_group (include/flowspec.h), so the stage
handoff (a10), in-flight row compaction (rows_compact_kernel, a14), pipeline
bubbles (R9) and the replicated prune on every stage run in the driver's 1-GPU
test pass.  Lockstep with the oracle pipeline of the same P (tests/lockstep.py):
every stage's replicated tree / schedule bit-exact, logits within the bar, KV
rows byte-identical across every fs_prune_and_compact (SURVEY §8(c)
"Compaction"), and the same committed stream at every P."""
import numpy as np
import pytest

from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES, reduced
from tests.lockstep import compare_tree, planted_trees, run_lockstep

pytestmark = pytest.mark.gpu
SEED = 0x5EED01


def _shape(name):
    if ":" in name:
        base, n = name.split(":")
        return reduced(base, int(n))
    return SHAPES[name]


def _local(name, P, max_ctx=1024, max_seg=16, prefix_len=40, mode="prefill"):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    shape = _shape(name)
    if P == 1:
        gp = F.Pipeline(shape, max_ctx=max_ctx, max_seg=max_seg)
        stages = [gp]
    else:
        gp = F.LocalPipeline(shape, P, max_ctx=max_ctx, max_seg=max_seg)
        stages = gp.stages
    gp.fs_load_random_weights(SEED)
    gp.enable_logits()
    lps = [st.state()["layer_end"] - st.state()["layer_begin"] for st in stages]
    op = OraclePipeline(shape, SEED, n_stages=P, layers_per_stage=lps, max_slots=max_ctx)
    prefix = gen.prefix_tokens(SEED, prefix_len, shape.vocab)
    xo = op.set_prefix(prefix, mode=mode, kv_seed=7)
    xg = gp.fs_set_prefix(prefix, F.FS_SYNTH_KV if mode == "synth" else F.FS_PREFILL, kv_seed=7)
    srt = np.sort(op.prefix_logits)
    assert xg == xo or srt[-1] - srt[-2] < 1e-2
    return F, shape, gp, stages, op


def _every_stage(stages):
    """After every prune: each stage's replica of the tree and schedule equals
    the oracle's ("local replicas of T")."""
    def check(gp, op):
        for st in stages:
            compare_tree(st, op, st.cfg.max_live // 32, f"stage {st.state()['rank']}")
    return check


@pytest.mark.parametrize("P", [1, 2])
def test_tiny_config1_two_stages(P):
    """configs[0]: tiny fp32, 2 stages, 32-token prefix, 15-node depth-4 trees,
    L_max 8 (segments 8 + 7), planted 3-token path: mid-flight prune of the
    in-flight segment at stage 0 and exit; same stream at P = 1 and 2."""
    F, shape, gp, stages, op = _local("tiny", P, prefix_len=32)
    st = run_lockstep(gp, op, planted_trees(shape, 15, 4, (0, 1, 2, 9), SEED), n_rounds=6, l_max=8,
                      tol=1e-4, check_kv=_every_stage(stages), kv_identity=stages)
    assert len(st.committed) == 4 * 6 and st.kv_rows_checked > 0
    ar = OraclePipeline(shape, SEED, max_slots=1024)
    ar.set_prefix(gen.prefix_tokens(SEED, 32, shape.vocab))
    assert st.committed == ar.greedy_stream(len(st.committed))[:len(st.committed)]
    gp.close()


@pytest.mark.parametrize("P,l_max", [(2, 3), (3, 5), (4, 2)])
def test_tiny_random_trees_bubbles(P, l_max):
    """Random 40-node trees with short segments: in-flight segments that prune
    to empty stay as bubbles (R9), queued ones are dropped, rows of in-flight
    segments are compacted at every stage > 0."""
    F, shape, gp, stages, op = _local("tiny" if P <= 2 else "tiny:4", P, prefix_len=24)

    def trees(r, op_):
        return gen.random_tree(300 + r, 40, 6, shape.vocab, op_.x_new)

    st = run_lockstep(gp, op, trees, n_rounds=5, l_max=l_max, tol=1e-4,
                      check_kv=_every_stage(stages), kv_identity=stages)
    assert st.decisions >= 5
    gp.close()


@pytest.mark.parametrize("name,P", [("small", 2), ("smallq", 2), ("small:4", 4), ("smallq:4", 4),
                                    ("small:8", 8)])
def test_bf16_local_pipeline_lockstep(name, P):
    """bf16 path (tcgen05 GEMMs, MHA and GQA+bias attention) split over P stages
    on one GPU, planted paths over several segments (mid-flight prunes)."""
    F, shape, gp, stages, op = _local(name, P)
    st = run_lockstep(gp, op, planted_trees(shape, 40, 6, (0, 2, 5, 17, 21, 33), SEED), n_rounds=3,
                      l_max=8, tol=2e-2, check_kv=_every_stage(stages), kv_identity=stages)
    assert st.max_abs <= 2e-2 and st.kv_rows_checked > 0
    print(f"{name} P={P}: max|dlogit| {st.max_abs:.2e} rows {st.rows} flagged {st.flagged} "
          f"kv rows {st.kv_rows_checked}")
    gp.close()


def test_7b_layers_two_stages():
    """configs[2] per-layer shapes (d 4096, 32 heads, ffn 11008), 64-node trees,
    L_max 16, two planted tokens per segment over segments 0-2, 2 stages."""
    F, shape, gp, stages, op = _local("7b_l2", 2, max_ctx=1200, prefix_len=64)
    st = run_lockstep(gp, op, planted_trees(shape, 64, 6, (0, 3, 9, 18, 25, 33, 40), SEED),
                      n_rounds=2, l_max=16, tol=2e-2, check_kv=_every_stage(stages),
                      kv_identity=stages)
    assert st.max_abs <= 2e-2
    gp.close()


def test_72b_layers_two_stages_compaction_stress():
    """configs[4] per-layer shapes (GQA 64/8, bias, 32-row segments) on 2 stages
    with a 16K synthetic-KV context, 256-node trees and the planted path spread
    so that each prune frees most of the cached draft rows (compaction stress)."""
    F, shape, gp, stages, op = _local("72b_l2", 2, max_ctx=17408, max_seg=32, prefix_len=16384,
                                      mode="synth")
    st = run_lockstep(gp, op, planted_trees(shape, 256, 8, (0, 3, 9, 40, 47, 70, 90, 100, 120), SEED),
                      n_rounds=1, l_max=32, tol=2e-2, check_kv=_every_stage(stages),
                      kv_identity=stages)
    assert st.max_abs <= 2e-2 and st.kv_rows_checked > 0
    gp.close()


@pytest.mark.parametrize("name,P,l_top", [("tiny", 2, 9), ("small", 1, 20)])
def test_top_l_selection(name, P, l_top):
    """Top-L_top by cumulative score before segmentation ("select the top
    L nodes"): the kept set is a score prefix, hence ancestor-closed."""
    F, shape, gp, stages, op = _local(name, P)
    n_nodes = 15 if name == "tiny" else 40
    planted = (0, 1, 2, 9) if name == "tiny" else (0, 2, 5, 17, 21, 33)
    st = run_lockstep(gp, op, planted_trees(shape, n_nodes, 5, planted, SEED), n_rounds=3,
                      l_max=4 if name == "tiny" else 8, tol=1e-4 if name == "tiny" else 2e-2,
                      check_kv=_every_stage(stages), kv_identity=stages, l_top=l_top)
    assert st.decisions >= 3
    gp.close()
