"""Per-layer shapes of BASELINE.json configs[3] (13B) and configs[4] (Qwen2-72B:
GQA 64/8, q/k/v bias, 32-row segments, long synthetic-KV context) with two
layers, in lockstep with the oracle (every S order / mask / prune / KV slot map
bit-exact, logits within 2e-2, accepted tokens identical except flagged)."""
import numpy as np
import pytest

from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES
from tests.lockstep import planted_trees, run_lockstep

pytestmark = pytest.mark.gpu
SEED = 0x5EED01


def _run(name, prefix_len, mode, max_seg, l_max, n_nodes, depth, planted, max_ctx, n_rounds,
         append_batches=0):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    shape = SHAPES[name]
    gp = F.Pipeline(shape, max_ctx=max_ctx, max_seg=max_seg)
    gp.fs_load_random_weights(SEED)
    gp.enable_logits()
    op = OraclePipeline(shape, SEED, max_slots=max_ctx)
    prefix = gen.prefix_tokens(SEED, prefix_len, shape.vocab)
    xo = op.set_prefix(prefix, mode=mode, kv_seed=7)
    xg = gp.fs_set_prefix(prefix, F.FS_SYNTH_KV if mode == "synth" else F.FS_PREFILL, kv_seed=7)
    srt = np.sort(op.prefix_logits)
    assert xg == xo or srt[-1] - srt[-2] < 1e-2
    append_fn = None
    appended = [0]
    if append_batches:
        from tests.test_gpu_parity import _append_batch
        rng = gen.Rng(91)

        def append_fn(r, ticks, gp_, op_):
            # steady expansion (configs[3], scenario S): a 16-node batch, its own
            # segment (L_exp = -1), after every tick while the round is live
            if not op_.live or appended[0] >= append_batches or len(op_.node) + 16 > 480:
                return
            parent, token, own = _append_batch(op_, rng, 16, shape.vocab)
            so = op_.submit(False, parent, token, own, l_max=16)
            sg = gp_.fs_submit_segment(F.FS_APPEND, parent, token, own, 16)
            assert sg["order"] == so["order"] and sg["bounds"] == [tuple(b) for b in so["bounds"]]
            appended[0] += 1

    st = run_lockstep(gp, op, planted_trees(shape, n_nodes, depth, planted, SEED), n_rounds=n_rounds,
                      l_max=l_max, tol=2e-2, append_fn=append_fn)
    if append_batches:
        assert appended[0] > 0
    print(f"{name}: max|dlogit| {st.max_abs:.3e} rows {st.rows} flagged {st.flagged} "
          f"overrides {st.overrides} committed {len(st.committed)}")
    return st


def test_13b_layers_expansion_shapes():
    """configs[3] per-layer shapes (d 5120, 40 heads, ffn 13824), 16-row segments."""
    _run("13b_l2", 300, "synth", 16, 16, 64, 6, (0, 2, 5, 17, 21), 1024, 2)


def test_13b_config4_long_context_steady_expansion():
    """configs[3] scenario on the per-layer shapes: 4096-token synthetic-KV
    context, 128-node initial trees, appended 16-node batches (own segments)
    while the round is live."""
    _run("13b_l2", 4096, "synth", 16, 16, 128, 6, (0, 2, 5, 17, 21, 40), 4800, 2, append_batches=6)


def test_72b_layers_gqa_bias_32row_segments_long_context():
    """configs[4] per-layer shapes: GQA 64/8 (8 query heads per KV head packed into
    M = 8 x 32 rows), q/k/v bias, 32-row segments (UMMA N = 64), 16K-token
    synthetic-KV context (130 attention chunks), 256-node trees."""
    _run("72b_l2", 16384, "synth", 32, 32, 256, 8, (0, 3, 9, 40, 47, 70, 90, 100, 120), 17408, 1)


def test_72b_gqa_online_softmax_rescale_path(monkeypatch):
    """The GQA kernel's lazy online-softmax rescale (running max raised, O rows
    rescaled in TMEM) normally triggers only on a > 2^8 jump of the row max;
    threshold 0 forces it at every increase of the max, so the path is checked
    against the oracle on the configs[4] per-layer shapes."""
    monkeypatch.setenv("FS_TCA_RESCALE", "0")
    _run("72b_l2", 16384, "synth", 32, 32, 256, 8, (0, 3, 9, 40, 47, 70, 90, 100, 120), 17408, 1)


def test_72b_gqa_f16_p_path(monkeypatch):
    """The fp16-P variant of the GQA kernel (V converted to fp16 in shared memory
    by the softmax warps, one P.V MMA; opt-in FS_TC_ATTN_P=f16) is parity-green
    on the configs[4] per-layer shapes."""
    monkeypatch.setenv("FS_TC_ATTN_P", "f16")
    _run("72b_l2", 16384, "synth", 32, 32, 256, 8, (0, 3, 9, 40, 47, 70, 90, 100, 120), 17408, 1)


@pytest.mark.parametrize("name,seg,env,fails", [
    ("72b_l2", 32, {"FS_TC_ATTN_P": "f16"}, True),     # GQA tcgen05 kernel, fp16 P (opt-in)
    ("72b_l2", 32, {}, False),                         # GQA, bf16 hi/lo P (default): reads bf16 V directly
    ("7b_l2", 16, {}, True),                           # MHA cluster kernel, fp16 P.V fragments
    ("7b_l2", 16, {"FS_MHA_TMA": "1"}, True),          # MHA TMA-ring kernel
])
def test_fp16_pv_v_range_fails_loudly(monkeypatch, name, seg, env, fails):
    """The fp16 P.V paths (the MHA kernels; the GQA kernel with
    FS_TC_ATTN_P=f16) convert V (bf16) to fp16 on chip: a V row outside fp16's
    range (|v| >= 65536) must fail the verify step with FS_ERANGE (and poison
    the context), never produce a silent inf; the default GQA hi/lo variant
    reads bf16 V directly and accepts the same row."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    shape = SHAPES[name]
    gp = F.Pipeline(shape, max_ctx=1024, max_seg=seg)
    gp.fs_load_random_weights(SEED)
    prefix = gen.prefix_tokens(SEED, 300, shape.vocab)
    gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
    kvh = min(3, shape.n_kv_heads - 1)
    row = gp.read_kv(0, 1, kvh, 17)
    row[5] = 1.0e5
    gp.debug_write_kv(0, 1, kvh, 17, row)
    assert gp.read_kv(0, 1, kvh, 17)[5] > 65536
    tree = gen.random_tree(3, seg, 6, shape.vocab, gp.state()["x_new"])
    gp.fs_submit_segment(F.FS_NEW_ROUND, tree["parent"], tree["token"], tree["own"], seg)
    if not fails:
        assert gp.fs_verify_step()["n_rows"] == seg
        return
    with pytest.raises(F.FlowSpecError) as e:
        gp.fs_verify_step()
    assert e.value.code == F.FS_ERANGE
    with pytest.raises(F.FlowSpecError) as e:
        gp.fs_verify_step()
    assert e.value.code == F.FS_EPOISONED


def test_gqa_many_splits_combine_batches():
    """smallq (GQA 8/2) with 32-row segments runs the tcgen05 GQA kernel with
    one split per 2 SMs of a kv head, capped by the workspace: at max_ctx 2048
    that is 64 splits, so the warp combine merges two 32-split batches (the
    running maximum raised between batches) and most splits are empty (neutral
    partials).  Lockstep with the oracle."""
    _run("smallq", 1400, "synth", 32, 32, 96, 6, (0, 2, 5, 17, 21, 40), 2048, 2)
