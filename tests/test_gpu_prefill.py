"""f3: chunked prefill at the prefill row width
(cfg.max_prefill rows per chunk: GEMM N = 2 x 32/64) pipelined over the stages
(stage p runs chunk t - p at step t), against the oracle's plain causal
prefill: the first sampled token, the KV rows of every prefix slot checked
at sampled positions, and the tree rounds that follow in lockstep."""
import numpy as np
import pytest

from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES, reduced
from tests.lockstep import planted_trees, run_lockstep

pytestmark = pytest.mark.gpu
SEED = 0x5EED01


@pytest.mark.parametrize("name,P,max_prefill,n_pre", [("tiny", 2, 64, 150), ("small", 1, 64, 200),
                                                      ("smallq:4", 2, 32, 150), ("small:4", 4, 64, 333),
                                                      ("72b_l2", 2, 64, 130)])
def test_chunked_prefill_matches_oracle(name, P, max_prefill, n_pre):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    shape = SHAPES[name] if ":" not in name else reduced(name.split(":")[0], int(name.split(":")[1]))
    kw = dict(max_ctx=1024, max_seg=16, max_prefill=max_prefill)
    if P == 1:
        gp = F.Pipeline(shape, **kw)
        stages = [gp]
    else:
        gp = F.LocalPipeline(shape, P, **kw)
        stages = gp.stages
    gp.fs_load_random_weights(SEED)
    gp.enable_logits()
    lps = [st.state()["layer_end"] - st.state()["layer_begin"] for st in stages]
    op = OraclePipeline(shape, SEED, n_stages=P, layers_per_stage=lps, max_slots=1024)
    prefix = gen.prefix_tokens(SEED + 5, n_pre, shape.vocab)
    xo = op.set_prefix(prefix)
    xg = gp.fs_set_prefix(prefix)
    srt = np.sort(op.prefix_logits)
    assert xg == xo or srt[-1] - srt[-2] < 1e-2
    tol = 1e-4 if not shape.bf16 else 2 ** -6
    for st in stages:
        s = st.state()
        for l in range(s["layer_begin"], s["layer_end"]):
            for slot in (0, 1, max_prefill - 1, max_prefill, n_pre // 2, n_pre - 1):
                for w in (0, 1):
                    a = st.read_kv(l, w, shape.n_kv_heads - 1, slot)
                    b = op.kv.get(l, w, shape.n_kv_heads - 1, slot)
                    assert float(np.abs(a - b).max()) <= tol * max(1.0, float(np.abs(b).max())), (l, slot, w)
    n_nodes, planted = (15, (0, 1, 2, 9)) if name == "tiny" else (30, (0, 2, 5, 17, 21))
    st = run_lockstep(gp, op, planted_trees(shape, n_nodes, 5, planted, SEED), n_rounds=2, l_max=8,
                      tol=1e-4 if not shape.bf16 else 2e-2)
    assert st.decisions >= 2
    gp.close()
