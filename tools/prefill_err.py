"""Max logit error of the 72B per-layer-shape prefill + tree-verify lockstep
(tests/test_gpu_prefill.py's 72b_l2 case) for the current environment."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_02620_b200 import flowspec as F
from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES
from tests.lockstep import planted_trees, run_lockstep
SEED = 0x5EED01
shape = SHAPES["72b_l2"]
gp = F.LocalPipeline(shape, 2, max_ctx=1024, max_seg=16, max_prefill=64)
gp.fs_load_random_weights(SEED)
gp.enable_logits()
lps = [st.state()["layer_end"] - st.state()["layer_begin"] for st in gp.stages]
op = OraclePipeline(shape, SEED, n_stages=2, layers_per_stage=lps, max_slots=1024)
prefix = gen.prefix_tokens(SEED + 5, 130, shape.vocab)
op.set_prefix(prefix)
gp.fs_set_prefix(prefix)
st = run_lockstep(gp, op, planted_trees(shape, 30, 5, (0, 2, 5, 17, 21), SEED), n_rounds=2, l_max=8, tol=1.0)
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FS_"))
print(f"max|dlogit| {st.max_abs:.5f}  {tag}", flush=True)
gp.close()
