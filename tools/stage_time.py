"""Stage-forward time (fs_bench_kernel kind 7) of the 7B configs[1] shape for
the current environment (used for env sweeps: FS_PF_*, FS_SPLIT_*)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
name = sys.argv[1] if len(sys.argv) > 1 else "7b"
shape = SHAPES[name]
gp = F.Pipeline(shape, max_ctx=2048, max_seg=16)
gp.fs_load_random_weights(1)
prefix = gen.prefix_tokens(1, 1024, shape.vocab)
gp.fs_set_prefix(prefix[:1024], F.FS_PREFILL)
best = 1e9
for rep in range(5):
    us, _ = gp.bench_kernel(7, 20)
    best = min(best, us)
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FS_"))
print(f"stage_us {best:9.2f}  {tag}", flush=True)
