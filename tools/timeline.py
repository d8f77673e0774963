"""Per-launch timeline of one non-graph 7B stage forward (fs_bench_kernel kind 8;
needs a diagnostic build: FS_NVCC_FLAGS=-DFS_DIAG python -m paper_2507_02620_b200.build --force).
--wide: at the prefill-chunk width on the last prefill chunk's rows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
args = [a for a in sys.argv[1:] if not a.startswith("--")]
wide = "--wide" in sys.argv
name = args[0] if args else "7b"
shape = SHAPES[name]
gp = F.Pipeline(shape, max_ctx=2048, max_seg=16, max_prefill=64)
gp.fs_load_random_weights(1)
prefix = gen.prefix_tokens(1, 1024, shape.vocab)
gp.fs_set_prefix(prefix[:1024], F.FS_PREFILL)
if not wide:
    tree = gen.random_tree(3, 16, 6, shape.vocab, gp.state()["x_new"])
    gp.fs_submit_segment(F.FS_NEW_ROUND, tree["parent"], tree["token"], tree["own"], 16)
flag = 0x100 if wide else 0
for _ in range(3):
    gp.bench_kernel(7 | flag, 5)
gp.bench_kernel(8 | flag, 1)
