import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
import bench
shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "small"]
gp = F.Pipeline(shape, max_ctx=2048, max_seg=16)
gp.fs_load_random_weights(bench.SEED)
prefix = gen.prefix_tokens(bench.SEED, 64, shape.vocab)
x = gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
print("x_new after prefix", x, gp.state()["x_new"])
for i in range(3):
    gp.fs_submit_segment(F.FS_NEW_ROUND, [-1], [gp.state()["x_new"]], [1.0], 1)
    o = gp.fs_verify_step()
    d = gp.fs_accept()
    print("step", i, "verify", o["seg_id"], o["n_rows"], o["am"], "accept", d.progress, d.n_acc, d.x_new, d.cont)
    gp.fs_prune_and_compact(d)
    print("  state x_new", gp.state()["x_new"])
