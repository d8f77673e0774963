import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
import bench
shape = SHAPES["7b"]
gp = F.Pipeline(shape, max_ctx=2048, max_seg=16)
gp.fs_load_random_weights(bench.SEED)
prefix = gen.prefix_tokens(bench.SEED, int(sys.argv[1]), shape.vocab)
x = gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
print("x_new after prefix", x, gp.state()["x_new"], flush=True)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    st = gp.state()
    try:
        gp.fs_submit_segment(F.FS_NEW_ROUND, [-1], [st["x_new"]], [1.0], 1)
    except Exception as e:
        print("FAIL at", i, st["x_new"], st["l_glo"], st["live"], st["n_live"], e, flush=True); break
    while True:
        o = gp.fs_verify_step()
        d = gp.fs_accept()
        if d.progress: break
    print("step", i, o["am"], d.x_new, d.cont, flush=True)
    gp.fs_prune_and_compact(d)
