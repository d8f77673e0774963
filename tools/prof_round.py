"""One SD round of the bench workload between cudaProfilerStart/Stop (for ncu
--profile-from-start off).  Synthetic-KV prefix for a fast setup."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
import bench

shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "7b"]
ranks = (0, 2, 5, 17, 21)
gp = F.Pipeline(shape, max_ctx=2048, max_seg=16)
gp.fs_load_random_weights(bench.SEED)
prefix = gen.prefix_tokens(bench.SEED, 1024, shape.vocab)
gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
stream = bench.greedy_stream(gp, 3 * 5 + 6)
gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
trees = [gen.planted_tree(bench.SEED + r, 64, 6, stream[r * 5: r * 5 + 6], ranks, shape.vocab) for r in range(3)]
bench.run_round(gp, trees[0], 16)
bench.run_round(gp, trees[1], 16)
torch.cuda.synchronize()
torch.cuda.profiler.start()
c, t = bench.run_round(gp, trees[2], 16)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("round committed", c, "ticks", t)
