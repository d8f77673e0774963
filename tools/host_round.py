"""Host-side time of every public API call in SD rounds of the bench workload
(where the per-round time beyond the stage forwards goes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
n_rounds = 8
stream = bench.greedy_stream(gp, n_rounds * 5 + 6)
gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
trees = [gen.planted_tree(bench.SEED + r, 64, 6, stream[r * 5: r * 5 + 6], ranks, shape.vocab)
         for r in range(n_rounds)]
acc = {}
def t(name, fn, *a):
    t0 = time.perf_counter()
    r = fn(*a)
    acc.setdefault(name, []).append((time.perf_counter() - t0) * 1e6)
    return r
rounds = []
for r, tree in enumerate(trees):
    t0 = time.perf_counter()
    t("submit", gp.fs_submit_segment, F.FS_NEW_ROUND, tree["parent"], tree["token"], tree["own"], 16)
    while True:
        t("verify_step", gp.fs_verify_step)
        d = t("accept", gp.fs_accept)
        if not d.progress:
            continue
        t("prune", gp.fs_prune_and_compact, d)
        if not d.cont:
            break
    rounds.append((time.perf_counter() - t0) * 1e6)
skip = 2
print("round us:", " ".join(f"{x:.0f}" for x in rounds[skip:]))
for k, v in acc.items():
    v2 = v[len(v) * skip // len(trees):]
    print(f"{k:12s} n={len(v2):3d} mean {sum(v2)/len(v2):8.1f} us  min {min(v2):8.1f}  max {max(v2):8.1f}")
us, _ = gp.bench_kernel(7, 20)
print("stage forward (graph) us", us)
