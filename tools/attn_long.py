"""Attention HBM bandwidth at the long-context configs (configs[3]
# timeline kinds 8-10 need a diagnostic build: FS_NVCC_FLAGS=-DFS_DIAG python -m paper_2507_02620_b200.build --force
13B with a 4096-token context, configs[4] 72B GQA with a 16384-token context),
on the full per-layer shapes with synthetic-KV prefixes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES, reduced

cases = [("7b", 1024, 16), ("13b", 4096, 16), ("72b", 16384, 32)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]] or cases
for name, ctx, seg in cases:
    shape = reduced(name, 1)
    gp = F.Pipeline(shape, max_ctx=ctx + 512, max_seg=seg)
    gp.fs_load_random_weights(1)
    prefix = gen.prefix_tokens(1, ctx, shape.vocab)
    gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
    # one full segment of tree rows so the tick has seg rows
    tree = gen.random_tree(3, seg, 6, shape.vocab, gp.state()["x_new"])
    gp.fs_submit_segment(F.FS_NEW_ROUND, tree["parent"], tree["token"], tree["own"], seg)
    gp.fs_verify_step()
    best = None
    for rep in range(5):
        us, by = gp.bench_kernel(5, 50)
        best = (us, by) if best is None or us < best[0] else best
    us, by = best
    print(f"{name}: ctx {ctx} rows {seg}: attention {us:8.2f} us/layer  {by/1e6:7.2f} MB  {by/us/1e3:7.1f} GB/s",
          flush=True)
    if "--probe" in sys.argv:
        gp.bench_kernel(9, 1)
    del gp
