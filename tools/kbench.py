import os, sys, json
# timeline kinds 8-10 need a diagnostic build: FS_NVCC_FLAGS=-DFS_DIAG python -m paper_2507_02620_b200.build --force
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
name = sys.argv[1] if len(sys.argv) > 1 else "7b"
shape = SHAPES[name]
gp = F.Pipeline(shape, max_ctx=2048, max_seg=16)
gp.fs_load_random_weights(1)
prefix = gen.prefix_tokens(1, 1024, shape.vocab)
gp.fs_set_prefix(prefix[:1009], F.FS_SYNTH_KV, kv_seed=7)   # leaves a 16-row tick? no: 1 row
# run a 16-row prefill chunk so the tick rows hold 16 rows
gp.fs_set_prefix(prefix[:1024], F.FS_PREFILL) if "--prefill" in sys.argv else None
names = ["qkv", "o", "gate_up", "down", "head", "attn(layer)", "rmsnorm", "stage"]
for k in range(8):
    for it in (1, 50):
        us, by = gp.bench_kernel(k, it)
    print(f"{names[k]:12s} {us:9.2f} us  {by/1e6:8.2f} MB  {by/us/1e3 if us else 0:8.1f} GB/s")
us, _ = gp.bench_kernel(8, 1)
print("timeline stage span us", us)
if "--attn" in sys.argv:
    gp.bench_kernel(9, 1)
if "--ogemm" in sys.argv:
    gp.bench_kernel(10, 1)
