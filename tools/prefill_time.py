"""Chunked prefill (f3) breakdown at the prefill row width: the whole prefill
(CUDA events around fs_set_prefix) and, on the last 64-row chunk, each GEMM
class, the attention and the whole stage forward (fs_bench_kernel kind |
FS_BENCH_WIDE, back-to-back launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES, reduced

name = sys.argv[1] if len(sys.argv) > 1 else "7b"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
mp = int(sys.argv[3]) if len(sys.argv) > 3 else 64
shape = SHAPES[name]
gp = F.Pipeline(shape, max_ctx=n + 600, max_seg=16, max_prefill=mp)
gp.fs_load_random_weights(1)
prefix = gen.prefix_tokens(1, n, shape.vocab)
gp.fs_set_prefix(prefix)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(gp.stream)
gp.fs_set_prefix(prefix)
b.record(gp.stream)
torch.cuda.synchronize()
print(f"{name}: prefill of {n} tokens in {mp}-row chunks: {a.elapsed_time(b):.2f} ms")
for k, nm in ((0, "qkv"), (1, "o"), (2, "gate_up"), (3, "down"), (4, "head"), (5, "attention"), (7, "stage forward")):
    us, by = gp.bench_kernel(k | 0x100, 10)
    print(f"  {nm:14s} {us:9.2f} us  ({by / us / 1e3 if by else 0:7.1f} GB/s)")
