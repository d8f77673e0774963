import sys, numpy as np
sys.path.insert(0, '.')
from oracle.pipeline import OraclePipeline
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
name = sys.argv[1] if len(sys.argv) > 1 else "7b_l2"
shape = SHAPES[name]
gp = F.Pipeline(shape, max_ctx=1024, max_seg=16); gp.fs_load_random_weights(0x5EED01); gp.enable_logits()
op = OraclePipeline(shape, 0x5EED01, max_slots=1024)
prefix = gen.prefix_tokens(0x5EED01, 40, shape.vocab)
xg = gp.fs_set_prefix(prefix); xo = op.set_prefix(prefix)
lg = gp.logits[:8].cpu().numpy()
d = lg[7] - op.prefix_logits
print("x_new", xg, xo, "last-row logits max|d| %.3e  std %.3e" % (np.abs(d).max(), d.std()))
for l in range(shape.n_layers):
  for w in range(2):
    diffs = []; nd = 0; tot = 0
    for s in range(40):
      for h in range(0, shape.n_kv_heads, max(1, shape.n_kv_heads // 4)):
        a = gp.read_kv(l, w, h, s); b = op.kv.get(l, w, h, s)
        diffs.append(np.abs(a - b).max()); nd += int((a != b).sum()); tot += a.size
    print(f"L{l} {'KV'[w]}: max|d| {max(diffs):.3e}  differing elems {nd}/{tot} ({nd/tot:.2%})")
