import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle.pipeline import OraclePipeline
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
name = sys.argv[1] if len(sys.argv) > 1 else "small"
shape = SHAPES[name]
gp = F.Pipeline(shape, max_ctx=1024, max_seg=16); gp.fs_load_random_weights(0x5EED01); gp.enable_logits()
op = OraclePipeline(shape, 0x5EED01, max_slots=1024)
prefix = gen.prefix_tokens(0x5EED01, 40, shape.vocab)
xg = gp.fs_set_prefix(prefix); xo = op.set_prefix(prefix)
print("x_new gpu", xg, "oracle", xo)
lg = gp.logits[:8].cpu().numpy()   # last chunk = rows 32..39
print("last-row logits max|d|", np.max(np.abs(lg[7] - op.prefix_logits)), "gpu top", np.sort(lg[7])[-3:], "orc top", np.sort(op.prefix_logits)[-3:])
for l in range(shape.n_layers):
  for w in range(2):
    for s in (0, 5, 39):
      a = gp.read_kv(l, w, 0, s); b = op.kv.get(l, w, 0, s)
      print(f"L{l} {'KV'[w]} slot{s}: max|d| {np.max(np.abs(a-b)):.3e} |b| {np.max(np.abs(b)):.3e}  a[:4]={a[:4]} b[:4]={b[:4]}")
