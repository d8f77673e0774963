import sys, numpy as np, dataclasses
sys.path.insert(0, '.')
from oracle.pipeline import OraclePipeline
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES
variants = {
 "small": SHAPES["small"],
 "small_gqa": dataclasses.replace(SHAPES["small"], n_kv_heads=1),
 "small_d1024": dataclasses.replace(SHAPES["small"], d_model=1024),
 "small_h8": dataclasses.replace(SHAPES["small"], n_heads=8, n_kv_heads=8),
}
for name, shape in variants.items():
  for plen, mseg in ((40, 64), (40, 16), (40, 32)):
    gp = F.Pipeline(shape, max_ctx=1024, max_seg=mseg); gp.fs_load_random_weights(0x5EED01)
    op = OraclePipeline(shape, 0x5EED01, max_slots=1024)
    prefix = gen.prefix_tokens(0x5EED01, plen, shape.vocab)
    xg = gp.fs_set_prefix(prefix); xo = op.set_prefix(prefix)
    errs = []
    for s in range(plen):
      a = gp.read_kv(1, 0, 0, s); b = op.kv.get(1, 0, 0, s); errs.append(float(np.max(np.abs(a-b))))
    bad = [s for s in range(plen) if errs[s] > 0.02]
    print(name, plen, mseg, "x", xg, xo, "bad slots", bad[:6], len(bad), "max %.3f" % max(errs))
    gp.close()
