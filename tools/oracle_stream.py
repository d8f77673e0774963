"""Oracle greedy stream artifact for the bench's planted draft trees (SURVEY
§8(d) "Trees (planted path)": the planted chain is the ORACLE's greedy output;
§8(d) "Oracle timing": expensive oracle records are precomputed and stored as
small repo artifacts).  Calls only oracle/ (test infrastructure).

    python tools/oracle_stream.py 7b 1024 320      # -> synth/streams/7b_p1024.json

Runs the oracle's real prefill of the seeded prompt (gen.prefix_tokens), then
greedy autoregressive decoding; records every token and its top-2 margin so
the bench can tell a flagged near-tie (margin < 1e-2, R22) from a mismatch."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import fso
from oracle import tree as T
from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES

SEED = 0x5EED01


def main():
    name, n_pre, count = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    shape = SHAPES[name]
    t0 = time.time()
    op = OraclePipeline(shape, SEED, n_stages=1, max_slots=n_pre + count + 8, cache_weights=True)
    prefix = gen.prefix_tokens(SEED, n_pre, shape.vocab)
    x_new = op.set_prefix(prefix)
    _, m0 = T.argmax_margin(op.prefix_logits)
    print(f"prefill {n_pre} in {time.time() - t0:.0f} s, x_new {x_new} margin {m0:.4f}", flush=True)
    toks, margins = [x_new], [float(m0)]
    out = os.path.join(ROOT, "synth", "streams", f"{name}_p{n_pre}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    for j in range(count):
        p = n_pre + j
        _, lg = fso.forward(op.model, op.kv, 0, shape.n_layers, [toks[-1]], [p], [p],
                            [list(range(p + 1))])
        t, m = T.argmax_margin(lg[0])
        toks.append(int(t))
        margins.append(float(m))
        if j % 20 == 19 or j == count - 1:
            with open(out, "w") as f:
                json.dump({"shape": name, "seed": hex(SEED), "prefix_len": n_pre,
                           "prefix_mode": "prefill", "stream": toks, "margin": margins,
                           "note": "oracle greedy AR stream [x_new, g1, ...] and each token's "
                                   "top-2 logit margin (tools/oracle_stream.py)"}, f)
            print(f"{len(toks)} tokens, {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
