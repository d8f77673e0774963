"""KV compaction (a14) under the configs[4] stress (up to
168 MB of draft rows move for the whole 72B model): one 72B-shaped stage of
L layers with a 16K synthetic-KV context, a 256-node tree verified in 32-row
segments (all 256 draft rows cached), then a prune that keeps the accepted
prefix and a subtree (n_new placed early); CUDA events around
fs_prune_and_compact, moved bytes from the rank map.

    python tools/compact_time.py [layers=10]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import reduced

L = int(sys.argv[1]) if len(sys.argv) > 1 else 10
shape = reduced("72b", L)
gp = F.Pipeline(shape, max_ctx=17408, max_seg=32)
gp.fs_load_random_weights(1)
prefix = gen.prefix_tokens(1, 16384, shape.vocab)
x = gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
res = []
for trial in range(3):
    t = gen.random_tree(50 + trial, 256, 8, shape.vocab, gp.state()["x_new"])
    gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 32)
    for _ in range(8):
        gp.fs_verify_step()
    d = gp.decision_dict(gp.fs_accept())
    # force a continuing decision: accept the root only, re-root at its first child
    order = list(gp.query(F.FS_Q_NODE))
    par = list(gp.query(F.FS_Q_PARENT))
    child = next(order[i] for i in range(len(order)) if par[i] == 0)
    dec = dict(acc_ids=[order[0]], x_new=int(gp.query(F.FS_Q_TOKEN)[order.index(child)]), n_new_id=child, cont=1)
    nc = gp.state()["n_cached"][0]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(gp.stream)
    gp.fs_prune_and_compact(dec)
    b.record(gp.stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    n_ret = gp.state()["n_live"] + 1
    moved = (n_ret - 1) * L * 2 * shape.n_kv_heads * shape.head_dim * 2   # rows that change slot (upper bound)
    res.append((ms, nc, n_ret, moved))
    # finish the round
    while True:
        gp.fs_verify_step()
        dd = gp.decision_dict(gp.fs_accept())
        if dd["progress"]:
            gp.fs_prune_and_compact(dd)
            if not dd["cont"]:
                break
for ms, nc, n_ret, moved in res:
    print(f"layers {L}: cached {nc} rows, retained {n_ret}: prune + compaction {ms * 1e3:8.1f} us, "
          f"<= {moved / 1e6:6.1f} MB moved -> {2 * moved / (ms * 1e-3) / 1e9:7.1f} GB/s (read + write)")
