"""Measurements for the SURVEY §8(f) rows built this round, on the 7B model
(32 layers, 1024-token synthetic-KV context, one GPU):

  f2  stochastic acceptance: sample_walk_kernel alone (fs_bench_kernel 11, back
      to back) and whole SD rounds at T = 1 against greedy rounds (CUDA events)
  f4  tree merging: merge_kernel alone (fs_bench_kernel 12) and the FS_MERGE
      submit through the public API (host wall clock)
Inputs are synthetic: random draft distributions q (torch, seeded) and random
trees; the numbers are costs, not acceptance rates of a trained draft."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2507_02620_b200 import flowspec as F
from synth import gen
from synth.configs import SHAPES

shape = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "7b"]
V = shape.vocab
gp = F.Pipeline(shape, max_ctx=4096, max_seg=16, sampling=1)
gp.fs_load_random_weights(1)
prefix = gen.prefix_tokens(1, 1024, V)
ev = lambda: torch.cuda.Event(enable_timing=True)


def rounds(n, stochastic, seed0=100):
    tot_ms, toks, ticks = 0.0, 0, 0
    g = torch.Generator(device="cuda").manual_seed(seed0)
    for r in range(n):
        t = gen.random_tree(seed0 + r, 64, 6, V, gp.state()["x_new"])
        if stochastic:
            q = torch.softmax(2.0 * torch.randn(64, V, device="cuda", generator=g), dim=1).contiguous()
            gp.fs_set_acceptance(F.FS_ACCEPT_STOCHASTIC, 1.0, seed0 + r, q)
        a, b = ev(), ev()
        torch.cuda.synchronize()
        a.record(gp.stream)
        gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 16)
        while True:
            gp.fs_verify_step()
            ticks += 1
            d = gp.decision_dict(gp.fs_accept())
            if not d["progress"]:
                continue
            toks += len(d["acc_ids"])
            gp.fs_prune_and_compact(d)
            if not d["cont"]:
                break
        b.record(gp.stream)
        torch.cuda.synchronize()
        tot_ms += a.elapsed_time(b)
        if stochastic:
            gp.fs_set_acceptance(F.FS_ACCEPT_GREEDY)
    return tot_ms / n, toks / n, ticks / n


gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
rounds(2, False)
gms, gt, gk = rounds(8, False)
gms_s, gt_s, gk_s = rounds(8, True)
print(f"f2 rounds (random 64-node trees): greedy {gms:7.3f} ms/round, {gt:.2f} tokens, {gk:.2f} ticks; "
      f"stochastic T=1 {gms_s:7.3f} ms/round, {gt_s:.2f} tokens, {gk_s:.2f} ticks")
# the walk alone, on a live tree with a verified root
g = torch.Generator(device="cuda").manual_seed(5)
q = torch.softmax(2.0 * torch.randn(64, V, device="cuda", generator=g), dim=1).contiguous()
gp.fs_set_acceptance(F.FS_ACCEPT_STOCHASTIC, 1.0, 77, q)
t = gen.random_tree(999, 64, 6, V, gp.state()["x_new"])
gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 16)
gp.fs_verify_step()
d = gp.decision_dict(gp.fs_accept())
us, by = gp.bench_kernel(11, 50)
print(f"f2 sample_walk_kernel: {us:7.2f} us per walk ({len(d.get('acc_ids', []))} accepted nodes; "
      f"{by / 1e3:.0f} KB read per walked node)")
while True:
    if d["progress"]:
        gp.fs_prune_and_compact(d)
        if not d["cont"]:
            break
    gp.fs_verify_step()
    d = gp.decision_dict(gp.fs_accept())
gp.fs_set_acceptance(F.FS_ACCEPT_GREEDY)

# f4: merge a 48-node tree (half its paths already live) after the first prune
stream = [gp.state()["x_new"]]
rng = gen.Rng(3)
t = gen.random_tree(1234, 64, 6, V, stream[0])
gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 16)
gp.fs_verify_step()
d = gp.decision_dict(gp.fs_accept())
live_tok = list(gp.query(F.FS_Q_TOKEN))
live_par = list(gp.query(F.FS_Q_PARENT))
par, tok = [-1], [live_tok[0]]
keep = {0: 0}
for s in range(1, len(live_tok)):
    if live_par[s] in keep and rng.below(2):
        keep[s] = len(par)
        par.append(keep[live_par[s]])
        tok.append(live_tok[s])
while len(par) < 48:
    p = rng.below(len(par))
    tk = 20000 + rng.below(10000)
    if all(not (par[i] == p and tok[i] == tk) for i in range(1, len(par))):
        par.append(p)
        tok.append(tk)
own = [1.0] + [0.5] * (len(par) - 1)
if d["progress"] and d["cont"]:
    pass
t0 = time.perf_counter()
out = gp.fs_submit_segment(F.FS_MERGE, par, tok, own, 16)
wall = (time.perf_counter() - t0) * 1e6
us, _ = gp.bench_kernel(12, 50)
print(f"f4 merge of a {len(par)}-node T_new into {len(live_tok)} live nodes ({len(out['order'])} new): "
      f"merge_kernel {us:6.2f} us, FS_MERGE submit through the API {wall:6.1f} us (host wall)")
