"""Full-size parity on BASELINE.json configs[1] (LLaMA2-7B shape, 32 layers,
prefix 1024, 64-node tree, segments of 16) in the launch configuration
bench.py times.  The oracle computes the sampled outputs one segment at a
time (synthetic-KV prefix so the CPU side stays within a minute)."""
import numpy as np
import pytest

from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES
from tests.lockstep import compare_tree

pytestmark = pytest.mark.gpu
SEED = 0x5EED01


def test_7b_full_size_sampled_segments():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    shape = SHAPES["7b"]
    gp = F.Pipeline(shape, max_ctx=2048, max_seg=16)
    gp.fs_load_random_weights(SEED)
    gp.enable_logits()
    op = OraclePipeline(shape, SEED, max_slots=2048)
    prefix = gen.prefix_tokens(SEED, 1024, shape.vocab)
    xo = op.set_prefix(prefix, mode="synth", kv_seed=7)
    xg = gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)
    srt = np.sort(op.prefix_logits)
    assert xg == xo or srt[-1] - srt[-2] < 1e-2
    stream = op.greedy_stream(5)
    t = gen.planted_tree(SEED, 64, 6, stream, (0, 2, 5, 17, 21), shape.vocab)
    so = op.submit(True, t["parent"], t["token"], t["own"], l_max=16)
    sg = gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 16)
    assert sg["order"] == so["order"] == list(t["order"])
    compare_tree(gp, op, 16, "submit")
    errs = []
    for tick in range(2):
        og, oo = gp.fs_verify_step(), op.verify_step()
        assert og["node"] == oo["node"]
        err = float(np.max(np.abs(og["logits"] - oo["logits"])))
        errs.append(err)
        for k in range(oo["n_rows"]):
            if oo["margin"][k] >= 1e-2:
                assert og["am"][k] == oo["am"][k]
        dg, do = gp.decision_dict(gp.fs_accept()), op.accept()
        want = dict(acc_ids=do["acc_ids"], x_new=do["x_new"], n_new_id=do["n_new_id"], cont=do["cont"])
        assert {k: dg[k] for k in want} == want
        gp.fs_prune_and_compact(want)
        op.prune(want)
        compare_tree(gp, op, 16, f"prune {tick}")
    print(f"7B full size: max|dlogit| per segment {errs}")
    assert max(errs) <= 2e-2


def test_7b_real_prefill_stream_matches_oracle():
    """The real-prefill path the bench times (configs[1]: 1024-token prefill
    through all 32 layers), checked against the ORACLE's own real prefill and
    greedy decoding (synth/streams/7b_p1024.json, written by
    tools/oracle_stream.py from oracle/ only): the first sampled token x_new,
    then tree verification of planted trees built from the oracle stream
    commits exactly that stream (R-def-2), up to the first oracle near-tie
    (margin < 1e-2, R22), after which the two may legitimately diverge."""
    import json
    import os
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_02620_b200 import flowspec as F
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "synth", "streams",
                        "7b_p1024.json")
    with open(path) as f:
        art = json.load(f)
    stream, margin = art["stream"], art["margin"]
    shape = SHAPES["7b"]
    gp = F.Pipeline(shape, max_ctx=2048, max_seg=16)
    gp.fs_load_random_weights(SEED)
    prefix = gen.prefix_tokens(SEED, art["prefix_len"], shape.vocab)
    assert gp.fs_set_prefix(prefix, F.FS_PREFILL) == stream[0]
    committed, r, a = [], 0, 4
    while len(committed) + a + 2 <= len(stream) and r < 24 and committed == stream[:len(committed)]:
        c = len(committed)
        x = gp.state()["x_new"]
        if x != stream[c]:       # the next root (not yet committed) already parts from the oracle
            committed.append(x)
            break
        t = gen.planted_tree(SEED + r, 64, 6, stream[c:c + a + 2], (0, 2, 5, 17, 21), shape.vocab)
        gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], 16)
        while True:
            gp.fs_verify_step()
            d = gp.decision_dict(gp.fs_accept())
            if not d["progress"]:
                continue
            committed += d["acc_tokens"]
            gp.fs_prune_and_compact(d)
            if not d["cont"]:
                break
        r += 1
    n = min(len(committed), len(stream))
    mism = [j for j in range(n) if committed[j] != stream[j]]
    print(f"7B real prefill: {n} committed tokens vs the oracle stream, first mismatch "
          f"{mism[0] if mism else None} (oracle margin {margin[mism[0]] if mism else None})")
    if mism:   # the stream may only part at an oracle near-tie (R22)
        assert margin[mism[0]] < 1e-2
    assert n >= 40 or mism
    gp.close()
