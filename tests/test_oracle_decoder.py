"""Pins of the oracle decoder and pipelined run (oracle/fso.c, oracle/pipeline.py).

* generator: published SplitMix64 outputs, value-grid structure, moments;
* decoder + tree attention: HF ``transformers`` LlamaForCausalLM /
  Qwen2ForCausalLM (fp32, eager) fed ``prefix ++ S`` with tree position ids and
  a custom 4D additive mask (library routine; SURVEY.md §8(c) "HF pin");
* R-def-1: tree-verification logits == plain causal forward over
  context ++ path(j) (brute force, PAPER.md:248 + north_star);
* R-def-2: the committed stream == greedy autoregressive decoding, for every
  segmentation L_max and stage count P ("ensure a correct
  inference output"; north_star "every segmentation must give the same
  accepted sequence");
* Fig. 3 prune applied to the pipelined state, compaction
  byte-identity and accepted rows landing at l_glo..l_glo'-1.
CPU only."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import fso
from oracle import tree as T
from oracle.pipeline import OraclePipeline
from synth import gen
from synth.configs import SHAPES

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SEED = 0x5EED01


# ------------------------------------------------------------------ generator
def test_splitmix64_published_values():
    with open(os.path.join(GOLD, "splitmix64.json")) as f:
        g = json.load(f)
    gamma = int(g["gamma"], 16)
    L = fso.lib()
    for k, want in enumerate(g["seed0_outputs"]):
        z = (k * gamma) & ((1 << 64) - 1)
        assert L.fso_mix64(z) == int(want, 16)
        assert gen.mix64(z) == int(want, 16)


def test_generator_grid_and_moments():
    L = fso.lib()
    sigma = 0.02
    c = np.float32(sigma * np.sqrt(3.0) / 2 ** 24)
    xs = np.array([L.fso_gen_value(7, 3, e, sigma, 0, 0) for e in range(20000)], np.float64)
    # every value is RN32(i * c) for an odd integer |i| < 2^24
    i0 = np.rint(xs / np.float64(c))
    ok = np.zeros(len(xs), bool)
    for di in (-1, 0, 1):
        i = i0 + di
        ok |= (np.abs(i) < 2 ** 24) & (i % 2 == 1) & \
            (np.float32(i.astype(np.float32) * c) == xs.astype(np.float32))
    assert ok.all()
    assert abs(xs.mean()) < 3 * sigma / np.sqrt(len(xs))
    assert abs(xs.std() - sigma) < 0.02 * sigma
    assert np.all(np.abs(xs) <= sigma * np.sqrt(3.0) * (1 + 1e-6))
    # bf16 variant is the round-to-nearest-even of the fp32 value
    for e in range(2000):
        a = L.fso_gen_value(7, 3, e, sigma, 0, 0)
        b = L.fso_gen_value(7, 3, e, sigma, 0, 1)
        t = torch.tensor([a], dtype=torch.float32).to(torch.bfloat16).float().item()
        assert b == t
    # gains: 1 + U(+-0.1)
    g = np.array([L.fso_gen_value(7, 0xFFFF2, e, 0.0, 1, 0) for e in range(5000)])
    assert g.min() >= 0.9 - 1e-6 and g.max() <= 1.1 + 1e-6 and abs(g.mean() - 1) < 0.01


# ------------------------------------------------------------------ HF pin
def _bf16_storage_attention(module, query, key, value, attention_mask, scaling,
                            dropout=0.0, **kw):
    """HF eager attention with q, K and V stored as bf16 after bias + RoPE — the
    storage points of the bf16 precision contract (R18: the KV cache
    and q are bf16); everything else stays HF's own fp32 arithmetic."""
    from transformers.models.llama.modeling_llama import eager_attention_forward
    r = lambda t: t.to(torch.bfloat16).to(t.dtype)
    return eager_attention_forward(module, r(query), r(key), r(value), attention_mask,
                                   scaling, dropout, **kw)


def _hf_model(shape, model):
    from transformers import LlamaConfig, LlamaForCausalLM, Qwen2Config, Qwen2ForCausalLM
    kw = dict(vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.ffn,
              num_hidden_layers=shape.n_layers, num_attention_heads=shape.n_heads,
              num_key_value_heads=shape.n_kv_heads, head_dim=shape.head_dim,
              rms_norm_eps=shape.rms_eps, tie_word_embeddings=False,
              max_position_embeddings=4096,
              rope_parameters={"rope_type": "default", "rope_theta": shape.rope_theta})
    if shape.qkv_bias:
        hf = Qwen2ForCausalLM(Qwen2Config(**kw))
    else:
        hf = LlamaForCausalLM(LlamaConfig(attention_bias=False, **kw))
    if shape.bf16:
        from transformers import AttentionInterface
        AttentionInterface.register("bf16_storage", _bf16_storage_attention)
        hf.config._attn_implementation = "bf16_storage"
        # the contract's RoPE tables: angle in fp64, cos/sin rounded to fp32
        # (DESIGN.md "RoPE tables"); HF's own fp32 angle differs by ~1e-6 at
        # position 40 and would only add bf16 rounding flips of q/K
        hd, theta = shape.head_dim, shape.rope_theta

        def rope64(x, position_ids):
            inv = theta ** (-torch.arange(0, hd, 2, dtype=torch.float64) / hd)
            ang = position_ids[0].to(torch.float64)[:, None] * inv[None, :]
            emb = torch.cat((ang, ang), dim=-1)[None]
            dt = x.dtype
            return emb.cos().float().to(dt), emb.sin().float().to(dt)
        hf.model.rotary_emb.forward = rope64
    else:
        hf.config._attn_implementation = "eager"
    sd = {"model.embed_tokens.weight": model.tensor(fso.EMBED),
          "lm_head.weight": model.tensor(fso.HEAD),
          "model.norm.weight": model.tensor(fso.FINAL_NORM)}
    for l in range(shape.n_layers):
        p = f"model.layers.{l}."
        sd[p + "self_attn.q_proj.weight"] = model.tensor(fso.Q, l)
        sd[p + "self_attn.k_proj.weight"] = model.tensor(fso.K, l)
        sd[p + "self_attn.v_proj.weight"] = model.tensor(fso.V, l)
        sd[p + "self_attn.o_proj.weight"] = model.tensor(fso.O, l)
        sd[p + "mlp.gate_proj.weight"] = model.tensor(fso.GATE, l)
        sd[p + "mlp.up_proj.weight"] = model.tensor(fso.UP, l)
        sd[p + "mlp.down_proj.weight"] = model.tensor(fso.DOWN, l)
        sd[p + "input_layernorm.weight"] = model.tensor(fso.ATTN_NORM, l)
        sd[p + "post_attention_layernorm.weight"] = model.tensor(fso.MLP_NORM, l)
        if shape.qkv_bias:
            sd[p + "self_attn.q_proj.bias"] = model.tensor(fso.BQ, l)
            sd[p + "self_attn.k_proj.bias"] = model.tensor(fso.BK, l)
            sd[p + "self_attn.v_proj.bias"] = model.tensor(fso.BV, l)
    sd = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in sd.items()}
    missing, unexpected = hf.load_state_dict(sd, strict=False)
    assert not unexpected and all("rotary" in m for m in missing), (missing, unexpected)
    return hf.eval()


def _hf_tree_logits(shape, name, mutant=0, hf64=False):
    """Oracle tree verification and HF over prefix ++ S with tree position ids
    and a custom 4D additive mask; returns (oracle prefix logits, oracle tree
    logits, HF logits, n_pre, x_new).  hf64: HF in fp64 arithmetic."""
    n_pre = 20
    fso.lib().fso_set_mutant(mutant)
    try:
        op = OraclePipeline(shape, SEED, n_stages=1)
        prefix = gen.prefix_tokens(11, n_pre, shape.vocab)
        x_new = op.set_prefix(prefix)
        t = gen.random_tree(5, 24, 5, shape.vocab, x_new)
        sub = op.submit(True, t["parent"], t["token"], t["own"], l_max=24)
        out = op.verify_step()
    finally:
        fso.lib().fso_set_mutant(0)
    snap = op.snapshot()
    m = len(sub["order"])
    hf = _hf_model(shape, op.model)
    dt = torch.float64 if hf64 else torch.float32
    hf = hf.to(dt)
    ids = list(prefix) + snap["token"]
    pos = list(range(n_pre)) + snap["pos"]
    L = n_pre + m
    mask = torch.full((1, 1, L, L), torch.finfo(dt).min, dtype=dt)
    for i in range(n_pre):
        mask[0, 0, i, :i + 1] = 0
    for k in range(m):
        mask[0, 0, n_pre + k, :n_pre] = 0
        for a in snap["anc"][k]:
            mask[0, 0, n_pre + k, n_pre + a] = 0
    with torch.no_grad():
        lg = hf(input_ids=torch.tensor([ids]), position_ids=torch.tensor([pos]),
                attention_mask=mask).logits[0].double().numpy()
    return op.prefix_logits, out["logits"], lg, n_pre, x_new


# bf16 bound.  The oracle (fp64 arithmetic, fp32 activations) and HF run in
# fp64 round q/K/V to bf16 at the same storage points, so they differ by the fp32
# rounding of the oracle's activations (relative 2^-24) and by the bf16 rounding
# flips that difference causes (a stored element whose two values straddle a
# bf16 boundary moves by one bf16 ulp, 2^-8 relative).  HF in fp32 arithmetic is
# a second correct implementation of the same contract with ~2^7x larger
# arithmetic error, hence more flips: |HF32 - HF64| is the contract's inherent
# spread, and the oracle must sit well inside it.  A hard cap keeps the pin
# meaningful on its own.
def _bf16_pin_errors(name, mutant=0):
    shape = SHAPES[name]
    pre, tree, lg64, n, _ = _hf_tree_logits(shape, name, mutant=mutant, hf64=True)
    _, _, lg32, _, _ = _hf_tree_logits(shape, name, hf64=False)
    o = np.concatenate([pre[None].astype(np.float64), tree.astype(np.float64)])
    return float(np.max(np.abs(o - lg64[n - 1:]))), float(np.max(np.abs(lg32[n - 1:] - lg64[n - 1:])))


@pytest.mark.parametrize("name", ["small", "smallq"])
def test_bf16_tree_verification_matches_hf(name):
    """bf16 branch of the oracle against HF on the same bf16-rounded weights,
    with q/K/V stored as bf16 and the contract's RoPE tables (R18):
    pins the plain RMSNorm -> linear order, the bias, RoPE and the storage
    points of the bf16 branch."""
    err, spread = _bf16_pin_errors(name)
    assert err <= 0.5 * spread and err <= 1e-3, (err, spread)


@pytest.mark.parametrize("mutant", [1, 2])
def test_bf16_hf_pin_catches_dropped_norm_scale(mutant):
    """A mistake in the bf16 branch (RMSNorm scale dropped before the head or
    before QKV) must fail the pin above by orders of magnitude."""
    err, _ = _bf16_pin_errors("small", mutant)
    assert err > 1.0, err      # the pin's cap is 1e-3


@pytest.mark.parametrize("name", ["tiny", "tinyq"])
def test_tree_verification_matches_hf(name):
    shape = SHAPES[name]
    n_pre = 20
    op = OraclePipeline(shape, SEED, n_stages=1)
    prefix = gen.prefix_tokens(11, n_pre, shape.vocab)
    x_new = op.set_prefix(prefix)
    t = gen.random_tree(5, 24, 5, shape.vocab, x_new)
    sub = op.submit(True, t["parent"], t["token"], t["own"], l_max=24)
    out = op.verify_step()
    snap = op.snapshot()
    m = len(sub["order"])
    hf = _hf_model(shape, op.model)
    ids = list(prefix) + snap["token"]
    pos = list(range(n_pre)) + snap["pos"]
    L = n_pre + m
    mask = torch.full((1, 1, L, L), torch.finfo(torch.float32).min)
    for i in range(n_pre):
        mask[0, 0, i, :i + 1] = 0
    for k in range(m):
        mask[0, 0, n_pre + k, :n_pre] = 0
        for a in snap["anc"][k]:
            mask[0, 0, n_pre + k, n_pre + a] = 0
    with torch.no_grad():
        lg = hf(input_ids=torch.tensor([ids]), position_ids=torch.tensor([pos]),
                attention_mask=mask).logits[0].numpy()
    np.testing.assert_allclose(op.prefix_logits, lg[n_pre - 1], atol=1e-4, rtol=0)
    np.testing.assert_allclose(out["logits"], lg[n_pre:], atol=1e-4, rtol=0)
    assert int(np.argmax(lg[n_pre - 1])) == x_new


# ------------------------------------------------------------------ R-def-1
@pytest.mark.parametrize("name", ["tiny", "small"])
def test_tree_logits_equal_per_path_autoregressive(name):
    shape = SHAPES[name]
    op = OraclePipeline(shape, SEED, n_stages=1, max_slots=256)
    prefix = gen.prefix_tokens(3, 16, shape.vocab)
    x_new = op.set_prefix(prefix)
    t = gen.random_tree(9, 15 if name == "tiny" else 10, 4, shape.vocab, x_new)
    op.submit(True, t["parent"], t["token"], t["own"], l_max=4)
    logits = {}
    while op.queue or any(s is not None for s in op.slot):
        o = op.verify_step()
        for k, nid in enumerate(o["node"]):
            logits[nid] = o["logits"][k]
    # brute force: fresh model + KV, causal forward over prefix ++ path(j)
    bf = OraclePipeline(shape, SEED, n_stages=1, max_slots=256)
    for j in range(len(t["parent"])):
        path, p = [], j
        while p >= 0:
            path.append(int(t["token"][p]))
            p = int(t["parent"][p])
        seq = list(prefix) + path[::-1]
        bf.set_prefix(seq)
        assert np.array_equal(bf.prefix_logits, logits[j]), j


# ------------------------------------------------------------------ R-def-2
def _run_rounds(shape, n_stages, l_max, n_rounds, planted=(0, 1, 2, 9), n_nodes=15,
                depth=4, trees=None, prefix_len=32):
    op = OraclePipeline(shape, SEED, n_stages=n_stages, max_slots=512)
    prefix = gen.prefix_tokens(SEED, prefix_len, shape.vocab)
    op.set_prefix(prefix)
    committed, used_trees, all_logits = [], [], {}
    for r in range(n_rounds):
        if trees is None:
            stream = op.greedy_stream(len(planted) + 1)
            t = gen.planted_tree(SEED + r, n_nodes, depth, stream, planted, shape.vocab)
        else:
            t = trees[r]
        used_trees.append(t)
        op.submit(True, t["parent"], t["token"], t["own"], l_max=l_max)
        while True:
            o = op.verify_step()
            d = op.accept()
            if not d["progress"]:
                continue
            committed += d["acc_tokens"]
            op.prune(dict(acc_ids=d["acc_ids"], x_new=d["x_new"], n_new_id=d["n_new_id"],
                          cont=d["cont"]))
            if not d["cont"]:
                break
    return committed, used_trees, op


def test_committed_stream_is_greedy_ar_and_segmentation_invariant():
    shape = SHAPES["tiny"]
    n_rounds = 6
    ref, trees, op = _run_rounds(shape, 1, 8, n_rounds)
    # planted scenario R: every round commits a+1 = 4 tokens
    assert len(ref) == 4 * n_rounds
    # greedy AR decoding from the prompt (R-def-2)
    ar = OraclePipeline(shape, SEED, n_stages=1, max_slots=512)
    ar.set_prefix(gen.prefix_tokens(SEED, 32, shape.vocab))
    stream = ar.greedy_stream(len(ref))
    assert ref == stream[:len(ref)]
    # every segmentation and P in {1, 2} commits the same stream
    for l_max in range(1, 16):
        for P in (1, 2):
            got, _, _ = _run_rounds(shape, P, l_max, n_rounds, trees=trees)
            assert got == ref, (l_max, P)


def test_fig3_prune_in_pipeline_state():
    """Fig. 3 applied to a live 2-stage pipeline after segment 0."""
    shape = SHAPES["tiny"]
    op = OraclePipeline(shape, SEED, n_stages=2, max_slots=256)
    x = op.set_prefix(gen.prefix_tokens(1, 12, shape.vocab))
    parent = [-1, 0, 0, 1, 1, 2, 3, 3]
    own = [1.0] + [np.float32((1 - 0.1 * (i + 1)) / (1 - 0.1 * i)) for i in range(1, 8)]
    # cu strictly decreasing with id -> S order is the id order
    own = [1.0] + [np.float32((1 - 0.1 * i) / (1 - 0.1 * parent[i])) for i in range(1, 8)]
    toks = [x, 11, 12, 13, 14, 15, 16, 17]
    sub = op.submit(True, parent, toks, own, l_max=3)
    assert sub["order"] == list(range(8)) and sub["bounds"] == [(0, 3), (3, 6), (6, 8)]
    l0 = op.l_glo
    op.verify_step()            # seg 0 at stage 0
    op.verify_step()            # seg 0 at stage 1 (verified), seg 1 at stage 0
    snap = op.snapshot()
    assert snap["n_cached"] == [6, 3]
    kv_before = {i: op.kv.get(0, 0, 0, l0 + i).copy() for i in range(6)}
    kv_before1 = {i: op.kv.get(1, 1, 1, l0 + i).copy() for i in range(3)}
    info = op.prune(dict(acc_ids=[0, 1], x_new=13, n_new_id=3, cont=1))
    assert info["i_acc"] == [0, 1] and info["i_pr"] == [3, 6, 7]
    snap = op.snapshot()
    assert op.l_glo == l0 + 2
    assert snap["node"] == [3, 6, 7]
    assert snap["pos"][0] == l0 + 2                  # node 3 depth 2: position unchanged (R4)
    assert snap["inflight"][1][1:] == (0, 1)           # segment {3,4,5} -> {3}
    assert snap["queue"][0][1:] == (1, 3)              # segment {6,7} -> S indices 1..2
    assert snap["n_cached"] == [1, 0]
    # compaction: accepted rows land at l_glo..l_glo'-1, retained draft rows move
    # byte-identically (stage 0 owns layer 0, stage 1 owns layer 1)
    assert np.array_equal(op.kv.get(0, 0, 0, l0 + 0), kv_before[0])
    assert np.array_equal(op.kv.get(0, 0, 0, l0 + 1), kv_before[1])
    assert np.array_equal(op.kv.get(0, 0, 0, l0 + 2), kv_before[3])
    assert np.array_equal(op.kv.get(1, 1, 1, l0 + 1), kv_before1[1])
