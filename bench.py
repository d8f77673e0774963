"""Benchmark: accepted tokens/s of pipelined tree verification (FlowSpec hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Default (every N): BASELINE.json configs[1] (LLaMA2-7B-shaped bf16, prefix
1024 with a real prefill, 64-node draft trees, segments of 16, planted accept
path a=4) -- at N>1 (torchrun, one rank per GPU) the same rounds run as an
N-stage pipeline, so the per-N values form a strong-scaling curve.  A step is
one SD round: submit the tree, pipeline ticks (verify_step), accept,
prune/compact, until the continuous condition fails (§3.1-3.3).
--workload picks the other configs: cfg3 (configs[2] planting), cfg4
(configs[3]: 13B, 4096-token synthetic-KV context, scenario S steady
expansion, a step = one tick), cfg5 (configs[4]: Qwen2-72B, 16384-token
context, 256-node trees), s7b (7B scenario S).

Draft trees are synthetic (the paper's draft model is out of scope): the
planted path is the oracle's greedy stream where one is stored
(synth/streams/, tools/oracle_stream.py), else the model's own greedy stream
through the same public API; untimed dry runs check that tree verification
commits the plan.  Weights >> L2 (126 MB): every tick streams them from HBM.
"""
import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 0x5EED01


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS),
                    help="cfg2 = configs[1] (default at every N), cfg3 = configs[2] planting, "
                         "cfg4 = configs[3] (13B, scenario S), cfg5 = configs[4] (72B), "
                         "s7b = 7B scenario S")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--real-prefill", action="store_true",
                    help="synthetic-KV workloads (cfg4/cfg5): real chunked prefill of the whole prefix instead")
    ap.add_argument("--max-prefill", type=int, default=64, help="rows per prefill chunk (<= 64)")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-attn-long", action="store_true")
    return ap.parse_args()


# BASELINE.json configs as bench workloads (SURVEY §8(d) per-config inputs).
# R = round-based (scenario R: each round commits a+1 tokens, then exits);
# S = steady expansion (scenario S: one long round, a 16-node batch carrying
# q planted chain nodes appended after every tick).
WORKLOADS = {
    "cfg2": dict(cfg="configs[1]", shape="7b", prefix=1024, mode="prefill", n_nodes=64, depth=6,
                 l_max=16, max_seg=16, ranks=(0, 2, 5, 17, 21), scenario="R"),
    "cfg3": dict(cfg="configs[2]", shape="7b", prefix=1024, mode="prefill", n_nodes=64, depth=6,
                 l_max=16, max_seg=16, ranks=(0, 3, 9, 18, 25, 33, 40), scenario="R"),
    "cfg4": dict(cfg="configs[3]", shape="13b", prefix=4096, mode="synth", n_nodes=128, depth=6,
                 l_max=16, max_seg=16, ranks=(0, 1, 2, 17, 18, 33, 34), scenario="S", q=2),
    "cfg5": dict(cfg="configs[4]", shape="72b", prefix=16384, mode="synth", n_nodes=256, depth=8,
                 l_max=32, max_seg=32, ranks=(0, 3, 9, 40, 47, 70, 90, 100, 120), scenario="R"),
    "s7b": dict(cfg="sweep 7B scenario S", shape="7b", prefix=1024, mode="prefill", n_nodes=64,
                depth=6, l_max=16, max_seg=16, ranks=(0, 1, 2, 17, 18, 33, 34), scenario="S", q=2),
}

# SURVEY §8(d) "Algorithmic work per verified segment" (bytes; 6.54 TB/s ideal
# tick at P=1/2/4/8, byte-balanced) -> xi ceilings of the two scenarios
IDEAL_TICK_MS = {"7b": (2.108, 1.074, 0.557, 0.299), "13b": (4.461, 2.255, 1.153, 0.601),
                 "72b": (22.69, 11.44, 5.86, 3.07)}


def xi_ceiling(wl, P):
    """Scenario S: q / tick.  Scenario R: (a+1) / (((P-1) + k_exit) * tick) with
    k_exit = the number of segments the planted path spans."""
    i = {1: 0, 2: 1, 4: 2, 8: 3}.get(P)
    if i is None:
        return None
    tick = IDEAL_TICK_MS[wl["shape"]][i] * 1e-3
    if wl["scenario"] == "S":
        return wl["q"] / tick
    a = len(wl["ranks"]) - 1
    k_exit = wl["ranks"][-1] // wl["l_max"] + 1
    return (a + 1) / (((P - 1) + k_exit) * tick)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), float(m["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def tflops_sustained():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops_sustained"]), "measured"
    except Exception:
        return 1590.0, "fallback"


def prefill_flops(shape, n):
    """Algorithmic FLOPs of a causal prefill of n tokens: the layer
    GEMMs 2 * params_per_layer * L per token, attention 4 * H * hd per
    visible key (QK^T and P V, causal: n(n+1)/2 keys), the head for the last
    token only."""
    d, hd = shape.d_model, shape.head_dim
    per_layer = (d * (shape.n_heads + 2 * shape.n_kv_heads) * hd + shape.n_heads * hd * d
                 + 3 * d * shape.ffn)
    return (2.0 * per_layer * shape.n_layers * n + 4.0 * shape.n_heads * hd * shape.n_layers * n * (n + 1) / 2
            + 2.0 * shape.vocab * d)


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.times = []
        self.proc = None
        self.t_from = 0.0

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)
                self.times.append(time.perf_counter())

    def count_since(self, t0):
        return sum(1 for t in self.times if t >= t0)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = [r for r, t in zip(self.rows, self.times) if t >= self.t_from] or self.rows
        sm = sorted(int(r[0]) for r in rows if r[0].isdigit())
        mx = max([int(r[1]) for r in rows if r[1].isdigit()] or [0])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None,
                "reasons": reasons, "samples": len(sm)}


# ------------------------------------------------------------------ our arm
PRUNES = [0]   # fs_prune_and_compact calls (host -> device decision copies)

# bytes the library copies per call (include/flowspec.h capacities: FS_MAX_LIVE
# 512, FS_MAX_SEG 64; csrc/state.cuh layouts): SubmitIn (5 ints + parent / token
# / own [512]) host -> device per submit; a synchronous submit reads the record
# prefix back (14 ints + order / merged [512]), an FS_SUBMIT_ASYNC one (every
# submit in the timed steps) nothing; the verify step's whole record (14 ints,
# 6 x [512] arrays, prune plan 1 + [512], 64 row results of 8 B and 64 node ids)
# back per tick; DecisionIn (4 ints + acc ids [512]) host -> device per prune
H2D_SUBMIT = 4 * (5 + 3 * 512)
D2H_SUBMIT = 0   # async submits in the timed steps (a synchronous one: 4 * (14 + 2 * 512))
D2H_TICK = 4 * (14 + 6 * 512 + 1 + 512) + 64 * 8 + 64 * 4   # sizeof(TreeRecord) = 15164
H2D_PRUNE = 4 * (4 + 512)


def run_round(gp, tree, l_max, tokens_out=None):
    """One SD round: submit, ticks, accept, prune until the round exits."""
    from paper_2507_02620_b200 import flowspec as F
    gp.fs_submit_segment(F.FS_NEW_ROUND | F.FS_SUBMIT_ASYNC, tree["parent"], tree["token"], tree["own"], l_max)
    committed = 0
    ticks = 0
    while True:
        gp.fs_verify_step()
        ticks += 1
        d = gp.fs_accept()
        if not d.progress:
            continue
        committed += d.n_acc
        if tokens_out is not None:
            tokens_out += list(d.acc_tokens[:d.n_acc])
        gp.fs_prune_and_compact(d)
        PRUNES[0] += 1
        if not d.cont:
            return committed, ticks


class Batches:
    """The appended batches of a scenario-S run, generated before the timed
    region (the draft side is out of scope; its host work is not the path's)."""

    def __init__(self, exp, n):
        self.items = [exp.next_batch() for _ in range(n)]
        self.i = 0

    def next_batch(self):
        b = self.items[self.i]
        self.i += 1
        return b


class SteadyRound:
    """Scenario S driver: one long round; every tick = verify, accept, prune,
    then append the next batch (a16).  end() stops appending and drains."""

    def __init__(self, gp, tree, exp, l_max):
        from paper_2507_02620_b200 import flowspec as F
        self.F, self.gp, self.exp, self.l_max = F, gp, exp, l_max
        gp.fs_submit_segment(F.FS_NEW_ROUND, tree["parent"], tree["token"], tree["own"], l_max)
        self.live = True

    def tick(self, tokens_out=None, append=True):
        gp = self.gp
        gp.fs_verify_step()
        d = gp.fs_accept()
        c = 0
        if d.progress:
            c = d.n_acc
            if tokens_out is not None:
                tokens_out += list(d.acc_tokens[:d.n_acc])
            gp.fs_prune_and_compact(d)
            PRUNES[0] += 1
            if not d.cont:
                self.live = False
                return c
        if append:
            par, tok, own = self.exp.next_batch()
            gp.fs_submit_segment(self.F.FS_APPEND | self.F.FS_SUBMIT_ASYNC, par, tok, own, self.l_max)
        return c

    def end(self, tokens_out=None):
        while self.live:
            self.tick(tokens_out, append=False)


def greedy_stream(gp, count):
    """AR decode through the API: one-node trees (root only)."""
    from paper_2507_02620_b200 import flowspec as F
    x = gp.state()["x_new"]
    out = [x]
    for _ in range(count):
        gp.fs_submit_segment(F.FS_NEW_ROUND, [-1], [out[-1]], [1.0], 1)
        while True:
            gp.fs_verify_step()
            d = gp.fs_accept()
            if d.progress:
                gp.fs_prune_and_compact(d)
                out.append(d.x_new)
                break
    return out


def oracle_stream(wl):
    """The oracle's greedy stream for this model / prompt (tools/oracle_stream.py
    artifact), or None when none is stored (synthetic-KV configs: a CPU
    prefill of 13B x 4096 / 72B x 16384 is out of reach)."""
    path = os.path.join(ROOT, "synth", "streams", f"{wl['shape']}_p{wl['prefix']}.json")
    if wl["mode"] != "prefill" or not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


def set_prefix(gp, wl, prefix):
    from paper_2507_02620_b200 import flowspec as F
    if wl["mode"] == "prefill":
        return gp.fs_set_prefix(prefix, F.FS_PREFILL)
    return gp.fs_set_prefix(prefix, F.FS_SYNTH_KV, kv_seed=7)


def plan_schedule(gp, wl, prefix, shape, n_rounds, n_ticks, max_iter=6):
    """Draft-provider stand-in (the paper's draft model is out of scope): trees
    whose planted path is the greedy continuation.  The plan starts as the
    oracle's greedy stream when one is stored, else the GPU's own
    AR stream; each untimed dry run replaces it with the stream tree
    verification actually commits plus an AR continuation, until a dry run
    follows its plan.  The timed steps replay exactly these inputs from the same
    prefix (deterministic).  Returns (inputs, plan record)."""
    from synth import gen
    ranks = wl["ranks"]
    a = len(ranks) - 1
    q = wl.get("q", 0)
    if wl["scenario"] == "R":
        need = n_rounds * (a + 1) + a + 2
    else:
        need = a + q * (n_ticks + 4) + q + 2
    orc = oracle_stream(wl)
    info = {"source": "gpu greedy AR through the public API"}
    if orc is not None and len(orc["stream"]) >= 2:
        plan = list(orc["stream"])
        info = {"source": f"oracle greedy stream (synth/streams/{wl['shape']}_p{wl['prefix']}.json)"}
        if len(plan) < need:
            set_prefix(gp, wl, prefix)
            plan = plan + greedy_stream_from(gp, plan, need - len(plan))
            info["source"] += f" + {need - len(orc['stream'])} gpu AR tokens"
    else:
        set_prefix(gp, wl, prefix)
        plan = greedy_stream(gp, need)
    first_plan = list(plan)
    for it in range(max_iter):
        set_prefix(gp, wl, prefix)
        committed, diverged = [], 0
        if wl["scenario"] == "R":
            inputs = []
            for r in range(n_rounds):
                c = len(committed)
                root = gp.state()["x_new"]
                if c + a + 2 <= len(plan) and plan[c] == root:
                    t = gen.planted_tree(SEED + r, wl["n_nodes"], wl["depth"], plan[c:c + a + 2], ranks,
                                         shape.vocab)
                else:  # off plan: unplanted tree rooted at the actual next token
                    diverged += 1
                    t = gen.random_tree(SEED + 7 * r, wl["n_nodes"], wl["depth"], shape.vocab, root)
                inputs.append(t)
                run_round(gp, t, wl["l_max"], committed)
        else:
            t = gen.planted_tree(SEED, wl["n_nodes"], wl["depth"], plan[:a + 2], ranks, shape.vocab)
            inputs = (t, plan)
            sr = SteadyRound(gp, t, gen.SteadyExpansion(SEED + 1, t, plan, q, 16, shape.vocab), wl["l_max"])
            for _ in range(n_ticks):
                sr.tick(committed)
                if not sr.live:
                    diverged += 1
                    break
            sr.end(committed)
        n = min(len(committed), len(first_plan))
        mism = [i for i in range(n) if committed[i] != first_plan[i]]
        if it == 0:
            info["tokens_checked"] = n
            info["mismatches_first_dry_run"] = len(mism)
            if mism and orc is not None and mism[0] < len(orc["margin"]):
                info["first_mismatch_oracle_margin"] = round(orc["margin"][mism[0]], 5)
        if diverged == 0 and committed == plan[:len(committed)]:
            info["dry_runs"] = it + 1
            return inputs, info
        plan = committed + greedy_stream(gp, need)
    info["dry_runs"] = max_iter
    info["unplanned_steps"] = diverged
    return inputs, info


def greedy_stream_from(gp, plan, count):
    """AR continuation after the tokens of `plan` (committed through one-node
    rounds first, so the context matches)."""
    from paper_2507_02620_b200 import flowspec as F
    for j in range(1, len(plan)):
        gp.fs_submit_segment(F.FS_NEW_ROUND, [-1], [plan[j - 1]], [1.0], 1)
        while True:
            gp.fs_verify_step()
            d = gp.fs_accept()
            if d.progress:
                gp.fs_prune_and_compact(d)
                break
    return greedy_stream(gp, count)[1:]


def ours(args):
    import torch
    import torch.distributed as dist
    from paper_2507_02620_b200 import flowspec as F
    from synth import gen
    from synth.configs import SHAPES

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    P = world
    assert P == args.gpus or world == 1, "launch N>1 with torchrun"
    torch.cuda.set_device(local)
    nccl_id = None
    if P > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [F.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    wl = dict(WORKLOADS[args.workload])
    if args.real_prefill:
        wl["mode"] = "prefill"
    shape = SHAPES[wl["shape"]]
    ranks = wl["ranks"]
    a = len(ranks) - 1
    l_max, n_nodes, depth = wl["l_max"], wl["n_nodes"], wl["depth"]
    W, K = args.warmup, args.steps
    S = wl["scenario"] == "S"
    if S:   # steady state: the initial tree's segments drained and the pipeline full
        W = max(W, P + wl["n_nodes"] // wl["l_max"] + 2)
    n_rounds = 0 if S else W + 2 * K
    n_ticks = W + 2 * K if S else 0
    grow = (n_rounds * (a + 1)) if not S else (a + wl["q"] * (n_ticks + 4))
    max_ctx = wl["prefix"] + grow + 1200
    clocks = Clocks(local)   # nvidia-smi needs ~1 s to start sampling
    clocks.start()
    gp = F.Pipeline(shape, n_stages=P, rank=rank, max_ctx=max_ctx, max_live=512, max_seg=wl["max_seg"],
                    device=local, nccl_id=nccl_id, max_prefill=args.max_prefill)
    gp.fs_load_random_weights(SEED)
    prefix = gen.prefix_tokens(SEED, wl["prefix"], shape.vocab)
    inputs, plan_info = plan_schedule(gp, wl, prefix, shape, n_rounds, n_ticks)
    set_prefix(gp, wl, prefix)
    st = gp.stream

    if S:
        t0_tree, plan = inputs
        sr = SteadyRound(gp, t0_tree, Batches(gen.SteadyExpansion(SEED + 1, t0_tree, plan, wl["q"], 16,
                                                                  shape.vocab), n_ticks), l_max)

        def step(i):
            return sr.tick(), 1
    else:
        def step(i):
            return run_round(gp, inputs[i], l_max)

    for r in range(W):
        step(r)
    # host hygiene for both timed regions (as timeit does): no cyclic-GC pause
    # inside them (collected before the barrier, so no rank enters the timed
    # region late and makes its peers wait inside it)
    gc.collect()
    gc.disable()
    launches0 = gp.state()["launches"]
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.t_from = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    tokens = ticks = 0
    prunes0 = PRUNES[0]
    for r in range(W, W + K):
        c, t = step(r)
        tokens += c
        ticks += t
    prunes = PRUNES[0] - prunes0
    e1.record(st)
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()
    launches = gp.state()["launches"] - launches0
    dev_ms = e0.elapsed_time(e1)
    if P > 1:
        tt = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms = float(tt.item())
    value = tokens / (dev_ms / 1e3)

    # e2e: the next K steps through the public API, host wall clock, host
    # buffers in (tree arrays) / records out
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e_tokens = 0
    for r in range(W + K, W + 2 * K):
        c, _ = step(r)
        e_tokens += c
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if P > 1:
        tt = torch.tensor([wall], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        wall = float(tt.item())
    e2e = e_tokens / wall
    gc.enable()
    if S:
        sr.end()
    # keep the same load (one-node verify rounds) until the sampler has seen
    # a few samples since the timed region started
    hold_t0 = time.perf_counter()
    while True:
        more = clocks.count_since(clocks.t_from) < 4 and time.perf_counter() - hold_t0 < 3.0
        if P > 1:  # every rank must run the same number of collective ticks
            flag = torch.tensor([1 if more else 0], device="cuda")
            dist.broadcast(flag, src=0)
            more = bool(flag.item())
        if not more:
            break
        greedy_stream(gp, 4)
    if P > 1:
        dist.barrier()
    clk = clocks.stop()

    # chunked prefill of the workload's prefix (f3): CUDA events on the
    # library stream, max over ranks
    pre = None
    if wl["mode"] == "prefill":
        if P > 1:
            dist.barrier()
        torch.cuda.synchronize()
        pa, pb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pa.record(st)
        gp.fs_set_prefix(prefix, F.FS_PREFILL)
        pb.record(st)
        torch.cuda.synchronize()
        p_ms = pa.elapsed_time(pb)
        if P > 1:
            tt = torch.tensor([p_ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            p_ms = float(tt.item())
        fl = prefill_flops(shape, wl["prefix"])
        sus, sus_src = tflops_sustained()
        pre = {"tokens": wl["prefix"], "ms": round(p_ms, 3), "tok_per_s": round(wl["prefix"] / p_ms * 1e3, 1),
               "tflops": round(fl / p_ms / 1e9, 1), "peak_bf16_sustained": sus, "peak_source": sus_src,
               "frac": round(fl / p_ms / 1e9 / sus, 4), "chunk_rows": args.max_prefill, "stages": P,
               "note": "algorithmic FLOPs (2*params*tokens + causal attention + last-token head); the "
                       "GEMMs carry activations as a bf16 hi/lo pair, so the tensor pipe executes 2x"}

    # roofline of the dominant kernel (weight-streaming GEMM)
    hbm, bf16_tf, peak_src = peaks()
    prof = None
    if not args.no_profile:
        set_prefix(gp, wl, prefix)
        gp.set_profiling(True)
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev_a.record(st)
        if S:
            sr_p = SteadyRound(gp, t0_tree, gen.SteadyExpansion(SEED + 1, t0_tree, plan, wl["q"], 16,
                                                                shape.vocab), l_max)
            for _ in range(W + 4):
                sr_p.tick()
            p_ticks = W + 4
        else:
            _, p_ticks = run_round(gp, inputs[0], l_max)
        ev_b.record(st)
        torch.cuda.synchronize()
        if S:
            sr_p.end()
        step_ms = ev_a.elapsed_time(ev_b)
        gp.set_profiling(False)
        prof = gp.get_profile()
        prof["step_ms"] = step_ms
        # per-launch GEMM time with launches back to back (programmatic overlap
        # between consecutive launches as in the step; the event pairs above
        # serialise every launch): tick rows of a full prefill chunk
        set_prefix(gp, wl, prefix)
        if rank == 0:
            prof["b2b"] = gemm_back_to_back(gp, last=(P == 1))
            prof["attn_b2b"] = min((gp.bench_kernel(5, 20) for _ in range(3)), key=lambda x: x[0])

    if rank != 0:
        gp.close()
        return
    ceil = xi_ceiling(wl, P)
    model = {"7b": "LLaMA2-7B-shaped (L32 d4096 H32 ffn11008 V32000)",
             "13b": "LLaMA2-13B-shaped (L40 d5120 H40 ffn13824 V32000)",
             "72b": "Qwen2-72B-shaped (L80 d8192 H64/KV8 ffn29568 V152064, q/k/v bias)"}[wl["shape"]]
    wname = f"{args.workload}_{wl['shape']}_p{P}"
    if S:
        desc = (f"{wl['cfg']}: {model} bf16, {P} pipeline stage(s), prefix {wl['prefix']} "
                f"({'real prefill' if wl['mode'] == 'prefill' else 'synthetic KV'}), {n_nodes}-node initial "
                f"tree depth {depth}, L_max {l_max}, scenario S: one 16-node batch with q={wl['q']} planted "
                f"chain nodes appended per tick; a step = one pipeline tick")
    else:
        desc = (f"{wl['cfg']}: {model} bf16, {P} pipeline stage(s), prefix {wl['prefix']} "
                f"({'real prefill' if wl['mode'] == 'prefill' else 'synthetic KV'}), {n_nodes}-node draft "
                f"tree depth {depth}, L_max {l_max}, planted accept path a={a} (scenario R); a step = one "
                f"SD round")
    rec = {
        "metric": "accepted tokens/s (pipelined tree verify)",
        "value": round(value, 3),
        "unit": "tok/s",
        "n_gpus": P,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(dev_ms / K, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights, counter-generated prompt and planted draft trees)",
        "config": {
            "workload": f"{wname} — {desc}",
            "model": model + ", random init",
            "stages": P,
            "tree_nodes": n_nodes,
            "segment": l_max,
            "prefix": wl["prefix"],
            "scaling_note": "the same workload at every N (strong scaling: fixed work, P splits the "
                            "layer stack)",
            "l2": "inputs larger than L2: the weights stream from HBM every tick",
            "host": "Python cyclic GC disabled inside the timed regions (as timeit does)",
            "tokens_per_step": tokens / K,
            "ticks_per_step": ticks / K,
            "planted_stream": plan_info,
            "xi_ceiling": round(ceil, 1) if ceil else None,
            "frac_of_xi_ceiling": round(value / ceil, 4) if ceil else None,
        },
        "clocks": clk,
        "e2e": {"value": round(e2e, 3), "unit": "tok/s",
                "h2d_bytes_per_step": round(H2D_SUBMIT + H2D_PRUNE * prunes / K),
                "d2h_bytes_per_step": round(D2H_SUBMIT + D2H_TICK * ticks / K),
                "bytes_note": "the library's whole-struct copies per submit / tick / prune (bench.py "
                              "H2D_SUBMIT, D2H_TICK, ...), not just the live entries"},
        "gpu_launches": int(launches),
    }
    if pre:
        rec["prefill"] = pre
    if prof:
        g_ms = prof["gemm_ms"] / max(prof["gemm_launches"], 1)
        g_bytes = prof["gemm_bytes"] / max(prof["gemm_launches"], 1)
        ach_ev = g_bytes / (g_ms / 1e3) / 1e9
        b2b = prof["b2b"]
        n_l = gp.state()["layer_end"] - gp.state()["layer_begin"]
        cnt = {k: (1 if k == "head" else n_l) for k in b2b}
        b_bytes = sum(cnt[k] * b2b[k]["bytes"] for k in b2b)
        b_us = sum(cnt[k] * b2b[k]["us"] for k in b2b)
        ach = b_bytes / (b_us * 1e-6) / 1e9
        rec["roofline"] = {
            "kernel": "gemm_cluster_kernel / gemm_tc_kernel (tcgen05 weight-streaming GEMMs, all layers + head)",
            "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(ach / hbm, 4), "traffic": ncu_traffic(g_bytes), "peak_source": peak_src,
            "per_kernel": {k: {"us": round(v["us"], 2), "bytes": v["bytes"],
                               "GB/s": round(v["bytes"] / v["us"] / 1e3, 1)} for k, v in b2b.items()},
            "event_pairs": {"achieved": round(ach_ev, 1), "frac": round(ach_ev / hbm, 4),
                            "note": "event pair around every launch of a profiled step (serialises launches)"},
            "launches_per_step": round(prof["gemm_launches"] / max(p_ticks, 1) * (ticks / K)),
            "share_of_step": round(min(1.0, b_us * 1e-3 * (ticks / K) / (dev_ms / K)), 4),
            "attention": {
                "achieved": round(prof["attn_b2b"][1] / prof["attn_b2b"][0] / 1e3, 1),
                "us_per_layer": round(prof["attn_b2b"][0], 2),
                "frac": round(prof["attn_b2b"][1] / prof["attn_b2b"][0] / 1e3 / hbm, 4),
                "unit": "GB/s", "launches_per_step": round(prof["attn_launches"] / max(p_ticks, 1) * (ticks / K)),
                "event_pairs_achieved": round(prof["attn_bytes"] / max(prof["attn_ms"], 1e-9) / 1e6, 1),
                "share_of_step": round(prof["attn_ms"] / prof["step_ms"], 4)},
            "measured": "GEMM: per launch = CUDA events around 20 back-to-back launches of each "
                        "weight GEMM (layer 0 of this stage, real epilogues, one prefill-chunk tick), "
                        "weighted by launches per tick; bytes = weights (dominant). Attention: 20 "
                        "back-to-back launches of layer 0's attention at the bench shape",
        }
    if P == 1 and not args.no_cpu_baseline:
        t_first = inputs[0] if not S else t0_tree
        rec["cpu_baseline"] = cpu_baseline(shape, wl, t_first, prefix, tokens / K, ticks / K)
    gp.close()
    if P == 1 and not args.no_attn_long and "roofline" in rec:
        try:
            rec["roofline"]["attention_long_context"] = attention_long_context(hbm)
        except Exception as ex:   # informative only: never costs the main line
            rec["roofline"]["attention_long_context"] = {"error": str(ex)[:200]}
    emit(rec)


def ncu_traffic(alg_bytes_per_launch):
    """roofline.traffic: DRAM bytes (read + write) per GEMM launch, from the committed
    ncu --set full capture of the same build (profiles/r2_ncu_traffic.json: per-class
    DRAM / algorithmic bytes, weighted over a tick) applied to this run's average
    algorithmic bytes per launch; null when the capture is absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")) as f:
            ratio = float(json.load(f)["ratio_weighted_per_tick"])
        return round(alg_bytes_per_launch * ratio)
    except Exception:
        return None


def gemm_back_to_back(gp, last):
    """Per-launch time of each weight GEMM class (fs_bench_kernel kinds 0-4:
    QKV, O, gate/up, down, head) over 20 back-to-back launches, best of 3."""
    out = {}
    for k, name in ((0, "qkv"), (1, "o"), (2, "gate_up"), (3, "down"), (4, "head")):
        if name == "head" and not last:
            continue
        best = None
        for _ in range(3):
            us, by = gp.bench_kernel(k, 20)
            best = (us, by) if best is None or us < best[0] else best
        out[name] = {"us": best[0], "bytes": best[1]}
    return out


def attention_long_context(hbm):
    """Tree attention where its bytes matter ("attention GB/s is
    meaningful on configs 4-5"): one layer of the configs[3] (13B, 4096-token
    context, 16-row segment) and configs[4] (72B GQA, 16384-token context,
    32-row segment) shapes, synthetic-KV prefix, bench_kernel kind 5 = that
    layer's attention launches back to back (CUDA events).  Achieved = K + V
    bytes of the context / time."""
    from paper_2507_02620_b200 import flowspec as F
    from synth import gen
    from synth.configs import reduced
    out = []
    for name, cfg, ctx, seg in (("13b", "configs[3] 13B MHA", 4096, 16), ("72b", "configs[4] 72B GQA", 16384, 32)):
        shape = reduced(name, 1)
        gp = F.Pipeline(shape, max_ctx=ctx + 600, max_seg=seg)
        try:
            gp.fs_load_random_weights(SEED)
            gp.fs_set_prefix(gen.prefix_tokens(SEED, ctx, shape.vocab), F.FS_SYNTH_KV, kv_seed=7)
            t = gen.random_tree(3, seg, 6, shape.vocab, gp.state()["x_new"])
            gp.fs_submit_segment(F.FS_NEW_ROUND, t["parent"], t["token"], t["own"], seg)
            gp.fs_verify_step()
            us = min(gp.bench_kernel(5, 20)[0] for _ in range(3))
            n_keys = ctx + seg
            kv = n_keys * shape.n_kv_heads * shape.head_dim * 2 * 2
            gbs = kv / (us * 1e-6) / 1e9
            out.append({"config": f"{cfg}, {n_keys} keys, {seg} query rows", "us_per_layer": round(us, 2),
                        "kv_bytes": kv, "achieved": round(gbs, 1), "unit": "GB/s",
                        "frac": round(gbs / hbm, 4)})
        finally:
            gp.close()
    return out


# ------------------------------------------------------------------ oracle arm
def oracle_pass_seconds(shape, wl, tree, prefix):
    """Seconds of one oracle pass (as it stands: fp64, weights regenerated) of
    one L_max-row segment of the step's tree through the whole model at the
    workload's prefix length (synthetic prefix KV: a CPU prefill is not what
    is being timed).  Models above 20 B parameters are timed on 1- and
    2-layer versions of the same shape and extrapolated linearly in the layer
    count (the oracle's cost per layer is the same at every depth)."""
    from oracle.pipeline import OraclePipeline
    from synth.configs import reduced

    def one(sh):
        op = OraclePipeline(sh, SEED, n_stages=1, max_slots=len(prefix) + 600)
        op.set_prefix(prefix, mode="synth", kv_seed=7)
        t = dict(tree)
        t["token"] = list(t["token"])
        t["token"][0] = op.x_new
        op.submit(True, t["parent"], t["token"], t["own"], l_max=wl["l_max"])
        t0 = time.perf_counter()
        op.verify_step()
        return time.perf_counter() - t0

    if shape.n_params <= 20e9:
        return one(shape), f"one pass of the full {shape.n_layers}-layer model"
    t1 = one(reduced(wl["shape"], 1))
    t2 = one(reduced(wl["shape"], 2))
    est = t1 + (shape.n_layers - 1) * (t2 - t1)
    return est, (f"1- and 2-layer passes of the same shape ({t1:.1f} s, {t2:.1f} s) extrapolated to "
                 f"{shape.n_layers} layers")


def cpu_baseline(shape, wl, tree, prefix, tok_per_step, ticks_per_step):
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    t_seg, how = oracle_pass_seconds(shape, wl, tree, prefix)
    return {"value": round(tok_per_step / (ticks_per_step * t_seg), 5), "unit": "tok/s", "cores": threads,
            "kind": "oracle",
            "sample": f"{how}: one {wl['l_max']}-row segment at prefix {len(prefix)} (synthetic KV, "
                      f"fp64, weights regenerated); {t_seg:.2f} s/segment, converted with the GPU run's "
                      f"{tok_per_step:.2f} tokens and {ticks_per_step:.2f} segment passes per step"}


def reference(args):
    """--impl reference: the oracle as it stands, same metric / workload, rank 0
    only.  Each step = one oracle segment pass; a step of the workload is
    (tokens per step) over (segment passes per step) of them — scenario R: a+1
    tokens over the segments the planted path spans; scenario S: q per pass."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import gen
    from synth.configs import SHAPES
    wl = WORKLOADS[args.workload]
    shape = SHAPES[wl["shape"]]
    P = args.gpus
    ranks = wl["ranks"]
    a = len(ranks) - 1
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    prefix = gen.prefix_tokens(SEED, wl["prefix"], shape.vocab)
    stream = [0] + list(range(1, a + 3))
    tree = gen.planted_tree(SEED, wl["n_nodes"], wl["depth"], stream, ranks, shape.vocab)
    if wl["scenario"] == "S":
        tok_per_pass = float(wl["q"])
    else:
        tok_per_pass = (a + 1) / (ranks[-1] // wl["l_max"] + 1)
    secs, how = [], ""
    for i in range(args.warmup + args.steps):
        dt, how = oracle_pass_seconds(shape, wl, tree, prefix)
        if i >= args.warmup:
            secs.append(dt)
    tot = sum(secs)
    value = tok_per_pass * len(secs) / tot
    emit({
        "impl": "reference", "metric": "accepted tokens/s (pipelined tree verify)",
        "value": round(value, 5), "unit": "tok/s", "n_gpus": P, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(secs), 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.workload}_{wl['shape']}_p{P} (oracle, CPU)"},
        "cpu_baseline": {"value": round(value, 5), "unit": "tok/s", "cores": threads,
                         "kind": "oracle",
                         "sample": f"each step = {how} of a {wl['l_max']}-row segment at the workload's "
                                   f"prefix length (synthetic KV); {tok_per_pass:.2f} accepted tokens per "
                                   "pass as in the GPU step"},
        "e2e": {"value": round(value, 5), "unit": "tok/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    })


_JSON_OUT = None


def emit(rec):
    """The one JSON line of the contract, on the process's original stdout
    (everything else -- including C-level prints such as NCCL's version banner
    -- goes to stderr)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(rec) + "\n")
    out.flush()


def _route_stdout_to_stderr():
    global _JSON_OUT
    try:
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        _JSON_OUT = os.fdopen(saved, "w")
    except OSError:
        _JSON_OUT = None


if __name__ == "__main__":
    _route_stdout_to_stderr()
    args = parse()
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)
