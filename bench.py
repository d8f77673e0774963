"""Benchmark: accepted tokens/s of pipelined tree verification (FlowSpec hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 runs BASELINE.json configs[1] (LLaMA2-7B-shaped bf16, prefix 1024 with a
real prefill, 64-node draft trees, segments of 16, planted accept path a=4).
N>1 (torchrun, one rank per GPU) runs the same model as an N-stage pipeline
(configs[2] planting: a=6, two planted nodes per segment over segments 0-2).
A step is one SD round: submit the tree, pipeline ticks (verify_step), accept,
prune/compact, until the continuous condition fails (§3.1-3.3).

Draft trees are synthetic: the planted path comes from the model's own greedy
stream, produced before the timed region by autoregressive decoding through
the same public API (a stand-in for the paper's draft model, which is out of
scope).  Weights (13.5 GB) >> L2 (126 MB): every step streams them from HBM.
"""
import argparse
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shape", default="7b")
    ap.add_argument("--prefix", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--no-attn-long", action="store_true")
    return ap.parse_args()


def workload(P):
    if P == 1:
        return dict(name="cfg2_7b_p1", ranks=(0, 2, 5, 17, 21))
    return dict(name=f"cfg3_7b_p{P}", ranks=(0, 3, 9, 18, 25, 33, 40))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), float(m["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


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
# 512, FS_MAX_SEG 64): SubmitIn (5 ints + parent / token / own [512]) host ->
# device per submit; the submit record prefix (11 ints + order [512]) back;
# the verify step's record (11 ints, 5 x [512] arrays, prune plan 1 + [512],
# 64 row results of 8 B and 64 node ids) back per tick; DecisionIn (4 ints +
# acc ids [512]) host -> device per prune
H2D_SUBMIT = 4 * (5 + 3 * 512)
D2H_SUBMIT = 4 * (11 + 512)
D2H_TICK = 4 * (11 + 5 * 512 + 1 + 512) + 64 * 8 + 64 * 4
H2D_PRUNE = 4 * (4 + 512)


def run_round(gp, tree, l_max, tokens_out=None):
    """One SD round: submit, ticks, accept, prune until the round exits."""
    from paper_2507_02620_b200 import flowspec as F
    gp.fs_submit_segment(F.FS_NEW_ROUND, tree["parent"], tree["token"], tree["own"], l_max)
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


def plan_schedule(gp, prefix, ranks, n_rounds, n_nodes, depth, l_max, shape, max_iter=6):
    """Draft-provider stand-in: trees whose planted path is the model's greedy
    continuation.  The plan starts as an AR greedy stream; each untimed dry run
    of all rounds replaces it with the stream tree verification actually
    commits (a flagged near-tie can make it differ from the AR stream) plus an
    AR continuation, until a dry run follows its plan.  The timed rounds then
    replay exactly these trees from the same prefix (deterministic)."""
    from paper_2507_02620_b200 import flowspec as F
    from synth import gen
    a = len(ranks) - 1
    need = n_rounds * (a + 1) + a + 2
    plan = greedy_stream(gp, need)
    trees, diverged = [], 0
    for it in range(max_iter):
        gp.fs_set_prefix(prefix, F.FS_PREFILL)
        trees, committed, diverged = [], [], 0
        for r in range(n_rounds):
            c = len(committed)
            root = gp.state()["x_new"]
            if c + a + 2 <= len(plan) and plan[c] == root:
                t = gen.planted_tree(SEED + r, n_nodes, depth, plan[c:c + a + 2], ranks, shape.vocab)
            else:  # off plan: unplanted tree rooted at the actual next token
                diverged += 1
                t = gen.random_tree(SEED + 7 * r, n_nodes, depth, shape.vocab, root)
            trees.append(t)
            run_round(gp, t, l_max, committed)
        if diverged == 0 and committed == plan[:len(committed)]:
            return trees, 0, it + 1
        plan = committed + greedy_stream(gp, need)
    return trees, diverged, max_iter


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
    shape = SHAPES[args.shape]
    wl = workload(P)
    ranks = wl["ranks"]
    a = len(ranks) - 1
    l_max, n_nodes, depth = 16, 64, 6
    W, K = args.warmup, args.steps
    max_ctx = args.prefix + (W + 2 * K + 4) * (a + 1) + 600
    clocks = Clocks(local)   # nvidia-smi needs ~1 s to start sampling
    clocks.start()
    gp = F.Pipeline(shape, n_stages=P, rank=rank, max_ctx=max_ctx, max_live=512, max_seg=16,
                    device=local, nccl_id=nccl_id)
    gp.fs_load_random_weights(SEED)
    prefix = gen.prefix_tokens(SEED, args.prefix, shape.vocab)
    gp.fs_set_prefix(prefix, F.FS_PREFILL)
    n_rounds = W + 2 * K
    trees, diverged, dry_runs = plan_schedule(gp, prefix, ranks, n_rounds, n_nodes, depth, l_max, shape)
    gp.fs_set_prefix(prefix, F.FS_PREFILL)

    def round_r(r):
        return run_round(gp, trees[r], l_max)

    st = gp.stream
    for r in range(W):
        round_r(r)
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = gp.state()["launches"]
    clocks.t_from = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    tokens = ticks = 0
    prunes0 = PRUNES[0]
    for r in range(W, W + K):
        c, t = round_r(r)
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

    # e2e: same rounds through the public API, host wall clock, host buffers in / records out
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e_tokens = 0
    for r in range(W + K, W + 2 * K):
        c, _ = round_r(r)
        e_tokens += c
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if P > 1:
        tt = torch.tensor([wall], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        wall = float(tt.item())
    e2e = e_tokens / wall
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

    # roofline of the dominant kernel (weight-streaming GEMM): CUDA-event pairs
    # around every GEMM / attention launch over K profiled rounds
    hbm, bf16_tf, peak_src = peaks()
    prof = None
    if not args.no_profile:
        gp.fs_set_prefix(prefix, F.FS_PREFILL)
        gp.set_profiling(True)
        ptree = trees[0]
        p_t0 = time.perf_counter()
        ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev_a.record(st)
        run_round(gp, ptree, l_max)
        ev_b.record(st)
        torch.cuda.synchronize()
        step_ms = ev_a.elapsed_time(ev_b)
        gp.set_profiling(False)
        prof = gp.get_profile()
        prof["step_ms"] = step_ms
        # per-launch GEMM time with launches back to back (programmatic overlap
        # between consecutive launches as in the step; the event pairs above
        # serialise every launch): tick rows of a full 16-row prefill chunk
        gp.fs_set_prefix(prefix, F.FS_PREFILL)
        if rank == 0:
            prof["b2b"] = gemm_back_to_back(gp, last=(P == 1))
            prof["attn_b2b"] = min((gp.bench_kernel(5, 20) for _ in range(3)), key=lambda x: x[0])

    if rank != 0:
        return
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
            "workload": wl["name"] + f": LLaMA2-7B-shaped bf16, {P} pipeline stage(s), prefix "
                        f"{args.prefix} (real prefill), {n_nodes}-node draft tree depth {depth}, "
                        f"L_max {l_max}, planted accept path a={a}",
            "model": "LLaMA2-7B-shaped (L32 d4096 H32 ffn11008 V32000), random init",
            "stages": P,
            "tree_nodes": n_nodes,
            "segment": l_max,
            "prefix": args.prefix,
            "l2": "inputs larger than L2: 13.5 GB of weights stream from HBM every step",
            "tokens_per_step": tokens / K,
            "ticks_per_step": ticks / K,
            "planted_path_divergences": diverged,
            "schedule_dry_runs": dry_runs,
        },
        "clocks": clk,
        "e2e": {"value": round(e2e, 3), "unit": "tok/s",
                "h2d_bytes_per_step": round(H2D_SUBMIT + H2D_PRUNE * prunes / K),
                "d2h_bytes_per_step": round(D2H_SUBMIT + D2H_TICK * ticks / K),
                "bytes_note": "the library's whole-struct copies per submit / tick / prune (bench.py "
                              "H2D_SUBMIT, D2H_TICK, ...), not just the live entries"},
        "gpu_launches": int(launches),
    }
    if prof:
        g_ms = prof["gemm_ms"] / max(prof["gemm_launches"], 1)
        g_bytes = prof["gemm_bytes"] / max(prof["gemm_launches"], 1)
        ach_ev = g_bytes / (g_ms / 1e3) / 1e9
        b2b = prof["b2b"]
        n_l = shape.n_layers // P
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
                            "note": "event pair around every launch of a profiled round (serialises launches)"},
            "launches_per_step": prof["gemm_launches"],
            "share_of_step": round(min(1.0, b_us * 1e-3 * (ticks / K) / (dev_ms / K)), 4),
            "attention": {
                "achieved": round(prof["attn_b2b"][1] / prof["attn_b2b"][0] / 1e3, 1),
                "us_per_layer": round(prof["attn_b2b"][0], 2),
                "frac": round(prof["attn_b2b"][1] / prof["attn_b2b"][0] / 1e3 / hbm, 4),
                "unit": "GB/s", "launches_per_step": prof["attn_launches"],
                "event_pairs_achieved": round(prof["attn_bytes"] / max(prof["attn_ms"], 1e-9) / 1e6, 1),
                "share_of_step": round(prof["attn_ms"] / prof["step_ms"], 4)},
            "measured": "GEMM: per launch = CUDA events around 20 back-to-back launches of each "
                        "weight GEMM (layer 0 of this stage, real epilogues, 16-row tick), weighted "
                        "by launches per tick; bytes = weights (dominant). Attention: 20 back-to-back launches "
                        "of layer 0's attention at the bench shape (1024-token context, 16 rows)",
        }
    if P == 1 and not args.no_cpu_baseline:
        rec["cpu_baseline"] = cpu_baseline(shape, trees[0], prefix, ranks, tokens / K, ticks / K,
                                           n_samples=1)
    gp.close()
    if P == 1 and not args.no_attn_long and "roofline" in rec:
        try:
            rec["roofline"]["attention_long_context"] = attention_long_context(hbm)
        except Exception as ex:   # informative only: never costs the main line
            rec["roofline"]["attention_long_context"] = {"error": str(ex)[:200]}
    emit(rec)


def ncu_traffic(alg_bytes_per_launch):
    """roofline.traffic: DRAM bytes (read + write) per GEMM launch, from the committed
    ncu --set full capture of the same build (profiles/r1_ncu_traffic.json: per-class
    DRAM / algorithmic bytes, weighted over a tick) applied to this run's average
    algorithmic bytes per launch; null when the capture is absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_ncu_traffic.json")) as f:
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
def oracle_segment_seconds(shape, tree, prefix, n_samples, n_rows=16):
    """Time the oracle as it stands verifying segments of the round's tree
    (synthetic prefix KV of the same length, 16-row segments)."""
    from oracle.pipeline import OraclePipeline
    op = OraclePipeline(shape, SEED, n_stages=1, max_slots=len(prefix) + 600)
    op.set_prefix(prefix, mode="synth", kv_seed=7)
    t = dict(tree)
    t["token"] = list(t["token"])
    t["token"][0] = op.x_new
    op.submit(True, t["parent"], t["token"], t["own"], l_max=n_rows)
    times = []
    for _ in range(n_samples):
        if not op.queue:
            break
        t0 = time.perf_counter()
        op.verify_step()
        times.append(time.perf_counter() - t0)
    return times


def cpu_baseline(shape, tree, prefix, ranks, tok_per_round, ticks_per_round, n_samples=1):
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    times = oracle_segment_seconds(shape, tree, prefix, n_samples)
    t_seg = sum(times) / len(times)
    segs = ticks_per_round  # P = 1: one segment pass per tick
    return {"value": round(tok_per_round / (segs * t_seg), 5), "unit": "tok/s", "cores": threads,
            "kind": "oracle",
            "sample": f"{len(times)} oracle pass(es) of one 16-row segment through the full "
                      f"{shape.n_layers}-layer model (weights regenerated, fp64) at prefix "
                      f"{len(prefix)} (synthetic KV); {t_seg:.2f} s/segment, converted with the "
                      f"GPU run's {tok_per_round:.2f} tokens and {segs:.2f} segment passes per round"}


def reference(args):
    """--impl reference: the oracle as it stands, same metric/config, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import gen
    from synth.configs import SHAPES
    shape = SHAPES[args.shape]
    P = args.gpus
    wl = workload(P)
    ranks = wl["ranks"]
    a = len(ranks) - 1
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    prefix = gen.prefix_tokens(SEED, args.prefix, shape.vocab)
    stream = [0] + list(range(1, a + 3))
    tree = gen.planted_tree(SEED, 64, 6, stream, ranks, shape.vocab)
    from oracle.pipeline import OraclePipeline
    op = OraclePipeline(shape, SEED, n_stages=1, max_slots=args.prefix + 600)
    op.set_prefix(prefix, mode="synth", kv_seed=7)
    tree["token"] = list(tree["token"])
    tree["token"][0] = op.x_new
    # one oracle step = one 16-row segment pass; a round of this workload is
    # (a+1) tokens over 2 segment passes at P=1 (P stages: same passes, no overlap on CPU)
    tok_per_pass = (a + 1) / (2 if P == 1 else 3)
    secs = []
    for i in range(args.warmup + args.steps):
        if not op.queue and not any(s is not None for s in op.slot):
            op.live = False
            op._reset_round()
            op.submit(True, tree["parent"], tree["token"], tree["own"], l_max=16)
        t0 = time.perf_counter()
        op.verify_step()
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            secs.append(dt)
    tot = sum(secs)
    value = tok_per_pass * len(secs) / tot
    emit({
        "impl": "reference", "metric": "accepted tokens/s (pipelined tree verify)",
        "value": round(value, 5), "unit": "tok/s", "n_gpus": P, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(secs), 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": wl["name"] + " (oracle, CPU)"},
        "cpu_baseline": {"value": round(value, 5), "unit": "tok/s", "cores": threads,
                         "kind": "oracle",
                         "sample": "each step = one oracle pass of a 16-row segment through the "
                                   "full model at the workload's prefix length (synthetic KV); "
                                   f"{tok_per_pass:.2f} accepted tokens per pass as in the round"},
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
