/*
 * flowspec.h — C-ABI of the B200-native FlowSpec pipelined tree-verification
 * hot path (arXiv 2507.02620).  libflowspec.so, sm_100a.
 *
 * Citations: P:NNN = /root/reference/PAPER.md line NNN (section / equation);
 * R# = reading of DESIGN.md.
 *
 * Execution model: SPMD, one process per GPU, rank p = pipeline stage p
 * ("the base LLM is partitioned into N consecutive layer blocks").
 * Every rank makes the same sequence of calls with identical host inputs; the
 * draft tree is replicated on every rank ("all stages need to perform pruning
 * over its local replicas of T").  Calls marked COLLECTIVE communicate
 * over NCCL (NVLink); all other calls are local.
 *
 * Conventions
 *  - Return: FS_OK (0) or a negative FS_E* code; no exception crosses the ABI.
 *    A failing call leaves the state unchanged, except FS_ECUDA/FS_ENCCL which
 *    poison the context (every later call returns FS_EPOISONED).
 *  - Host arrays passed in are caller-owned and copied before return.  Output
 *    structs are caller-owned, fixed capacity.
 *  - Device memory comes only from the caller's arena (fs_config.arena, e.g.
 *    a torch.empty(uint8) tensor); the library allocates no device memory.
 *  - Work is issued on fs_config.stream; calls that return results to the host
 *    synchronise that stream before returning.
 *  - A context is single-owner and not thread-safe.
 */
#ifndef FLOWSPEC_H
#define FLOWSPEC_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define FS_OK 0
#define FS_EINVAL (-1)     /* bad argument / malformed tree */
#define FS_ENOMEM (-2)     /* arena too small */
#define FS_ESTATE (-3)     /* call not valid in the current state */
#define FS_ECAPACITY (-4)  /* max_ctx / max_live / max_seg exceeded */
#define FS_ECUDA (-5)      /* CUDA error: context poisoned */
#define FS_ENCCL (-6)      /* NCCL error: context poisoned */
#define FS_EPOISONED (-7)  /* an earlier CUDA/NCCL error poisoned the context */
#define FS_ERANGE (-8)     /* a value outside the range of a kernel-internal format (GQA
                              attention with fp16 P converts V to fp16: |V| >= 65536 or a
                              non-finite V); poisons the context */

#define FS_MAX_LIVE 512    /* hard cap on live draft nodes (ancestor bitsets) */
#define FS_MAX_SEG 64      /* hard cap on rows per segment */
#define FS_MAX_STAGES 8

/* Single-process transport between the stage contexts of one pipeline (one
 * context per stage, each driven by its own host thread, SPMD as with NCCL):
 * the collective calls (fs_set_prefix, fs_verify_step) exchange the hidden
 * rows p -> p+1 ("the intermediate result ... sent to V2") and the last
 * stage's row results as device-to-device copies ordered by CUDA events — the
 * same schedule and bytes as the NCCL path, so a P-stage pipeline runs (and is
 * tested) on one GPU.  Every stage's collective call must be in flight
 * concurrently (one thread per context); a peer that does not arrive within
 * 120 s fails the call with FS_ENCCL and poisons the context. */
typedef struct fs_local_group fs_local_group;
/* Create a group for n_stages contexts.  FS_EINVAL for n_stages outside
 * 2..FS_MAX_STAGES.  The caller owns it; destroy after every member context. */
int fs_local_group_create(int32_t n_stages, fs_local_group** out);
void fs_local_group_destroy(fs_local_group* g);

typedef struct fs_config {
  /* model shape (LLaMA2 / Qwen2 decoder, App. B.1; R19) */
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, ffn, vocab;
  int32_t qkv_bias;         /* 1: q/k/v projections carry a bias (Qwen2) */
  int32_t bf16;             /* 1: bf16 weights/activations, fp32 accumulate and
                               residual (precision contract R18); 0: fp32
                               everywhere, no TF32 */
  double rms_eps, rope_theta;
  /* pipeline */
  int32_t n_stages;         /* 1..FS_MAX_STAGES */
  int32_t rank;             /* this process' stage, 0..n_stages-1 */
  const int32_t* layers_per_stage; /* n_stages entries summing to n_layers, or
                               NULL = byte-balanced consecutive blocks (head
                               bytes counted on the last stage) */
  /* capacities */
  int32_t max_ctx;          /* KV slots (context + live drafts) */
  int32_t max_live;         /* live draft nodes, <= FS_MAX_LIVE, multiple of 32 */
  int32_t max_seg;          /* rows per segment / prefill chunk, <= FS_MAX_SEG */
  /* plumbing (PyTorch: device memory, stream, process group bootstrap) */
  int32_t device;
  void* arena;              /* device pointer, >= fs_arena_bytes(cfg) bytes, 256-B aligned */
  size_t arena_bytes;
  void* stream;             /* cudaStream_t the library issues all work on */
  const uint8_t* nccl_id;   /* 128-byte ncclUniqueId from rank 0 (n_stages > 1) */
  fs_local_group* local_group; /* n_stages > 1 without NCCL: all stages are
                               contexts of THIS process (same or peer-accessible
                               devices), the stage transport (a10) is a device
                               copy through the group.  Exactly one of nccl_id /
                               local_group must be set when n_stages > 1. */
  int32_t sampling;         /* 1: the last stage keeps every verified node's fp32
                               logits ([max_live][vocab], arena) so that
                               fs_set_acceptance can switch to stochastic
                               acceptance; 0: greedy only */
  int32_t max_prefill;      /* rows per prefill chunk (P:214 chunked prefill;
                               <= FS_MAX_SEG; 0 = max_seg).  Chunks run at their
                               own row width (GEMM N = 2 x 16/32/64) and are
                               pipelined over the stages: at step t stage p
                               processes chunk t - p. */
} fs_config;

typedef struct fs_ctx fs_ctx;

/* Bytes of device arena the configuration needs (weights of this rank's layer
 * block, KV cache, activations, tree state, workspaces).  0 if cfg invalid. */
size_t fs_arena_bytes(const fs_config* cfg);

/* Host only.  Layers per stage the configuration uses (cfg->layers_per_stage,
 * or the byte-balanced consecutive blocks, head bytes counted on the last
 * stage).  out: n_stages entries.  FS_EINVAL if invalid. */
int fs_layers_per_stage(const fs_config* cfg, int32_t* out);

/* Fill out[128] with a fresh ncclUniqueId (call on rank 0, broadcast it). */
int fs_nccl_unique_id(uint8_t* out);

/* Create a context.  Validates cfg (FS_EINVAL), checks the arena
 * (FS_ENOMEM), joins the NCCL communicator (or registers as stage `rank` of
 * cfg->local_group, FS_EINVAL if that rank is taken) when n_stages > 1. */
int fs_init(const fs_config* cfg, fs_ctx** out);

/* Fill this rank's weights (its layer block; embedding on stage 0; final norm
 * and head on the last stage) on the device with the counter-based generator
 * of DESIGN.md "Input recipe": uniform, std sigma, bf16 RNE.
 * No host buffers.  FS_ESTATE if called twice. */
int fs_load_random_weights(fs_ctx* ctx, uint64_t seed);

#define FS_PREFILL 0  /* chain-mask passes of <= max_seg rows (P:214 chunked prefill) */
#define FS_SYNTH_KV 1 /* slots [0,n-1) synthetic K/V, last token real (configs 4-5) */
/* COLLECTIVE.  Build the prefix KV cache and the first sampled token
 * (FS_PREFILL: chunks of cfg.max_prefill rows, causal, pipelined over the
 * stages — stage p runs chunk t - p at step t, hidden rows move p -> p+1 as
 * in a verify tick):
 * l_glo = n, *x_new_out = argmax of the last prefix token's logits
 * ("compute the initial KV cache and generate the first sampled token
 * x_new").  Drops any live round.  FS_EINVAL: n < 1, bad token, bad mode;
 * FS_ECAPACITY: n + max_live > max_ctx. */
int fs_set_prefix(fs_ctx* ctx, const int32_t* tok, int32_t n, int32_t mode,
                  uint64_t kv_seed, int32_t* x_new_out);

#define FS_NEW_ROUND 1 /* draft initialization step */
#define FS_APPEND 2    /* expansion: S <- S || S_app */
/* OR-ed into flags: order the batch breadth-first (depth asc, id asc) instead
 * of by cumulative score -- the "FlowSpec w/o Score-Based Draft" ablation
 * (Table 2; SPEC S:506 reading).
 * Still topological, so every prefix stays ancestor-closed. */
#define FS_ORDER_BFS 4
/* Expansion by tree merging (P:383-392 context-aware expansion; with L_top =
 * L_se the score-aware expansion of P:399-402): (parent, token, own) is a
 * tree T_new with parent indices WITHIN T_new (parent[0] = -1, parent[i] <
 * i), rooted at the current root token.  Nodes whose root path already
 * exists in the live tree are dropped (path-hash table + exact path check);
 * the new ones get ids next_id, next_id+1, ... in T_new order and are
 * appended like an APPEND batch (cumulative-score order in the merged tree,
 * optional top-L_top of them, own segments: S_mer = S_pr || S_app).
 * out->merged[i] = node id of T_new node i (existing or new). */
#define FS_MERGE 8
/* OR-ed into NEW_ROUND / APPEND flags (L_top 0): do not wait for the device.
 * The segments are enqueued from n alone; validation still runs on the device
 * and a rejected batch poisons the context at the next fs_verify_step
 * (FS_EPOISONED afterwards).  out (optional) then gets n, s_base and the
 * segment bounds but no order. */
#define FS_SUBMIT_ASYNC 16
typedef struct fs_submit_out {
  int32_t n;                     /* nodes added (after optional top-L) */
  int32_t s_base;                /* S index of the first added node */
  int32_t order[FS_MAX_LIVE];    /* node ids of the batch in S order */
  int32_t n_segs;                /* segments enqueued */
  int32_t seg_begin[FS_MAX_LIVE + 1]; /* S-index bounds, n_segs+1 entries */
  int32_t seg_id0;               /* id of the first enqueued segment */
  int32_t merged[FS_MAX_LIVE];   /* FS_MERGE: node id of every T_new node */
} fs_submit_out;
/* Local.  Submit a draft tree (NEW_ROUND) or an appended batch (APPEND) and
 * enqueue it as segments:
 *   Eq. 1: cu = own * cu(parent), fp32, root cu = 1 (R11);
 *   score order: cu descending, node id ascending (R10); optional
 *   top-L_top (L_top = 0: keep all); S-order prefixes are ancestor-closed
 *   (P:284);  segments: consecutive slices of <= L_max (R12); an
 *   appended batch forms its own segments;  positions pos = l_glo + depth
 *   (R4) and ancestor-or-self bitsets.
 * parent[i]: node id of the parent (NEW_ROUND: ids are 0..n-1, node 0 is the
 * root with parent -1 and token == current x_new; APPEND: ids continue the
 * round's sequence, parents are live ids or earlier ids of the batch);
 * token[i] vocabulary id; own[i] draft score in (0, 1].
 * FS_EINVAL: n < 1, L_max < 1 or > max_seg, L_top < 0, parent[i] >= id(i),
 * unknown/pruned parent, duplicate sibling token, own outside (0,1], bad
 * token, root token != x_new.  FS_ESTATE: APPEND without a live round,
 * NEW_ROUND while a round is live.  FS_ECAPACITY: live nodes > max_live. */
int fs_submit_segment(fs_ctx* ctx, int32_t flags, const int32_t* parent,
                      const int32_t* token, const float* own, int32_t n,
                      int32_t L_top, int32_t L_max, fs_submit_out* out);

typedef struct fs_step_out {
  int32_t seg_id;            /* segment that left the last stage, -1 if none */
  int32_t s_begin, n_rows;   /* its S range (n_rows 0: pruned-empty bubble) */
  int32_t node[FS_MAX_SEG];  /* node ids of the rows */
  int32_t am[FS_MAX_SEG];    /* greedy target token (argmax, lowest id on ties) */
  float margin[FS_MAX_SEG];  /* top-1 minus top-2 logit */
} fs_step_out;
/* COLLECTIVE.  One pipeline tick (P:228 step-wise pipelined verification):
 * stage 0 takes the next queued segment; every stage runs its in-flight
 * segment through its layer block (tree-masked attention over the prefix KV
 * plus ancestor drafts), hidden rows move p -> p+1 (NCCL send/recv);
 * the last stage computes final norm + head + argmax/top-2 (R7) and the
 * per-row results are broadcast to every rank.  Every rank gets the same
 * *out. */
int fs_verify_step(fs_ctx* ctx, fs_step_out* out);

/* Optional parity readback: device buffer of rows_cap x vocab fp32 where the
 * last stage writes the logits of each verified segment (NULL disables). */
int fs_set_logits_buffer(fs_ctx* ctx, float* dev_logits, int32_t rows_cap);

typedef struct fs_accept_out {
  int32_t progress;          /* 0: the current root is not verified yet (R23) */
  int32_t n_acc;             /* |S_acc|, root included (R2) */
  int32_t acc_ids[FS_MAX_LIVE];
  int32_t acc_tokens[FS_MAX_LIVE];
  int32_t x_new;             /* token sampled after S_acc */
  int32_t n_new;             /* node id with path S_acc||x_new, or -1 */
  int32_t cont;              /* Eq. 2 continuous condition */
  int32_t n_flagged;         /* walked nodes with top-2 margin < 1e-2 */
  int32_t flagged_ids[FS_MAX_LIVE];
} fs_accept_out;
#define FS_ACCEPT_GREEDY 0
#define FS_ACCEPT_STOCHASTIC 1
/* Acceptance rule of the following rounds (no live round: FS_ESTATE).
 * GREEDY (default): child c of v is accepted iff token(c) = argmax of v
 * (R1).  STOCHASTIC: multi-branch speculative rejection sampling at
 * temperature `temperature` > 0 ("aligned distribution", Table 1 T=1,
 * P:461; reading R24): at the walk's node v, p = softmax(logits_v / T) and
 * q = row node_id(v) of q_dev; children in draw order (node id ascending)
 * are accepted iff u < p(t)/q(t), else p <- norm(max(p - q, 0)),
 * q(t) <- 0, q <- norm(q); all rejected: x_new ~ p and the round exits.
 * u = mix(mix(seed ^ 0x5EED5A3C) ^ (node_id * 2^16 + attempt)) >> 40 / 2^24.
 * The walk runs in the verify step on the last stage (its logits) and its
 * decision is broadcast with the row results; fs_accept returns it until the
 * tree changes.  Nodes whose decision margin (|u - ratio|, or the sample's
 * distance to a CDF boundary) is below 1e-6 are flagged.
 * q_dev: DEVICE, caller-owned, [q_rows][vocab] fp32, row = node id of the
 * round (every node that has children needs its row before that node's
 * segment is verified); fs_submit_segment fails with FS_ECAPACITY for node
 * ids >= q_rows.  STOCHASTIC needs cfg.sampling = 1 (FS_ESTATE otherwise).
 * The prefix's first token x_new stays the argmax (fs_set_prefix). */
int fs_set_acceptance(fs_ctx* ctx, int32_t mode, float temperature, uint64_t seed,
                      const float* q_dev, int32_t q_rows);

/* Local (deterministic on replicated state, so every rank computes the same
 * record).  Greedy acceptance + Eq. 2 over all verified nodes (R1,
 * R3): from the root, descend while the child carrying the argmax exists and
 * is verified.  Stochastic mode (fs_set_acceptance): returns the decision the
 * last verify step took (FS_ESTATE if the tree changed under a verified root
 * since then). */
int fs_accept(fs_ctx* ctx, fs_accept_out* out);

/* Local.  Apply a decision (normally fs_accept's; the parity harness may pass
 * the oracle's after a flagged near-tie):
 *  cont = 1: tree pruning: I_retain = I_acc ∪ I_pr; each stage keeps
 *    retained draft KV rows (I_incache) by a stable
 *    stream-compaction gather slot l_glo+i -> l_glo+rank(i), prunes its
 *    in-flight hidden rows and queued segments (I_local),
 *    re-roots S at n_new, then l_glo += |S_acc|.
 *  cont = 0: round exit: S_acc becomes context, everything else drops.
 * FS_ESTATE: no live round, progress = 0, ids not live, S_acc not a root path,
 * n_new not a child of the last accepted node. */
int fs_prune_and_compact(fs_ctx* ctx, const fs_accept_out* decision);

/* ---- parity / introspection ---- */
typedef struct fs_state {
  int32_t l_glo, x_new, live, n_live, next_id;
  int32_t n_stages, rank, layer_begin, layer_end;
  int32_t n_cached[FS_MAX_STAGES];   /* per stage: S indices < n_cached have KV */
  int32_t layers_per_stage[FS_MAX_STAGES];
  int32_t n_queue;                   /* queued (undispatched) segments */
  int32_t queue[FS_MAX_LIVE][3];     /* {seg_id, s_begin, s_end} */
  int32_t inflight[FS_MAX_STAGES][3];/* segment each stage runs next tick, seg_id -1 = none */
  uint64_t launches;                 /* kernels this rank launched so far */
} fs_state;
#define FS_Q_STATE 0   /* fs_state */
#define FS_Q_NODE 1    /* int32[n_live] node ids in S order */
#define FS_Q_TOKEN 2   /* int32[n_live] */
#define FS_Q_PARENT 3  /* int32[n_live] parent S index (-1 root) */
#define FS_Q_POS 4     /* int32[n_live] l_glo + depth */
#define FS_Q_ANC 5     /* uint32[n_live][max_live/32] ancestor-or-self bitsets */
#define FS_Q_CU 6      /* float[n_live] cumulative scores relative to the root */
#define FS_Q_RETAIN 7  /* uint32[max_live/32] I_retain of the last prune */
/* Copy item `what` into buf (bytes capacity); *needed receives the size. */
int fs_query(fs_ctx* ctx, int32_t what, void* buf, size_t bytes, size_t* needed);

/* Read one K (which=0) or V (which=1) row (head_dim values as fp32) of a
 * layer owned by this rank.  FS_EINVAL otherwise. */
int fs_read_kv(fs_ctx* ctx, int32_t layer, int32_t which, int32_t kv_head,
               int32_t slot, float* out);

/* Test hook: overwrite one K (which=0) or V (which=1) row of a layer owned by
 * this rank with `in` (head_dim fp32 values, rounded to the cache format,
 * bf16 round-to-nearest-even).  Synchronous.  FS_EINVAL on a bad index. */
int fs_debug_write_kv(fs_ctx* ctx, int32_t layer, int32_t which, int32_t kv_head,
                      int32_t slot, const float* in);

/* ---- measurement ---- */
typedef struct fs_profile {
  uint64_t gemm_launches;   /* tcgen05 weight-GEMM launches (bf16) / fp32 GEMMs */
  double gemm_ms;           /* sum of their CUDA-event durations */
  double gemm_bytes;        /* algorithmic bytes: weights + bf16 activation
                               pair (2 x npad x K x 2) + outputs (rows x N x 4) */
  uint64_t attn_launches;   /* tree-attention launches (split-KV kernel) */
  double attn_ms;
  double attn_bytes;        /* K and V rows of all visible-key chunks + Q + partials */
} fs_profile;
/* on != 0: record a CUDA event pair (on the library stream) around every
 * weight-GEMM and attention launch; off by default (no events recorded). */
int fs_set_profiling(fs_ctx* ctx, int32_t on);
/* Synchronise, sum the recorded event pairs into *out and reset. */
int fs_get_profile(fs_ctx* ctx, fs_profile* out);

/* Kernel microbenchmark on the rows of the last tick / prefill chunk:
 * kind 0..3 = layer-0 QKV / O / gate-up / down GEMM, 4 = head GEMM (last
 * stage), 5 = layer-0 attention, 6 = RMSNorm, 7 = whole stage forward.
 * Launches back to back `iters` times on the library stream and returns the
 * mean CUDA-event time per launch in *us and the algorithmic bytes per
 * launch in *bytes.  Overwrites activations (not the KV context).  kind |
 * FS_BENCH_WIDE runs them at the prefill-chunk width on the rows of the last
 * prefill chunk (f3 measurements).  11 = the stochastic accept walk on the
 * live tree (f2; *bytes = the bytes read per walked node), 12 = the merge
 * kernel on the last FS_MERGE batch (f4).  Kinds 8-10
 * (timeline probes, printed to stderr) exist only in a -DFS_DIAG build, which
 * allocates its probe buffers; the product build allocates no device memory. */
#define FS_BENCH_WIDE 0x100
int fs_bench_kernel(fs_ctx* ctx, int32_t kind, int32_t iters, double* us, double* bytes);

/* GEMM numerics check (layer `layer` of this rank, which = 0 QKV, 1 O,
 * 2 gate/up (interleaved rows), 3 down, 4 head): X (host, n x K fp32, n <=
 * max_seg) is staged as the bf16 hi/lo activation pair, Y_dev (DEVICE,
 * caller-allocated, n x N_out fp32) receives the raw GEMM output (no
 * epilogue).  Synchronous.  bf16 configs only. */
int fs_debug_gemm(fs_ctx* ctx, int32_t layer, int32_t which, const float* X, int32_t n, float* Y_dev);

void fs_destroy(fs_ctx* ctx);
const char* fs_last_error(const fs_ctx* ctx);
const char* fs_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif
