// api.cu — the fs_* C-ABI (include/flowspec.h): per-rank stage runtime, tick
// scheduler, NCCL stage transport and the launch sequences of the kernels.
//
// Host code here does bookkeeping only (which segment each stage runs this
// tick, arena carving, argument marshalling); every step of the path —
// tree metadata, decoder layers, argmax, acceptance, pruning, compaction —
// runs in the kernels of k_*.cuh.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <deque>
#include <string>
#include <vector>

#include "../../include/flowspec.h"
#include "common.cuh"
#include "k_fwd.cuh"
#include "k_gemm.cuh"
#include "k_attn_tc.cuh"
#include "k_attn_mha.cuh"
#include "k_gen.cuh"
#include "k_tree.cuh"
#include "k_sample.cuh"
#include "state.cuh"

using namespace fs;

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

struct Seg {
  int id = -1, b = 0, e = 0;
  bool valid() const { return id >= 0; }
  int n() const { return e - b; }
};

struct GemmOp {
  CUtensorMap ta, tb;   // weights, bf16 hi/lo activations
  GemmShape sh;
  int grid = 0;
  int split = 0;        // > 0: cluster split-K with this many CTAs per tile
  bool ok = false;
};

struct LayerW {
  void *wqkv = nullptr, *bqkv = nullptr, *wo = nullptr, *wgu = nullptr, *wd = nullptr;
  void *g1 = nullptr, *g2 = nullptr;
  GemmOp qkv, o, gu, dn;
  GemmOp qkv_w, o_w, gu_w, dn_w;   // the other row width (prefill chunks vs tree segments; use_width)
  CUtensorMap tk, tv;   // this layer's K / V cache planes [Hkv * max_ctx][128] (GQA tcgen05 attention)
  CUtensorMap mk, mv;   // the same planes in 64-key boxes (MHA attention, TMA ring)
};

}  // namespace

// Single-process stage transport (include/flowspec.h fs_local_group): a
// channel per (src, dst) pair carries one posted buffer at a time; the
// receiver pulls it with a device copy on its own stream after the sender's
// ready event and acknowledges with its own done event, on which the sender's
// stream then waits (the sender may not overwrite the buffer before the copy).
struct fs_local_group {
  int P = 0;
  std::mutex mu;
  std::condition_variable cv;
  struct Chan {
    uint64_t posted = 0, taken = 0;
    const void* ptr = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr, done = nullptr;
  } ch[FS_MAX_STAGES][FS_MAX_STAGES];
  fs_ctx* member[FS_MAX_STAGES] = {};
};

struct fs_ctx {
  fs_config cfg;
  int lps[FS_MAX_STAGES];
  int P = 1, rank = 0, L0 = 0, L1 = 0, nl = 0;
  bool first = true, last = true, bf = true;
  int esz = 2, npad = 16, n_sms = 148, ancw = 16, max_ids = 65536, gemm_ctas = 2;
  // row widths: tree segments (npad of max_seg) and prefill chunks (npad of
  // max_prefill); buffers are carved for the larger, GemmOps exist for both
  int npad_tick = 16, npad_pre = 16, ctas_tick = 2, ctas_pre = 2;
  bool wide = false;                // the prefill-chunk width is active
  int att_dbg_ends = 0;
  int att_nsplit[3] = {0, 0, 0};   // MHA attention key splits per m-tile count (planned once)
  int mha_nsplit[5] = {0, 0, 0, 0, 0};   // TMA MHA attention: splits per m-tile count (SM-count sized)
  cudaStream_t st = nullptr;
  ncclComm_t comm = nullptr;
  fs_local_group* lg = nullptr;           // single-process stage transport (else NCCL)
  cudaEvent_t ev_ready = nullptr;         // local transport: this rank's outgoing data ready
  cudaEvent_t ev_sub = nullptr;           // the last submit's host -> device copy (async submits)
  cudaEvent_t ev_done[FS_MAX_STAGES] = {}; // local transport: copy from rank q finished
  // arena
  char* base = nullptr;
  size_t off = 0, cap = 0;
  // weights
  std::vector<LayerW> lw;
  void *emb = nullptr, *wh = nullptr, *gf = nullptr;
  GemmOp head, head_w;
  // kv / rope
  char* kv = nullptr;
  size_t kv_plane_elems = 0;  // Hkv * max_ctx * hd
  float2* rope = nullptr;
  // activations
  float *x = nullptr, *hin = nullptr, *yf = nullptr;
  void *y = nullptr, *q = nullptr, *att = nullptr, *act = nullptr;
  float *gws = nullptr;
  float* ssq = nullptr;   // [d/32][npad] per-32-column sums of squares of the residual
  int* gcnt = nullptr;
  Top2* head_part = nullptr;
  RowResult* res = nullptr;
  float *aws_o = nullptr, *aws_ml = nullptr;
  int* att_cnt = nullptr;
  unsigned long long* att_dbg = nullptr;  // FS_ATT_DEBUG diagnostics only
  unsigned long long* gemm_dbg = nullptr;
  unsigned long long* tl_buf = nullptr;     // timeline diagnostics (fs_bench_kernel kind 8)
  std::vector<std::string> tl_names;
  // CUDA graph of one tick's stage forward (replayed every tick)
  cudaGraphExec_t fwd_exec = nullptr;
  uint64_t fwd_kernels = 0;
  float* fwd_logits = nullptr;
  int fwd_mha_tma = -1;   // the MHA kernel choice baked into the graph (by context length)
  bool use_graph = true;
  int att_chunk_cap = 0;
  size_t gws_floats = 0;
  // tree
  TreeDev tree;
  SubmitIn* d_sub = nullptr;
  SubmitIn* d_sub2 = nullptr;   // merge: the APPEND batch of T_new's new nodes
  DecisionIn* d_dec = nullptr;
  TreeRecord* d_rec = nullptr;
  TickRows* d_rows = nullptr;
  // pinned host staging
  SubmitIn* h_sub = nullptr;
  DecisionIn* h_dec = nullptr;
  TreeRecord* h_rec = nullptr;
  TickRows* h_rows = nullptr;
  RowResult* h_res = nullptr;
  int32_t* h_node = nullptr;
  // schedule (replicated on every rank)
  int l_glo = 0, x_new = -1, live = 0, n_live = 0, next_id = 0, seg_counter = 0;
  // the accept walk (a12) enqueued by verify_step right after the commit; its
  // record in h_rec is valid until the tree changes (submit / prune / prefix)
  bool acc_ready = false;
  std::deque<Seg> queue;
  Seg slot[FS_MAX_STAGES];
  int n_cached[FS_MAX_STAGES] = {0};
  bool weights = false, poisoned = false, prefixed = false;
  bool plan_ready = false;   // h_rec->spec_* match the tree (set by the verify step's accept)
  std::string err;
  uint64_t launches = 0;
  float* logits_buf = nullptr;
  int logits_cap = 0;
  // stochastic acceptance (k_sample.cuh): per-S-index logits of verified nodes
  // (last stage, cfg.sampling), fp64 walk scratch, the broadcast decision
  float* lstore = nullptr;
  double *samp_r = nullptr, *samp_q = nullptr;
  SampleDecision* dec = nullptr;
  int samp_mode = 0;          // 0 greedy, 1 stochastic
  double inv_temp = 1.0;
  uint64_t samp_seed = 0;
  const float* q_dev = nullptr;
  int q_rows = 0;
  // profiling: event pairs around GEMM / attention launches
  bool prof = false;
  // FS_XCHG_TIMING (diagnostics): CUDA-event pairs around every NCCL tick exchange and
  // every stage forward, summarised to stderr at fs_destroy
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> xt_x, xt_f;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, double>> ev_used;  // (kind 0 gemm / 1 attn, bytes) per pair
  size_t ev_next = 0;
};

namespace {


int fail(fs_ctx* c, int code, const char* msg) {
  if (c) c->err = msg;
  return code;
}

#define CK_CUDA(c, expr)                                                    \
  do {                                                                      \
    cudaError_t e_ = (expr);                                                \
    if (e_ != cudaSuccess) {                                                \
      (c)->poisoned = true;                                                 \
      (c)->err = std::string(#expr) + ": " + cudaGetErrorString(e_);        \
      return FS_ECUDA;                                                      \
    }                                                                       \
  } while (0)
#define CK_NCCL(c, expr)                                                    \
  do {                                                                      \
    ncclResult_t r_ = (expr);                                               \
    if (r_ != ncclSuccess) {                                                \
      (c)->poisoned = true;                                                 \
      (c)->err = std::string(#expr) + ": " + ncclGetErrorString(r_);        \
      return FS_ENCCL;                                                      \
    }                                                                       \
  } while (0)
#define CK_LAUNCH(c)                                                        \
  do {                                                                      \
    (c)->launches++;                                                        \
    cudaError_t e_ = cudaGetLastError();                                    \
    if (e_ != cudaSuccess) {                                                \
      (c)->poisoned = true;                                                 \
      (c)->err = std::string("launch: ") + cudaGetErrorString(e_);          \
      return FS_ECUDA;                                                      \
    }                                                                       \
  } while (0)

// ---------------------------------------------------------------- validation
bool cfg_valid(const fs_config* c, std::string* why) {
  auto bad = [&](const char* s) {
    if (why) *why = s;
    return false;
  };
  if (!c) return bad("null cfg");
  if (c->n_layers < 1 || c->d_model < 1 || c->n_heads < 1 || c->n_kv_heads < 1 ||
      c->head_dim < 2 || c->ffn < 1 || c->vocab < 2)
    return bad("bad model shape");
  if (c->n_heads % c->n_kv_heads) return bad("n_heads % n_kv_heads");
  if (c->head_dim % 2) return bad("odd head_dim");
  if (c->ffn % 64) return bad("ffn must be a multiple of 64 (interleaved gate/up tiles)");
  if (c->bf16) {
    if (c->head_dim != 128) return bad("bf16 path needs head_dim 128");
    if (c->d_model % 64 || (c->n_heads * c->head_dim) % 64) return bad("K dims must be multiples of 64");
  } else {
    if (c->head_dim * 4 % 16) return bad("fp32 head_dim must be a multiple of 4");
  }
  if (c->n_stages < 1 || c->n_stages > FS_MAX_STAGES) return bad("n_stages");
  if (c->rank < 0 || c->rank >= c->n_stages) return bad("rank");
  if (c->n_stages > c->n_layers) return bad("more stages than layers");
  if (c->layers_per_stage) {
    int s = 0;
    for (int p = 0; p < c->n_stages; p++) {
      if (c->layers_per_stage[p] < 1) return bad("layers_per_stage entry < 1");
      s += c->layers_per_stage[p];
    }
    if (s != c->n_layers) return bad("layers_per_stage does not sum to n_layers");
  }
  if (c->max_live < 32 || c->max_live > FS_MAX_LIVE || c->max_live % 32) return bad("max_live");
  if (c->max_seg < 1 || c->max_seg > FS_MAX_SEG) return bad("max_seg");
  if (c->max_prefill < 0 || c->max_prefill > FS_MAX_SEG) return bad("max_prefill");
  if (c->max_ctx < c->max_live + 2) return bad("max_ctx");
  if (!c->bf16 && c->max_ctx > 50000) return bad("fp32 path: max_ctx <= 50000 (attention scores in smem)");
  if (c->rms_eps <= 0 || c->rope_theta <= 0) return bad("eps/theta");
  return true;
}

// byte-balanced consecutive layer blocks; the head (V*d) counts on the last stage
void balance(const fs_config* c, int* out) {
  const int P = c->n_stages, L = c->n_layers;
  if (c->layers_per_stage) {
    for (int p = 0; p < P; p++) out[p] = c->layers_per_stage[p];
    return;
  }
  const double layer = (double)c->d_model * (c->n_heads + 2 * c->n_kv_heads) * c->head_dim +
                       (double)c->n_heads * c->head_dim * c->d_model + 3.0 * c->d_model * c->ffn;
  const double head = (double)c->vocab * c->d_model / layer;
  int last = (int)std::lround((L + head) / P - head);
  last = std::max(1, std::min(last, L - (P - 1)));
  if (P == 1) last = L;
  const int rest = L - last;
  for (int p = 0; p < P - 1; p++) out[p] = rest / (P - 1) + (p < rest % (P - 1) ? 1 : 0);
  out[P - 1] = last;
}

int npad_of(int max_seg) { return max_seg <= 16 ? 16 : (max_seg <= 32 ? 32 : 64); }

// ---------------------------------------------------------------- arena
struct Carver {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

void plan_gemm(GemmOp& g, int n_out, int K, int n_sms, int ctas_per_sm, const char* env = nullptr,
               int def_split = -1, bool wide = false) {
  g.sh.n_out = n_out;
  g.sh.K = K;
  g.sh.kb_total = K / 64;
  g.sh.n_tiles = (n_out + 127) / 128;
  g.sh.units = g.sh.n_tiles * g.sh.kb_total;
  g.sh.late_trigger = getenv("FS_LATE_TRIGGER") ? 1 : 0;
  // Many tiles, gemm_tc_kernel: one CTA per output tile when all tiles fit one
  // wave (no split-K, no fix-up; 7B gate/up: 172 CTAs, tick 2.88 -> 2.79 ms),
  // else stream-K over one CTA per SM (two per SM measured 3.15 vs 2.92 ms:
  // the next GEMM's CTAs then find no free slot to prefetch into)
  g.grid = std::min(n_sms, g.sh.units);
  if (g.sh.n_tiles > n_sms && g.sh.n_tiles <= ctas_per_sm * n_sms && !getenv("FS_NO_TILE_GRID"))
    g.grid = g.sh.n_tiles;
  // Prefill-width rows with fewer tiles than SMs: one CTA per tile (no 64-column
  // stream-K fix-up) is faster (7B QKV 33.6 vs 38.1 us) but changes the fp32
  // summation order, and the 72B 2-layer prefill lockstep then sits at 0.0200 of
  // its 2e-2 logit bar (0.0180 with stream-K): opt-in only (FS_WIDE_TILES)
  if (wide && g.sh.n_tiles <= ctas_per_sm * n_sms && getenv("FS_WIDE_TILES")) g.grid = g.sh.n_tiles;
  // Few output tiles: tile-aligned cluster split-K with S CTAs per tile.  Two
  // CTAs fit per SM (NT 16): S = the largest power of two keeping the grid in
  // one wave of 2 x SMs slots; otherwise S = floor(SMs / tiles).  Many tiles:
  // stream-K.  (Measured on the 7B stage forward with windowed epilogues:
  // QKV 2, O 8, down 8, gate/up and head stream-K -- 3.02 ms vs 3.11 ms with
  // O / down at 4, 3.44 ms at 16.)
  int S;
  if (ctas_per_sm >= 2) {
    const int cap = ctas_per_sm * n_sms / std::max(1, g.sh.n_tiles);
    S = 1;
    while (S * 2 <= cap) S *= 2;
  } else {
    S = n_sms / std::max(1, g.sh.n_tiles);
  }
  if (S < 2 && ctas_per_sm >= 2 && g.sh.n_tiles <= n_sms) S = 2;
  S = std::min({S, 16, g.sh.kb_total});
  g.split = (S >= 2 && !getenv("FS_NO_CLUSTER_GEMM")) ? S : 0;
  if (def_split >= 0) g.split = def_split;          // tuned default for this GEMM
  if (env && getenv(env)) g.split = atoi(getenv(env));  // tuning override
  if (g.split == 1 || g.split > std::min(16, g.sh.kb_total)) g.split = 0;
  int mc = 1;
  const int U = g.sh.units, G = g.grid, KB = g.sh.kb_total;
  auto cta = [&](int u) { return (int)(((long long)(u + 1) * G + U - 1) / U) - 1; };
  for (int t = 0; t < g.sh.n_tiles; t++) mc = std::max(mc, cta((t + 1) * KB - 1) - cta(t * KB) + 1);
  g.sh.max_contrib = mc;
}

// carve every buffer; with base == nullptr only measures
size_t carve(fs_ctx* c, char* base) {
  const fs_config& f = c->cfg;
  Carver cv{base};
  const int d = f.d_model, H = f.n_heads, Hkv = f.n_kv_heads, hd = f.head_dim, ffn = f.ffn,
            V = f.vocab;
  const int nq = (H + 2 * Hkv) * hd;
  const int es = c->esz;
  // bf16 GEMM weights are box-tiled (gen_weight_kernel): rows padded to 128
  auto wr = [&](int64_t r) -> size_t { return (size_t)(c->bf ? (r + 127) / 128 * 128 : r); };
  c->lw.assign(c->nl, LayerW());
  for (int l = 0; l < c->nl; l++) {
    LayerW& w = c->lw[l];
    w.wqkv = cv.take<char>(wr(nq) * d * es);
    if (f.qkv_bias) w.bqkv = cv.take<char>((size_t)nq * es);
    w.wo = cv.take<char>(wr(d) * H * hd * es);
    w.wgu = cv.take<char>(wr(2 * ffn) * d * es);
    w.wd = cv.take<char>(wr(d) * ffn * es);
    w.g1 = cv.take<char>((size_t)d * es);
    w.g2 = cv.take<char>((size_t)d * es);
    plan_gemm(w.qkv, nq, d, c->n_sms, c->ctas_tick, "FS_SPLIT_QKV");
    plan_gemm(w.o, d, H * hd, c->n_sms, c->ctas_tick, "FS_SPLIT_O");
    plan_gemm(w.gu, 2 * ffn, d, c->n_sms, c->ctas_tick, "FS_SPLIT_GU");
    plan_gemm(w.dn, d, ffn, c->n_sms, c->ctas_tick, "FS_SPLIT_DN");
    plan_gemm(w.qkv_w, nq, d, c->n_sms, c->ctas_pre, nullptr, -1, true);
    plan_gemm(w.o_w, d, H * hd, c->n_sms, c->ctas_pre, nullptr, -1, true);
    plan_gemm(w.gu_w, 2 * ffn, d, c->n_sms, c->ctas_pre, nullptr, -1, true);
    plan_gemm(w.dn_w, d, ffn, c->n_sms, c->ctas_pre, nullptr, -1, true);
  }
  c->emb = c->first ? cv.take<char>((size_t)V * d * es) : nullptr;
  if (c->last) {
    c->wh = cv.take<char>(wr(V) * d * es);
    c->gf = cv.take<char>((size_t)d * es);
    plan_gemm(c->head, V, d, c->n_sms, c->ctas_tick, "FS_SPLIT_HEAD");
    plan_gemm(c->head_w, V, d, c->n_sms, c->ctas_pre, nullptr, -1, true);
  }
  c->kv_plane_elems = (size_t)Hkv * f.max_ctx * hd;
  c->kv = cv.take<char>((size_t)c->nl * 2 * c->kv_plane_elems * es);
  c->rope = cv.take<float2>((size_t)f.max_ctx * (hd / 2));
  const int np = std::max(c->npad_tick, c->npad_pre);
  c->x = cv.take<float>((size_t)np * d);
  c->hin = cv.take<float>((size_t)np * d);
  // GEMM B operands: 2*np rows (bf16 hi rows, then lo rows)
  c->y = cv.take<char>((size_t)2 * np * d * es);
  c->q = cv.take<char>((size_t)np * H * hd * es);
  c->att = cv.take<char>((size_t)2 * np * H * hd * es);
  c->act = cv.take<char>((size_t)2 * np * ffn * es);
  // fp32 path scratch: GEMM output [np][max(nq, 2ffn, V, d)]
  size_t ymax = std::max({(size_t)nq, (size_t)2 * ffn, (size_t)V, (size_t)d});
  c->yf = c->bf ? nullptr : cv.take<float>((size_t)np * ymax);
  // GEMM stream-K workspace / counters (shared by the sequential GEMMs)
  size_t wsf = 0;
  int max_tiles = 1;
  auto acc = [&](const GemmOp& g) {
    wsf = std::max(wsf, (size_t)g.sh.n_tiles * g.sh.max_contrib * 128 * np);
    max_tiles = std::max(max_tiles, g.sh.n_tiles);
  };
  for (auto& w : c->lw) {
    acc(w.qkv);
    acc(w.o);
    acc(w.gu);
    acc(w.dn);
    acc(w.qkv_w);
    acc(w.o_w);
    acc(w.gu_w);
    acc(w.dn_w);
  }
  if (c->last) {
    acc(c->head);
    acc(c->head_w);
  }
  c->gws_floats = wsf;
  c->gws = c->bf ? cv.take<float>(wsf) : nullptr;
  c->gcnt = cv.take<int>(max_tiles);
  c->ssq = cv.take<float>((size_t)((d + 127) / 128) * 4 * np);
  c->head_part = cv.take<Top2>((size_t)((V + 127) / 128) * np);
  c->res = cv.take<RowResult>(FS_MAX_SEG);
  c->dec = cv.take<SampleDecision>(1);   // directly after res: one broadcast covers both
  if (f.sampling && c->last) {
    c->lstore = cv.take<float>((size_t)f.max_live * V);
    c->samp_r = cv.take<double>(V);
    c->samp_q = cv.take<double>(V);
  }
  c->att_chunk_cap = (f.max_ctx + ATT_KC - 1) / ATT_KC;
  const int G = H / Hkv;
  c->aws_o = c->bf ? cv.take<float>((size_t)c->att_chunk_cap * 4 * Hkv * G * np * ATT_HD) : nullptr;
  c->aws_ml = c->bf ? cv.take<float>((size_t)c->att_chunk_cap * 4 * Hkv * G * np * 2) : nullptr;
  c->att_cnt = cv.take<int>(Hkv);
  // tree
  const int ML = f.max_live;
  TreeDev& t = c->tree;
  t.max_live = ML;
  t.ancw = ML / 32;
  t.max_ids = c->max_ids;
  t.node = cv.take<int32_t>(ML);
  t.token = cv.take<int32_t>(ML);
  t.par = cv.take<int32_t>(ML);
  t.own = cv.take<float>(ML);
  t.cu = cv.take<float>(ML);
  t.depth = cv.take<int32_t>(ML);
  t.anc = cv.take<uint32_t>((size_t)ML * (ML / 32));
  t.verified = cv.take<int32_t>(ML);
  t.am = cv.take<int32_t>(ML);
  t.margin = cv.take<float>(ML);
  t.id2s = cv.take<int32_t>(c->max_ids);
  t.rank = cv.take<int32_t>(ML);
  t.retain = cv.take<uint32_t>(ML / 32);
  c->d_sub = cv.take<SubmitIn>(1);
  c->d_sub2 = cv.take<SubmitIn>(1);
  c->d_dec = cv.take<DecisionIn>(1);
  c->d_rec = cv.take<TreeRecord>(1);
  c->d_rows = cv.take<TickRows>(1);
  return cv.off + 256;
}

bool setup_ctx(fs_ctx* c, const fs_config* f) {
  c->cfg = *f;
  c->P = f->n_stages;
  c->rank = f->rank;
  balance(f, c->lps);
  c->cfg.layers_per_stage = nullptr;
  c->L0 = 0;
  for (int p = 0; p < c->rank; p++) c->L0 += c->lps[p];
  c->nl = c->lps[c->rank];
  c->L1 = c->L0 + c->nl;
  c->first = c->rank == 0;
  c->last = c->rank == c->P - 1;
  c->bf = f->bf16 != 0;
  c->esz = c->bf ? 2 : 4;
  c->npad_tick = npad_of(f->max_seg);
  c->npad_pre = npad_of(std::max(f->max_seg, f->max_prefill));
  // grouped-query heads pack G * npad query rows per kv head; the attention
  // kernels take at most 256 (two tcgen05 M-tiles): cap the prefill width
  const int G = f->n_kv_heads > 0 ? f->n_heads / f->n_kv_heads : 1;
  while (f->bf16 && c->npad_pre > c->npad_tick && G * c->npad_pre > 256) c->npad_pre /= 2;
  c->ctas_tick = c->npad_tick <= 16 ? GemmCfg<16>::MIN_CTAS : 1;
  c->ctas_pre = c->npad_pre <= 16 ? GemmCfg<16>::MIN_CTAS : 1;
  c->npad = c->npad_tick;
  c->gemm_ctas = c->ctas_tick;
  c->ancw = f->max_live / 32;
  return true;
}

bool encode_map(CUtensorMap* m, void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                uint32_t box_outer, bool f32 = false);

// box-tiled weight [ceil(R/128)][K/64][128][64]: a 64-wide map whose row u*128 is box u
bool encode_wmap(CUtensorMap* m, void* ptr, uint64_t K, uint64_t R) {
  return encode_map(m, ptr, 64, (R + 127) / 128 * 128 * (K / 64), 64, 128);
}

bool encode_map(CUtensorMap* m, void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner,
                uint32_t box_outer, bool f32) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims,
             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             f32 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

char* kv_plane(fs_ctx* c, int local_layer, int which);

bool build_maps(fs_ctx* c) {
  const fs_config& f = c->cfg;
  const int d = f.d_model, H = f.n_heads, Hkv = f.n_kv_heads, hd = f.head_dim, ffn = f.ffn;
  const int nq = (H + 2 * Hkv) * hd;
  bool ok = true;
  for (auto& w : c->lw) {
    for (int wide = 0; wide < 2; wide++) {
      const int np = wide ? c->npad_pre : c->npad_tick;
      GemmOp& qkv = wide ? w.qkv_w : w.qkv;
      GemmOp& o = wide ? w.o_w : w.o;
      GemmOp& gu = wide ? w.gu_w : w.gu;
      GemmOp& dn = wide ? w.dn_w : w.dn;
      ok &= encode_wmap(&qkv.ta, w.wqkv, d, nq);
      ok &= encode_map(&qkv.tb, c->y, d, 2 * np, 64, 2 * np);
      ok &= encode_wmap(&o.ta, w.wo, H * hd, d);
      ok &= encode_map(&o.tb, c->att, H * hd, 2 * np, 64, 2 * np);
      ok &= encode_wmap(&gu.ta, w.wgu, d, 2 * ffn);
      ok &= encode_map(&gu.tb, c->y, d, 2 * np, 64, 2 * np);
      ok &= encode_wmap(&dn.ta, w.wd, ffn, d);
      ok &= encode_map(&dn.tb, c->act, ffn, 2 * np, 64, 2 * np);
      qkv.ok = o.ok = gu.ok = dn.ok = ok;
    }
  }
  for (int l = 0; l < c->nl; l++) {
    LayerW& w = c->lw[l];
    const uint64_t kv_rows = (uint64_t)Hkv * f.max_ctx;
    ok &= encode_map(&w.tk, kv_plane(c, l, 0), hd, kv_rows, 64, 128);
    ok &= encode_map(&w.tv, kv_plane(c, l, 1), hd, kv_rows, 64, 128);
    ok &= encode_map(&w.mk, kv_plane(c, l, 0), hd, kv_rows, 64, ATT_SUB);
    ok &= encode_map(&w.mv, kv_plane(c, l, 1), hd, kv_rows, 64, ATT_SUB);
  }
  if (c->last) {
    ok &= encode_wmap(&c->head.ta, c->wh, d, f.vocab);
    ok &= encode_map(&c->head.tb, c->y, d, 2 * c->npad_tick, 64, 2 * c->npad_tick);
    ok &= encode_wmap(&c->head_w.ta, c->wh, d, f.vocab);
    ok &= encode_map(&c->head_w.tb, c->y, d, 2 * c->npad_pre, 64, 2 * c->npad_pre);
    c->head.ok = c->head_w.ok = ok;
  }
  return ok;
}

// switch the active row width: prefill chunks (wide) or tree segments; the
// GemmOps of the two widths trade places so every launch site stays as is
void use_width(fs_ctx* c, bool wide) {
  if (wide == c->wide) return;
  for (auto& w : c->lw) {
    std::swap(w.qkv, w.qkv_w);
    std::swap(w.o, w.o_w);
    std::swap(w.gu, w.gu_w);
    std::swap(w.dn, w.dn_w);
  }
  std::swap(c->head, c->head_w);
  c->wide = wide;
  c->npad = wide ? c->npad_pre : c->npad_tick;
  c->gemm_ctas = wide ? c->ctas_pre : c->ctas_tick;
}

// ---------------------------------------------------------------- profiling
// returns the index of the event pair whose start was recorded, or -1
int prof_begin(fs_ctx* c, int kind, double bytes) {
  if (!c->prof) return -1;
  if (c->ev_next + 2 > c->ev_pool.size()) {
    for (int i = 0; i < 512; i++) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      c->ev_pool.push_back(e);
    }
  }
  const int idx = (int)(c->ev_next / 2);
  cudaEventRecord(c->ev_pool[c->ev_next], c->st);
  c->ev_next += 2;
  c->ev_used.push_back({kind, bytes});
  return idx;
}
void prof_end(fs_ctx* c, int idx) {
  if (idx < 0) return;
  cudaEventRecord(c->ev_pool[2 * idx + 1], c->st);
}

// ---------------------------------------------------------------- launches
// kernel attributes are per device: set them once on every device a context uses
// (double-checked under a lock: contexts of a local group launch from several threads)
template <typename F>
void once_per_device(std::atomic<uint64_t>& done, const fs_ctx* c, F set) {
  static std::mutex mu;
  const uint64_t bit = 1ull << (c->cfg.device & 63);
  if (done.load() & bit) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done.load() & bit) return;
  set();
  done.fetch_or(bit);
}

template <int NT>
int launch_gemm_nt(fs_ctx* c, const GemmOp& g, const GemmEpi& ep) {
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, c, [] {
    cudaFuncSetAttribute(gemm_tc_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         GemmCfg<NT>::SMEM);
    cudaFuncSetAttribute(gemm_cluster_kernel<NT, NT / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         GemmCfg<NT>::SMEM);
    cudaFuncSetAttribute(gemm_cluster_kernel<NT, NT / 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(gemm_cluster_kernel<NT, NT / 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         GemmCfg<NT>::SMEM);
    cudaFuncSetAttribute(gemm_cluster_kernel<NT, NT / 4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  });
  if (g.split > 0) {
    GemmShape sh = g.sh;
    sh.dbg = nullptr;
    if (c->tl_buf) {
      sh.dbg = c->tl_buf + c->tl_names.size() * 8192;
      c->tl_names.push_back("gemm");
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(g.sh.n_tiles * g.split);
    lc.blockDim = dim3(192);   // gemm_cluster_kernel: TMA, MMA, 4 epilogue warps at every width
    lc.dynamicSmemBytes = GemmCfg<NT>::SMEM;
    lc.stream = c->st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = g.split;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 2;
    // column window per rank: NT / 2 covers S <= 3, NT / 4 covers S >= 4
    if (g.split <= 3)
      cudaLaunchKernelEx(&lc, gemm_cluster_kernel<NT, NT / 2>, g.ta, g.tb, sh, ep);
    else
      cudaLaunchKernelEx(&lc, gemm_cluster_kernel<NT, NT / 4>, g.ta, g.tb, sh, ep);
    CK_LAUNCH(c);
    return FS_OK;
  }
  GemmShape sh = g.sh;
  sh.ws = c->gws;
  sh.counters = c->gcnt;
  sh.dbg = c->gemm_dbg;
  if (c->tl_buf) {
    sh.dbg = c->tl_buf + c->tl_names.size() * 8192;
    c->tl_names.push_back("gemm");
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(g.grid);
  lc.blockDim = dim3(GemmCfg<NT>::THREADS);
  lc.dynamicSmemBytes = GemmCfg<NT>::SMEM;
  lc.stream = c->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaLaunchKernelEx(&lc, gemm_tc_kernel<NT>, g.ta, g.tb, sh, ep);
  CK_LAUNCH(c);
  return FS_OK;
}

int launch_gemm(fs_ctx* c, const GemmOp& g, const GemmEpi& ep) {
  const double bytes = (double)g.sh.n_out * g.sh.K * 2 + 2.0 * c->npad * g.sh.K * 2 +
                       (double)c->h_rows->n_rows * g.sh.n_out * 4;
  const int pi = prof_begin(c, 0, bytes);
  int rc;
  switch (c->npad) {
    case 16: rc = launch_gemm_nt<16>(c, g, ep); break;
    case 32: rc = launch_gemm_nt<32>(c, g, ep); break;
    default: rc = launch_gemm_nt<64>(c, g, ep); break;
  }
  prof_end(c, pi);
  return rc;
}

GemmEpi base_epi(fs_ctx* c) {
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.rows = c->d_rows;
  e.H = c->cfg.n_heads;
  e.Hkv = c->cfg.n_kv_heads;
  e.max_ctx = c->cfg.max_ctx;
  e.rope = c->rope;
  e.ffn = c->cfg.ffn;
  e.d = c->cfg.d_model;
  e.vocab = c->cfg.vocab;
  return e;
}

// epilogue params of a GEMM fed by an RMSNorm applied by linearity: B = (x*g)
// as a hi/lo pair (written by the producer of x), accumulator rows *= inv[m]
GemmEpi norm_input(fs_ctx* c) {
  GemmEpi e = base_epi(c);
  e.scale_ssq = c->ssq;
  e.scale_n = c->cfg.d_model / 32;   // one partial per 32 residual columns (an epilogue warp's rows)
  e.eps = (float)c->cfg.rms_eps;
  return e;
}

// the gain of the RMSNorm that follows local layer l's residual update
// (down-proj): next layer's attention norm, the final norm, or none at a
// stage boundary (the next stage prepares its own input)
const bf16* next_gain_after_down(fs_ctx* c, int l) {
  if (l + 1 < c->nl) return (const bf16*)c->lw[l + 1].g1;
  if (c->last) return (const bf16*)c->gf;
  return nullptr;
}

char* kv_plane(fs_ctx* c, int local_layer, int which) {
  return c->kv + ((size_t)local_layer * 2 + which) * c->kv_plane_elems * c->esz;
}

// merge of the split partials (programmatic launch): one warp per (row, head),
// or one CTA per (row, head) (FS_COMBINE_CTA)
void launch_combine(fs_ctx* c, const AttnArgs& a, cudaLaunchAttribute* pdl, int nsplit) {
  static const bool cta = getenv("FS_COMBINE_CTA") != nullptr;
  cudaLaunchConfig_t cc = {};
  cc.stream = c->st;
  cc.attrs = pdl;
  cc.numAttrs = 1;
  if (cta) {
    cc.gridDim = dim3(c->npad, c->cfg.n_heads);
    cc.blockDim = dim3(ATT_HD);
    cudaLaunchKernelEx(&cc, attn_combine_kernel, a, (bf16*)c->att, 1, nsplit);
  } else {
    cc.gridDim = dim3(c->npad, (c->cfg.n_heads + 3) / 4);
    cc.blockDim = dim3(128);
    cudaLaunchKernelEx(&cc, attn_combine_warp_kernel, a, (bf16*)c->att, nsplit);
  }
}

// tree-masked attention of local layer l on the current rows -> c->att (hi/lo)
int launch_attention(fs_ctx* c, int l) {
  const fs_config& f = c->cfg;
  const int H = f.n_heads, Hkv = f.n_kv_heads, hd = f.head_dim;
  const int np = c->npad;
    AttnArgs a;
    a.q = (const bf16*)c->q;
    a.kc = (const bf16*)kv_plane(c, l, 0);
    a.vc = (const bf16*)kv_plane(c, l, 1);
    a.rows = c->d_rows;
    a.anc = c->tree.anc;
    a.ws_o = c->aws_o;
    a.ws_ml = c->aws_ml;
    a.ancw = c->ancw;
    a.max_live = f.max_live;
    a.H = H;
    a.Hkv = Hkv;
    a.max_ctx = f.max_ctx;
    a.npad = np;
    a.n_chunk_cap = c->att_chunk_cap;
    a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)hd));
    a.resc_log2 = getenv("FS_TCA_RESCALE") ? (float)atof(getenv("FS_TCA_RESCALE")) : 8.f;
    a.dbg = c->att_dbg;
    a.dbg_ends = c->att_dbg_ends;
    a.num_err = &c->d_rec->num_err;
    if (c->tl_buf) {
      a.dbg = c->tl_buf + c->tl_names.size() * 8192;
      c->tl_names.push_back("attn");
    }
    const int G = H / Hkv, QR = G * np, MT = QR / 16;
    const int KS = MT >= 4 ? 1 : 4 / MT;
    const int n_keys = c->h_rows->n_keys;
    // MHA: short contexts run the cluster kernel (split merge through DSMEM, no
    // second kernel: 7B 1K context 2.72 vs 2.86 ms per tick), long contexts the
    // TMA ring + combine (13B 4K context 16.4 vs 23.0 us per layer)
    const bool mha_tma = getenv("FS_MHA_CP_ASYNC") ? false
                         : getenv("FS_MHA_TMA") ? true
                         : n_keys > MHA_TMA_MIN_KEYS;
    // prefill chunks of an MHA model (64 query rows, MT 4) also take the TMA kernel
    if ((MT <= 2 && hd == ATT_HD && mha_tma) || (MT == 4 && hd == ATT_HD && !getenv("FS_MHA_CP_ASYNC"))) {
      // MHA path: TMA-staged K/V ring, splits sized to fill every SM slot,
      // partials merged by attn_combine_kernel (programmatic launch)
      const size_t smem = mha_tma_smem(np, c->ancw, QR);
      static std::atomic<uint64_t> tattr{0};
      once_per_device(tattr, c, [] {   // the largest any context needs (npad 64, max_live 512, QR 64)
        const int mx = (int)mha_tma_smem(64, FS_MAX_LIVE / 32, 64);
        cudaFuncSetAttribute(attn_mha_tma_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(attn_mha_tma_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(attn_mha_tma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      });
      if (c->mha_nsplit[MT] == 0) {
        int occ = 0;
        if ((MT == 1   ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, attn_mha_tma_kernel<16>, MHA_THREADS, smem)
             : MT == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, attn_mha_tma_kernel<32>, MHA_THREADS, smem)
                       : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, attn_mha_tma_kernel<64>, MHA_THREADS, smem)) !=
                cudaSuccess ||
            occ < 1) {
          cudaGetLastError();
          occ = 1;
        }
        int ns = std::max(1, occ * c->n_sms / Hkv);
        ns = std::min(ns, (f.max_ctx + ATT_SUB - 1) / ATT_SUB);   // at least one sub-chunk of keys each
        ns = std::min(ns, c->att_chunk_cap * 4);                   // workspace capacity
        ns = std::min(ns, getenv("FS_MHA_NSPLIT_CAP") ? atoi(getenv("FS_MHA_NSPLIT_CAP")) : 8);
        if (getenv("FS_ATT_NSPLIT")) ns = std::max(1, std::min(ns, atoi(getenv("FS_ATT_NSPLIT"))));
        c->mha_nsplit[MT] = ns;
      }
      const int nsplit = c->mha_nsplit[MT];
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(nsplit, Hkv);
      lc.blockDim = dim3(MHA_THREADS);
      lc.dynamicSmemBytes = smem;
      lc.stream = c->st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      const int api = prof_begin(c, 1, (double)n_keys * Hkv * hd * 2 * 2 + (double)QR * Hkv * hd * 2 * 3);
      if (MT == 1)
        cudaLaunchKernelEx(&lc, attn_mha_tma_kernel<16>, c->lw[l].mk, c->lw[l].mv, a);
      else if (MT == 2)
        cudaLaunchKernelEx(&lc, attn_mha_tma_kernel<32>, c->lw[l].mk, c->lw[l].mv, a);
      else
        cudaLaunchKernelEx(&lc, attn_mha_tma_kernel<64>, c->lw[l].mk, c->lw[l].mv, a);
      CK_LAUNCH(c);
      launch_combine(c, a, at, nsplit);
      prof_end(c, api);
      CK_LAUNCH(c);
    } else if (MT <= 2) {
      // MHA path (FS_MHA_CP_ASYNC): key splits of one kv head form a cluster (DSMEM merge), PDL launch
      AttnMhaArgs ma;
      ma.a = a;
      ma.out = (bf16*)c->att;
      const size_t smem = (size_t)QR * ATT_LD * 2 + (size_t)ATT_NBUF * 2 * ATT_SUB * ATT_LD * 2 +
                          (size_t)np * c->ancw * 4 + 16;
      static std::atomic<uint64_t> mattr{0};
      once_per_device(mattr, c, [] {
        cudaFuncSetAttribute(attn_mha_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(attn_mha_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      });
      // cluster of key splits per kv head (sizes read on device): the largest
      // split count <= 8 whose Hkv clusters are all co-resident (one wave;
      // clusters must fit inside a GPC, so this is below 2 * SMs / Hkv)
      if (c->att_nsplit[MT] == 0) {
        int ns = 8;
        for (; ns > 1; ns--) {
          cudaLaunchConfig_t oc = {};
          oc.gridDim = dim3(ns, Hkv);
          oc.blockDim = dim3(128);
          oc.dynamicSmemBytes = smem;
          cudaLaunchAttribute oa[1];
          oa[0].id = cudaLaunchAttributeClusterDimension;
          oa[0].val.clusterDim.x = ns;
          oa[0].val.clusterDim.y = 1;
          oa[0].val.clusterDim.z = 1;
          oc.attrs = oa;
          oc.numAttrs = 1;
          int nclu = 0;
          const cudaError_t oe = MT == 1
              ? cudaOccupancyMaxActiveClusters(&nclu, attn_mha_kernel<16>, &oc)
              : cudaOccupancyMaxActiveClusters(&nclu, attn_mha_kernel<32>, &oc);
          if (oe != cudaSuccess) {
            cudaGetLastError();
            ns = std::max(1, std::min(8, 2 * c->n_sms / std::max(1, Hkv)));
            break;
          }
          if (nclu >= Hkv) break;
        }
        if (getenv("FS_ATT_NSPLIT")) ns = std::max(1, std::min(ns, atoi(getenv("FS_ATT_NSPLIT"))));
        c->att_nsplit[MT] = ns;
      }
      const int nsplit = c->att_nsplit[MT];
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(nsplit, Hkv);
      lc.blockDim = dim3(128);
      lc.dynamicSmemBytes = smem;
      lc.stream = c->st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      at[1].id = cudaLaunchAttributeClusterDimension;
      at[1].val.clusterDim.x = nsplit;
      at[1].val.clusterDim.y = 1;
      at[1].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 2;
      const int api = prof_begin(c, 1, (double)n_keys * Hkv * hd * 2 * 2 + (double)QR * Hkv * hd * 2 * 3);
      if (MT == 1)
        cudaLaunchKernelEx(&lc, attn_mha_kernel<16>, ma);
      else
        cudaLaunchKernelEx(&lc, attn_mha_kernel<32>, ma);
      prof_end(c, api);
      CK_LAUNCH(c);
    } else {
    if ((QR == 128 || QR == 256) && hd == ATT_HD && !getenv("FS_NO_TC_ATTN")) {
      // grouped-query rows fill 128-row M-tiles: tcgen05 attention, one CTA per SM
      int nsplit = std::max(1, std::min(c->n_sms / Hkv, c->att_chunk_cap * 4));
      if (getenv("FS_GQA_NSPLIT")) nsplit = std::max(1, std::min(c->att_chunk_cap * 4, atoi(getenv("FS_GQA_NSPLIT"))));
      TcAttnArgs ta;
      ta.a = a;
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(nsplit, Hkv);
      lc.stream = c->st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      const int api = prof_begin(c, 1, (double)n_keys * Hkv * hd * 2 * 2 + (double)QR * Hkv * hd * 2 +
                                           (double)nsplit * Hkv * QR * (hd + 2) * 4 * 2);
      // P format of P.V: the bf16 hi/lo pair (default: two P.V MMAs, 72B 16K layer
      // 37.4 us with the warp combine), fp16 with V converted to fp16 in shared memory
      // by the softmax warps (FS_TC_ATTN_P=f16: one P.V MMA, 3-4 us less per layer, but
      // the 80-layer 72B logits reach 0.0212 > 2e-2, hi/lo 0.019) or plain bf16
      // (FS_TC_ATTN_P=bf16: 0.027 > 2e-2 on 2 layers).  f16 P with bf16 V is not a
      // valid kind::f16 instruction (A and B formats must match); with f16, a V outside
      // fp16's range fails the call with FS_ERANGE
      const char* pfe = getenv("FS_TC_ATTN_P");
      const int pf = getenv("FS_TC_ATTN_P_BF16") ? TCA_P_BF16
                     : !pfe ? TCA_P_HILO
                     : !strcmp(pfe, "f16") ? TCA_P_F16
                     : !strcmp(pfe, "bf16") ? TCA_P_BF16 : TCA_P_HILO;
      auto go = [&](auto kern, int threads, int smem_bytes) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
        lc.blockDim = dim3(threads);
        lc.dynamicSmemBytes = smem_bytes;
        cudaLaunchKernelEx(&lc, kern, c->lw[l].tk, c->lw[l].tv, ta);
      };
      if (QR == 128) {
        if (pf == TCA_P_HILO) go(attn_gqa_tc_kernel<1, TCA_P_HILO>, TcAttnCfg<1>::THREADS, TcAttnCfg<1>::SMEM);
        else if (pf == TCA_P_F16) go(attn_gqa_tc_kernel<1, TCA_P_F16>, TcAttnCfg<1>::THREADS, TcAttnCfg<1>::SMEM);
        else go(attn_gqa_tc_kernel<1, TCA_P_BF16>, TcAttnCfg<1>::THREADS, TcAttnCfg<1>::SMEM);
      } else {
        if (pf == TCA_P_HILO) go(attn_gqa_tc_kernel<2, TCA_P_HILO>, TcAttnCfg<2>::THREADS, TcAttnCfg<2>::SMEM);
        else if (pf == TCA_P_F16) go(attn_gqa_tc_kernel<2, TCA_P_F16>, TcAttnCfg<2>::THREADS, TcAttnCfg<2>::SMEM);
        else go(attn_gqa_tc_kernel<2, TCA_P_BF16>, TcAttnCfg<2>::THREADS, TcAttnCfg<2>::SMEM);
      }
      prof_end(c, api);
      CK_LAUNCH(c);
      launch_combine(c, a, at, nsplit);
      CK_LAUNCH(c);
      return FS_OK;
    }
    const int n_chunks = (n_keys + ATT_KC - 1) / ATT_KC;
    const size_t smem = (size_t)QR * ATT_LD * 2 + 2 * ATT_KC * ATT_LD * 2 + (size_t)np * c->ancw * 4;
    static std::atomic<uint64_t> attr{0};
    once_per_device(attr, c, [] {
      cudaFuncSetAttribute(attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    const int api = prof_begin(c, 1, (double)n_keys * Hkv * hd * 2 * 2 + (double)QR * Hkv * hd * 2 +
                                         (double)n_chunks * KS * Hkv * QR * (hd + 2) * 4);
    attn_mma_kernel<<<dim3(c->att_chunk_cap, Hkv), 128, smem, c->st>>>(a);
    prof_end(c, api);
    CK_LAUNCH(c);
    attn_combine_kernel<<<dim3(np, H), ATT_HD, 0, c->st>>>(a, (bf16*)c->att, KS);
    CK_LAUNCH(c);
    }
  return FS_OK;
}

// one decoder layer on the current tick rows (x in place)
int layer_forward(fs_ctx* c, int l) {
  const fs_config& f = c->cfg;
  LayerW& w = c->lw[l];
  const int d = f.d_model, H = f.n_heads, Hkv = f.n_kv_heads, hd = f.head_dim, ffn = f.ffn;
  const int np = c->npad;
  const int nq = (H + 2 * Hkv) * hd;
  int rc;
  if (c->bf) {
    // RMSNorm fused into the GEMM B operand (norm_input): no separate launch
    GemmEpi e = norm_input(c);
    e.mode = EPI_QKV;
    e.bias = (const bf16*)w.bqkv;
    e.q_out = (bf16*)c->q;
    e.k_cache = (bf16*)kv_plane(c, l, 0);
    e.v_cache = (bf16*)kv_plane(c, l, 1);
    if ((rc = launch_gemm(c, w.qkv, e))) return rc;
    if ((rc = launch_attention(c, l))) return rc;
    e = base_epi(c);
    e.mode = EPI_RESID;
    e.x = c->x;
    e.ssq_out = c->ssq;
    e.z_gain = (const bf16*)w.g2;
    e.z_out = (bf16*)c->y;
    if ((rc = launch_gemm(c, w.o, e))) return rc;
    e = norm_input(c);
    e.mode = EPI_GLU;
    e.act = (bf16*)c->act;
    if ((rc = launch_gemm(c, w.gu, e))) return rc;
    e = base_epi(c);
    e.mode = EPI_RESID;
    e.x = c->x;
    const bf16* gn = next_gain_after_down(c, l);
    e.ssq_out = gn ? c->ssq : nullptr;
    e.z_gain = gn;
    e.z_out = gn ? (bf16*)c->y : nullptr;
    if ((rc = launch_gemm(c, w.dn, e))) return rc;
  } else {
    float* yf = c->yf;
    rmsnorm_kernel<float, float, false><<<np, 128, 0, c->st>>>(c->x, (const float*)w.g1, (float*)c->y, d,
                                                       (float)f.rms_eps, c->d_rows);
    CK_LAUNCH(c);
    gemm_f32_kernel<<<(nq + 127) / 128, 128, 0, c->st>>>((const float*)w.wqkv, (const float*)c->y, yf,
                                                         nq, d, c->d_rows);
    CK_LAUNCH(c);
    epi_qkv_f32_kernel<<<dim3(((H + 2 * Hkv) * hd / 2 + 127) / 128, FS_MAX_SEG), 128, 0, c->st>>>(
        yf, (const float*)w.bqkv, c->rope, (float*)c->q, (float*)kv_plane(c, l, 0),
        (float*)kv_plane(c, l, 1), H, Hkv, hd, f.max_ctx, c->d_rows);
    CK_LAUNCH(c);
    static std::atomic<uint64_t> sattr{0};
    once_per_device(sattr, c, [] {
      cudaFuncSetAttribute(attn_simple_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    // scores for up to max_ctx keys (fixed size: the launch is graph-replayed)
    attn_simple_kernel<float><<<dim3(H, FS_MAX_SEG), 128, (size_t)f.max_ctx * 4, c->st>>>(
        (const float*)c->q, (const float*)kv_plane(c, l, 0), (const float*)kv_plane(c, l, 1),
        (float*)c->att, c->d_rows, c->tree.anc, c->ancw, f.max_live, H, Hkv, hd, f.max_ctx,
        (float)(1.0 / std::sqrt((double)hd)));
    CK_LAUNCH(c);
    gemm_f32_kernel<<<(d + 127) / 128, 128, 0, c->st>>>((const float*)w.wo, (const float*)c->att, yf,
                                                        d, H * hd, c->d_rows);
    CK_LAUNCH(c);
    epi_resid_f32_kernel<<<dim3((d + 127) / 128, FS_MAX_SEG), 128, 0, c->st>>>(yf, c->x, d, c->d_rows);
    CK_LAUNCH(c);
    rmsnorm_kernel<float, float, false><<<np, 128, 0, c->st>>>(c->x, (const float*)w.g2, (float*)c->y, d,
                                                       (float)f.rms_eps, c->d_rows);
    CK_LAUNCH(c);
    gemm_f32_kernel<<<(2 * ffn + 127) / 128, 128, 0, c->st>>>((const float*)w.wgu, (const float*)c->y,
                                                              yf, 2 * ffn, d, c->d_rows);
    CK_LAUNCH(c);
    epi_glu_f32_kernel<<<dim3((ffn + 127) / 128, FS_MAX_SEG), 128, 0, c->st>>>(yf, (float*)c->act, ffn,
                                                                             c->d_rows);
    CK_LAUNCH(c);
    gemm_f32_kernel<<<(d + 127) / 128, 128, 0, c->st>>>((const float*)w.wd, (const float*)c->act, yf,
                                                        d, ffn, c->d_rows);
    CK_LAUNCH(c);
    epi_resid_f32_kernel<<<dim3((d + 127) / 128, FS_MAX_SEG), 128, 0, c->st>>>(yf, c->x, d, c->d_rows);
    CK_LAUNCH(c);
  }
  return FS_OK;
}

// the stochastic accept walk (f2): a cluster of SWC CTAs, each with its slice
// of the vocabulary in shared memory (FS_SAMPLE_ONE_CTA: the single-CTA kernel)
int launch_sample_walk(fs_ctx* c, const SampleArgs& sa) {
  if (getenv("FS_SAMPLE_ONE_CTA")) {
    sample_walk_kernel<<<1, SAMPLE_THREADS, 0, c->st>>>(sa);
    CK_LAUNCH(c);
    return FS_OK;
  }
  const int per = (c->cfg.vocab + SWC - 1) / SWC;
  const size_t smem = (size_t)2 * per * sizeof(double);
  static std::atomic<uint64_t> wattr{0};
  once_per_device(wattr, c, [] {
    cudaFuncSetAttribute(sample_walk_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(sample_walk_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(SWC);
  lc.blockDim = dim3(SWT);
  lc.dynamicSmemBytes = smem;
  lc.stream = c->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = SWC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaLaunchKernelEx(&lc, sample_walk_cluster_kernel, sa);
  CK_LAUNCH(c);
  return FS_OK;
}

// where the head writes fp32 logits: the per-S-index store in stochastic
// mode (the walk needs every verified node's distribution), else the
// caller's parity buffer (or nowhere)
float* head_logits(fs_ctx* c) { return c->samp_mode ? c->lstore : c->logits_buf; }

// final RMSNorm + head + argmax/top-2 on the last stage -> c->res
int head_forward(fs_ctx* c) {
  const fs_config& f = c->cfg;
  const int d = f.d_model, V = f.vocab, np = c->npad;
  if (c->bf) {
    GemmEpi e = norm_input(c);
    e.mode = EPI_HEAD;
    e.head_part = c->head_part;
    e.logits = head_logits(c);
    e.logits_by_s = c->samp_mode ? 1 : 0;
    int rc = launch_gemm(c, c->head, e);
    if (rc) return rc;
    argmax_final_kernel<<<FS_MAX_SEG, 32, 0, c->st>>>(c->head_part, c->head.sh.n_tiles, np, c->d_rows,
                                                      c->res);
    CK_LAUNCH(c);
  } else {
    rmsnorm_kernel<float, float, false><<<np, 128, 0, c->st>>>(c->x, (const float*)c->gf, (float*)c->y, d,
                                                       (float)f.rms_eps, c->d_rows);
    CK_LAUNCH(c);
    gemm_f32_kernel<<<(V + 127) / 128, 128, 0, c->st>>>((const float*)c->wh, (const float*)c->y, c->yf,
                                                        V, d, c->d_rows);
    CK_LAUNCH(c);
    argmax_rows_kernel<<<FS_MAX_SEG, 256, 0, c->st>>>(c->yf, V, c->d_rows, c->res, head_logits(c),
                                                      c->samp_mode ? 1 : 0);
    CK_LAUNCH(c);
  }
  return FS_OK;
}

// this stage's forward of the rows in d_rows (h_rows mirrors it on the host)
int stage_forward(fs_ctx* c, bool from_hin) {
  const int d = c->cfg.d_model;
  if (c->bf) {  // embedding / received rows -> x, and the first RMSNorm's inputs (one kernel)
    const bf16* g0 = c->nl > 0 ? (const bf16*)c->lw[0].g1 : (const bf16*)c->gf;
    const float* src = (!c->first && from_hin) ? c->hin : c->x;
    norm_prep_kernel<bf16><<<dim3(c->npad, std::max(1, d / 512)), 128, 0, c->st>>>(c->first ? (const bf16*)c->emb : nullptr, src, c->x,
                                                       g0, (bf16*)c->y, c->ssq, d, c->d_rows);
    CK_LAUNCH(c);
  } else if (c->first) {
    embed_kernel<float><<<FS_MAX_SEG, 256, 0, c->st>>>((const float*)c->emb, d, c->d_rows, c->x);
    CK_LAUNCH(c);
  } else if (from_hin) {
    CK_CUDA(c, cudaMemcpyAsync(c->x, c->hin, (size_t)c->npad * d * 4, cudaMemcpyDeviceToDevice, c->st));
  }
  for (int l = 0; l < c->nl; l++) {
    int rc = layer_forward(c, l);
    if (rc) return rc;
  }
  if (c->last) return head_forward(c);
  return FS_OK;
}

// the tick's stage forward: replay a captured CUDA graph (sizes live in
// d_rows, so one graph serves every tick); direct launches when profiling
int tick_forward(fs_ctx* c) {
  if (!c->use_graph || c->prof) return stage_forward(c, true);
  const int want_tma = c->h_rows->n_keys > MHA_TMA_MIN_KEYS ? 1 : 0;
  if (c->fwd_exec && (c->fwd_logits != head_logits(c) || c->fwd_mha_tma != want_tma)) {
    cudaGraphExecDestroy(c->fwd_exec);
    c->fwd_exec = nullptr;
  }
  if (!c->fwd_exec) {
    cudaGraph_t g;
    const uint64_t l0 = c->launches;
    CK_CUDA(c, cudaStreamBeginCapture(c->st, cudaStreamCaptureModeRelaxed));
    int rc = stage_forward(c, true);
    cudaError_t e = cudaStreamEndCapture(c->st, &g);
    if (rc) return rc;
    CK_CUDA(c, e);
    CK_CUDA(c, cudaGraphInstantiate(&c->fwd_exec, g, 0));
    cudaGraphDestroy(g);
    c->fwd_kernels = c->launches - l0;
    c->launches = l0;
    c->fwd_logits = head_logits(c);
    c->fwd_mha_tma = want_tma;
  }
  CK_CUDA(c, cudaGraphLaunch(c->fwd_exec, c->st));
  c->launches += c->fwd_kernels;
  return FS_OK;
}

int upload_rows(fs_ctx* c) {
  CK_CUDA(c, cudaMemcpyAsync(c->d_rows, c->h_rows, sizeof(TickRows), cudaMemcpyHostToDevice, c->st));
  return FS_OK;
}

int sync(fs_ctx* c) {
  CK_CUDA(c, cudaStreamSynchronize(c->st));
  return FS_OK;
}

// ---------------------------------------------------------------- stage transport (a10)
// One grouped exchange of this rank (R8): send `sw` 4-byte words from
// sptr to rank+1, receive `rw` words into rptr from rank-1, and broadcast `bw`
// words at bptr from the last rank to every rank.  Zero counts skip a leg; all
// ranks agree on the legs because the schedule is replicated.  NCCL: one group
// (one launch).  Local group: post every outgoing buffer first, then pull every
// incoming one, then wait for the acknowledgements (no cycle can block).
int exchange(fs_ctx* c, const void* sptr, size_t sw, void* rptr, size_t rw, void* bptr, size_t bw) {
  const int p = c->rank, P = c->P;
  if (P == 1 || (!sw && !rw && !bw)) return FS_OK;
  if (!c->lg) {
    static const bool xt = getenv("FS_XCHG_TIMING") != nullptr;
    cudaEvent_t xa = nullptr, xb = nullptr;
    if (xt) {
      cudaEventCreate(&xa);
      cudaEventCreate(&xb);
      cudaEventRecord(xa, c->st);
    }
    CK_NCCL(c, ncclGroupStart());
    if (sw) CK_NCCL(c, ncclSend(sptr, sw, ncclFloat32, p + 1, c->comm, c->st));
    if (rw) CK_NCCL(c, ncclRecv(rptr, rw, ncclFloat32, p - 1, c->comm, c->st));
    if (bw) CK_NCCL(c, ncclBroadcast(bptr, bptr, bw, ncclInt32, P - 1, c->comm, c->st));
    CK_NCCL(c, ncclGroupEnd());
    if (xt) {
      cudaEventRecord(xb, c->st);
      c->xt_x.push_back({xa, xb});
    }
    return FS_OK;
  }
  fs_local_group* g = c->lg;
  const bool root = p == P - 1;
  auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
  auto fail_tx = [&](const char* why) {
    c->poisoned = true;
    c->err = std::string("local transport: ") + why;
    return FS_ENCCL;
  };
  // 1. posts
  int posts[FS_MAX_STAGES], n_posts = 0;
  if (sw) posts[n_posts++] = p + 1;
  if (bw && root)
    for (int q = 0; q < P - 1; q++) posts[n_posts++] = q;
  if (n_posts) {
    CK_CUDA(c, cudaEventRecord(c->ev_ready, c->st));
    std::lock_guard<std::mutex> lk(g->mu);
    for (int k = 0; k < n_posts; k++) {
      auto& ch = g->ch[p][posts[k]];
      // the last stage only broadcasts, every other stage only sends
      ch.ptr = root ? bptr : sptr;
      ch.bytes = 4 * (root ? bw : sw);
      ch.ready = c->ev_ready;
      ch.posted++;
    }
    g->cv.notify_all();
  }
  // 2. pulls (recv from p-1, broadcast from the root)
  auto pull = [&](int src, void* dst, size_t bytes) -> int {
    auto& ch = g->ch[src][p];
    const void* from;
    cudaEvent_t ready;
    {
      std::unique_lock<std::mutex> lk(g->mu);
      if (!g->cv.wait_until(lk, deadline, [&] { return ch.posted > ch.taken; }))
        return fail_tx("peer did not post in time");
      if (ch.bytes != bytes) return fail_tx("peer posted a different size");
      from = ch.ptr;
      ready = ch.ready;
    }
    CK_CUDA(c, cudaStreamWaitEvent(c->st, ready, 0));
    CK_CUDA(c, cudaMemcpyAsync(dst, from, bytes, cudaMemcpyDefault, c->st));
    CK_CUDA(c, cudaEventRecord(c->ev_done[src], c->st));
    std::lock_guard<std::mutex> lk(g->mu);
    ch.done = c->ev_done[src];
    ch.taken++;
    g->cv.notify_all();
    return FS_OK;
  };
  int rc;
  // a non-root rank that also sends posted the send first; broadcast and
  // recv pulls come from different channels ([P-1][p] vs [p-1][p])
  if (rw && (rc = pull(p - 1, rptr, 4 * rw))) return rc;
  if (bw && !root && (rc = pull(P - 1, bptr, 4 * bw))) return rc;
  // 3. acknowledgements: the stream may not overwrite a posted buffer before
  // the receiver's copy has run
  for (int k = 0; k < n_posts; k++) {
    auto& ch = g->ch[p][posts[k]];
    cudaEvent_t done;
    {
      std::unique_lock<std::mutex> lk(g->mu);
      if (!g->cv.wait_until(lk, deadline, [&] { return ch.taken == ch.posted; }))
        return fail_tx("peer did not receive in time");
      done = ch.done;
    }
    CK_CUDA(c, cudaStreamWaitEvent(c->st, done, 0));
  }
  return FS_OK;
}

bool check(fs_ctx* c, int* rc) {
  if (!c) {
    *rc = FS_EINVAL;
    return false;
  }
  if (c->poisoned) {
    *rc = FS_EPOISONED;
    return false;
  }
  // the calling thread may not have this context's device current (local
  // groups drive one context per thread)
  cudaSetDevice(c->cfg.device);
  return true;
}

}  // namespace

// =====================================================================  ABI
extern "C" {

size_t fs_arena_bytes(const fs_config* cfg) {
  if (!cfg_valid(cfg, nullptr)) return 0;
  fs_ctx tmp;
  setup_ctx(&tmp, cfg);
  return carve(&tmp, nullptr);
}

int fs_layers_per_stage(const fs_config* cfg, int32_t* out) {
  if (!out || !cfg_valid(cfg, nullptr)) return FS_EINVAL;
  int lps[FS_MAX_STAGES];
  balance(cfg, lps);
  for (int p = 0; p < cfg->n_stages; p++) out[p] = lps[p];
  return FS_OK;
}

int fs_nccl_unique_id(uint8_t* out) {
  if (!out) return FS_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return FS_ENCCL;
  memcpy(out, id.internal, 128);
  return FS_OK;
}

int fs_init(const fs_config* cfg, fs_ctx** out) {
  if (!out) return FS_EINVAL;
  *out = nullptr;
  std::string why;
  if (!cfg_valid(cfg, &why)) {
    fprintf(stderr, "fs_init: %s\n", why.c_str());
    return FS_EINVAL;
  }
  if (!cfg->arena || !cfg->stream) return FS_EINVAL;
  if (cfg->n_stages > 1 && !cfg->nccl_id == !cfg->local_group) return FS_EINVAL;
  if (cfg->local_group && cfg->local_group->P != cfg->n_stages) return FS_EINVAL;
  fs_ctx* c = new fs_ctx();
  setup_ctx(c, cfg);
  if (cudaSetDevice(cfg->device) != cudaSuccess) {
    delete c;
    return FS_ECUDA;
  }
  cudaDeviceGetAttribute(&c->n_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  c->st = (cudaStream_t)cfg->stream;
  c->use_graph = getenv("FS_NO_GRAPH") == nullptr;
  const size_t need = carve(c, nullptr);
  if (cfg->arena_bytes < need) {
    delete c;
    return FS_ENOMEM;
  }
  c->base = (char*)cfg->arena;
  c->cap = cfg->arena_bytes;
  carve(c, c->base);
  if ((char*)c->dec != (char*)c->res + sizeof(RowResult) * FS_MAX_SEG) {  // one broadcast covers both
    delete c;
    return FS_EINVAL;
  }
  if (c->bf && !build_maps(c)) {
    delete c;
    return FS_ECUDA;
  }
  if (cudaMallocHost(&c->h_sub, sizeof(SubmitIn)) || cudaMallocHost(&c->h_dec, sizeof(DecisionIn)) ||
      cudaMallocHost(&c->h_rec, sizeof(TreeRecord)) || cudaMallocHost(&c->h_rows, sizeof(TickRows)) ||
      cudaMallocHost(&c->h_res, sizeof(RowResult) * FS_MAX_SEG) ||
      cudaMallocHost(&c->h_node, sizeof(int32_t) * FS_MAX_SEG)) {
    delete c;
    return FS_ECUDA;
  }
  memset(c->h_rows, 0, sizeof(TickRows));
  // zero activations / tree; id2s = -1; counters = 0
  cudaMemsetAsync(c->base, 0, need - 256, c->st);
  cudaMemsetAsync(c->tree.id2s, 0xff, sizeof(int32_t) * c->max_ids, c->st);
  if (cudaStreamSynchronize(c->st) != cudaSuccess) {
    delete c;
    return FS_ECUDA;
  }
  if (c->P > 1 && cfg->local_group) {
    fs_local_group* g = cfg->local_group;
    if (cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming) != cudaSuccess) {
      delete c;
      return FS_ECUDA;
    }
    for (int q = 0; q < c->P; q++)
      if (cudaEventCreateWithFlags(&c->ev_done[q], cudaEventDisableTiming) != cudaSuccess) {
        fs_destroy(c);
        return FS_ECUDA;
      }
    std::lock_guard<std::mutex> lk(g->mu);
    if (g->member[c->rank]) {
      fs_destroy(c);
      return FS_EINVAL;
    }
    g->member[c->rank] = c;
    c->lg = g;
  } else if (c->P > 1) {
    ncclUniqueId id;
    memcpy(id.internal, cfg->nccl_id, 128);
    if (ncclCommInitRank(&c->comm, c->P, id, c->rank) != ncclSuccess) {
      delete c;
      return FS_ENCCL;
    }
  }
  *out = c;
  return FS_OK;
}

int fs_load_random_weights(fs_ctx* c, uint64_t seed) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (c->weights) return fail(c, FS_ESTATE, "weights already loaded");
  const fs_config& f = c->cfg;
  const int d = f.d_model, H = f.n_heads, Hkv = f.n_kv_heads, hd = f.head_dim, ffn = f.ffn,
            V = f.vocab, L = f.n_layers;
  auto key = [&](uint64_t tid) {
    // tensor key: mix(seed ^ tid * 0xD1B54A32D192ED03) (host copy of the recipe)
    uint64_t z = seed ^ (tid * 0xD1B54A32D192ED03ull);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  auto scale = [](double sigma, int gain) {
    return gain ? (float)(0.1 / 16777216.0) : (float)(sigma * std::sqrt(3.0) / 16777216.0);
  };
  auto gen = [&](void* dst, uint64_t tid, double sigma, int gain, int64_t rows, int64_t cols,
                 int mode, int64_t off, int tiled = 0) -> int {
    tiled &= c->bf ? 1 : 0;
    const int64_t n = rows * cols;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (c->bf)
      gen_weight_kernel<bf16><<<blocks, 256, 0, c->st>>>((bf16*)dst, key(tid), scale(sigma, gain), gain,
                                                         rows, cols, mode, off, tiled);
    else
      gen_weight_kernel<float><<<blocks, 256, 0, c->st>>>((float*)dst, key(tid), scale(sigma, gain),
                                                          gain, rows, cols, mode, off, 0);
    CK_LAUNCH(c);
    return FS_OK;
  };
  const double s = 0.02, so = 0.02 / std::sqrt(2.0 * L);
  // a ragged last 128-row box of a tiled weight: zero its padding rows
  auto pad0 = [&](void* p, int64_t R, int64_t K) {
    if (c->bf && R % 128) cudaMemsetAsync((char*)p + (size_t)(R / 128) * 128 * K * 2, 0, (size_t)128 * K * 2, c->st);
  };
  for (int l = 0; l < c->nl; l++) {
    const uint64_t gl = (uint64_t)(c->L0 + l) * 16;
    LayerW& w = c->lw[l];
    pad0(w.wqkv, (int64_t)(H + 2 * Hkv) * hd, d);
    pad0(w.wo, d, (int64_t)H * hd);
    pad0(w.wd, d, ffn);
    if ((rc = gen(w.wqkv, gl + 0, s, 0, (int64_t)H * hd, d, 0, 0, 1))) return rc;
    if ((rc = gen(w.wqkv, gl + 1, s, 0, (int64_t)Hkv * hd, d, 0, (int64_t)H * hd, 1))) return rc;
    if ((rc = gen(w.wqkv, gl + 2, s, 0, (int64_t)Hkv * hd, d, 0, (int64_t)(H + Hkv) * hd, 1))) return rc;
    if (f.qkv_bias) {
      if ((rc = gen(w.bqkv, gl + 9, s, 0, 1, (int64_t)H * hd, 0, 0))) return rc;
      char* bk = (char*)w.bqkv + (size_t)H * hd * c->esz;
      if ((rc = gen(bk, gl + 10, s, 0, 1, (int64_t)Hkv * hd, 0, 0))) return rc;
      char* bv = bk + (size_t)Hkv * hd * c->esz;
      if ((rc = gen(bv, gl + 11, s, 0, 1, (int64_t)Hkv * hd, 0, 0))) return rc;
    }
    if ((rc = gen(w.wo, gl + 3, so, 0, d, (int64_t)H * hd, 0, 0, 1))) return rc;
    if ((rc = gen(w.wgu, gl + 4, s, 0, ffn, d, 1, 0, 1))) return rc;
    if ((rc = gen(w.wgu, gl + 5, s, 0, ffn, d, 2, 0, 1))) return rc;
    if ((rc = gen(w.wd, gl + 6, so, 0, d, ffn, 0, 0, 1))) return rc;
    if ((rc = gen(w.g1, gl + 7, 0, 1, 1, d, 0, 0))) return rc;
    if ((rc = gen(w.g2, gl + 8, 0, 1, 1, d, 0, 0))) return rc;
  }
  if (c->first && (rc = gen(c->emb, 0xFFFF0, s, 0, V, d, 0, 0))) return rc;
  if (c->last) {
    pad0(c->wh, V, d);
    if ((rc = gen(c->wh, 0xFFFF1, 2.0 / std::sqrt((double)d), 0, V, d, 0, 0, 1))) return rc;
    if ((rc = gen(c->gf, 0xFFFF2, 0, 1, 1, d, 0, 0))) return rc;
  }
  rope_table_kernel<<<148 * 4, 256, 0, c->st>>>(c->rope, f.max_ctx, hd / 2, f.rope_theta, hd);
  CK_LAUNCH(c);
  if ((rc = sync(c))) return rc;
  c->weights = true;
  return FS_OK;
}

int fs_set_logits_buffer(fs_ctx* c, float* dev_logits, int32_t rows_cap) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (dev_logits && rows_cap < c->cfg.max_seg) return fail(c, FS_EINVAL, "rows_cap < max_seg");
  c->logits_buf = dev_logits;
  c->logits_cap = rows_cap;
  return FS_OK;
}

static void reset_round(fs_ctx* c) {
  c->acc_ready = false;
  c->plan_ready = false;
  c->live = 0;
  c->n_live = 0;
  c->next_id = 0;
  c->queue.clear();
  for (int p = 0; p < FS_MAX_STAGES; p++) {
    c->slot[p] = Seg();
    c->n_cached[p] = 0;
  }
}

int fs_set_prefix(fs_ctx* c, const int32_t* tok, int32_t n, int32_t mode, uint64_t kv_seed,
                  int32_t* x_new_out) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (!c->weights) return fail(c, FS_ESTATE, "weights not loaded");
  if (!tok || n < 1 || (mode != FS_PREFILL && mode != FS_SYNTH_KV)) return fail(c, FS_EINVAL, "bad prefix");
  for (int i = 0; i < n; i++)
    if (tok[i] < 0 || tok[i] >= c->cfg.vocab) return fail(c, FS_EINVAL, "bad prefix token");
  if (n + c->cfg.max_live > c->cfg.max_ctx) return fail(c, FS_ECAPACITY, "prefix too long");
  reset_round(c);
  int start = 0;
  if (mode == FS_SYNTH_KV) {
    const fs_config& f = c->cfg;
    for (int l = 0; l < c->nl; l++)
      for (int w = 0; w < 2; w++) {
        uint64_t tid = 0x200000ull + (uint64_t)(c->L0 + l) * 2 + w;
        uint64_t z = kv_seed ^ (tid * 0xD1B54A32D192ED03ull);
        z += 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const float cc = (float)(1.0 * std::sqrt(3.0) / 16777216.0);
        if (c->bf)
          gen_kv_kernel<bf16><<<148 * 8, 256, 0, c->st>>>((bf16*)kv_plane(c, l, w), z, cc, f.n_kv_heads,
                                                          f.max_ctx, f.head_dim, n - 1);
        else
          gen_kv_kernel<float><<<148 * 8, 256, 0, c->st>>>((float*)kv_plane(c, l, w), z, cc, f.n_kv_heads,
                                                           f.max_ctx, f.head_dim, n - 1);
        CK_LAUNCH(c);
      }
    start = n - 1;
  }
  // chunked prefill at the prefill row width, pipelined over the
  // stages: at step t stage p runs chunk t - p; its input rows arrive from
  // p-1 at the end of step t-1 (the same exchange as a verify tick)
  const int M = std::min(std::max(c->cfg.max_seg, c->cfg.max_prefill), c->npad_pre);
  use_width(c, true);
  const int n_chunks = (n - start + M - 1) / M;
  const int p = c->rank, P = c->P, d = c->cfg.d_model;
  rc = FS_OK;
  for (int t = 0; t < n_chunks + P - 1; t++) {
    const int ch = t - p;                       // this stage's chunk this step
    const bool has = ch >= 0 && ch < n_chunks;
    const int b0 = start + ch * M;
    const int m = has ? std::min(M, n - b0) : 0;
    if (has) {
      TickRows* r = c->h_rows;
      r->n_rows = m;
      r->l_glo = b0;
      r->s_begin = 0;
      r->n_keys = b0 + m;
      for (int i = 0; i < m; i++) {
        r->token[i] = tok[b0 + i];
        r->pos[i] = b0 + i;
        r->slot[i] = b0 + i;
        r->ctx_lim[i] = b0 + i + 1;
        r->sidx[i] = -1;
      }
      if ((rc = upload_rows(c))) break;
      if ((rc = stage_forward(c, true))) break;
    }
    if (P > 1) {
      const int chp = t - (p - 1);              // the chunk stage p-1 ran this step
      const bool recv = p > 0 && chp >= 0 && chp < n_chunks;
      const int mr = recv ? std::min(M, n - (start + chp * M)) : 0;
      const int chl = t - (P - 1);              // the last stage's chunk: only the final one's rows matter
      const bool bc = chl == n_chunks - 1;
      const int mb = bc ? std::min(M, n - (start + chl * M)) : 0;
      if ((rc = exchange(c, c->x, (has && !c->last) ? (size_t)m * d : 0, c->hin, (size_t)mr * d, c->res,
                         (size_t)mb * 2)))
        break;
    }
    // h_rows (pinned) is rewritten next step: the async H2D copy must have run
    if ((rc = sync(c))) break;
  }
  use_width(c, false);
  if (rc) return rc;
  {
    const int mlast = n - (start + (n_chunks - 1) * M);
    CK_CUDA(c, cudaMemcpyAsync(c->h_res, c->res, sizeof(RowResult) * mlast, cudaMemcpyDeviceToHost, c->st));
    CK_CUDA(c, cudaMemcpyAsync(&c->h_rec->num_err, &c->d_rec->num_err, sizeof(int32_t), cudaMemcpyDeviceToHost,
                               c->st));
    if ((rc = sync(c))) return rc;
    if (c->h_rec->num_err) {
      c->poisoned = true;
      return fail(c, FS_ERANGE, "attention V outside the fp16 range of the f16-P kernel (FS_TC_ATTN_P=hilo)");
    }
    c->x_new = c->h_res[mlast - 1].am;
  }
  c->l_glo = n;
  c->prefixed = true;
  if (x_new_out) *x_new_out = c->x_new;
  return FS_OK;
}

int fs_submit_segment(fs_ctx* c, int32_t flags, const int32_t* parent, const int32_t* token,
                      const float* own, int32_t n, int32_t L_top, int32_t L_max, fs_submit_out* out) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (!c->prefixed) return fail(c, FS_ESTATE, "no prefix");
  const int32_t kind = flags & ~(FS_ORDER_BFS | FS_SUBMIT_ASYNC);
  const bool async = (flags & FS_SUBMIT_ASYNC) != 0;
  if (async && (kind == FS_MERGE || (L_top > 0 && L_top < n))) return fail(c, FS_EINVAL, "async submit: no merge / top-L");
  if (kind != FS_NEW_ROUND && kind != FS_APPEND && kind != FS_MERGE) return fail(c, FS_EINVAL, "bad flags");
  const bool merge = kind == FS_MERGE;
  if (merge && parent && n >= 1) {   // T_new: parent indices within T_new, node 0 the root
    if (parent[0] != -1) return fail(c, FS_EINVAL, "merge: T_new node 0 must be the root");
    for (int i = 1; i < n; i++)
      if (parent[i] < 0 || parent[i] >= i) return fail(c, FS_EINVAL, "merge: parent must precede child");
  }
  if (!parent || !token || !own || n < 1 || n > FS_MAX_LIVE || L_max < 1 || L_max > c->cfg.max_seg ||
      L_top < 0)
    return fail(c, FS_EINVAL, "bad submit arguments");
  const bool nr = kind == FS_NEW_ROUND;
  c->acc_ready = false;
  c->plan_ready = false;
  if (nr && c->live) return fail(c, FS_ESTATE, "round live");
  if (!nr && !c->live) return fail(c, FS_ESTATE, "no live round");
  const int base = nr ? 0 : c->next_id;
  if (base + n > c->max_ids) return fail(c, FS_ECAPACITY, "node id space exhausted");
  const int n_keep = (L_top > 0 && L_top < n) ? L_top : n;
  if (c->samp_mode && base + n > c->q_rows) return fail(c, FS_ECAPACITY, "node id beyond the draft distributions (q_rows)");
  if ((nr ? 0 : c->n_live) + n_keep > c->cfg.max_live) return fail(c, FS_ECAPACITY, "max_live");
  if (c->l_glo + (nr ? 0 : c->n_live) + n_keep > c->cfg.max_ctx) return fail(c, FS_ECAPACITY, "max_ctx");
  // the pinned staging struct is reused: the previous (asynchronous) copy must have run
  if (c->ev_sub) CK_CUDA(c, cudaEventSynchronize(c->ev_sub));
  SubmitIn* s = c->h_sub;
  s->n = n;
  s->flags = flags;
  s->l_top = L_top;
  s->l_max = L_max;
  s->base_id = base;
  memcpy(s->parent, parent, sizeof(int32_t) * n);
  memcpy(s->token, token, sizeof(int32_t) * n);
  memcpy(s->own, own, sizeof(float) * n);
  CK_CUDA(c, cudaMemcpyAsync(c->d_sub, s, sizeof(SubmitIn), cudaMemcpyHostToDevice, c->st));
  if (merge) {
    merge_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->d_sub, c->d_sub2, c->d_rec, c->n_live, base);
    CK_LAUNCH(c);
  }
  submit_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, merge ? c->d_sub2 : c->d_sub, c->d_rec,
                                               nr ? 0 : c->n_live, c->cfg.vocab, c->x_new, nr ? 1 : 0);
  CK_LAUNCH(c);
  if (async) {
    if (!c->ev_sub) CK_CUDA(c, cudaEventCreateWithFlags(&c->ev_sub, cudaEventDisableTiming));
    CK_CUDA(c, cudaEventRecord(c->ev_sub, c->st));
    const int s_base = nr ? 0 : c->n_live;
    if (out) {
      out->n = n;
      out->s_base = s_base;
      out->seg_id0 = c->seg_counter;
    }
    int k = 0;
    for (int b = 0; b < n; b += L_max, k++) {
      Seg sg;
      sg.id = c->seg_counter++;
      sg.b = s_base + b;
      sg.e = s_base + std::min(b + L_max, n);
      c->queue.push_back(sg);
      if (out) out->seg_begin[k] = sg.b;
    }
    if (out) {
      out->n_segs = k;
      out->seg_begin[k] = s_base + n;
    }
    c->n_live = s_base + n;
    c->next_id = base + n;
    c->live = 1;
    return FS_OK;
  }
  CK_CUDA(c, cudaMemcpyAsync(c->h_rec, c->d_rec, offsetof(TreeRecord, acc_s), cudaMemcpyDeviceToHost, c->st));
  if ((rc = sync(c))) return rc;
  const TreeRecord* r = c->h_rec;
  if (r->err) return fail(c, r->err == -4 ? FS_ECAPACITY : FS_EINVAL, "submit rejected by validation");
  const int s_base = nr ? 0 : c->n_live;
  const int n_ids = merge ? r->n_batch : n;   // ids the call consumed
  if (out) {
    out->n = r->n;
    out->s_base = s_base;
    memcpy(out->order, r->order, sizeof(int32_t) * r->n);
    if (merge) memcpy(out->merged, r->merged, sizeof(int32_t) * n);
    out->n_segs = 0;
    out->seg_id0 = c->seg_counter;
  }
  // segmentation (R12): consecutive slices of <= L_max; a batch forms its own segments
  int k = 0;
  for (int b = 0; b < r->n; b += L_max, k++) {
    Seg sg;
    sg.id = c->seg_counter++;
    sg.b = s_base + b;
    sg.e = s_base + std::min(b + L_max, r->n);
    c->queue.push_back(sg);
    if (out) out->seg_begin[k] = sg.b;
  }
  if (out) {
    out->n_segs = k;
    out->seg_begin[k] = s_base + r->n;
  }
  c->n_live = r->n_live;
  c->next_id = base + n_ids;
  c->live = 1;
  return FS_OK;
}

int fs_verify_step(fs_ctx* c, fs_step_out* out) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (!c->prefixed) return fail(c, FS_ESTATE, "no prefix");
  const int P = c->P, p = c->rank, d = c->cfg.d_model;
  if (!c->slot[0].valid() && !c->queue.empty()) {
    c->slot[0] = c->queue.front();
    c->queue.pop_front();
  }
  const Seg cur = c->slot[p];
  const bool has = cur.valid() && cur.n() > 0;
  if (has) {
    tick_setup_kernel<<<1, FS_MAX_SEG, 0, c->st>>>(c->tree, c->d_rows, cur.b, cur.n(), c->l_glo);
    CK_LAUNCH(c);
    // host mirror of the sizes the launch configuration needs
    c->h_rows->n_rows = cur.n();
    c->h_rows->n_keys = c->l_glo + cur.e;
    if ((rc = tick_forward(c))) return rc;
  }
  // stage transport: p -> p+1 hidden rows (fp32), NCCL over NVLink, grouped
  // with the broadcast of the last stage's row results (one NCCL launch per tick)
  const Seg outseg = c->slot[P - 1];
  const bool out_rows = outseg.valid() && outseg.n() > 0;
  const bool acc = out_rows && c->live && c->n_live > 0;
  const bool stoch = c->samp_mode != 0;
  if (stoch && c->last && out_rows) {
    // stochastic acceptance needs this stage's logits: commit the rows, run the
    // walk, and broadcast its decision with the row results
    post_tick_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->res, outseg.b, outseg.n(), c->d_rec, c->n_live,
                                                    0, 1e-2f);
    CK_LAUNCH(c);
    if (acc) {
      SampleArgs sa;
      sa.t = c->tree;
      sa.lstore = c->lstore;
      sa.q = c->q_dev;
      sa.q_rows = c->q_rows;
      sa.V = c->cfg.vocab;
      sa.n_live = c->n_live;
      sa.inv_temp = c->inv_temp;
      sa.seed = c->samp_seed;
      sa.flag = 1e-6;
      sa.r = c->samp_r;
      sa.qs = c->samp_q;
      sa.dec = c->dec;
      if ((rc = launch_sample_walk(c, sa))) return rc;
    }
    if (c->logits_buf)   // parity copy of this tick's rows
      CK_CUDA(c, cudaMemcpyAsync(c->logits_buf, c->lstore + (size_t)outseg.b * c->cfg.vocab,
                                 (size_t)outseg.n() * c->cfg.vocab * 4, cudaMemcpyDeviceToDevice, c->st));
  }
  if (P > 1) {
    const Seg prev = c->slot[p > 0 ? p - 1 : 0];
    const bool recv = p > 0 && prev.valid() && prev.n() > 0;
    const bool send = !c->last && has;
    // stochastic: res[FS_MAX_SEG] and the decision that follows it in one broadcast
    const size_t bw = !out_rows ? 0 : stoch ? (sizeof(RowResult) * FS_MAX_SEG + sizeof(SampleDecision)) / 4
                                            : (size_t)outseg.n() * 2;
    if ((rc = exchange(c, c->x, send ? (size_t)cur.n() * d : 0, c->hin, recv ? (size_t)prev.n() * d : 0,
                       c->res, bw)))
      return rc;
  }
  for (int q = 0; q < P; q++)
    if (c->slot[q].valid()) c->n_cached[q] = std::max(c->n_cached[q], c->slot[q].e);
  if (out) {
    out->seg_id = outseg.valid() ? outseg.id : -1;
    out->s_begin = outseg.b;
    out->n_rows = outseg.valid() ? outseg.n() : 0;
  }
  if (out_rows) {
    const int n = outseg.n();
    c->acc_ready = false;
    c->plan_ready = false;
    if (stoch) {
      // commit (the last stage did already) and take the broadcast decision
      if (!c->last) {
        post_tick_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->res, outseg.b, n, c->d_rec, c->n_live, 0,
                                                        1e-2f);
        CK_LAUNCH(c);
      }
      if (acc) {
        apply_decision_kernel<<<1, 256, 0, c->st>>>(c->tree, c->dec, c->d_rec);
        CK_LAUNCH(c);
        // the prune plan of this decision, so fs_prune_and_compact needs no read-back
        prune_plan_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->d_rec, c->n_live);
        CK_LAUNCH(c);
      }
      CK_CUDA(c, cudaMemcpyAsync(c->h_rec, c->d_rec, sizeof(TreeRecord), cudaMemcpyDeviceToHost, c->st));
      c->acc_ready = acc;
      c->plan_ready = acc;
    } else {
      // commit the rows, then the accept walk over the updated tree and the
      // prune plan of its decision (fs_accept / fs_prune_and_compact consume them
      // without another device round trip): one kernel, one read-back
      post_tick_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->res, outseg.b, n, c->d_rec, c->n_live,
                                                      acc ? 1 : 0, 1e-2f);
      CK_LAUNCH(c);
      CK_CUDA(c, cudaMemcpyAsync(c->h_rec, c->d_rec, sizeof(TreeRecord), cudaMemcpyDeviceToHost, c->st));
      c->acc_ready = acc;
      c->plan_ready = acc;
    }
    if ((rc = sync(c))) return rc;
    if (c->h_rec->sub_err) {
      c->poisoned = true;
      return fail(c, FS_EINVAL, "an asynchronous submit was rejected by validation");
    }
    if (c->h_rec->num_err) {
      c->poisoned = true;
      return fail(c, FS_ERANGE, "attention V outside the fp16 range of the f16-P kernel (FS_TC_ATTN_P=hilo)");
    }
    if (out)
      for (int m = 0; m < n; m++) {
        out->node[m] = c->h_rec->tick_node[m];
        out->am[m] = c->h_rec->tick_res[m].am;
        out->margin[m] = c->h_rec->tick_res[m].margin;
      }
  } else {
    if ((rc = sync(c))) return rc;
  }
  for (int q = P - 1; q > 0; q--) c->slot[q] = c->slot[q - 1];
  c->slot[0] = Seg();
  return FS_OK;
}

int fs_accept(fs_ctx* c, fs_accept_out* out) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (!out) return fail(c, FS_EINVAL, "null out");
  memset(out, 0, offsetof(fs_accept_out, acc_ids));
  if (!c->live || c->n_live == 0) {
    out->progress = 0;
    return FS_OK;
  }
  if (!c->acc_ready) {
    c->plan_ready = false;
    accept_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->d_rec, c->n_live, 1e-2f);
    CK_LAUNCH(c);
    CK_CUDA(c, cudaMemcpyAsync(c->h_rec, c->d_rec, sizeof(TreeRecord), cudaMemcpyDeviceToHost, c->st));
    if ((rc = sync(c))) return rc;
    // stochastic decisions are taken by the verify step (the last stage's
    // logits); with the root verified and no such decision pending, the tree
    // changed after it (the greedy walk above only tells whether the root is
    // verified)
    if (c->samp_mode && c->h_rec->progress) return fail(c, FS_ESTATE, "stochastic decision not pending");
  }
  c->acc_ready = false;
  const TreeRecord* r = c->h_rec;
  out->progress = r->progress;
  if (!r->progress) return FS_OK;
  out->n_acc = r->n_acc;
  memcpy(out->acc_ids, r->acc_id, sizeof(int32_t) * r->n_acc);
  memcpy(out->acc_tokens, r->acc_tok, sizeof(int32_t) * r->n_acc);
  out->x_new = r->x_new;
  out->n_new = r->n_new_id;
  out->cont = r->cont;
  out->n_flagged = r->n_flagged;
  memcpy(out->flagged_ids, r->flagged, sizeof(int32_t) * r->n_flagged);
  return FS_OK;
}

int fs_prune_and_compact(fs_ctx* c, const fs_accept_out* dcs) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (!dcs) return fail(c, FS_EINVAL, "null decision");
  if (!c->live) return fail(c, FS_ESTATE, "no live round");
  if (!dcs->progress || dcs->n_acc < 1 || dcs->n_acc > c->n_live) return fail(c, FS_ESTATE, "no progress");
  if (dcs->x_new < 0 || dcs->x_new >= c->cfg.vocab) return fail(c, FS_ESTATE, "x_new outside the vocabulary");
  c->acc_ready = false;
  // the decision fs_accept returned from the verify step: its rank map is
  // already on the host (prune_plan_kernel), so no device round trip here
  const TreeRecord* hr = c->h_rec;
  const bool planned = c->plan_ready && hr->progress && hr->spec_n_pr >= 0 && dcs->n_acc == hr->n_acc &&
                       (dcs->cont != 0) == (hr->cont != 0) && dcs->x_new == hr->x_new &&
                       (!dcs->cont || dcs->n_new == hr->n_new_id) &&
                       !memcmp(dcs->acc_ids, hr->acc_id, sizeof(int32_t) * dcs->n_acc);
  c->plan_ready = false;
  DecisionIn* di = c->h_dec;
  di->n_acc = dcs->n_acc;
  di->n_new_id = dcs->cont ? dcs->n_new : -1;
  di->cont = dcs->cont ? 1 : 0;
  di->x_new = dcs->x_new;
  memcpy(di->acc_id, dcs->acc_ids, sizeof(int32_t) * dcs->n_acc);
  CK_CUDA(c, cudaMemcpyAsync(c->d_dec, di, sizeof(DecisionIn), cudaMemcpyHostToDevice, c->st));
  const int n_live_old = c->n_live;
  prune_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->d_dec, c->d_rec, n_live_old);
  CK_LAUNCH(c);
  // rank map -> host (to re-map the replicated segment schedule)
  static thread_local std::vector<int32_t> hrank;
  hrank.resize(c->cfg.max_live);
  int n_pr_new;
  if (planned) {
    memcpy(hrank.data(), hr->spec_rank, sizeof(int32_t) * c->cfg.max_live);
    n_pr_new = hr->spec_n_pr;
  } else {
    CK_CUDA(c, cudaMemcpyAsync(c->h_rec, c->d_rec, offsetof(TreeRecord, order), cudaMemcpyDeviceToHost, c->st));
    CK_CUDA(c, cudaMemcpyAsync(hrank.data(), c->tree.rank, sizeof(int32_t) * c->cfg.max_live,
                               cudaMemcpyDeviceToHost, c->st));
    if ((rc = sync(c))) return rc;
    if (c->h_rec->err) return fail(c, FS_ESTATE, "inconsistent decision");
    n_pr_new = c->h_rec->n_pr;
  }
  const int a = dcs->n_acc;
  const bool cont = dcs->cont != 0;
  // KV-cache pruning of this stage's layers
  const int nc = c->n_cached[c->rank];
  if (nc > 0) {
    const int chunks = c->cfg.head_dim * c->esz / 16;
    const int planes = c->nl * 2 * c->cfg.n_kv_heads;
    const size_t sm = (size_t)nc * chunks * 16;
    if (chunks == 16 && !getenv("FS_KV_COMPACT_SERIAL")) {
      // one round trip per plane through shared memory (<= 512 rows x 256 B)
      static std::atomic<uint64_t> kattr{0};
      once_per_device(kattr, c, [] {
        cudaFuncSetAttribute(kv_compact_smem_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FS_MAX_LIVE * 16 * 16);
      });
      kv_compact_smem_kernel<16><<<planes, 256, sm, c->st>>>((uint4*)c->kv, c->cfg.max_ctx, c->tree.rank, nc,
                                                             c->l_glo);
    } else if (chunks == 16)
      kv_compact_kernel<16><<<planes, 16, 0, c->st>>>((uint4*)c->kv, c->cfg.max_ctx, c->tree.rank, nc, c->l_glo);
    else if (chunks == 4)
      kv_compact_kernel<4><<<planes, 4, 0, c->st>>>((uint4*)c->kv, c->cfg.max_ctx, c->tree.rank, nc, c->l_glo);
    else if (chunks == 8)
      kv_compact_kernel<8><<<planes, 8, 0, c->st>>>((uint4*)c->kv, c->cfg.max_ctx, c->tree.rank, nc, c->l_glo);
    else if (chunks == 32)
      kv_compact_kernel<32><<<planes, 32, 0, c->st>>>((uint4*)c->kv, c->cfg.max_ctx, c->tree.rank, nc, c->l_glo);
    else
      return fail(c, FS_EINVAL, "unsupported head_dim for compaction");
    CK_LAUNCH(c);
  }
  // per-S-index logits of the pruned tree's verified nodes (stochastic mode)
  if (cont && c->samp_mode && c->lstore) {
    const int v4 = c->cfg.vocab / 4;
    lstore_compact_kernel<<<(v4 + 255) / 256, 256, 0, c->st>>>((float4*)c->lstore, v4, c->tree.rank, n_live_old, a);
    CK_LAUNCH(c);
  }
  // pruned S-index prefix: count of I_pr entries below x
  auto pr_below = [&](int x) {
    int k = 0;
    for (int s = 0; s < x && s < n_live_old; s++)
      if (hrank[s] >= 0 && hrank[s] >= a) k++;
    return k;
  };
  if (cont) {
    // in-flight rows at this stage (I_local)
    const Seg sg = c->slot[c->rank];
    if (c->rank > 0 && sg.valid() && sg.n() > 0) {
      const int d4 = c->cfg.d_model / 4;
      rows_compact_kernel<<<(d4 + 255) / 256, 256, 0, c->st>>>((float4*)c->hin, d4, c->tree.rank, sg.b, sg.n());
      CK_LAUNCH(c);
    }
    for (int q = 0; q < c->P; q++) {
      c->n_cached[q] = pr_below(c->n_cached[q]);
      if (c->slot[q].valid()) {
        c->slot[q].b = pr_below(c->slot[q].b);
        c->slot[q].e = pr_below(c->slot[q].e);
      }
    }
    std::deque<Seg> nq;
    for (Seg s : c->queue) {
      s.b = pr_below(s.b);
      s.e = pr_below(s.e);
      if (s.e > s.b) nq.push_back(s);
    }
    c->queue.swap(nq);
    c->n_live = n_pr_new;
    c->l_glo += a;
  } else {
    c->l_glo += a;
    c->x_new = dcs->x_new;
    reset_round(c);
  }
  // no sync: the compaction kernels are stream-ordered before any later call,
  // and no host buffer they touch is reused before the next sync
  return FS_OK;
}

int fs_query(fs_ctx* c, int32_t what, void* buf, size_t bytes, size_t* needed) {
  int rc;
  if (!check(c, &rc)) return rc;
  size_t need = 0;
  const int nl = c->n_live;
  void* src = nullptr;
  switch (what) {
    case FS_Q_STATE: need = sizeof(fs_state); break;
    case FS_Q_NODE: need = 4 * nl; src = c->tree.node; break;
    case FS_Q_TOKEN: need = 4 * nl; src = c->tree.token; break;
    case FS_Q_PARENT: need = 4 * nl; src = c->tree.par; break;
    case FS_Q_POS: need = 4 * nl; src = c->tree.depth; break;
    case FS_Q_ANC: need = (size_t)4 * nl * c->ancw; src = c->tree.anc; break;
    case FS_Q_CU: need = 4 * nl; src = c->tree.cu; break;
    case FS_Q_RETAIN: need = (size_t)4 * c->ancw; src = c->tree.retain; break;
    default: return fail(c, FS_EINVAL, "bad query");
  }
  if (needed) *needed = need;
  if (!buf) return FS_OK;
  if (bytes < need) return fail(c, FS_EINVAL, "buffer too small");
  if (what == FS_Q_STATE) {
    fs_state* s = (fs_state*)buf;
    memset(s, 0, sizeof(*s));
    s->l_glo = c->l_glo;
    s->x_new = c->x_new;
    s->live = c->live;
    s->n_live = c->n_live;
    s->next_id = c->next_id;
    s->n_stages = c->P;
    s->rank = c->rank;
    s->layer_begin = c->L0;
    s->layer_end = c->L1;
    for (int p = 0; p < c->P; p++) {
      s->n_cached[p] = c->n_cached[p];
      s->layers_per_stage[p] = c->lps[p];
      s->inflight[p][0] = c->slot[p].id;
      s->inflight[p][1] = c->slot[p].b;
      s->inflight[p][2] = c->slot[p].e;
    }
    s->n_queue = (int)c->queue.size();
    for (int i = 0; i < s->n_queue && i < FS_MAX_LIVE; i++) {
      s->queue[i][0] = c->queue[i].id;
      s->queue[i][1] = c->queue[i].b;
      s->queue[i][2] = c->queue[i].e;
    }
    s->launches = c->launches;
    return FS_OK;
  }
  if (need) {
    CK_CUDA(c, cudaMemcpyAsync(buf, src, need, cudaMemcpyDeviceToHost, c->st));
    if ((rc = sync(c))) return rc;
  }
  if (what == FS_Q_POS)
    for (int i = 0; i < nl; i++) ((int32_t*)buf)[i] += c->l_glo;
  return FS_OK;
}

int fs_read_kv(fs_ctx* c, int32_t layer, int32_t which, int32_t kvh, int32_t slot, float* out) {
  int rc;
  if (!check(c, &rc)) return rc;
  const fs_config& f = c->cfg;
  if (!out || layer < c->L0 || layer >= c->L1 || which < 0 || which > 1 || kvh < 0 ||
      kvh >= f.n_kv_heads || slot < 0 || slot >= f.max_ctx)
    return fail(c, FS_EINVAL, "bad kv index");
  const char* src = kv_plane(c, layer - c->L0, which) + ((size_t)kvh * f.max_ctx + slot) * f.head_dim * c->esz;
  std::vector<char> tmp((size_t)f.head_dim * c->esz);
  CK_CUDA(c, cudaMemcpyAsync(tmp.data(), src, tmp.size(), cudaMemcpyDeviceToHost, c->st));
  if ((rc = sync(c))) return rc;
  for (int j = 0; j < f.head_dim; j++) {
    if (c->bf) {
      uint32_t u = (uint32_t)((uint16_t*)tmp.data())[j] << 16;
      memcpy(&out[j], &u, 4);
    } else {
      out[j] = ((float*)tmp.data())[j];
    }
  }
  return FS_OK;
}

int fs_debug_write_kv(fs_ctx* c, int32_t layer, int32_t which, int32_t kvh, int32_t slot, const float* in) {
  int rc;
  if (!check(c, &rc)) return rc;
  const fs_config& f = c->cfg;
  if (!in || layer < c->L0 || layer >= c->L1 || which < 0 || which > 1 || kvh < 0 ||
      kvh >= f.n_kv_heads || slot < 0 || slot >= f.max_ctx)
    return fail(c, FS_EINVAL, "bad kv index");
  char* dst = kv_plane(c, layer - c->L0, which) + ((size_t)kvh * f.max_ctx + slot) * f.head_dim * c->esz;
  std::vector<char> tmp((size_t)f.head_dim * c->esz);
  for (int j = 0; j < f.head_dim; j++) {
    if (c->bf) {
      uint32_t u;
      memcpy(&u, &in[j], 4);
      u += 0x7FFFu + ((u >> 16) & 1u);   // round to nearest even (finite inputs)
      ((uint16_t*)tmp.data())[j] = (uint16_t)(u >> 16);
    } else {
      ((float*)tmp.data())[j] = in[j];
    }
  }
  CK_CUDA(c, cudaMemcpyAsync(dst, tmp.data(), tmp.size(), cudaMemcpyHostToDevice, c->st));
  return sync(c);
}

int fs_set_profiling(fs_ctx* c, int32_t on) {
  int rc;
  if (!check(c, &rc)) return rc;
  c->prof = on != 0;
  return FS_OK;
}

int fs_get_profile(fs_ctx* c, fs_profile* out) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (!out) return fail(c, FS_EINVAL, "null out");
  memset(out, 0, sizeof(*out));
  if ((rc = sync(c))) return rc;
  for (size_t i = 0; i < c->ev_used.size(); i++) {
    float ms = 0.f;
    CK_CUDA(c, cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]));
    if (c->ev_used[i].first == 0) {
      out->gemm_launches++;
      out->gemm_ms += ms;
      out->gemm_bytes += c->ev_used[i].second;
    } else {
      out->attn_launches++;
      out->attn_ms += ms;
      out->attn_bytes += c->ev_used[i].second;
    }
  }
  c->ev_used.clear();
  c->ev_next = 0;
  return FS_OK;
}

static int bench_kernel_impl(fs_ctx* c, int32_t kind, int32_t iters, double* us, double* bytes);

int fs_bench_kernel(fs_ctx* c, int32_t kind, int32_t iters, double* us, double* bytes) {
  int rc;
  if (!check(c, &rc)) return rc;
  // kind | FS_BENCH_WIDE: the same launches at the prefill-chunk row width, on
  // the rows of the last prefill chunk
  const bool wide = (kind & FS_BENCH_WIDE) != 0;
  use_width(c, wide);
  rc = bench_kernel_impl(c, kind & ~FS_BENCH_WIDE, iters, us, bytes);
  use_width(c, false);
  return rc;
}

static int bench_kernel_impl(fs_ctx* c, int32_t kind, int32_t iters, double* us, double* bytes) {
  int rc;
  if (kind == 11 || kind == 12) {
    // 11: the stochastic accept walk (f2) on the current tree; 12: the merge
    // kernel (f4) on the T_new of the last FS_MERGE submit.  Back-to-back
    // launches; they only rewrite the decision / merge scratch.
    if (!c->live || iters < 1 || !us || !bytes) return fail(c, FS_EINVAL, "bad bench request");
    if (kind == 11 && !(c->samp_mode && c->lstore)) return fail(c, FS_ESTATE, "stochastic mode on the last stage");
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    SampleArgs sa;
    if (kind == 11) {
      sa.t = c->tree;
      sa.lstore = c->lstore;
      sa.q = c->q_dev;
      sa.q_rows = c->q_rows;
      sa.V = c->cfg.vocab;
      sa.n_live = c->n_live;
      sa.inv_temp = c->inv_temp;
      sa.seed = c->samp_seed;
      sa.flag = 1e-6;
      sa.r = c->samp_r;
      sa.qs = c->samp_q;
      sa.dec = c->dec;
    }
    cudaEventRecord(a, c->st);
    for (int i = 0; i < iters; i++) {
      if (kind == 11) {
        if ((rc = launch_sample_walk(c, sa))) return rc;
      } else {
        merge_kernel<<<1, TREE_THREADS, 0, c->st>>>(c->tree, c->d_sub, c->d_sub2, c->d_rec, c->n_live, c->next_id);
        CK_LAUNCH(c);
      }
    }
    cudaEventRecord(b, c->st);
    CK_CUDA(c, cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *us = 1e3 * ms / iters;
    *bytes = kind == 11 ? (double)c->cfg.vocab * 8 : 0.0;   // per walked node: a logits row + a q row
    return FS_OK;
  }
#ifdef FS_DIAG  // timeline diagnostics (build with -DFS_DIAG): probe buffers allocated here
  if (kind == 9 || kind == 10) {
    // diagnostics: phase probes of attention (9) or O-projection GEMM with its
    // residual epilogue (10) launches running alone
    const size_t per = 8192, nl = 8;
    CK_CUDA(c, cudaMalloc(&c->tl_buf, per * nl * 8));
    cudaMemsetAsync(c->tl_buf, 0, per * nl * 8, c->st);
    c->tl_names.clear();
    rc = FS_OK;
    for (int i = 0; i < 6 && rc == FS_OK; i++) {
      c->att_dbg_ends = i >= 4;   // launches 4, 5: end probes only (probe cost check)
      if (kind == 9) {
        rc = launch_attention(c, 0);
      } else {
        GemmEpi e = base_epi(c);
        e.mode = EPI_RESID;
        e.x = c->x;
        e.ssq_out = c->ssq;
        e.z_gain = (const bf16*)c->lw[0].g2;
        e.z_out = (bf16*)c->y;
        rc = launch_gemm(c, c->lw[0].o, e);
      }
      cudaStreamSynchronize(c->st);
    }
    c->att_dbg_ends = 0;
    std::vector<unsigned long long> h(per * nl);
    cudaMemcpyAsync(h.data(), c->tl_buf, h.size() * 8, cudaMemcpyDeviceToHost, c->st);
    cudaStreamSynchronize(c->st);
    cudaFree(c->tl_buf);
    c->tl_buf = nullptr;
    for (size_t i = 2; i < c->tl_names.size() && i < nl; i++) {
      unsigned long long t00 = ~0ull;
      for (size_t cta = 0; cta < 512; cta++) {
        const unsigned long long v = h[i * per + cta * 16];
        if (v) t00 = std::min(t00, v);
      }
      {
        double cyc = 0, ns = 0;
        int n = 0;
        for (size_t cta = 0; cta < 512; cta++) {
          const unsigned long long* pr = &h[i * per + cta * 16];
          if (pr[0] && pr[14] && pr[15]) {
            cyc += (double)pr[15];
            ns += (double)(pr[14] - pr[0]);
            n++;
          }
        }
        fprintf(stderr, "%s launch %zu (isolated): SM clock %.0f MHz over %d CTAs\n",
                kind == 9 ? "attention" : "O-proj gemm", i, n ? cyc / ns * 1e3 : 0.0, n);
      }
      for (int k = 0; k < 15; k++) {
        std::vector<double> vals;
        for (size_t cta = 0; cta < 512; cta++) {
          const unsigned long long v = h[i * per + cta * 16 + k];
          if (v && v >= t00) vals.push_back((v - t00) / 1e3);
        }
        if (vals.empty()) continue;
        std::sort(vals.begin(), vals.end());
        fprintf(stderr, "      aprobe %2d: min %8.2f p10 %8.2f med %8.2f p90 %8.2f max %8.2f (n=%zu)\n", k,
                vals[0], vals[vals.size() / 10], vals[vals.size() / 2], vals[vals.size() * 9 / 10],
                vals.back(), vals.size());
      }
    }
    // raw per-CTA probe deltas (ns) of the last launch: timer granularity check
    {
      const size_t i = std::min(c->tl_names.size(), nl) - 1;
      for (size_t cta = 0; cta < 4; cta++) {
        const unsigned long long* pr = &h[i * per + cta * 16];
        fprintf(stderr, "cta %zu raw deltas ns:", cta);
        for (int k = 1; k < 15; k++)
          if (pr[k] && pr[0]) fprintf(stderr, " %d:%lld", k, (long long)(pr[k] - pr[0]));
        fprintf(stderr, "\n");
      }
    }
    c->tl_names.clear();
    *us = 0;
    *bytes = 0;
    return rc;
  }
  if (kind == 8) {
    // timeline of one (non-graph) stage forward: per probed launch, first CTA start and last
    // CTA end relative to the first launch's start
    const size_t per = 8192, nl = 400;
    CK_CUDA(c, cudaMalloc(&c->tl_buf, per * nl * 8));
    cudaMemsetAsync(c->tl_buf, 0, per * nl * 8, c->st);
    c->tl_names.clear();
    rc = stage_forward(c, false);
    std::vector<unsigned long long> h(per * nl);
    cudaMemcpyAsync(h.data(), c->tl_buf, h.size() * 8, cudaMemcpyDeviceToHost, c->st);
    cudaStreamSynchronize(c->st);
    cudaFree(c->tl_buf);
    c->tl_buf = nullptr;
    unsigned long long t00 = 0;
    double prev_end = 0;
    for (size_t i = 0; i < c->tl_names.size() && i < nl; i++) {
      unsigned long long st = ~0ull, en = 0;
      const bool g = c->tl_names[i] == "gemm";
      for (size_t k = 0; k < per; k++) {
        unsigned long long v = h[i * per + k];
        if (!v) continue;
        const size_t slot = k % 16;
        if (g && slot >= 7) continue;
        if (slot == 0) st = std::min(st, v);
        en = std::max(en, v);
      }
      if (st == ~0ull) continue;
      if (!t00) t00 = st;
      const double s0 = (st - t00) / 1e3, e0 = (en - t00) / 1e3;
      if (i < 24 || i + 3 >= c->tl_names.size()) {
        fprintf(stderr, "%3zu %-5s start %8.2f end %8.2f dur %6.2f gap-from-prev-end %6.2f\n", i,
                c->tl_names[i].c_str(), s0, e0, e0 - s0, s0 - prev_end);
        if (!g && i >= 6 && i <= 11) {  // attention phases over CTAs (one layer)
          for (int k = 0; k < 15; k++) {
            std::vector<double> vals;
            for (size_t cta = 0; cta < 512; cta++) {
              unsigned long long v = h[i * per + cta * 16 + k];
              if (v) vals.push_back((v - t00) / 1e3);
            }
            if (vals.empty()) continue;
            std::sort(vals.begin(), vals.end());
            fprintf(stderr, "      aprobe %2d: min %8.2f p10 %8.2f med %8.2f p90 %8.2f max %8.2f (n=%zu)\n", k,
                    vals[0], vals[vals.size() / 10], vals[vals.size() / 2], vals[vals.size() * 9 / 10],
                    vals.back(), vals.size());
          }
        }
        if (g && i >= 7 && i <= 11) {  // per-probe distribution over CTAs for one layer
          for (int k = 0; k < 13; k++) {
            std::vector<double> vals;
            for (size_t cta = 0; cta < 512; cta++) {
              unsigned long long v = h[i * per + cta * 16 + k];
              if (v) vals.push_back((v - t00) / 1e3);
            }
            if (vals.empty()) continue;
            std::sort(vals.begin(), vals.end());
            fprintf(stderr, "      probe %d: min %8.2f p10 %8.2f med %8.2f p90 %8.2f max %8.2f\n", k, vals[0],
                    vals[vals.size() / 10], vals[vals.size() / 2], vals[vals.size() * 9 / 10], vals.back());
          }
        }
      }
      prev_end = e0;
    }
    c->tl_names.clear();
    *us = prev_end;
    *bytes = 0;
    return rc;
  }
#else
  if (kind >= 8) return fail(c, FS_EINVAL, "diagnostic kinds need a -DFS_DIAG build");
#endif
  if (!c->weights || !c->prefixed || iters < 1 || !us || !bytes || kind < 0 || kind > 7)  // 8-10: above
    return fail(c, FS_EINVAL, "bad bench request");
  if (kind <= 5 && !c->bf) return fail(c, FS_EINVAL, "bf16 path only");
  if (kind == 4 && !c->last) return fail(c, FS_EINVAL, "head lives on the last stage");
  const fs_config& f = c->cfg;
  LayerW& w = c->lw[0];
  GemmEpi e = base_epi(c);
  const GemmOp* g = nullptr;
  switch (kind) {
    case 0: e = norm_input(c); g = &w.qkv; e.mode = EPI_QKV; e.bias = (const bf16*)w.bqkv; e.q_out = (bf16*)c->q;
            e.k_cache = (bf16*)kv_plane(c, 0, 0); e.v_cache = (bf16*)kv_plane(c, 0, 1); break;
    // O / down: the real residual epilogue (x += ., next norm operand, sums of
    // squares); x drifts over the iterations (timing only)
    case 1: g = &w.o; e.mode = EPI_RESID; e.x = c->x; e.ssq_out = c->ssq;
            e.z_gain = (const bf16*)w.g2; e.z_out = (bf16*)c->y; break;
    case 2: e = norm_input(c); g = &w.gu; e.mode = EPI_GLU; e.act = (bf16*)c->act; break;
    case 3: g = &w.dn; e.mode = EPI_RESID; e.x = c->x; e.ssq_out = c->ssq;
            e.z_gain = (const bf16*)w.g1; e.z_out = (bf16*)c->y; break;
    case 4: e = norm_input(c); g = &c->head; e.mode = EPI_HEAD; e.head_part = c->head_part; break;
    default: break;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double by = 0;
  if (kind == 5) {  // algorithmic bytes from one profiled launch; the timed loop runs unprofiled
    bool pr = c->prof;  // (per-launch event pairs would break the programmatic-launch overlap)
    c->prof = true;
    size_t before = c->ev_used.size();
    if ((rc = launch_attention(c, 0))) return rc;
    by = c->ev_used.size() > before ? c->ev_used.back().second : 0;
    c->ev_used.resize(before);
    c->ev_next = before * 2;
    c->prof = pr;
  }
  cudaEventRecord(a, c->st);
  for (int i = 0; i < iters; i++) {
    if (g) {
      if ((rc = launch_gemm(c, *g, e))) return rc;
      by = (double)g->sh.n_out * g->sh.K * 2;
    } else if (kind == 5 || kind == 7) {
      if (kind == 7) {
        if ((rc = tick_forward(c))) return rc;
      } else {
        if ((rc = launch_attention(c, 0))) return rc;
      }
    } else {
      rmsnorm_kernel<bf16, bf16, true><<<c->npad, 256, 0, c->st>>>(c->x, (const bf16*)w.g1, (bf16*)c->y,
                                                                   f.d_model, (float)f.rms_eps, c->d_rows);
      CK_LAUNCH(c);
      by = (double)c->h_rows->n_rows * f.d_model * 4;
    }
  }
  cudaEventRecord(b, c->st);
  CK_CUDA(c, cudaEventSynchronize(b));
#ifdef FS_DIAG
  if (g && getenv("FS_ATT_DEBUG")) {
    const int ncta = 148;
    cudaMalloc(&c->gemm_dbg, sizeof(unsigned long long) * 8 * ncta);
    cudaMemsetAsync(c->gemm_dbg, 0, sizeof(unsigned long long) * 8 * ncta, c->st);
    launch_gemm(c, *g, e);
    std::vector<unsigned long long> h(8 * ncta);
    cudaMemcpyAsync(h.data(), c->gemm_dbg, h.size() * 8, cudaMemcpyDeviceToHost, c->st);
    cudaStreamSynchronize(c->st);
    unsigned long long t0 = ~0ull, tend = 0;
    for (int i = 0; i < g->grid; i++) { t0 = std::min(t0, h[i * 8]); tend = std::max(tend, h[i * 8 + 6]); }
    for (int k = 0; k < 7; k++) {
      double sum = 0, mx = 0, mn = 1e30; int n = 0;
      for (int i = 0; i < g->grid; i++)
        if (h[i * 8 + k]) { double v = (h[i * 8 + k] - t0) / 1e3; sum += v; mx = std::max(mx, v); mn = std::min(mn, v); n++; }
      if (n) fprintf(stderr, "gemm probe %d: min %7.2f mean %7.2f max %7.2f us (n=%d)\n", k, mn, sum / n, mx, n);
    }
    fprintf(stderr, "gemm kernel span %.2f us\n", (tend - t0) / 1e3);
    cudaFree(c->gemm_dbg);
    c->gemm_dbg = nullptr;
  }
  if (kind == 5 && getenv("FS_ATT_DEBUG")) {
    // one more probed launch: per-phase times (us from CTA start), mean/max over CTAs
    const int ncta = 8 * c->cfg.n_kv_heads;
    if (!c->att_dbg) cudaMalloc(&c->att_dbg, sizeof(unsigned long long) * 16 * ncta);
    cudaMemsetAsync(c->att_dbg, 0, sizeof(unsigned long long) * 16 * ncta, c->st);
    launch_attention(c, 0);
    std::vector<unsigned long long> h(16 * ncta);
    cudaMemcpyAsync(h.data(), c->att_dbg, h.size() * 8, cudaMemcpyDeviceToHost, c->st);
    cudaStreamSynchronize(c->st);
    unsigned long long t0 = ~0ull, tend = 0;
    for (int i = 0; i < ncta; i++)
      if (h[i * 16]) { t0 = std::min(t0, h[i * 16]); tend = std::max(tend, h[i * 16 + 14]); }
    for (int k = 0; k < 15; k++) {
      double sum = 0, mx = 0; int n = 0;
      for (int i = 0; i < ncta; i++)
        if (h[i * 16] && h[i * 16 + k]) { double v = (h[i * 16 + k] - t0) / 1e3; sum += v; mx = std::max(mx, v); n++; }
      if (n) fprintf(stderr, "probe %2d: mean %7.2f us  max %7.2f us  (n=%d)\n", k, sum / n, mx, n);
    }
    fprintf(stderr, "kernel span %.2f us\n", (tend - t0) / 1e3);
    cudaFree(c->att_dbg);
    c->att_dbg = nullptr;
  }
#endif
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *us = 1e3 * ms / iters;
  *bytes = by;
  return FS_OK;
}

int fs_debug_gemm(fs_ctx* c, int32_t layer, int32_t which, const float* X, int32_t n, float* Y_dev) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (!c->bf || !c->weights || !X || !Y_dev || n < 1 || n > c->cfg.max_seg || which < 0 || which > 4 ||
      layer < c->L0 || layer >= c->L1 || (which == 4 && !c->last))
    return fail(c, FS_EINVAL, "bad debug gemm request");
  LayerW& w = c->lw[layer - c->L0];
  const GemmOp* g = which == 0 ? &w.qkv : which == 1 ? &w.o : which == 2 ? &w.gu : which == 3 ? &w.dn : &c->head;
  const int K = g->sh.K, N = g->sh.n_out, np = c->npad;
  // hi/lo bf16 pair of X into the B-operand buffer of this GEMM
  void* bbuf = (which == 1) ? c->att : (which == 3) ? c->act : c->y;
  std::vector<uint16_t> hb((size_t)2 * np * K, 0);
  for (int m = 0; m < n; m++)
    for (int k = 0; k < K; k++) {
      float v = X[(size_t)m * K + k];
      uint32_t u;
      memcpy(&u, &v, 4);
      uint32_t hi = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
      float hf;
      memcpy(&hf, &hi, 4);
      float lo = v - hf;
      uint32_t ul;
      memcpy(&ul, &lo, 4);
      uint32_t lob = (ul + 0x7fffu + ((ul >> 16) & 1u)) & 0xffff0000u;
      hb[(size_t)m * K + k] = (uint16_t)(hi >> 16);
      hb[(size_t)(np + m) * K + k] = (uint16_t)(lob >> 16);
    }
  CK_CUDA(c, cudaMemcpyAsync(bbuf, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice, c->st));
  c->h_rows->n_rows = n;
  c->h_rows->n_keys = 1;
  if ((rc = upload_rows(c))) return rc;
  GemmEpi e = base_epi(c);
  e.mode = EPI_STORE;
  e.out = Y_dev;
  e.ldo = N;
  if ((rc = launch_gemm(c, *g, e))) return rc;
  return sync(c);
}

int fs_set_acceptance(fs_ctx* c, int32_t mode, float temperature, uint64_t seed, const float* q_dev,
                      int32_t q_rows) {
  int rc;
  if (!check(c, &rc)) return rc;
  if (c->live) return fail(c, FS_ESTATE, "round live");
  if (mode == FS_ACCEPT_GREEDY) {
    c->samp_mode = 0;
    return FS_OK;
  }
  if (mode != FS_ACCEPT_STOCHASTIC || !(temperature > 0.f) || !q_dev || q_rows < 1)
    return fail(c, FS_EINVAL, "bad acceptance mode");
  if (!c->cfg.sampling) return fail(c, FS_ESTATE, "context built without cfg.sampling");
  if (c->cfg.vocab % 4) return fail(c, FS_EINVAL, "stochastic mode needs vocab % 4 == 0");
  c->samp_mode = 1;
  c->inv_temp = 1.0 / (double)temperature;
  c->samp_seed = seed;
  c->q_dev = q_dev;
  c->q_rows = q_rows;
  return FS_OK;
}

int fs_local_group_create(int32_t n_stages, fs_local_group** out) {
  if (!out) return FS_EINVAL;
  *out = nullptr;
  if (n_stages < 2 || n_stages > FS_MAX_STAGES) return FS_EINVAL;
  fs_local_group* g = new fs_local_group();
  g->P = n_stages;
  *out = g;
  return FS_OK;
}

void fs_local_group_destroy(fs_local_group* g) { delete g; }

void fs_destroy(fs_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->cfg.device);
  if (!c->xt_x.empty()) {
    cudaDeviceSynchronize();
    std::vector<double> d;
    for (auto& e : c->xt_x) {
      float ms = 0;
      cudaEventElapsedTime(&ms, e.first, e.second);
      d.push_back(1e3 * ms);
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    std::sort(d.begin(), d.end());
    fprintf(stderr, "[rank %d] NCCL tick exchanges: %zu, min %.1f us, median %.1f us, p90 %.1f us\n", c->rank,
            d.size(), d[0], d[d.size() / 2], d[d.size() * 9 / 10]);
  }
  if (c->lg) {
    std::lock_guard<std::mutex> lk(c->lg->mu);
    if (c->lg->member[c->rank] == c) c->lg->member[c->rank] = nullptr;
  }
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_sub) cudaEventDestroy(c->ev_sub);
  for (int q = 0; q < FS_MAX_STAGES; q++)
    if (c->ev_done[q]) cudaEventDestroy(c->ev_done[q]);
  if (c->fwd_exec) cudaGraphExecDestroy(c->fwd_exec);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->h_sub) cudaFreeHost(c->h_sub);
  if (c->h_dec) cudaFreeHost(c->h_dec);
  if (c->h_rec) cudaFreeHost(c->h_rec);
  if (c->h_rows) cudaFreeHost(c->h_rows);
  if (c->h_res) cudaFreeHost(c->h_res);
  if (c->h_node) cudaFreeHost(c->h_node);
  delete c;
}

const char* fs_last_error(const fs_ctx* c) { return c ? c->err.c_str() : "null context"; }

const char* fs_strerror(int code) {
  switch (code) {
    case FS_OK: return "ok";
    case FS_EINVAL: return "invalid argument";
    case FS_ENOMEM: return "arena too small";
    case FS_ESTATE: return "invalid state for this call";
    case FS_ECAPACITY: return "capacity exceeded";
    case FS_ECUDA: return "CUDA error (context poisoned)";
    case FS_ENCCL: return "NCCL error (context poisoned)";
    case FS_EPOISONED: return "context poisoned by an earlier CUDA/NCCL error";
    case FS_ERANGE: return "value outside a kernel-internal format's range (context poisoned)";
  }
  return "unknown error";
}

}  // extern "C"
