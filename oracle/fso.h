/*
 * fso.h — CPU ORACLE for the FlowSpec pipelined tree-verification hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2507_02620_b200/, libflowspec.so) never links or
 * calls it, and this file shares no code, header or constant generator with
 * the CUDA path.
 *
 * What it computes (plain definitions, fp64 arithmetic, storage rounding at
 * the precision-contract points of SURVEY.md §8(d) / DESIGN.md "readings"):
 *   - the counter-based synthetic weight generator (SURVEY §8(d) "Generators");
 *   - a LLaMA2/Qwen2-shaped decoder forward (App. B.1 "embedding
 *     -> stacked decoder layers (self-attention + FFN + residual) ->
 *     classification head") over an explicit per-row visibility set of KV slots.
 *     Tree attention (§3.1 "tree position IDs and tree attention
 *     mask") is this function with visibility = context ∪ ancestors-or-self;
 *     prefill is the same with a causal chain.
 *   - a KV store with slot moves (§3.3 KV cache pruning).
 * The tree algorithms (Eq. 1, ordering, segmentation, accept, prune) live in
 * oracle/tree.py.
 */
#ifndef FSO_H
#define FSO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct fso_cfg {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, ffn, vocab;
  int32_t qkv_bias;  /* 1: Qwen2-style q/k/v bias */
  int32_t bf16;      /* 1: bf16 storage contract; 0: fp32 everywhere (no TF32) */
  int32_t cache_weights; /* 1: materialise weights once; 0: regenerate per use */
  double rms_eps, rope_theta;
  uint64_t seed;
} fso_cfg;

/* tensor ids: layer*16 + which; globals below */
enum { FSO_Q = 0, FSO_K = 1, FSO_V = 2, FSO_O = 3, FSO_GATE = 4, FSO_UP = 5,
       FSO_DOWN = 6, FSO_ATTN_NORM = 7, FSO_MLP_NORM = 8, FSO_BQ = 9,
       FSO_BK = 10, FSO_BV = 11,
       FSO_EMBED = 16, FSO_HEAD = 17, FSO_FINAL_NORM = 18 };

typedef struct fso_model fso_model;
typedef struct fso_kv fso_kv;

/* generator primitives (exposed for pins) */
uint64_t fso_mix64(uint64_t z);
float fso_gen_value(uint64_t seed, uint64_t tid, uint64_t e, double sigma,
                    int32_t gain, int32_t bf16);
float fso_round_bf16(float x);

fso_model* fso_model_create(const fso_cfg* cfg);
void fso_model_free(fso_model* m);
/* generate every tensor once into memory (only when cfg.cache_weights) */
int32_t fso_model_materialise(fso_model* m);
/* number of elements of a tensor, and the full tensor in HF [out,in] layout */
int64_t fso_tensor_numel(const fso_model* m, int32_t which);
int32_t fso_gen_tensor(fso_model* m, int32_t layer, int32_t which, float* out);

fso_kv* fso_kv_create(const fso_model* m, int32_t max_slots);
void fso_kv_free(fso_kv* kv);
/* read one K (which=0) or V (which=1) row of head_dim values */
int32_t fso_kv_get(const fso_kv* kv, int32_t layer, int32_t which, int32_t kvh,
                   int32_t slot, float* out);
/* stable gather of rows: for every layer in [layer_begin,layer_end), K and V,
 * every kv head: row to[i] <- row from[i] (all reads happen before all
 * writes).  PAPER.md:347 KV cache pruning. */
int32_t fso_kv_move(fso_kv* kv, int32_t layer_begin, int32_t layer_end,
                    const int32_t* from, const int32_t* to, int32_t n);
/* synthetic prefix KV for slots [0,n): sigma 1, tid 0x200000+layer*2+which,
 * e = (kvh*2^32 + slot)*head_dim + j (SURVEY §8(d) "Prefix", configs 4-5) */
int32_t fso_kv_synth(fso_kv* kv, int32_t n, uint64_t kv_seed);

/* Decoder forward over layers [layer_begin, layer_end) for n_rows rows.
 *  tokens[m]   token id (used when layer_begin == 0: x = E[token])
 *  pos[m]      RoPE position
 *  slot[m]     KV slot row m writes its K/V into (before attention)
 *  vis_off[m..m+1) indexes vis_slot: the KV slots row m attends to, in order
 *  h_in        [n_rows, d] fp32 residual input when layer_begin > 0
 *  h_out       [n_rows, d] fp32 residual output (may be NULL)
 *  logits      [n_rows, vocab] fp32 (computed iff layer_end == n_layers and
 *              logits != NULL): final RMSNorm + head.
 * Returns 0, or -1 on bad arguments. */
int32_t fso_forward(fso_model* m, fso_kv* kv, int32_t layer_begin,
                    int32_t layer_end, int32_t n_rows, const int32_t* tokens,
                    const int32_t* pos, const int32_t* slot,
                    const int32_t* vis_off, const int32_t* vis_slot,
                    const float* h_in, float* h_out, float* logits);

/* Pin tests only: 1 = drop inv of the final RMSNorm (head), 2 = drop inv of
 * the attention RMSNorm (QKV); 0 = the oracle as specified.  Lets a test show
 * that its pin fails on a plausible mistake. */
void fso_set_mutant(int32_t which);

#ifdef __cplusplus
}
#endif
#endif
