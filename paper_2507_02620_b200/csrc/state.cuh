// state.cuh — device-resident data structures of one pipeline stage.
#pragma once
#include "common.cuh"

namespace fs {

constexpr int MAXSEG = 64;     // FS_MAX_SEG
constexpr int MAXLIVE = 512;   // FS_MAX_LIVE
constexpr int ANCW_MAX = MAXLIVE / 32;

// Row descriptor of the rows a stage runs this tick (tree segment or prefill
// chunk).  Kernels read sizes from here, so a tick is graph-replayable.
struct TickRows {
  int32_t n_rows;          // rows in the segment (0 = nothing to do)
  int32_t l_glo;           // committed context length
  int32_t n_keys;          // attention key slots [0, n_keys) may be visible
  int32_t s_begin;         // S index of row 0 (tree mode)
  int32_t token[MAXSEG];
  int32_t pos[MAXSEG];     // RoPE position (l_glo + depth, or prefill index)
  int32_t slot[MAXSEG];    // KV slot the row writes (l_glo + S index)
  int32_t ctx_lim[MAXSEG]; // key slots < ctx_lim are visible (context / causal)
  int32_t sidx[MAXSEG];    // S index whose ancestor bitset masks the draft keys, -1 none
};

// Replicated draft-tree state (every rank holds the same), capacity max_live.
struct TreeDev {
  int32_t* node;      // node id per S index
  int32_t* token;
  int32_t* par;       // parent S index, -1 root
  float* own;         // draft score c(n)
  float* cu;          // Eq. 1 cumulative score relative to the current root
  int32_t* depth;
  uint32_t* anc;      // [max_live][ancw] ancestor-or-self bitsets over S indices
  int32_t* verified;
  int32_t* am;        // argmax of the base model at the node
  float* margin;      // top-1 minus top-2
  int32_t* id2s;      // node id -> S index, -1 if not live; capacity max_ids
  int32_t* rank;      // last prune: S index -> rank in I_retain, -1 not retained
  uint32_t* retain;   // last prune: I_retain bitset
  int32_t max_live, ancw, max_ids;
};

// Per-segment result record, broadcast from the last stage.
struct RowResult {
  int32_t am;
  float margin;
};

// Small control record written by the tree kernels and read back by the host.
struct TreeRecord {
  int32_t err;              // 0 ok, else FS_E* code
  int32_t n;                // nodes added (submit)
  int32_t n_live;           // live nodes after the call
  int32_t progress, n_acc, x_new, n_new_s, n_new_id, cont, n_flagged;
  int32_t n_pr;             // |I_pr| (prune)
  int32_t n_batch;          // merge: nodes of T_new whose path is new (ids base .. base+n_batch-1)
  int32_t sub_err;          // sticky: an asynchronous submit's validation error (read by the next verify)
  int32_t num_err;          // sticky: a value outside a kernel-internal format's range (fp16 V of the f16-P attention)
  int32_t order[MAXLIVE];   // submit: batch node ids in S order
  int32_t merged[MAXLIVE];  // merge: node id of every T_new node (existing or new)
  int32_t acc_s[MAXLIVE];   // accept: S indices of S_acc
  int32_t acc_id[MAXLIVE];
  int32_t acc_tok[MAXLIVE];
  int32_t flagged[MAXLIVE];
  // accept (verify step): the prune rank map this decision implies, computed
  // ahead so fs_prune_and_compact needs no device round trip when the caller
  // passes the decision fs_accept returned (prune_plan_kernel)
  int32_t spec_n_pr;
  int32_t spec_rank[MAXLIVE];
  // verify step: the output segment's row results and node ids (one D2H with the record)
  RowResult tick_res[FS_MAX_SEG];
  int32_t tick_node[FS_MAX_SEG];
};

// Input of the submit kernel (copied host -> device)
struct SubmitIn {
  int32_t n, flags, l_top, l_max;
  int32_t base_id;          // id of batch node 0
  int32_t parent[MAXLIVE];  // parent node ids
  int32_t token[MAXLIVE];
  float own[MAXLIVE];
};

struct DecisionIn {
  int32_t n_acc, n_new_id, cont, x_new;
  int32_t acc_id[MAXLIVE];
};

}  // namespace fs
