// k_tree.cuh — draft-tree kernels: metadata (Eq. 1, score order, segments,
// positions, ancestor bitsets), acceptance + Eq. 2, pruning with rank maps,
// KV-cache and in-flight-row stream compaction.
//
// Single-CTA kernels (<= 512 live nodes, one thread per node) for the
// latency-bound tree bookkeeping; grid-wide kernels for the byte moves.
#pragma once
#include "state.cuh"

namespace fs {

constexpr int TREE_THREADS = 512;

// Block-wide exclusive prefix count of a predicate over threadIdx.x using
// warp ballots + popc, and the total.  All TREE_THREADS threads must call.
FS_DEV int block_excl_count(bool pred, int* s_warp, int* total) {
  const int w = warp_id(), l = lane_id();
  uint32_t m = __ballot_sync(0xffffffffu, pred);
  int before_in_warp = __popc(m & ((1u << l) - 1u));
  if (l == 0) s_warp[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < TREE_THREADS / 32; i++) {
      int c = s_warp[i];
      s_warp[i] = acc;
      acc += c;
    }
    s_warp[TREE_THREADS / 32] = acc;
  }
  __syncthreads();
  int r = s_warp[w] + before_in_warp;
  *total = s_warp[TREE_THREADS / 32];
  __syncthreads();
  return r;
}

// ancestor-or-self bitset of S entry s by walking parents (P:248 tree mask)
FS_DEV void build_anc(const TreeDev& t, int s) {
  uint32_t* a = t.anc + (size_t)s * t.ancw;
  for (int w = 0; w < t.ancw; w++) a[w] = 0u;
  for (int j = s; j >= 0; j = t.par[j]) a[j >> 5] |= 1u << (j & 31);
}

// ---------------------------------------------------------------- submit
// Rows a1-a3 of SURVEY §8(a).  Validates first; on error writes rec->err and
// leaves the state untouched.
__global__ void __launch_bounds__(TREE_THREADS) submit_kernel(TreeDev t, const SubmitIn* in,
                                                              TreeRecord* rec, int32_t n_live,
                                                              int32_t vocab, int32_t x_new,
                                                              int32_t new_round) {
  __shared__ int s_err;
  __shared__ float s_cu[MAXLIVE];
  __shared__ int s_depth[MAXLIVE];
  __shared__ int s_done[MAXLIVE];
  __shared__ int s_rank[MAXLIVE];
  __shared__ int s_flag;
  const int i = threadIdx.x;
  const int n = in->n;
  const int base = in->base_id;
  if (n < 0) return;   // the merge kernel rejected the batch (rec->err set)
  if (i == 0) s_err = 0;
  __syncthreads();
  int p = 0, tok = 0, id = base + i;
  float own = 0.f;
  bool is_root = false;
  if (i < n) {
    p = in->parent[i];
    tok = in->token[i];
    own = in->own[i];
    is_root = new_round && i == 0;
    int e = 0;
    if (tok < 0 || tok >= vocab) e = -1;
    if (id >= t.max_ids) e = -4;
    if (is_root) {
      if (p != -1 || tok != x_new) e = -1;
    } else {
      if (!(own > 0.f && own <= 1.f)) e = -1;  // NaN fails as well
      if (p < 0 || p >= id) {
        e = -1;
      } else if (p < base) {
        if (p >= t.max_ids || t.id2s[p] < 0) e = -1;
      }
      if (e == 0) {  // duplicate sibling tokens (paths must be unique)
        for (int j = 0; j < i; j++)
          if (!(new_round && j == 0) && in->parent[j] == p && in->token[j] == tok) e = -1;
        if (p < base) {
          int ps = t.id2s[p];
          for (int s = 0; s < n_live; s++)
            if (t.par[s] == ps && t.token[s] == tok) e = -1;
        }
      }
    }
    if (e) atomicExch(&s_err, e);
  }
  __syncthreads();
  if (s_err) {
    if (i == 0) {
      rec->err = s_err;
      if (in->flags & FS_SUBMIT_ASYNC) rec->sub_err = s_err;
    }
    return;
  }
  // Eq. 1: cu = own * cu(parent), fp32 RN, folded root -> node;
  // depth = depth(parent) + 1.  Level-synchronous over in-batch parents.
  float cu = 0.f;
  int depth = 0, done = 0;
  if (i < n) {
    if (is_root) {
      cu = 1.0f;
      depth = 0;
      done = 1;
    } else if (p < base) {
      int ps = t.id2s[p];
      cu = __fmul_rn(t.cu[ps], own);
      depth = t.depth[ps] + 1;
      done = 1;
    }
    s_cu[i] = cu;
    s_depth[i] = depth;
    s_done[i] = done;
  }
  __syncthreads();
  while (true) {
    int ready = 0;
    float ncu = 0.f;
    int nd = 0;
    if (i < n && !done) {
      int pb = p - base;
      if (s_done[pb]) {
        ncu = __fmul_rn(s_cu[pb], own);
        nd = s_depth[pb] + 1;
        ready = 1;
      }
    }
    __syncthreads();
    if (ready) {
      cu = ncu;
      depth = nd;
      done = 1;
      s_cu[i] = cu;
      s_depth[i] = depth;
      s_done[i] = 1;
    }
    if (!__syncthreads_or(ready)) break;
  }
  // score order: rank by count over (cu desc, id asc) (R10); or the
  // breadth-first ablation order (FS_ORDER_BFS: depth asc, id asc)
  int rank = 0;
  if (i < n) {
    if (in->flags & FS_ORDER_BFS) {
      for (int j = 0; j < n; j++) {
        const int dj = s_depth[j];
        rank += (dj < depth) || (dj == depth && j < i);
      }
    } else {
      for (int j = 0; j < n; j++) {
        float cj = s_cu[j];
        rank += (cj > cu) || (cj == cu && j < i);
      }
    }
    s_rank[i] = rank;
  }
  const int l_top = in->l_top;
  const int n_keep = (l_top > 0 && l_top < n) ? l_top : n;
  if (i == 0) s_flag = (n_live + n_keep > t.max_live) ? -4 : 0;
  __syncthreads();
  if (s_flag) {
    if (i == 0) {
      rec->err = s_flag;
      if (in->flags & FS_SUBMIT_ASYNC) rec->sub_err = s_flag;
    }
    return;
  }
  const bool keep = i < n && rank < n_keep;
  if (keep) {
    int s = n_live + rank;
    int ps = is_root ? -1 : (p < base ? t.id2s[p] : n_live + s_rank[p - base]);
    t.node[s] = id;
    t.token[s] = tok;
    t.par[s] = ps;
    t.own[s] = is_root ? 1.0f : own;
    t.cu[s] = cu;
    t.depth[s] = depth;
    t.verified[s] = 0;
    t.am[s] = -1;
    t.margin[s] = __int_as_float(0x7f800000);
    t.id2s[id] = s;
    rec->order[rank] = id;
  }
  __syncthreads();
  if (keep) build_anc(t, n_live + rank);
  if (i == 0) {
    rec->err = 0;
    rec->n = n_keep;
    rec->n_live = n_live + n_keep;
  }
}

// ---------------------------------------------------------------- merge (f4)
// Context-aware tree expansion (§3.4): T_new, rooted at the current
// root, is merged into the live tree T_pr.  A node of T_new is new iff its
// root path is not a path of T_pr (N_new = {n | path(n) not in P_pr}).  As in
// the paper, P_pr is a hash table of path hashes, here in shared memory
// (h(root) = mix(K ^ token), h(n) = mix(h(parent) ^ (token+1) * C), open
// addressing); a hit is confirmed by comparing the two root paths token by
// token, so a hash collision cannot merge distinct paths.  Output: the APPEND
// batch of the new nodes in T_new order (parents mapped to live ids or to the
// batch's new ids base + rank) for submit_kernel, which orders it by
// cumulative score, applies top-L_se (score-aware expansion) and
// enqueues S_app (S_mer = S_pr || S_app).
FS_DEV uint64_t path_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
FS_DEV uint64_t path_step(uint64_t h_parent, int32_t tok) {
  return path_mix(h_parent ^ ((uint64_t)(tok + 1) * 0xD1B54A32D192ED03ull)) | 1ull;   // 0 = empty slot
}
constexpr int MERGE_SLOTS = 2048;

__global__ void __launch_bounds__(TREE_THREADS) merge_kernel(TreeDev t, const SubmitIn* in, SubmitIn* out,
                                                             TreeRecord* rec, int32_t n_live, int32_t base) {
  __shared__ unsigned long long s_hpr[MAXLIVE];
  __shared__ unsigned long long s_hnew[MAXLIVE];
  __shared__ int s_ok_pr[MAXLIVE];
  __shared__ int s_ok_new[MAXLIVE];
  __shared__ unsigned long long s_key[MERGE_SLOTS];
  __shared__ int s_val[MERGE_SLOTS];
  __shared__ int s_match[MAXLIVE];
  __shared__ int s_rank[MAXLIVE];
  __shared__ int s_warp[TREE_THREADS / 32 + 1];
  __shared__ int s_err;
  const int i = threadIdx.x;
  const int n = in->n;
  if (i == 0) s_err = (n < 1 || in->parent[0] != -1 || n_live < 1 || in->token[0] != t.token[0]) ? -1 : 0;
  for (int k = i; k < MERGE_SLOTS; k += TREE_THREADS) s_key[k] = 0ull;
  if (i < MAXLIVE) {
    s_ok_pr[i] = 0;
    s_ok_new[i] = 0;
  }
  __syncthreads();
  if (s_err) {
    if (i == 0) {
      rec->err = -1;
      out->n = -1;
    }
    return;
  }
  // path hashes of both trees, level-synchronous (parents precede children)
  while (true) {
    int prog_pr = 0, prog_new = 0;
    if (i < n_live && !s_ok_pr[i]) {
      const int p = t.par[i];
      if (p < 0 || s_ok_pr[p]) {
        s_hpr[i] = p < 0 ? path_step(0x5A3C5EEDull, t.token[i]) : path_step(s_hpr[p], t.token[i]);
        prog_pr = 1;
      }
    }
    if (i < n && !s_ok_new[i]) {
      const int p = in->parent[i];
      if (p < 0 || s_ok_new[p]) {
        s_hnew[i] = p < 0 ? path_step(0x5A3C5EEDull, in->token[i]) : path_step(s_hnew[p], in->token[i]);
        prog_new = 1;
      }
    }
    __syncthreads();
    if (prog_pr) s_ok_pr[i] = 1;
    if (prog_new) s_ok_new[i] = 1;
    if (!__syncthreads_or(prog_pr | prog_new)) break;
  }
  // P_pr: hash table of T_pr's path hashes -> S index
  if (i < n_live) {
    const unsigned long long h = s_hpr[i];
    for (int k = 0; k < MERGE_SLOTS; k++) {
      const int slot = (int)((h + k) & (MERGE_SLOTS - 1));
      const unsigned long long prev = atomicCAS(&s_key[slot], 0ull, h);
      if (prev == 0ull) {
        s_val[slot] = i;
        break;
      }
    }
  }
  __syncthreads();
  // N_new: lookup + exact path comparison of every candidate with the same hash
  int m = -1;
  if (i < n) {
    const unsigned long long h = s_hnew[i];
    for (int k = 0; k < MERGE_SLOTS && m < 0; k++) {
      const int slot = (int)((h + k) & (MERGE_SLOTS - 1));
      const unsigned long long key = s_key[slot];
      if (key == 0ull) break;
      if (key != h) continue;
      int a = i, b = s_val[slot];
      while (a >= 0 && b >= 0 && in->token[a] == t.token[b]) {
        a = in->parent[a];
        b = t.par[b];
      }
      if (a < 0 && b < 0) m = s_val[slot];
    }
    s_match[i] = m;
  }
  if (i == 0 && s_match[0] != 0) s_err = -1;   // (i == 0 wrote s_match[0] above)
  int n_new;
  const int r = block_excl_count(i < n && m < 0, s_warp, &n_new);
  if (i < n) s_rank[i] = r;
  __syncthreads();
  if (s_err) {
    if (i == 0) {
      rec->err = -1;
      out->n = -1;
    }
    return;
  }
  if (i < n) {
    rec->merged[i] = m >= 0 ? t.node[m] : base + r;
    if (m < 0) {
      const int p = in->parent[i];
      out->parent[r] = s_match[p] >= 0 ? t.node[s_match[p]] : base + s_rank[p];
      out->token[r] = in->token[i];
      out->own[r] = in->own[i];
    }
  }
  if (i == 0) {
    out->n = n_new;
    out->flags = FS_APPEND | (in->flags & FS_ORDER_BFS);
    out->l_top = in->l_top;
    out->l_max = in->l_max;
    out->base_id = base;
    rec->n_batch = n_new;
  }
}

// ---------------------------------------------------------------- accept
// Greedy acceptance + continuous condition (Eq. 2; R1, R3, R23).
FS_DEV void accept_walk(TreeDev t, TreeRecord* rec, int32_t n_live, float flag_margin) {
  __shared__ int s_child;
  __shared__ int s_v;
  __shared__ int s_nacc;
  __shared__ int s_stop;
  const int i = threadIdx.x;
  if (n_live <= 0 || !t.verified[0]) {
    if (i == 0) {
      rec->err = 0;
      rec->progress = 0;
    }
    return;
  }
  if (i == 0) {
    s_v = 0;
    s_nacc = 1;
    rec->acc_s[0] = 0;
    s_stop = 0;
  }
  __syncthreads();
  int c = -1;
  while (true) {
    const int v = s_v;
    const int target = t.am[v];
    if (i == 0) s_child = 0x7fffffff;
    __syncthreads();
    if (i < n_live && t.par[i] == v && t.token[i] == target) atomicMin(&s_child, i);
    __syncthreads();
    c = s_child;
    if (i == 0) {
      if (c != 0x7fffffff && t.verified[c]) {
        s_v = c;
        rec->acc_s[s_nacc++] = c;
      } else {
        s_stop = 1;
      }
    }
    __syncthreads();
    if (s_stop) break;
  }
  if (i == 0) {
    const int v = s_v;
    const int na = s_nacc;
    rec->err = 0;
    rec->progress = 1;
    rec->n_acc = na;
    rec->x_new = t.am[v];
    rec->n_new_s = (c == 0x7fffffff) ? -1 : c;
    rec->n_new_id = (c == 0x7fffffff) ? -1 : t.node[c];
    rec->cont = (c != 0x7fffffff);
    int nf = 0;
    for (int k = 0; k < na; k++) {
      int s = rec->acc_s[k];
      rec->acc_id[k] = t.node[s];
      rec->acc_tok[k] = t.token[s];
      if (t.margin[s] < flag_margin) rec->flagged[nf++] = t.node[s];
    }
    rec->n_flagged = nf;
  }
}

// ---------------------------------------------------------------- prune
// Tree pruning: I_retain = I_acc ∪ I_pr, rank map r(i) by ballot +
// popc prefix counts, S_pr in original order re-rooted at n_new (R4, R11).
// On exit (cont = 0): I_retain = I_acc, S becomes empty (R16).
__global__ void __launch_bounds__(TREE_THREADS) prune_kernel(TreeDev t, const DecisionIn* d,
                                                             TreeRecord* rec, int32_t n_live) {
  __shared__ int s_err;
  __shared__ int s_acc_s[MAXLIVE];
  __shared__ unsigned char s_is_acc[MAXLIVE];
  __shared__ int s_warp[TREE_THREADS / 32 + 1];
  __shared__ int s_nn;
  __shared__ int s_maxd;
  const int i = threadIdx.x;
  const int n_acc = d->n_acc;
  const int cont = d->cont;
  if (i == 0) {
    s_err = 0;
    s_maxd = 0;
    s_nn = -1;
    if (n_acc < 1 || n_acc > n_live) s_err = -3;
  }
  if (i < MAXLIVE) s_is_acc[i] = 0;
  __syncthreads();
  if (s_err) {
    if (i == 0) rec->err = s_err;
    return;
  }
  if (i < n_acc) {
    int id = d->acc_id[i];
    int s = (id >= 0 && id < t.max_ids) ? t.id2s[id] : -1;
    s_acc_s[i] = s;
    if (s < 0 || s >= n_live) atomicExch(&s_err, -3);
  }
  if (i == 0 && cont) {
    int id = d->n_new_id;
    int s = (id >= 0 && id < t.max_ids) ? t.id2s[id] : -1;
    if (s < 0 || s >= n_live) s_err = -3;
    s_nn = s;
  }
  __syncthreads();
  if (!s_err && i < n_acc) {
    int s = s_acc_s[i];
    if (i == 0 ? (s != 0) : (t.par[s] != s_acc_s[i - 1])) atomicExch(&s_err, -3);
    // only verified nodes can be accepted (R3): an unverified accepted node
    // would commit KV that later stages never computed
    if (!t.verified[s]) atomicExch(&s_err, -3);
    s_is_acc[s] = 1;
  }
  if (!s_err && i == 0 && cont && t.par[s_nn] != s_acc_s[n_acc - 1]) s_err = -3;
  __syncthreads();
  if (s_err) {
    if (i == 0) rec->err = s_err;
    return;
  }
  const int nn = s_nn;
  // membership: I_pr = n_new and its descendants (ancestor bitset test)
  bool in_pr = false, in_acc = false;
  if (i < n_live) {
    in_acc = s_is_acc[i];
    if (cont) in_pr = (t.anc[(size_t)i * t.ancw + (nn >> 5)] >> (nn & 31)) & 1u;
  }
  const bool ret = in_acc || in_pr;
  int n_ret, n_pr;
  const int r = block_excl_count(ret, s_warp, &n_ret);
  const int newidx = block_excl_count(in_pr, s_warp, &n_pr);
  // I_retain bitset and rank map (consumed by the KV / row compaction kernels)
  {
    uint32_t m = __ballot_sync(0xffffffffu, ret && i < n_live);
    if (lane_id() == 0 && warp_id() < t.ancw) t.retain[warp_id()] = m;
  }
  if (i < t.max_live) t.rank[i] = (i < n_live && ret) ? r : -1;
  // load the old entry, then rewrite S_pr in place
  int node = 0, tok = 0, par = -1, ver = 0, am = -1, dep = 0;
  float own = 1.f, mg = 0.f;
  if (i < n_live) {
    node = t.node[i];
    tok = t.token[i];
    par = t.par[i];
    ver = t.verified[i];
    am = t.am[i];
    dep = t.depth[i];
    own = t.own[i];
    mg = t.margin[i];
  }
  const int D = cont ? t.depth[nn] : 0;
  // new index of the old parent: count of I_pr entries before it
  __shared__ int s_newidx[MAXLIVE];
  if (i < MAXLIVE) s_newidx[i] = (i < n_live && in_pr) ? newidx : -1;
  __syncthreads();
  if (i < n_live) {
    if (in_pr) {
      const int ns = newidx;
      t.node[ns] = node;
      t.token[ns] = tok;
      t.par[ns] = (i == nn) ? -1 : s_newidx[par];
      t.own[ns] = (i == nn) ? 1.0f : own;
      t.verified[ns] = ver;
      t.am[ns] = am;
      t.margin[ns] = mg;
      t.depth[ns] = dep - D;
      t.id2s[node] = ns;
      atomicMax(&s_maxd, dep - D);
    } else {
      t.id2s[node] = -1;
    }
  }
  __syncthreads();
  // Eq. 1 relative to the new root, level by level (root -> node fold, R11)
  if (i < n_pr && t.par[i] < 0) t.cu[i] = 1.0f;
  __syncthreads();
  for (int lvl = 1; lvl <= s_maxd; lvl++) {
    if (i < n_pr && t.depth[i] == lvl) t.cu[i] = __fmul_rn(t.cu[t.par[i]], t.own[i]);
    __syncthreads();
  }
  if (i < n_pr) build_anc(t, i);
  if (i == 0) {
    rec->err = 0;
    rec->n_pr = n_pr;
    rec->n_live = n_pr;
  }
}

// The rank map and |I_pr| prune_kernel derives from the decision accept_kernel
// just recorded (same membership rule: I_acc, plus n_new and its descendants
// by the ancestor bitset when the round continues), without touching the tree.
FS_DEV void prune_plan(TreeDev t, TreeRecord* rec, int32_t n_live) {
  __shared__ unsigned char s_is_acc[MAXLIVE];
  __shared__ int s_warp[TREE_THREADS / 32 + 1];
  const int i = threadIdx.x;
  const bool ok = n_live > 0 && rec->progress && !rec->err;
  if (i < MAXLIVE) s_is_acc[i] = 0;
  __syncthreads();
  const int n_acc = ok ? rec->n_acc : 0;
  if (i < n_acc) s_is_acc[rec->acc_s[i]] = 1;
  __syncthreads();
  const int cont = ok && rec->cont, nn = cont ? rec->n_new_s : 0;
  bool in_pr = false, in_acc = false;
  if (ok && i < n_live) {
    in_acc = s_is_acc[i];
    if (cont) in_pr = (t.anc[(size_t)i * t.ancw + (nn >> 5)] >> (nn & 31)) & 1u;
  }
  const bool ret = in_acc || in_pr;
  int n_ret, n_pr;
  const int r = block_excl_count(ret, s_warp, &n_ret);
  block_excl_count(in_pr, s_warp, &n_pr);
  if (i < MAXLIVE) rec->spec_rank[i] = (i < n_live && ret) ? r : -1;
  if (i == 0) rec->spec_n_pr = ok ? n_pr : -1;
}

__global__ void __launch_bounds__(TREE_THREADS) accept_kernel(TreeDev t, TreeRecord* rec, int32_t n_live,
                                                              float flag_margin) {
  accept_walk(t, rec, n_live, flag_margin);
}

__global__ void __launch_bounds__(TREE_THREADS) prune_plan_kernel(TreeDev t, TreeRecord* rec, int32_t n_live) {
  prune_plan(t, rec, n_live);
}

// The verify step's tail in one launch: commit the output segment's row
// results into the tree (am, margin, verified) and copy them with the node
// ids into the record; then (do_accept) the accept walk and the prune plan
// of its decision.  The record is read back with one copy.
__global__ void __launch_bounds__(TREE_THREADS) post_tick_kernel(TreeDev t, const RowResult* res, int32_t s_begin,
                                                                 int32_t n_rows, TreeRecord* rec, int32_t n_live,
                                                                 int32_t do_accept, float flag_margin) {
  const int m = threadIdx.x;
  if (m < n_rows) {
    const int s = s_begin + m;
    const RowResult r = res[m];
    t.am[s] = r.am;
    t.margin[s] = r.margin;
    t.verified[s] = 1;
    rec->tick_res[m] = r;
    rec->tick_node[m] = t.node[s];
  }
  if (!do_accept) return;
  __syncthreads();   // the committed rows are visible to the whole block
  accept_walk(t, rec, n_live, flag_margin);
  __syncthreads();
  prune_plan(t, rec, n_live);
}

// ---------------------------------------------------------------- KV compaction
// Stable stream-compaction gather over this stage's KV planes:
// for retained S index i < n_cached, row l_glo+i -> l_glo+rank(i).  rank(i) <= i
// and each thread owns one 16-B column chunk of every row, visiting rows in
// increasing i and loading a batch before storing it, so the in-place move
// never overwrites a row it has not read yet.  Context rows are untouched.
template <int CHUNKS>
__global__ void kv_compact_kernel(uint4* kv, int64_t plane_rows, const int32_t* rank,
                                  int32_t n_cached, int32_t l_glo) {
  const int c = threadIdx.x;
  if (c >= CHUNKS) return;
  uint4* base = kv + (size_t)blockIdx.x * plane_rows * CHUNKS;
  constexpr int B = 8;
  for (int s0 = 0; s0 < n_cached; s0 += B) {
    uint4 buf[B];
    int dst[B];
#pragma unroll
    for (int k = 0; k < B; k++) {
      int s = s0 + k;
      int r = (s < n_cached) ? rank[s] : -1;
      dst[k] = (r >= 0 && r != s) ? r : -1;
      if (dst[k] >= 0) buf[k] = base[(size_t)(l_glo + s) * CHUNKS + c];
    }
#pragma unroll
    for (int k = 0; k < B; k++)
      if (dst[k] >= 0) base[(size_t)(l_glo + dst[k]) * CHUNKS + c] = buf[k];
  }
}

// The same gather with one round trip per plane: a 256-thread CTA loads every
// moving chunk of its plane into shared memory (all loads in flight, coalesced
// along the row), then stores them at their ranks.  Reads complete before any
// write, so overlapping source / destination rows are safe.  Dynamic shared
// memory: n_cached * CHUNKS * 16 bytes (<= max_live rows).
template <int CHUNKS>
__global__ void __launch_bounds__(256) kv_compact_smem_kernel(uint4* kv, int64_t plane_rows,
                                                              const int32_t* rank, int32_t n_cached,
                                                              int32_t l_glo) {
  extern __shared__ uint4 kv_stage[];
  uint4* base = kv + (size_t)blockIdx.x * plane_rows * CHUNKS;
  const int n = n_cached * CHUNKS;
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int s = idx / CHUNKS;
    const int r = rank[s];
    if (r >= 0 && r != s) kv_stage[idx] = base[(size_t)(l_glo + s) * CHUNKS + idx % CHUNKS];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int s = idx / CHUNKS;
    const int r = rank[s];
    if (r >= 0 && r != s) base[(size_t)(l_glo + r) * CHUNKS + idx % CHUNKS] = kv_stage[idx];
  }
}

// In-flight hidden rows of a segment (S range [s_b, s_b+n_rows)) keep the
// rows whose S index is retained (I_local); order preserved.
__global__ void rows_compact_kernel(float4* h, int32_t d4, const int32_t* rank, int32_t s_b,
                                    int32_t n_rows) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d4) return;
  int k = 0;
  for (int m = 0; m < n_rows; m++) {
    if (rank[s_b + m] >= 0) {
      if (k != m) h[(size_t)k * d4 + c] = h[(size_t)m * d4 + c];
      k++;
    }
  }
}

// ---------------------------------------------------------------- tick
// Row descriptor of a tree segment: pos = l_glo + depth (R4), slot = l_glo + S
// index (R6), context visibility [0, l_glo) plus ancestor drafts.
__global__ void tick_setup_kernel(TreeDev t, TickRows* rows, int32_t s_begin, int32_t n_rows,
                                  int32_t l_glo) {
  const int m = threadIdx.x;
  if (m < n_rows) {
    const int s = s_begin + m;
    rows->token[m] = t.token[s];
    rows->pos[m] = l_glo + t.depth[s];
    rows->slot[m] = l_glo + s;
    rows->ctx_lim[m] = l_glo;
    rows->sidx[m] = s;
  }
  if (m == 0) {
    rows->n_rows = n_rows;
    rows->l_glo = l_glo;
    rows->n_keys = l_glo + s_begin + n_rows;
    rows->s_begin = s_begin;
  }
}

}  // namespace fs
