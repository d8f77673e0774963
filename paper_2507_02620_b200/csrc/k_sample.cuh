// k_sample.cuh — stochastic acceptance (temperature T > 0) of the verified
// draft tree: multi-branch speculative rejection sampling, the lossless form
// for children drawn from the draft distribution without replacement
// ("tokens that lead to an aligned distribution", evaluated at
// T = 1 in Table 1; reading R24 in DESIGN.md §2).
//
// At the current node v (verified), p = softmax(logits_v / T), q = the draft
// distribution of v; for the children c_1..c_k of v in draw order (node id
// ascending):
//     accept c_i iff u_i < p(t_i) / q(t_i)
//     else  p <- norm(max(p - q, 0)),  q(t_i) <- 0, q <- norm(q)
// all rejected: x_new ~ p (inverse CDF with u_k), the round exits (Eq. 2
// false); accepted and verified: descend; accepted but unverified: x_new =
// token(c), n_new = c (Eq. 2 true).  No progress while the root is unverified
// (R23).  u(seed, node id, attempt) = mix(mix(seed ^ 0x5EED5A3C) ^
// (id * 2^16 + attempt)) >> 40, / 2^24 — the counter-based generator both
// sides implement independently.  The walk's arithmetic is fp64 (latency
// bound, one CTA; B200 runs fp64 on the CUDA cores).
#pragma once
#include "common.cuh"
#include "state.cuh"

namespace fs {

constexpr int SAMPLE_THREADS = 1024;

// the walk's outcome, broadcast from the last stage (every rank applies it to
// its replica of the tree; only the last stage holds the logits)
struct SampleDecision {
  int32_t progress, n_acc, x_new, n_new_s, cont, n_flagged;
  int32_t acc_s[MAXLIVE];
  int32_t flagged[MAXLIVE];   // S indices whose decision margin < flag
};

struct SampleArgs {
  TreeDev t;
  const float* lstore;   // [max_live][V] fp32 logits of verified nodes, by S index
  const float* q;        // [q_rows][V] draft distributions, row = node id
  int32_t q_rows;
  int32_t V;
  int32_t n_live;
  double inv_temp;
  uint64_t seed;
  double flag;
  double* r;             // [V] scratch: residual distribution
  double* qs;            // [V] scratch: draft distribution
  SampleDecision* dec;
};

FS_DEV uint64_t smix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

FS_DEV double sample_uniform(uint64_t seed, int32_t node_id, int32_t attempt) {
  const uint64_t h = smix64(smix64(seed ^ 0x5EED5A3Cull) ^ (((uint64_t)node_id << 16) + (uint64_t)attempt));
  return (double)(h >> 40) / 16777216.0;
}

// block-wide reductions over SAMPLE_THREADS threads (result on every thread)
FS_DEV double block_sum_d(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane_id() == 0) sh[warp_id()] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll 4
  for (int w = 0; w < SAMPLE_THREADS / 32; w++) s += sh[w];
  return s;
}

FS_DEV double block_max_d(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane_id() == 0) sh[warp_id()] = v;
  __syncthreads();
  double s = -INFINITY;
  for (int w = 0; w < SAMPLE_THREADS / 32; w++) s = fmax(s, sh[w]);
  return s;
}

__global__ void __launch_bounds__(SAMPLE_THREADS) sample_walk_kernel(SampleArgs a) {
  __shared__ double sh[SAMPLE_THREADS / 32];
  __shared__ double s_scan[SAMPLE_THREADS];
  __shared__ int32_t s_kids[MAXLIVE];
  __shared__ int s_nk, s_v, s_nacc, s_nflag, s_done, s_pick;
  const int tid = threadIdx.x;
  const TreeDev& t = a.t;
  const int V = a.V, n = a.n_live;
  SampleDecision* d = a.dec;
  if (n <= 0 || !t.verified[0]) {
    if (tid == 0) d->progress = 0;
    return;
  }
  if (tid == 0) {
    s_v = 0;
    s_nacc = 1;
    s_nflag = 0;
    s_done = 0;
    d->acc_s[0] = 0;
  }
  __syncthreads();
  while (true) {
    const int v = s_v;
    // children of v in draw order (node id ascending)
    if (tid == 0) s_nk = 0;
    __syncthreads();
    if (tid < n && t.par[tid] == v) {
      int rk = 0;
      const int my = t.node[tid];
      for (int j = 0; j < n; j++)
        if (t.par[j] == v && t.node[j] < my) rk++;
      s_kids[rk] = tid;
      atomicAdd(&s_nk, 1);
    }
    // p_v = softmax(logits_v / T) in fp64; q_v as given
    const float* lg = a.lstore + (size_t)v * V;
    const float* qv = a.q + (size_t)t.node[v] * V;
    double m = -INFINITY;
    for (int s = tid; s < V; s += SAMPLE_THREADS) m = fmax(m, (double)lg[s] * a.inv_temp);
    m = block_max_d(m, sh);
    double z = 0.0;
    for (int s = tid; s < V; s += SAMPLE_THREADS) {
      const double e = exp((double)lg[s] * a.inv_temp - m);
      a.r[s] = e;
      a.qs[s] = (double)qv[s];
      z += e;
    }
    z = block_sum_d(z, sh);
    for (int s = tid; s < V; s += SAMPLE_THREADS) a.r[s] /= z;
    __syncthreads();
    const int nk = s_nk;
    double margin = INFINITY;
    int acc = -1;
    for (int k = 0; k < nk; k++) {
      const int c = s_kids[k];
      const int tok = t.token[c];
      const double qt = a.qs[tok];
      const double ratio = qt > 0.0 ? a.r[tok] / qt : INFINITY;
      const double u = sample_uniform(a.seed, t.node[v], k);
      margin = fmin(margin, fabs(u - ratio));
      if (u < ratio) {
        acc = k;
        break;
      }
      // rejection: p <- norm(max(p - q, 0)); q(tok) <- 0, q <- norm(q)
      double sr = 0.0, sq = 0.0;
      for (int s = tid; s < V; s += SAMPLE_THREADS) {
        const double nr = fmax(a.r[s] - a.qs[s], 0.0);
        a.r[s] = nr;
        sr += nr;
        if (s != tok) sq += a.qs[s];
      }
      sr = block_sum_d(sr, sh);
      sq = block_sum_d(sq, sh);
      for (int s = tid; s < V; s += SAMPLE_THREADS) {
        a.r[s] /= sr;
        a.qs[s] = (s == tok) ? 0.0 : (sq > 0.0 ? a.qs[s] / sq : a.qs[s]);
      }
      __syncthreads();
    }
    if (acc < 0) {
      // x_new ~ residual: smallest t with cumsum(r)[t] > u * sum(r)
      const double u = sample_uniform(a.seed, t.node[v], nk);
      const int per = (V + SAMPLE_THREADS - 1) / SAMPLE_THREADS;
      const int b0 = min(V, tid * per), b1 = min(V, b0 + per);
      double loc = 0.0;
      for (int s = b0; s < b1; s++) loc += a.r[s];
      s_scan[tid] = loc;
      __syncthreads();
      for (int o = 1; o < SAMPLE_THREADS; o <<= 1) {   // inclusive scan (Hillis-Steele)
        const double x = tid >= o ? s_scan[tid - o] : 0.0;
        __syncthreads();
        s_scan[tid] += x;
        __syncthreads();
      }
      const double total = s_scan[SAMPLE_THREADS - 1];
      const double target = u * total;
      if (tid == 0) {
        s_pick = V - 1;
        sh[0] = 0.0;   // u * total at or beyond the last boundary: flag
      }
      __syncthreads();
      double run = s_scan[tid] - loc;
      if (b0 < b1 && run <= target && target < s_scan[tid]) {
        int pick = b1 - 1;
        double mg = 0.0;   // rounding moved the crossing out of this chunk: flag
        for (int s = b0; s < b1; s++) {
          const double lo = run;
          run += a.r[s];
          if (run > target) {
            pick = s;
            mg = fmin(target - lo, run - target) / total;
            break;
          }
        }
        s_pick = pick;
        sh[0] = mg;
      }
      __syncthreads();
      if (tid == 0) {
        margin = fmin(margin, sh[0]);
        if (margin < a.flag) d->flagged[s_nflag++] = v;
        d->progress = 1;
        d->n_acc = s_nacc;
        d->x_new = s_pick;
        d->n_new_s = -1;
        d->cont = 0;
        d->n_flagged = s_nflag;
      }
      return;
    }
    if (tid == 0) {
      if (margin < a.flag) d->flagged[s_nflag++] = v;
      const int c = s_kids[acc];
      if (!t.verified[c]) {
        d->progress = 1;
        d->n_acc = s_nacc;
        d->x_new = t.token[c];
        d->n_new_s = c;
        d->cont = 1;
        d->n_flagged = s_nflag;
        s_done = 1;
      } else {
        d->acc_s[s_nacc++] = c;
        s_v = c;
      }
    }
    __syncthreads();
    if (s_done) return;
  }
}

// Every rank: the broadcast decision -> the accept record (as accept_walk
// writes it; no prune plan: fs_prune_and_compact reads the rank map back).
__global__ void apply_decision_kernel(TreeDev t, const SampleDecision* d, TreeRecord* rec) {
  const int i = threadIdx.x;
  const int na = d->progress ? d->n_acc : 0;
  for (int k = i; k < na; k += blockDim.x) {
    const int s = d->acc_s[k];
    rec->acc_s[k] = s;
    rec->acc_id[k] = t.node[s];
    rec->acc_tok[k] = t.token[s];
  }
  const int nf = d->progress ? d->n_flagged : 0;
  for (int k = i; k < nf; k += blockDim.x) rec->flagged[k] = t.node[d->flagged[k]];
  if (i == 0) {
    rec->err = 0;
    rec->progress = d->progress;
    rec->n_acc = na;
    rec->x_new = d->x_new;
    rec->n_new_s = d->progress ? d->n_new_s : -1;
    rec->n_new_id = (d->progress && d->n_new_s >= 0) ? t.node[d->n_new_s] : -1;
    rec->cont = d->progress ? d->cont : 0;
    rec->n_flagged = nf;
    rec->spec_n_pr = -1;
  }
}

// Logits rows of the retained pruned-tree nodes follow their S index (I_pr:
// i -> rank(i) - a <= i): each thread owns one 16-byte column chunk and moves
// rows in increasing i, so the in-place move never overwrites an unread row.
__global__ void lstore_compact_kernel(float4* L, int32_t v4, const int32_t* rank, int32_t n_live, int32_t a) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= v4) return;
  for (int i = 0; i < n_live; i++) {
    const int r = rank[i];
    if (r >= a && r - a != i) L[(size_t)(r - a) * v4 + col] = L[(size_t)i * v4 + col];
  }
}

}  // namespace fs
