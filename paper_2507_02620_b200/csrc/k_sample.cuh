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


// ---------------------------------------------------------------- cluster walk
// The same walk spread over a cluster of SWC CTAs: CTA c keeps its slice of
// the vocabulary's residual r and draft q in shared memory (fp64), the
// reductions over V are block reductions combined in rank order through
// distributed shared memory (deterministic), and every CTA takes the same
// accept / reject decisions from the same reduced values; rank 0 writes the
// decision.  One CTA streamed the whole V through L2 for every pass (200 us
// per 7B walk); here each pass touches V / SWC elements per SM.
constexpr int SWC = 16;                 // CTAs per walk (non-portable cluster size)
constexpr int SWT = 512;                // threads per CTA

FS_DEV double ld_dsmem_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
FS_DEV void cluster_sync_acqrel() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// all-reduce of two values over the cluster (sum or max per value), rank order
template <bool MAX0, bool MAX1>
FS_DEV void cl_reduce2(double& v0, double& v1, double* sh, double* slot, double* bc) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double a0 = __shfl_xor_sync(0xffffffffu, v0, o), a1 = __shfl_xor_sync(0xffffffffu, v1, o);
    v0 = MAX0 ? fmax(v0, a0) : v0 + a0;
    v1 = MAX1 ? fmax(v1, a1) : v1 + a1;
  }
  __syncthreads();
  if (lane_id() == 0) {
    sh[2 * warp_id()] = v0;
    sh[2 * warp_id() + 1] = v1;
  }
  __syncthreads();
  if (tid == 0) {
    double b0 = MAX0 ? -INFINITY : 0.0, b1 = MAX1 ? -INFINITY : 0.0;
    for (int w = 0; w < SWT / 32; w++) {
      b0 = MAX0 ? fmax(b0, sh[2 * w]) : b0 + sh[2 * w];
      b1 = MAX1 ? fmax(b1, sh[2 * w + 1]) : b1 + sh[2 * w + 1];
    }
    slot[0] = b0;
    slot[1] = b1;
  }
  cluster_sync_acqrel();
  if (tid == 0) {
    double b0 = MAX0 ? -INFINITY : 0.0, b1 = MAX1 ? -INFINITY : 0.0;
    for (int c = 0; c < SWC; c++) {
      const double x0 = ld_dsmem_f64(dsmem_addr(slot, (uint32_t)c));
      const double x1 = ld_dsmem_f64(dsmem_addr(slot + 1, (uint32_t)c));
      b0 = MAX0 ? fmax(b0, x0) : b0 + x0;
      b1 = MAX1 ? fmax(b1, x1) : b1 + x1;
    }
    bc[0] = b0;
    bc[1] = b1;
  }
  cluster_sync_acqrel();   // every slot read before any CTA rewrites it; bc visible
  v0 = bc[0];
  v1 = bc[1];
}

__global__ void __launch_bounds__(SWT) sample_walk_cluster_kernel(SampleArgs a) {
  extern __shared__ double wsm[];
  __shared__ double sh[2 * (SWT / 32)];
  __shared__ double slot[6];   // [0,2) reductions, [2] slice total, [4] sample, [5] its margin
  __shared__ double bc[2];
  __shared__ int32_t s_kids[MAXLIVE];
  __shared__ int s_nk, s_v, s_nacc, s_nflag, s_done, s_pick;
  const int tid = threadIdx.x;
  const uint32_t rank = blockIdx.x;     // the grid is one cluster
  const TreeDev& t = a.t;
  const int V = a.V, n = a.n_live;
  const int per = (V + SWC - 1) / SWC;
  const int lo = min(V, (int)rank * per), hi = min(V, lo + per), ns = hi - lo;
  double* r = wsm;
  double* qs = wsm + per;
  SampleDecision* d = a.dec;
  if (n <= 0 || !t.verified[0]) {
    if (rank == 0 && tid == 0) d->progress = 0;
    return;   // every CTA returns: no cluster barrier follows
  }
  if (tid == 0) {
    s_v = 0;
    s_nacc = 1;
    s_nflag = 0;
    s_done = 0;
  }
  if (rank == 0 && tid == 0) d->acc_s[0] = 0;
  __syncthreads();
  // the slice owner of token tok and its local index
  auto ld_r = [&](int tok) { return ld_dsmem_f64(dsmem_addr(r + (tok - (tok / per) * per), (uint32_t)(tok / per))); };
  auto ld_q = [&](int tok) { return ld_dsmem_f64(dsmem_addr(qs + (tok - (tok / per) * per), (uint32_t)(tok / per))); };
  while (true) {
    const int v = s_v;
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
    const float* lg = a.lstore + (size_t)v * V;
    const float* qv = a.q + (size_t)t.node[v] * V;
    double m = -INFINITY, dummy = -INFINITY;
    for (int i = tid; i < ns; i += SWT) m = fmax(m, (double)lg[lo + i] * a.inv_temp);
    cl_reduce2<true, true>(m, dummy, sh, slot, bc);
    double z = 0.0, z2 = 0.0;
    for (int i = tid; i < ns; i += SWT) {
      const double e = exp((double)lg[lo + i] * a.inv_temp - m);
      r[i] = e;
      qs[i] = (double)qv[lo + i];
      z += e;
    }
    cl_reduce2<false, false>(z, z2, sh, slot, bc);
    for (int i = tid; i < ns; i += SWT) r[i] /= z;
    cluster_sync_acqrel();   // r normalised in every slice before remote reads
    const int nk = s_nk;
    double margin = INFINITY;
    int acc = -1;
    for (int k = 0; k < nk; k++) {
      const int c = s_kids[k];
      const int tok = t.token[c];
      const double qt = ld_q(tok);
      const double ratio = qt > 0.0 ? ld_r(tok) / qt : INFINITY;
      const double u = sample_uniform(a.seed, t.node[v], k);
      margin = fmin(margin, fabs(u - ratio));
      if (u < ratio) {
        acc = k;
        break;
      }
      cluster_sync_acqrel();   // every CTA read r(tok), q(tok) before the slices change
      double sr = 0.0, sq = 0.0;
      for (int i = tid; i < ns; i += SWT) {
        const double nr = fmax(r[i] - qs[i], 0.0);
        r[i] = nr;
        sr += nr;
        if (lo + i != tok) sq += qs[i];
      }
      cl_reduce2<false, false>(sr, sq, sh, slot, bc);
      for (int i = tid; i < ns; i += SWT) {
        r[i] /= sr;
        qs[i] = (lo + i == tok) ? 0.0 : (sq > 0.0 ? qs[i] / sq : qs[i]);
      }
      cluster_sync_acqrel();
    }
    if (acc < 0) {
      // x_new ~ residual: cluster prefix over the slice totals, then the owner
      // slice's block scan (the single-CTA kernel's search, on its slice)
      const double u = sample_uniform(a.seed, t.node[v], nk);
      const int pt = (ns + SWT - 1) / SWT;
      const int b0 = min(ns, tid * pt), b1 = min(ns, b0 + pt);
      double loc = 0.0;
      for (int i = b0; i < b1; i++) loc += r[i];
      // slice total (block sum) published in slot[2]
      double tot = loc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
      __syncthreads();
      if (lane_id() == 0) sh[warp_id()] = tot;
      __syncthreads();
      if (tid == 0) {
        double b = 0.0;
        for (int w = 0; w < SWT / 32; w++) b += sh[w];
        slot[2] = b;
        slot[5] = 1e300;   // this CTA's sample margin (set by the owner only)
        s_pick = -1;
      }
      cluster_sync_acqrel();
      double before = 0.0, total = 0.0;
      if (tid == 0) {
        for (int c = 0; c < SWC; c++) {
          const double x = ld_dsmem_f64(dsmem_addr(slot + 2, (uint32_t)c));
          if (c < (int)rank) before += x;
          total += x;
        }
        bc[0] = before;
        bc[1] = total;
      }
      __syncthreads();
      before = bc[0];
      total = bc[1];
      const double target = u * total;
      const double mine = slot[2];
      if (target >= before && (target < before + mine || (rank == SWC - 1 && !(target < total)))) {
        // this slice holds the crossing: block inclusive scan of the thread chunks
        double* scan = sh;   // reuse as [SWT/32] warp totals
        double incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane_id() >= o) incl += y;
        }
        __syncthreads();
        if (lane_id() == 31) scan[warp_id()] = incl;
        __syncthreads();
        double wbefore = 0.0;
        for (int w = 0; w < warp_id(); w++) wbefore += scan[w];
        double run = before + wbefore + incl - loc;   // cumulative sum before this thread's chunk
        if (b0 < b1 && run <= target && target < run + loc) {
          int pick = lo + b1 - 1;
          double mg = 0.0;
          for (int i = b0; i < b1; i++) {
            const double lo_c = run;
            run += r[i];
            if (run > target) {
              pick = lo + i;
              mg = fmin(target - lo_c, run - target) / total;
              break;
            }
          }
          s_pick = pick;
          bc[0] = mg;
        }
        __syncthreads();
        if (tid == 0) {
          if (s_pick < 0) {   // rounding moved the crossing out of every chunk: flag
            s_pick = hi - 1;
            bc[0] = 0.0;
          }
          slot[4] = (double)s_pick;   // publish the sample and its margin
          slot[5] = bc[0];
        }
      }
      cluster_sync_acqrel();
      if (rank == 0 && tid == 0) {
        // the owner: the first CTA (rank order) whose slot[3] was set below 1e300
        int pick = V - 1;
        double mg = 0.0;
        for (int c = 0; c < SWC; c++) {
          const double mgc = ld_dsmem_f64(dsmem_addr(slot + 5, (uint32_t)c));
          if (mgc < 1e299) {
            pick = (int)ld_dsmem_f64(dsmem_addr(slot + 4, (uint32_t)c));
            mg = mgc;
            break;
          }
        }
        margin = fmin(margin, mg);
        if (margin < a.flag) d->flagged[s_nflag++] = v;
        d->progress = 1;
        d->n_acc = s_nacc;
        d->x_new = pick;
        d->n_new_s = -1;
        d->cont = 0;
        d->n_flagged = s_nflag;
      }
      cluster_sync_acqrel();   // keep every CTA's shared memory alive for rank 0's reads
      return;
    }
    if (tid == 0) {
      if (margin < a.flag) s_nflag++;   // the same count in every CTA
      const int c = s_kids[acc];
      if (rank == 0 && margin < a.flag) d->flagged[s_nflag - 1] = v;
      if (!t.verified[c]) {
        if (rank == 0) {
          d->progress = 1;
          d->n_acc = s_nacc;
          d->x_new = t.token[c];
          d->n_new_s = c;
          d->cont = 1;
          d->n_flagged = s_nflag;
        }
        s_done = 1;
      } else {
        if (rank == 0) d->acc_s[s_nacc] = c;
        s_nacc++;
        s_v = c;
      }
    }
    __syncthreads();
    if (s_done) {
      cluster_sync_acqrel();   // no CTA exits while another may still read its slice
      return;
    }
    cluster_sync_acqrel();     // slices are rewritten for the next node
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
