// k_gemm.cuh — small-M weight-streaming GEMM on 5th-gen tensor cores.
//
//   Y[m][n] = sum_k W[n][k] * X[m][k]     W: [N_out, K] bf16 (HF [out,in]),
//                                          X: [NT, K] bf16 activations
// Swap-AB: the weight tile is the UMMA A operand (M = 128 output rows), the
// NT (16/32/64) segment rows are the UMMA N dimension, the accumulator lives in
// TMEM (128 lanes x NT fp32 columns).  A and B tiles (64 K-elements, 128-byte
// swizzle) are staged by TMA into a STAGES-deep mbarrier ring; one elected
// thread issues tcgen05.mma; 4 epilogue warps read TMEM with tcgen05.ld.
//
// Work split: stream-K over units = (128-row tile, 64-wide k block).  Grid =
// min(#SMs, units); CTA c owns units [c*U/G, (c+1)*U/G), so every SM streams
// the same number of weight bytes (HBM-bound: M=16..64 is far below the ridge).
// A tile split across CTAs is reduced deterministically: every contributor
// writes an fp32 partial, the last to arrive (atomic counter) sums them in
// contributor order and runs the fused epilogue:
//   EPI_QKV   + bias, rotate-half RoPE at the row's position, bf16 -> Q / K
//             cache / V cache at the row's slot (K/V appended before attention)
//   EPI_GLU   silu(gate) * up with 64-row interleaved gate/up weights -> bf16
//   EPI_RESID residual += (fp32), one writer per element
//   EPI_HEAD  logits (optional fp32 copy) + per-tile top-2 for the argmax
//   EPI_STORE plain fp32 store (unit tests)
#pragma once
#include <cooperative_groups.h>

#include "state.cuh"

namespace fs {

enum { EPI_QKV = 0, EPI_GLU = 1, EPI_RESID = 2, EPI_HEAD = 3, EPI_STORE = 4 };

struct GemmShape {
  int n_out, K, kb_total, n_tiles, units, max_contrib;
  float* ws;       // [n_tiles][max_contrib][128][NT] fp32 partials
  int* counters;   // [n_tiles], zero between launches
  int late_trigger; // diagnostics: trigger dependents at exit instead of at start
  unsigned long long* dbg;  // optional phase timestamps [cta][8] (diagnostics)
};
FS_DEV unsigned long long g_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef FS_DIAG  // timeline probes (diagnostic builds only)
#define GEMM_PROBE(k)                                        \
  do {                                                       \
    if (sh.dbg) sh.dbg[(size_t)blockIdx.x * 16 + (k)] = g_gtimer(); \
  } while (0)
#else
#define GEMM_PROBE(k) do {} while (0)
#endif

struct GemmEpi {
  int mode;
  const TickRows* rows;
  // QKV
  const bf16* bias;
  const float2* rope;  // [max_ctx][64] (cos, sin)
  bf16* q_out;         // [npad][H*128]
  bf16* k_cache;       // this layer: [Hkv][max_ctx][128]
  bf16* v_cache;
  int H, Hkv, max_ctx;
  // GLU
  bf16* act;
  int ffn;
  // RESID
  float* x;
  int d;
  // HEAD
  Top2* head_part;     // [n_tiles][NT]
  float* logits;       // optional [rows][vocab]
  int vocab;
  int logits_by_s;     // 1: row m goes to logits row rows->s_begin + m (per-S-index store)
  // STORE
  float* out;
  int ldo;
  // RMSNorm feeding this GEMM, applied by linearity: the B operand is the hi/lo
  // pair of x*g and the accumulator row m is scaled by inv[m] = 1/sqrt(ss/K+eps),
  // ss summed from the producer's per-128-column partials (QKV / gate-up / head)
  const float* scale_ssq;   // [scale_n][npad] or null
  int scale_n;
  float eps;
  // RESID: per-tile sums of squares of the updated residual, and the next
  // norm's B operand z = x_new * g_next as a bf16 hi/lo pair [2*npad][d]
  float* ssq_out;           // [n_tiles][npad] or null
  const bf16* z_gain;       // g of the next RMSNorm, or null
  bf16* z_out;
};

// The activation operand carries each fp32 value as two bf16 rows (hi, lo:
// rows [0,NT) and [NT,2NT) of the B tile), so UMMA N = 2*NT and the epilogue
// adds the two accumulator halves: the GEMM sees ~16-bit-mantissa activations
// at no HBM cost (the weights dominate the bytes).
#ifndef FS_GEMM_STAGES16
#define FS_GEMM_STAGES16 5
#endif
// NT=64 (the prefill-chunk width): one CTA per SM, a deep ring so the
// 32 KB stages (weight box + 128-row activation box) keep enough bytes in flight
#ifndef FS_GEMM_STAGES32
#define FS_GEMM_STAGES32 6
#endif
#ifndef FS_GEMM_STAGES64
#define FS_GEMM_STAGES64 5
#endif
#ifndef FS_GEMM_CTAS16
#define FS_GEMM_CTAS16 2
#endif
template <int NT>
struct GemmCfg {
  static constexpr int BN = 2 * NT;                      // UMMA N
  static constexpr int A_BYTES = 128 * 64 * 2;           // 16 KB weight tile
  static constexpr int B_BYTES = BN * 64 * 2;            // activation tile (hi|lo)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // NT=16: 5 stages -> ~110 KB, two CTAs per SM (the next GEMM's CTA starts
  // streaming its weights while this one drains: early PDL trigger)
  static constexpr int STAGES = NT <= 16 ? FS_GEMM_STAGES16 : (NT <= 32 ? FS_GEMM_STAGES32 : FS_GEMM_STAGES64);
  static constexpr int MIN_CTAS = NT <= 16 ? FS_GEMM_CTAS16 : 1;   // ~110 KB: two CTAs per SM
  // two accumulator buffers (segment s uses buffer s&1) so the MMA of the next
  // tile segment never waits for the epilogue of the previous one
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int XCH_BYTES = 128 * (NT + 1) * 4;
  static constexpr int TOP_BYTES = 4 * NT * (int)sizeof(Top2);
  static constexpr int INV_BYTES = 64 * 4;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256 + XCH_BYTES + TOP_BYTES + INV_BYTES;
  // TMA producer, MMA issuer, 4 epilogue warps (8 at NT 64: two groups of 4,
  // each finishing half of the 16-column windows of a prefill-width tile)
  static constexpr int EPW = NT > 32 ? 8 : 4;
  static constexpr int THREADS = 64 + 32 * EPW;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

FS_DEV int cta_of_unit(int u, int units, int G) {
  // largest c with floor(c*U/G) <= u
  return (int)(((long long)(u + 1) * G + units - 1) / units) - 1;
}

// Epilogue operands that do not depend on the accumulator, loaded by the
// epilogue warps while the mainloop streams (they idle until acc_full): the
// dependent L2 round trips (n_rows -> pos -> rope, bias, slot, residual, gain)
// then stay off the critical path between the last MMA and the stores.
template <int W>
struct EpiPre {
  static constexpr int NP = W <= 16 ? W : 1;   // register budget: windows of <= 16 columns
  int n_rows;
  bool tile;          // bias / gv / x hold tile t's values
  float bias, gv;
  float2 cs[NP];
  int slot[NP];
  float x[NP];
};

// window j <-> token column mlo + j
template <int NT, int W, bool PFR = true>
FS_DEV void epi_prefetch(const GemmShape& sh, const GemmEpi& ep, int t, int row, int mlo, int mhi,
                         bool tile, EpiPre<W>& p) {
  const TickRows* rows = ep.rows;
  p.n_rows = rows->n_rows;
  p.tile = tile;
  p.bias = 0.f;
  p.gv = 0.f;
  const int ng = t * 128 + row;
  const int jend = min(mhi, p.n_rows) - mlo;
  if (ep.mode == EPI_QKV) {
    if (tile && ep.bias) p.bias = to_f32(ep.bias[ng]);
    if constexpr (PFR && W <= 16) {
      const int i = row & 63;
#pragma unroll
      for (int j = 0; j < W; j++) {
        const bool live = j < jend;
        p.slot[j] = live ? rows->slot[mlo + j] : 0;
        p.cs[j] = live ? ep.rope[(size_t)rows->pos[mlo + j] * 64 + i] : make_float2(0.f, 0.f);
      }
    }
  } else if (ep.mode == EPI_RESID) {
    if (tile && ep.z_gain && ng < sh.n_out) p.gv = __bfloat162float(ep.z_gain[ng]);
    if constexpr (PFR && W <= 16) {
#pragma unroll
      for (int j = 0; j < W; j++)
        p.x[j] = (tile && j < jend && ng < sh.n_out) ? ep.x[(size_t)(mlo + j) * ep.d + ng] : 0.f;
    }
  }
}

// Per-column sums over the 32 lanes (rows) of a warp for W columns: a
// reduce-scatter butterfly (each step keeps half of the columns and adds the
// partner lane's copy), then a plain butterfly; the lane's column is returned
// in col.  W <= 16 shuffles in total, no branches.
template <int W, int LVL>
FS_DEV float warp_colsum(const float* v, int lane, int& col) {
  if constexpr (W == 1) {
    float z = v[0];
#pragma unroll
    for (int o = 16 >> LVL; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    return z;
  } else {
    constexpr int O = 16 >> LVL, H = W / 2;
    const bool up = lane & O;
    float u[H];
#pragma unroll
    for (int k = 0; k < H; k++) {
      const float send = up ? v[k] : v[k + H];
      u[k] = (up ? v[k + H] : v[k]) + __shfl_xor_sync(0xffffffffu, send, O);
    }
    if (up) col += H;
    return warp_colsum<H, LVL + 1>(u, lane, col);
  }
}

// Fused epilogue for output rows (weights) t*128+row and token columns
// [mlo, mhi): v[j] holds column mlo + j (W = NT, mlo = 0 for stream-K; a
// W = NT / S window for cluster split-K rank r).
template <int NT, int W, bool PFR = true>
FS_DEV void gemm_epilogue(const GemmShape& sh, const GemmEpi& ep, int t, int row, float* v,
                          float* xch, Top2* stop, int mlo, int mhi, const EpiPre<W>& p, int bar = 1) {
  const TickRows* rows = ep.rows;
  const int n_rows = p.n_rows;
  constexpr bool PF = PFR && W <= 16;   // per-row operands prefetched
  const int ng = t * 128 + row;
  const int lane = lane_id(), q = warp_id() & 3;
  const int jend = min(mhi, n_rows) - mlo, jhi = mhi - mlo;
  if (ep.mode == EPI_QKV) {
    const int H = ep.H, Hkv = ep.Hkv;
    if (ep.bias) {
      const float b = p.tile ? p.bias : to_f32(ep.bias[ng]);
#pragma unroll
      for (int j = 0; j < W; j++) v[j] += b;
    }
    const int hh = t;  // one head (128 rows) per tile
    if (hh < H + Hkv) {  // rotate-half RoPE on q and k heads (partner row ^ 64)
#pragma unroll
      for (int j = 0; j < W; j++) xch[row * (W + 1) + j] = v[j];
      named_bar_sync(bar, 128);
      const int i = row & 63;
#pragma unroll
      for (int j = 0; j < W; j++) {
        const float pv = xch[(row ^ 64) * (W + 1) + j];
        if (j < jend) {
          const float2 cs = PF ? p.cs[PF ? j : 0] : ep.rope[(size_t)rows->pos[mlo + j] * 64 + i];
          v[j] = (row < 64) ? (v[j] * cs.x - pv * cs.y) : (v[j] * cs.x + pv * cs.y);
        }
      }
      named_bar_sync(bar, 128);
    }
#pragma unroll
    for (int j = 0; j < W; j++) {
      if (j >= jend) continue;
      const int m = mlo + j;
      const bf16 o = __float2bfloat16_rn(v[j]);
      if (hh < H) {
        ep.q_out[((size_t)m * H + hh) * 128 + row] = o;
      } else if (hh < H + Hkv) {
        const int sl = PF ? p.slot[PF ? j : 0] : rows->slot[m];
        ep.k_cache[((size_t)(hh - H) * ep.max_ctx + sl) * 128 + row] = o;
      } else {
        const int sl = PF ? p.slot[PF ? j : 0] : rows->slot[m];
        ep.v_cache[((size_t)(hh - H - Hkv) * ep.max_ctx + sl) * 128 + row] = o;
      }
    }
  } else if (ep.mode == EPI_GLU) {
#pragma unroll
    for (int j = 0; j < W; j++) xch[row * (W + 1) + j] = v[j];
    named_bar_sync(bar, 128);
    if (row < 64) {
#pragma unroll
      for (int j = 0; j < W; j++) {
        if (j >= jend) continue;
        const int m = mlo + j;
        const float g = v[j], u = xch[(row + 64) * (W + 1) + j];
        const float a = g / (1.0f + expf(-g)) * u;
        const bf16 hi = __float2bfloat16_rn(a);
        ep.act[(size_t)m * ep.ffn + t * 64 + row] = hi;
        ep.act[(size_t)(NT + m) * ep.ffn + t * 64 + row] = __float2bfloat16_rn(a - __bfloat162float(hi));
      }
    }
    named_bar_sync(bar, 128);
  } else if (ep.mode == EPI_RESID) {
    float sq[W], xn[W];
    // old residual values first (all loads in flight), then the update
#pragma unroll
    for (int j = 0; j < W; j++) {
      xn[j] = 0.f;
      if (j < jend && ng < sh.n_out) xn[j] = (PF && p.tile) ? p.x[PF ? j : 0] : ep.x[(size_t)(mlo + j) * ep.d + ng];
    }
#pragma unroll
    for (int j = 0; j < W; j++) {
      sq[j] = 0.f;
      if (j < jend && ng < sh.n_out) {
        xn[j] += v[j];
        ep.x[(size_t)(mlo + j) * ep.d + ng] = xn[j];
        sq[j] = xn[j] * xn[j];
      }
    }
    if (threadIdx.x == 64 && sh.dbg) GEMM_PROBE(10);
    if (ep.z_out && ng < sh.n_out) {  // next norm's B operand: x_new * g as a bf16 hi/lo pair
      const float gv = p.tile ? p.gv : __bfloat162float(ep.z_gain[ng]);
#pragma unroll
      for (int j = 0; j < W; j++) {
        if (j >= jhi) continue;
        const int m = mlo + j;
        const float zv = (m < n_rows) ? xn[j] * gv : 0.f;
        const bf16 hi = __float2bfloat16_rn(zv);
        ep.z_out[(size_t)m * ep.d + ng] = hi;
        ep.z_out[(size_t)(NT + m) * ep.d + ng] = __float2bfloat16_rn(zv - __bfloat162float(hi));
      }
    }
    if (threadIdx.x == 64 && sh.dbg) GEMM_PROBE(11);
    if (ep.ssq_out) {  // deterministic sums of squares of the new residual rows: one
      // partial per warp (32 output columns); the consumer sums d / 32 of them
      if constexpr (W <= 16) {
        int col = 0;
        const float z = warp_colsum<W, 0>(sq, lane, col);
        if ((lane % (32 / W)) == 0 && col < jhi) ep.ssq_out[((size_t)t * 4 + q) * NT + mlo + col] = z;
      } else {
#pragma unroll
        for (int j = 0; j < W; j++) {
          if (j >= jhi) continue;
          float z = sq[j];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
          if (lane == 0) ep.ssq_out[((size_t)t * 4 + q) * NT + mlo + j] = z;
        }
      }
    }
  } else if (ep.mode == EPI_HEAD) {
    const bool valid = ng < ep.vocab;
    if (ep.logits && valid) {
      const size_t r0 = ep.logits_by_s ? (size_t)ep.rows->s_begin : 0;
#pragma unroll
      for (int j = 0; j < W; j++)
        if (j < jend) ep.logits[(r0 + mlo + j) * ep.vocab + ng] = v[j];
    }
#pragma unroll
    for (int j = 0; j < W; j++) {
      Top2 tt;
      tt.v1 = valid ? v[j] : -INFINITY;
      tt.i1 = valid ? ng : 0x7fffffff;
      tt.v2 = -INFINITY;
      tt = top2_warp(tt);
      if (lane == 0) stop[q * W + j] = tt;
    }
    named_bar_sync(bar, 128);
    if (row < jhi) {
      Top2 r = stop[row];
      for (int w = 1; w < 4; w++) r = top2_merge(r, stop[w * W + row]);
      ep.head_part[(size_t)t * NT + mlo + row] = r;
    }
    named_bar_sync(bar, 128);
  } else {  // EPI_STORE
    if (ng < sh.n_out)
#pragma unroll
      for (int j = 0; j < W; j++)
        if (j < jend) ep.out[(size_t)(mlo + j) * ep.ldo + ng] = v[j];
  }
}

template <int NT>
__global__ void __launch_bounds__(GemmCfg<NT>::THREADS, GemmCfg<NT>::MIN_CTAS)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   GemmShape sh, GemmEpi ep) {
  using C = GemmCfg<NT>;
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;      // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int* s_flag = reinterpret_cast<int*>(tmem_holder + 1);
  float* xch = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 256);
  Top2* stop = reinterpret_cast<Top2*>(reinterpret_cast<uint8_t*>(xch) + C::XCH_BYTES);
  float* s_inv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(stop) + C::TOP_BYTES);

  const int warp = warp_id(), lane = lane_id();
  const int G = gridDim.x, c = blockIdx.x;
  const int U = sh.units, KB = sh.kb_total;
  const int u0 = (int)((long long)c * U / G), u1 = (int)((long long)(c + 1) * U / G);

  if (threadIdx.x == 0) GEMM_PROBE(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 32 * C::EPW);
    }
    fence_barrier_init();
  }
  __syncwarp();
  if (warp == 1) tmem_alloc(tmem_holder, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // dependents may launch now: they prefetch their weights and wait on
  // griddepcontrol.wait (full completion of this grid) before reading outputs
  if (!sh.late_trigger) pdl_trigger();

  if (warp == 0) {
    // ---------------- TMA producer: weights never depend on the previous
    // kernel, so they stream before the grid dependency resolves (PDL).
    if (lane == 0) {
      const uint64_t polA = l2_evict_first_policy();
      const uint64_t polB = l2_evict_last_policy();
      int stage = 0;
      uint32_t phase = 0;
      const int pre = min(u1 - u0, C::STAGES);
      const uint32_t tx = C::STAGE_BYTES;
      for (int i = 0; i < pre; i++) {
        const int u = u0 + i;
        mbar_arrive_expect_tx(&full[i], tx);
        tma_load_2d(sA + i * C::A_BYTES, &tmA, &full[i], 0, u * 128, polA);  // box-tiled weights: box u
      }
      GEMM_PROBE(1);
      pdl_wait();  // activations / residual are produced by the previous kernel
      GEMM_PROBE(2);
      for (int i = 0; i < pre; i++) {
        const int u = u0 + i;
        tma_load_2d(sB + i * C::B_BYTES, &tmB, &full[i], (u % KB) * 64, 0, polB);
      }
      stage = pre % C::STAGES;
      phase = (pre == C::STAGES) ? 1 : 0;
      for (int u = u0 + pre; u < u1; u++) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], tx);
        tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], 0, u * 128, polA);
        tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], (u % KB) * 64, 0, polB);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, C::BN);
      int stage = 0, seg = 0;
      uint32_t phase = 0;
      int u = u0;
      while (u < u1) {
        const int t = u / KB;
        const int seg_start = u, seg_end = min(u1, (t + 1) * KB);
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&acc_empty[buf], ((seg >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t tacc = tmem + (uint32_t)(buf * C::BN);
        for (; u < seg_end; u++) {
          mbar_wait(&full[stage], phase);
          if (u == u0) GEMM_PROBE(3);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < 4; k++)
            umma_bf16(tacc, umma_sdesc_sw128(a0 + k * 32), umma_sdesc_sw128(b0 + k * 32), idesc,
                      (u > seg_start || k > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&acc_full[buf]);
        seg++;
      }
      GEMM_PROBE(4);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2.. (TMEM lane quarter = warp % 4; group
    // grp of 4 warps at NT 64)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int grp = (warp - 2) >> 2;
    constexpr int EPT = 32 * C::EPW;   // epilogue threads
    // previous kernels complete (their outputs are this epilogue's inputs, and
    // their reads of this epilogue's outputs are done); then prefetch
    pdl_wait();
    EpiPre<NT> pf;
    epi_prefetch<NT, NT, false>(sh, ep, 0, row, 0, NT, false, pf);
    if (ep.scale_ssq) {
      // inv[m] of the RMSNorm applied by linearity (rows >= n_rows: padding)
      if (row < NT && grp == 0) {
        float ss = 0.f;
        for (int i = 0; i < ep.scale_n; i++) ss += ep.scale_ssq[(size_t)i * NT + row];
        s_inv[row] = 1.0f / sqrtf(ss / (float)sh.K + ep.eps);
      }
      named_bar_sync(1, EPT);
    }
    int seg = 0, u = u0;
    while (u < u1) {
      const int t = u / KB;
      const int seg_start = u, seg_end = min(u1, (t + 1) * KB);
      const int buf = seg & 1;
      const bool whole = (seg_start == t * KB) && (seg_end == (t + 1) * KB);
      const int cf = whole ? c : cta_of_unit(t * KB, U, G);
      const int cl = whole ? c : cta_of_unit((t + 1) * KB - 1, U, G);
      const int j = c - cf, nc = cl - cf + 1;
      // Two contributors (the common case: a CTA's run is longer than a tile):
      // the head contributor j = 0 always finishes the tile.  Its head segment
      // is the last of its run while the tail contributor's is the first of
      // its, so the partial is published long before; the head's epilogue
      // warps wait for it and pull it into registers while the MMA still
      // streams, keeping both L2 round trips off the tail.
      if constexpr (NT > 32) {
        // Wide rows (prefill chunks): the tile's accumulator stays in TMEM and
        // every step runs over 16-column windows (register budget: 64 columns of
        // own / partial / sum values do not fit one thread), partials summed in
        // contributor order as below; the buffer is released after its last read.
        constexpr int EW = 16;
        // per-column epilogue operands (RoPE cos/sin, KV slots, residual rows) of
        // window 0, loaded while the mainloop still streams; later windows load
        // theirs (all 16 columns in flight) just before use
        EpiPre<EW> pw;
        const int wbeg = grp * (NT / 2), wend = (grp + 1) * (NT / 2);   // this group's windows
        epi_prefetch<NT, EW, true>(sh, ep, t, row, wbeg, wbeg + EW, true, pw);
        mbar_wait(&acc_full[buf], (seg >> 1) & 1);
        tc_fence_after();
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * C::BN);
        auto own_window = [&](int wlo, float* v) {
          tmem_ld16(tl + wlo, v);
          float w[EW];
          tmem_ld16(tl + NT + wlo, w);
#pragma unroll
          for (int i = 0; i < EW; i++) v[i] += w[i];
        };
        if (threadIdx.x == 64) GEMM_PROBE(8 + 2 * (seg & 1));
        bool run_epi = whole;
        if (!whole) {
          // the head of a two-contributor tile waits for the tail's partial
          // (published at the start of the tail's run); otherwise the last
          // contributor to arrive finishes the tile
          bool publish = !(nc == 2 && j == 0);
          if (publish && nc > 2) {
            if (warp == 2 && lane == 0) *s_flag = (ld_acquire_gpu(&sh.counters[t]) == nc - 1) ? 2 : 0;
            named_bar_sync(1, EPT);
            publish = *s_flag != 2;
          }
          if (publish) {
            float* wp = sh.ws + (((size_t)t * sh.max_contrib + j) * 128 + row) * NT;
            for (int wlo = grp * (NT / 2); wlo < (grp + 1) * (NT / 2); wlo += EW) {   // this group's half
              float v[EW];
              own_window(wlo, v);
#pragma unroll
              for (int m = 0; m < EW; m += 4)
                __stcg(reinterpret_cast<float4*>(wp + wlo + m), make_float4(v[m], v[m + 1], v[m + 2], v[m + 3]));
            }
            named_bar_sync(1, EPT);
            if (warp == 2 && lane == 0) {
              __threadfence();
              const int last = (atomicAdd(&sh.counters[t], 1) == nc - 1);
              if (last) __threadfence();   // acquire: every contributor's partial is visible
              *s_flag = last;
            }
            named_bar_sync(1, EPT);
            run_epi = nc > 2 && *s_flag;
          } else {
            run_epi = true;
          }
          if (run_epi && nc == 2) {   // head: the tail's partial is published (or about to be)
            if (warp == 2 && lane == 0)
              while (ld_acquire_gpu(&sh.counters[t]) < 1) __nanosleep(64);
            named_bar_sync(1, EPT);
          }
        }
        if (run_epi) {
          for (int wlo = wbeg; wlo < wend; wlo += EW) {
            if (wlo > wbeg) epi_prefetch<NT, EW, true>(sh, ep, t, row, wlo, wlo + EW, true, pw);
            float v[EW];
            if (whole) {
              own_window(wlo, v);
            } else {
#pragma unroll
              for (int m = 0; m < EW; m++) v[m] = 0.f;
              for (int jj = 0; jj < nc; jj++) {   // contributor order (deterministic)
                float x[EW];
                if (jj == j) {
                  own_window(wlo, x);
                } else {
                  const float* rp = sh.ws + (((size_t)t * sh.max_contrib + jj) * 128 + row) * NT + wlo;
#pragma unroll
                  for (int m = 0; m < EW / 4; m++) {
                    const float4 q4 = __ldcg(reinterpret_cast<const float4*>(rp) + m);
                    x[4 * m] = q4.x;
                    x[4 * m + 1] = q4.y;
                    x[4 * m + 2] = q4.z;
                    x[4 * m + 3] = q4.w;
                  }
                }
#pragma unroll
                for (int m = 0; m < EW; m++) v[m] += x[m];
              }
            }
            if (ep.scale_ssq) {
#pragma unroll
              for (int m = 0; m < EW; m++) v[m] *= s_inv[wlo + m];
            }
            gemm_epilogue<NT, EW, true>(sh, ep, t, row, v, xch + grp * 128 * (EW + 1), stop + grp * 4 * EW, wlo,
                                        wlo + EW, pw, 2 + grp);
          }
          if (!whole && warp == 2 && lane == 0) sh.counters[t] = 0;
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
        if (threadIdx.x == 64) GEMM_PROBE(12 + (seg & 1));
      } else {
        float pre[NT];
        if (nc == 2 && j == 0) {
          if (warp == 2 && lane == 0)
            while (ld_acquire_gpu(&sh.counters[t]) < 1) __nanosleep(64);
          named_bar_sync(1, 128);
          const float* rp = sh.ws + (((size_t)t * sh.max_contrib + 1) * 128 + row) * NT;
  #pragma unroll
          for (int m = 0; m < NT / 4; m++) {
            const float4 q4 = __ldcg(reinterpret_cast<const float4*>(rp) + m);
            pre[4 * m] = q4.x;
            pre[4 * m + 1] = q4.y;
            pre[4 * m + 2] = q4.z;
            pre[4 * m + 3] = q4.w;
          }
          if (warp == 2 && lane == 0) sh.counters[t] = 0;
        }
        mbar_wait(&acc_full[buf], (seg >> 1) & 1);
        tc_fence_after();
        float v[NT];
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * C::BN);
  #pragma unroll
        for (int jc = 0; jc < NT; jc += 16) tmem_ld16(tl + jc, v + jc);
  #pragma unroll
        for (int jc = 0; jc < NT; jc += 16) {  // + lo half of the activation pair
          float w[16];
          tmem_ld16(tl + NT + jc, w);
  #pragma unroll
          for (int i = 0; i < 16; i++) v[jc + i] += w[i];
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
        if (threadIdx.x == 64) GEMM_PROBE(8 + 2 * (seg & 1));
        bool run_epi = whole;
        if (nc == 2) {
          if (j == 0) {
  #pragma unroll
            for (int m = 0; m < NT; m++) v[m] += pre[m];   // own + partial 1: contributor order
            run_epi = true;
          } else {  // tail contributor: publish (one gpu-scope release) and leave
            float* wp = sh.ws + (((size_t)t * sh.max_contrib + 1) * 128 + row) * NT;
  #pragma unroll
            for (int m = 0; m < NT; m += 4)
              __stcg(reinterpret_cast<float4*>(wp + m), make_float4(v[m], v[m + 1], v[m + 2], v[m + 3]));
            named_bar_sync(1, 128);
            if (warp == 2 && lane == 0) {
              __threadfence();
              atomicAdd(&sh.counters[t], 1);
            }
          }
        } else if (!whole) {
          // every other contributor already published (the common case for the CTA
          // finishing a tile last): reduce from registers, no partial round trip
          if (warp == 2 && lane == 0) *s_flag = (ld_acquire_gpu(&sh.counters[t]) == nc - 1) ? 2 : 0;
          named_bar_sync(1, 128);
          const bool fast = *s_flag == 2;
          if (!fast) {
            float* wp = sh.ws + (((size_t)t * sh.max_contrib + j) * 128 + row) * NT;
  #pragma unroll
            for (int m = 0; m < NT; m += 4)
              __stcg(reinterpret_cast<float4*>(wp + m), make_float4(v[m], v[m + 1], v[m + 2], v[m + 3]));
            // one gpu-scope release by the counting thread: bar.sync orders the other
            // threads' partial stores before it (fence cumulativity)
            named_bar_sync(1, 128);
            if (warp == 2 && lane == 0) {
              __threadfence();
              const int last = (atomicAdd(&sh.counters[t], 1) == nc - 1);
              if (last) __threadfence();   // acquire: every contributor's partial is visible
              *s_flag = last;
            }
            named_bar_sync(1, 128);
            run_epi = *s_flag;
          } else {
            run_epi = true;
          }
          if (run_epi) {
            float own[NT];
  #pragma unroll
            for (int m = 0; m < NT; m++) {
              own[m] = v[m];
              v[m] = 0.f;
            }
            // partials summed in contributor order (deterministic, whichever CTA is
            // last); loads of up to four contributors are in flight together
            for (int j0 = 0; j0 < nc; j0 += 4) {
              float4 pv[4][NT / 4];
  #pragma unroll
              for (int jj = 0; jj < 4; jj++) {
                if (j0 + jj < nc && j0 + jj != j) {
                  const float* rp = sh.ws + (((size_t)t * sh.max_contrib + j0 + jj) * 128 + row) * NT;
  #pragma unroll
                  for (int m = 0; m < NT / 4; m++) pv[jj][m] = __ldcg(reinterpret_cast<const float4*>(rp) + m);
                }
              }
  #pragma unroll
              for (int jj = 0; jj < 4; jj++) {
                if (j0 + jj < nc) {
                  if (j0 + jj == j) {
  #pragma unroll
                    for (int m = 0; m < NT; m++) v[m] += own[m];
                  } else {
  #pragma unroll
                    for (int m = 0; m < NT / 4; m++) {
                      v[4 * m] += pv[jj][m].x;
                      v[4 * m + 1] += pv[jj][m].y;
                      v[4 * m + 2] += pv[jj][m].z;
                      v[4 * m + 3] += pv[jj][m].w;
                    }
                  }
                }
              }
            }
            if (warp == 2 && lane == 0) sh.counters[t] = 0;
          }
          named_bar_sync(1, 128);
        }
        if (threadIdx.x == 64) GEMM_PROBE(12 + (seg & 1));
        if (run_epi) {
          if (ep.scale_ssq) {
  #pragma unroll
            for (int m = 0; m < NT; m++) v[m] *= s_inv[m];
          }
          gemm_epilogue<NT, NT, false>(sh, ep, t, row, v, xch, stop, 0, NT, pf);
        }
      }
      if (threadIdx.x == 64) GEMM_PROBE(9 + 2 * (seg & 1));
      u = seg_end;
      seg++;
    }
  }
  if (threadIdx.x == 64) GEMM_PROBE(5);
  __syncthreads();
  if (threadIdx.x == 0) GEMM_PROBE(6);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}


// ---------------------------------------------------------------- cluster split-K
// Tile-aligned split-K for GEMMs with few output tiles (QKV, O, down): the S
// CTAs splitting one 128-row weight tile over K form a thread-block cluster.
// Each CTA streams its K range into its TMEM accumulator, parks the fp32
// partial in its own shared memory, and after a cluster barrier CTA rank r
// sums the S partials of its share of token columns through distributed
// shared memory (rank order: deterministic) and runs the fused epilogue for
// them.  No global partials, atomics or fences on the epilogue path.
// W: the per-rank column window (>= ceil(NT / S)): NT / 2 for S <= 3, NT / 4 for S >= 4
template <int NT, int W>
__global__ void __launch_bounds__(192, GemmCfg<NT>::MIN_CTAS)
    gemm_cluster_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        GemmShape sh, GemmEpi ep) {
  namespace cg = cooperative_groups;
  using C = GemmCfg<NT>;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ uint8_t gsm_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* acc_full = empty + C::STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(acc_full + 2);
  float* xch = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES + 256);
  Top2* stop = reinterpret_cast<Top2*>(reinterpret_cast<uint8_t*>(xch) + C::XCH_BYTES);
  float* s_inv = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(stop) + C::TOP_BYTES);
  float* part = reinterpret_cast<float*>(sA);   // [NT][128] partial (column-major), after the mainloop

  const int warp = warp_id(), lane = lane_id();
  const int S = (int)cluster.num_blocks(), r = (int)cluster.block_rank();
  const int t = blockIdx.x / S;
  const int KB = sh.kb_total;
  const int kb0 = (int)((long long)r * KB / S), kb1 = (int)((long long)(r + 1) * KB / S);
  const int nu = kb1 - kb0;
  if (threadIdx.x == 0) GEMM_PROBE(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_full[0], 1);
    fence_barrier_init();
  }
  __syncwarp();
  if (warp == 1) tmem_alloc(tmem_holder, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (!sh.late_trigger) pdl_trigger();
  EpiPre<W> pf;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: weights before the grid dependency, activations after
      const uint64_t polA = l2_evict_first_policy();
      const uint64_t polB = l2_evict_last_policy();
      const int pre = min(nu, C::STAGES);
      for (int i = 0; i < pre; i++) {
        mbar_arrive_expect_tx(&full[i], C::STAGE_BYTES);
        tma_load_2d(sA + i * C::A_BYTES, &tmA, &full[i], 0, (t * KB + kb0 + i) * 128, polA);
      }
      GEMM_PROBE(1);
      pdl_wait();
      GEMM_PROBE(2);
      for (int i = 0; i < pre; i++) tma_load_2d(sB + i * C::B_BYTES, &tmB, &full[i], (kb0 + i) * 64, 0, polB);
      int stage = pre % C::STAGES;
      uint32_t phase = (pre == C::STAGES) ? 1 : 0;
      for (int i = pre; i < nu; i++) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
        tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], 0, (t * KB + kb0 + i) * 128, polA);
        tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], (kb0 + i) * 64, 0, polB);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(128, C::BN);
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nu; i++) {
        mbar_wait(&full[stage], phase);
        if (i == 0) GEMM_PROBE(3);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
        const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < 4; k++)
          umma_bf16(tmem, umma_sdesc_sw128(a0 + k * 32), umma_sdesc_sw128(b0 + k * 32), idesc,
                    (i > 0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[stage]);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(&acc_full[0]);
      GEMM_PROBE(4);
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    pdl_wait();
    epi_prefetch<NT, W>(sh, ep, t, row, r * NT / S, (r + 1) * NT / S, true, pf);
    if (threadIdx.x == 64 && sh.dbg) {  // diagnostics: prefetched operands have landed
      float z = pf.gv + pf.bias;
#pragma unroll
      for (int m = 0; m < EpiPre<W>::NP; m++) z += pf.x[m] + pf.cs[m].x + (float)pf.slot[m];
      if (z == 12345.f) sh.dbg[0] = 0;
      GEMM_PROBE(7);
    }
    if (ep.scale_ssq) {
      if (row < NT) {
        float ss = 0.f;
        for (int i = 0; i < ep.scale_n; i++) ss += ep.scale_ssq[(size_t)i * NT + row];
        s_inv[row] = 1.0f / sqrtf(ss / (float)sh.K + ep.eps);
      }
    }
    // pass 0 runs the reduction + epilogue code on an empty column range while
    // the mainloop streams: every global / DSMEM access is predicated off, the
    // only effect is a warm instruction cache for pass 1 (the straight-line
    // epilogue otherwise executes from cold i-cache lines, ~1 us per phase)
#pragma unroll 1
    for (int pass = 0; pass < 2; pass++) {
      if (pass == 1) {
        mbar_wait(&acc_full[0], 0);
        tc_fence_after();
        float v[NT];
        const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int j = 0; j < NT; j += 16) tmem_ld16(tl + j, v + j);
#pragma unroll
        for (int j = 0; j < NT; j += 16) {
          float w[16];
          tmem_ld16(tl + NT + j, w);
#pragma unroll
          for (int i = 0; i < 16; i++) v[j + i] += w[i];
        }
        // every MMA has completed (acc_full): the stage buffers are free for the partial
#pragma unroll
        for (int m = 0; m < NT; m++) part[m * 128 + row] = v[m];
        cluster.sync();
        if (threadIdx.x == 64) GEMM_PROBE(8);
      }
      const int mlo = r * NT / S, mhi = pass ? (r + 1) * NT / S : mlo;
      // DSMEM partials of every rank for my column window: issue up to 4
      // ranks' loads together, accumulate in rank order (deterministic)
      float acc[W];
#pragma unroll
      for (int j = 0; j < W; j++) acc[j] = 0.f;
      for (int c0 = 0; c0 < S; c0 += 4) {
        float pv[4][W];
#pragma unroll
        for (int cc = 0; cc < 4; cc++) {
          if (c0 + cc < S) {
            const uint32_t pc = dsmem_addr(part + mlo * 128 + row, (uint32_t)(c0 + cc));
#pragma unroll
            for (int j = 0; j < W; j++)
              if (mlo + j < mhi) pv[cc][j] = ld_dsmem_f32(pc + j * 128 * 4);
          }
        }
#pragma unroll
        for (int cc = 0; cc < 4; cc++) {
          if (c0 + cc < S) {
#pragma unroll
            for (int j = 0; j < W; j++) acc[j] += (mlo + j < mhi) ? pv[cc][j] : 0.f;
          }
        }
      }
      if (threadIdx.x == 64 && sh.dbg) {  // diagnostics: DSMEM loads complete
        if (acc[0] + acc[W - 1] == 12345.f) sh.dbg[1] = 0;
        GEMM_PROBE(9);
      }
      if (ep.scale_ssq) {
        named_bar_sync(1, 128);  // s_inv visible to all epilogue warps
#pragma unroll
        for (int j = 0; j < W; j++) acc[j] *= s_inv[min(mlo + j, NT - 1)];
      }
      gemm_epilogue<NT, W>(sh, ep, t, row, acc, xch, stop, mlo, mhi, pf);
    }
  }
  // matches the epilogue warps' pass-1 barrier (these warps published nothing)
  if (warp < 2) cluster_sync_relaxed();
  if (threadIdx.x == 64) GEMM_PROBE(5);
  // peers are done reading this CTA's partial (their DSMEM loads were consumed
  // before they arrive): no release needed, the epilogue stores need not drain
  cluster_sync_relaxed();
  if (threadIdx.x == 0) GEMM_PROBE(6);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

}  // namespace fs
