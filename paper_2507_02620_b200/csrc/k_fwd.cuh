// k_fwd.cuh — decoder-layer kernels other than the tcgen05 weight GEMM:
// embedding gather, RMSNorm, tree-masked attention (bf16 tensor-core
// mma.sync flash-decoding with split-KV, and an fp32 CUDA-core variant for
// the fp32 configuration), split combine, argmax/top-2, and the fp32
// CUDA-core GEMM + epilogues used by the fp32 (no-TF32) configuration.
#pragma once
#include <cooperative_groups.h>

#include "state.cuh"

namespace fs {


// ---------------------------------------------------------------- embedding
template <typename T>
__global__ void embed_kernel(const T* __restrict__ E, int d, const TickRows* rows, float* x) {
  const int m = blockIdx.x;
  if (m >= rows->n_rows) return;
  const size_t tok = (size_t)rows->token[m];
  for (int k = threadIdx.x; k < d; k += blockDim.x) x[(size_t)m * d + k] = to_f32(E[tok * d + k]);
}

// First RMSNorm input of a stage's forward: x = the embedding rows (E != null),
// the received rows (src != x) or x as it is; then per-32-column sums of
// squares of x [d/32][npad] and z = x*g as the bf16 hi/lo B operand [2*npad][d]
// (RMSNorm applied by linearity in the GEMM).  CTA (m, y) covers the 32-column
// groups g = 4 * (y + gridDim.y * i) + w (warp w) with coalesced loads, so a row
// is spread over gridDim.y CTAs (latency: every load of a row in flight);
// rows >= n_rows give z = 0.
template <typename TE>
__global__ void __launch_bounds__(128) norm_prep_kernel(const TE* __restrict__ E, const float* src, float* x,
                                                        const bf16* __restrict__ g, bf16* z, float* ssq, int d,
                                                        const TickRows* rows) {
  const int m = blockIdx.x, np = gridDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cy = blockIdx.y, ny = gridDim.y;
  const bool live = m < rows->n_rows;
  const TE* er = (E && live) ? E + (size_t)rows->token[m] * d : nullptr;
  const float* xs = (E ? x : src) + (size_t)m * d;
  float* xr = x + (size_t)m * d;
  const int ng = d / 32;   // d % 32 == 0 (cfg_valid): whole groups, warp-uniform bound
#pragma unroll 2
  for (int i = 0; (cy + ny * i) * 4 + warp < ng; i++) {
    const int grp = (cy + ny * i) * 4 + warp;
    const int k = grp * 32 + lane;
    float v = 0.f;
    if (live) {
      v = er ? to_f32(er[k]) : xs[k];
      if (er || src != x) xr[k] = v;
    }
    const float gv = v * __bfloat162float(g[k]);
    const bf16 hi = __float2bfloat16_rn(gv);
    z[(size_t)m * d + k] = hi;
    z[(size_t)(np + m) * d + k] = __float2bfloat16_rn(gv - __bfloat162float(hi));
    float s = v * v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) ssq[(size_t)grp * np + m] = s;
  }
}

// ---------------------------------------------------------------- RMSNorm
// y = round(x * 1/sqrt(mean(x^2) + eps) * g)  (LLaMA RMSNorm; R18 rounding)
// Rows >= n_rows are zero-filled (they are the padding columns of the GEMM).
// SPLIT (bf16 path): y holds 2*npad rows, row m = bf16(v), row npad+m =
// bf16(v - bf16(v)) (the hi/lo activation pair of the GEMM B operand).
template <typename TW, typename TO, bool SPLIT>
__global__ void rmsnorm_kernel(const float* __restrict__ x, const TW* __restrict__ g, TO* y,
                               int d, float eps, const TickRows* rows) {
  const int m = blockIdx.x;
  TO* yr = y + (size_t)m * d;
  TO* yl = y + (size_t)(gridDim.x + m) * d;
  if (m >= rows->n_rows) {
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
      yr[k] = from_f32<TO>(0.f);
      if (SPLIT) yl[k] = from_f32<TO>(0.f);
    }
    return;
  }
  const float* xr = x + (size_t)m * d;
  float ss = 0.f;
  for (int k = threadIdx.x; k < d; k += blockDim.x) ss += xr[k] * xr[k];
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane_id() == 0) red[warp_id()] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const float v = xr[k] * inv * to_f32(g[k]);
    const TO h = from_f32<TO>(v);
    yr[k] = h;
    if (SPLIT) yl[k] = from_f32<TO>(v - to_f32(h));
  }
}

// ---------------------------------------------------------------- visibility
// Key slot k is visible to row m iff it is committed context below ctx_lim
// (causal in prefill) or a draft slot l_glo+a with a in anc(row).
FS_DEV bool key_visible(const TickRows* rows, int m, int k, const uint32_t* anc, int ancw,
                        int max_live) {
  if (k < rows->ctx_lim[m]) return true;
  const int s = rows->sidx[m];
  const int a = k - rows->l_glo;
  if (s < 0 || a < 0 || a >= max_live) return false;
  return (anc[(size_t)s * ancw + (a >> 5)] >> (a & 31)) & 1u;
}

// ---------------------------------------------------------------- fp32 attention
// CUDA-core attention for the fp32 configuration (launch-bound sizes).
// grid (H, MAXSEG), block 128, dyn smem n_keys_cap floats.
template <typename T>
__global__ void attn_simple_kernel(const T* __restrict__ q, const T* __restrict__ kc,
                                   const T* __restrict__ vc, T* o, const TickRows* rows,
                                   const uint32_t* anc, int ancw, int max_live, int H, int Hkv,
                                   int hd, int max_ctx, float scale) {
  extern __shared__ float sc[];
  const int h = blockIdx.x, m = blockIdx.y;
  if (m >= rows->n_rows) return;
  const int kvh = h / (H / Hkv);
  const int nk = rows->n_keys;
  const T* qr = q + ((size_t)m * H + h) * hd;
  const T* kb = kc + (size_t)kvh * max_ctx * hd;
  const T* vb = vc + (size_t)kvh * max_ctx * hd;
  __shared__ float red[32];
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < nk; k += blockDim.x) {
    float s = -INFINITY;
    if (key_visible(rows, m, k, anc, ancw, max_live)) {
      float dot = 0.f;
      for (int j = 0; j < hd; j++) dot += to_f32(qr[j]) * to_f32(kb[(size_t)k * hd + j]);
      s = dot * scale;
    }
    sc[k] = s;
    mx = fmaxf(mx, s);
  }
  for (int of = 16; of > 0; of >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, of));
  if (lane_id() == 0) red[warp_id()] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < (int)blockDim.x / 32; w++) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float den = 0.f;
  for (int k = threadIdx.x; k < nk; k += blockDim.x) {
    float p = (sc[k] == -INFINITY) ? 0.f : expf(sc[k] - mx);
    sc[k] = p;
    den += p;
  }
  for (int of = 16; of > 0; of >>= 1) den += __shfl_xor_sync(0xffffffffu, den, of);
  if (lane_id() == 0) red[warp_id()] = den;
  __syncthreads();
  den = 0.f;
  for (int w = 0; w < (int)blockDim.x / 32; w++) den += red[w];
  for (int j = threadIdx.x; j < hd; j += blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < nk; k++)
      if (sc[k] != 0.f) acc += sc[k] * to_f32(vb[(size_t)k * hd + j]);
    o[((size_t)m * H + h) * hd + j] = from_f32<T>(acc / den);
  }
}

// ---------------------------------------------------------------- bf16 attention
// Split-KV flash-decoding on tensor cores (mma.sync m16n8k16 bf16 -> fp32).
// CTA = (key chunk of ATT_KC slots, kv head).  Query rows of the CTA are the
// G = H/Hkv heads sharing the kv head times the padded segment rows (GQA
// packing into M).  Each CTA writes an unnormalised partial (O, m, l) per row;
// attn_combine_kernel merges the chunks.
constexpr int ATT_KC = 128;     // keys per CTA
constexpr int ATT_HD = 128;     // head dim (all bf16 configs)
constexpr int ATT_LD = ATT_HD + 8;  // padded smem row (bf16 elements): conflict-free ldmatrix

FS_DEV void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
FS_DEV void ldsm_x2(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(p)));
}
FS_DEV void ldsm_x2_t(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(p)));
}
FS_DEV void mma_bf16_16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                           uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
FS_DEV void mma_f16_16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                          uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// two bf16 (one 32-bit register) -> two fp16, exact in fp16's normal range
FS_DEV uint32_t bf16x2_to_f16x2(uint32_t v) {
  const __half2 h = __floats2half2_rn(__uint_as_float(v << 16), __uint_as_float(v & 0xFFFF0000u));
  return *reinterpret_cast<const uint32_t*>(&h);
}
// nonzero if either bf16 of the pair is outside fp16's finite range (biased
// exponent >= 127 + 16: |v| >= 65536; every smaller bf16 converts finitely) or
// not finite: the fp16 P.V paths flag it (AttnArgs::num_err -> FS_ERANGE)
FS_DEV uint32_t f16_range_check(uint32_t x) {
  return (uint32_t)(((x >> 7) & 0xFFu) >= 143u) | (uint32_t)(((x >> 23) & 0xFFu) >= 143u);
}
#ifndef FS_MHA_P16
#define FS_MHA_P16 1
#endif
FS_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
FS_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
FS_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct AttnArgs {
  const bf16* q;        // [npad][H*128]
  const bf16* kc;       // layer K cache [Hkv][max_ctx][128]
  const bf16* vc;
  const TickRows* rows;
  const uint32_t* anc;
  float* ws_o;          // [n_chunk_cap][Hkv][QR][128]
  float* ws_ml;         // [n_chunk_cap][Hkv][QR][2]
  int ancw, max_live, H, Hkv, max_ctx, npad, n_chunk_cap;
  float scale_log2;     // log2(e) / sqrt(hd)
  float resc_log2;      // GQA online softmax: raise the running max when a tile exceeds it by more
                        // than 2^resc_log2 (8; FS_TCA_RESCALE overrides, 0 = at every increase: tests)
  unsigned long long* dbg;  // optional phase timestamps [cta][16] (diagnostics)
  int dbg_ends;             // diagnostics: record only the first and last probe
  int32_t* num_err;         // sticky range flag (TreeRecord::num_err)
};
FS_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef FS_DIAG  // timeline probes (diagnostic builds only)
#define ATT_PROBE(k)                                                               \
  do {                                                                             \
    if (a.dbg && threadIdx.x == 0 && (!a.dbg_ends || (k) == 0 || (k) == 14))      \
      a.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (k)] = gtimer();  \
  } while (0)
#else
#define ATT_PROBE(k) do {} while (0)
#endif

// block 128 threads (4 warps); dyn smem: Q [QR][LD] + K,V [KC][LD] + anc rows
__global__ void __launch_bounds__(128) attn_mma_kernel(AttnArgs a) {
  extern __shared__ __align__(16) uint8_t att_smem[];
  const int chunk = blockIdx.x, kvh = blockIdx.y;
  const TickRows* rows = a.rows;
  const int n_rows = rows->n_rows;
  const int nk = rows->n_keys;
  const int k0 = chunk * ATT_KC;
  const int G = a.H / a.Hkv;
  const int QR = G * a.npad;           // query rows (multiple of 16)
  const int MT = QR / 16;              // m16 tiles
  bf16* sQ = reinterpret_cast<bf16*>(att_smem);
  bf16* sK = sQ + (size_t)QR * ATT_LD;
  bf16* sV = sK + ATT_KC * ATT_LD;
  uint32_t* sAnc = reinterpret_cast<uint32_t*>(sV + ATT_KC * ATT_LD);  // [npad][ancw]
  if (k0 >= nk || n_rows == 0) return;   // grid is sized for max_ctx (graph replay)
  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  // ---- stage Q (GQA-packed), K, V chunk, ancestor rows
  for (int idx = tid; idx < QR * (ATT_HD / 8); idx += 128) {
    const int r = idx / (ATT_HD / 8), c = idx % (ATT_HD / 8);
    const int g = r / a.npad, m = r % a.npad;
    const bf16* src = a.q + ((size_t)m * a.H + kvh * G + g) * ATT_HD + c * 8;
    cp_async16(sQ + (size_t)r * ATT_LD + c * 8, src);
  }
  const bf16* kbase = a.kc + ((size_t)kvh * a.max_ctx) * ATT_HD;
  const bf16* vbase = a.vc + ((size_t)kvh * a.max_ctx) * ATT_HD;
  for (int idx = tid; idx < ATT_KC * (ATT_HD / 8); idx += 128) {
    const int r = idx / (ATT_HD / 8), c = idx % (ATT_HD / 8);
    const int slot = min(k0 + r, a.max_ctx - 1);
    cp_async16(sK + (size_t)r * ATT_LD + c * 8, kbase + (size_t)slot * ATT_HD + c * 8);
    cp_async16(sV + (size_t)r * ATT_LD + c * 8, vbase + (size_t)slot * ATT_HD + c * 8);
  }
  for (int idx = tid; idx < a.npad * a.ancw; idx += 128) {
    const int m = idx / a.ancw, w = idx % a.ancw;
    const int s = (m < n_rows) ? rows->sidx[m] : -1;
    sAnc[idx] = (s >= 0) ? a.anc[(size_t)s * a.ancw + w] : 0u;
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- work split: m-tiles x key splits over the 4 warps
  const int KS = (MT >= 4) ? 1 : 4 / MT;            // key splits per m-tile
  const int keys_per = ATT_KC / KS;                 // 32, 64 or 128
  const int g_row = lane >> 2, t4 = lane & 3;
  for (int mt = (MT >= 4 ? warp : warp % MT); mt < MT; mt += (MT >= 4 ? 4 : MT)) {
    const int ks = (MT >= 4) ? 0 : warp / MT;
    const int kbeg = ks * keys_per;
    float oacc[16][4];
#pragma unroll
    for (int j = 0; j < 16; j++) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    // query rows of this thread (two rows: g_row, g_row+8)
    int qm[2], ctx[2], sl[2];
    for (int h2 = 0; h2 < 2; h2++) {
      const int r = mt * 16 + g_row + 8 * h2;
      qm[h2] = r % a.npad;
      ctx[h2] = (qm[h2] < n_rows) ? rows->ctx_lim[qm[h2]] : 0;
      sl[h2] = (qm[h2] < n_rows) ? rows->sidx[qm[h2]] : -1;
    }
    for (int kb = kbeg; kb < kbeg + keys_per; kb += 32) {
      if (k0 + kb >= nk) break;
      float sacc[4][4];
#pragma unroll
      for (int j = 0; j < 4; j++) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < ATT_HD / 16; kk++) {
        uint32_t a0, a1, a2, a3;
        const bf16* qa = sQ + (size_t)(mt * 16 + (lane & 15)) * ATT_LD + kk * 16 + (lane >> 4) * 8;
        ldsm_x4(a0, a1, a2, a3, qa);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint32_t b0, b1;
          const bf16* kp = sK + (size_t)(kb + j * 8 + (lane & 7)) * ATT_LD + kk * 16 + ((lane >> 3) & 1) * 8;
          ldsm_x2(b0, b1, kp);
          mma_bf16_16816(sacc[j], a0, a1, a2, a3, b0, b1);
        }
      }
      // mask + scale (log2 domain), online softmax
      float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int h2 = e >> 1;
          const int key = k0 + kb + j * 8 + t4 * 2 + (e & 1);
          bool vis = key < nk && qm[h2] < n_rows;
          if (vis && key >= ctx[h2]) {
            const int aa = key - rows->l_glo;
            vis = sl[h2] >= 0 && aa >= 0 && aa < a.max_live &&
                  ((sAnc[qm[h2] * a.ancw + (aa >> 5)] >> (aa & 31)) & 1u);
          }
          const float v = vis ? sacc[j][e] * a.scale_log2 : -INFINITY;
          sacc[j][e] = v;
          mnew[h2] = fmaxf(mnew[h2], v);
        }
#pragma unroll
      for (int h2 = 0; h2 < 2; h2++) {
        mnew[h2] = fmaxf(mnew[h2], __shfl_xor_sync(0xffffffffu, mnew[h2], 1));
        mnew[h2] = fmaxf(mnew[h2], __shfl_xor_sync(0xffffffffu, mnew[h2], 2));
      }
      float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
      for (int h2 = 0; h2 < 2; h2++) {
        corr[h2] = (mnew[h2] == -INFINITY) ? 1.f : exp2f(mrow[h2] - mnew[h2]);
        mrow[h2] = mnew[h2];
      }
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const int h2 = e >> 1;
          const float p = (sacc[j][e] == -INFINITY) ? 0.f : exp2f(sacc[j][e] - mrow[h2]);
          sacc[j][e] = p;
          rs[h2] += p;
        }
#pragma unroll
      for (int h2 = 0; h2 < 2; h2++) lrow[h2] = lrow[h2] * corr[h2] + rs[h2];
#pragma unroll
      for (int j = 0; j < 16; j++) {
        oacc[j][0] *= corr[0];
        oacc[j][1] *= corr[0];
        oacc[j][2] *= corr[1];
        oacc[j][3] *= corr[1];
      }
      // O += P V  (P from registers as the A operand, V via ldmatrix.trans).
      // P is split into bf16 hi + lo parts (two MMAs) so the probabilities keep
      // ~16 mantissa bits: rounding P to one bf16 would perturb the bf16-stored
      // attention output by a fraction of an ulp and flip its rounding often
      // (precision contract R18: fp32 softmax and accumulation).
#pragma unroll
      for (int kk = 0; kk < 2; kk++) {
        uint32_t ph[4], pl[4];
#pragma unroll
        for (int f = 0; f < 4; f++) {
          const int jt = 2 * kk + (f >> 1), e0 = (f & 1) * 2;
          const float x0 = sacc[jt][e0], x1 = sacc[jt][e0 + 1];
          const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
          ph[f] = *reinterpret_cast<const uint32_t*>(&h);
          pl[f] = pack_bf16(x0 - __bfloat162float(h.x), x1 - __bfloat162float(h.y));
        }
#pragma unroll
        for (int j = 0; j < 16; j++) {
          uint32_t b0, b1;
          const bf16* vp = sV + (size_t)(kb + kk * 16 + (lane & 15)) * ATT_LD + j * 8;
          ldsm_x2_t(b0, b1, vp);
          mma_bf16_16816(oacc[j], ph[0], ph[1], ph[2], ph[3], b0, b1);
          mma_bf16_16816(oacc[j], pl[0], pl[1], pl[2], pl[3], b0, b1);
        }
      }
    }
    // row sums across the quad
#pragma unroll
    for (int h2 = 0; h2 < 2; h2++) {
      lrow[h2] += __shfl_xor_sync(0xffffffffu, lrow[h2], 1);
      lrow[h2] += __shfl_xor_sync(0xffffffffu, lrow[h2], 2);
    }
    // write the partial of (chunk, key split): slot = chunk * KS + ks
    const int part = chunk * KS + ks;
    for (int h2 = 0; h2 < 2; h2++) {
      const int r = mt * 16 + g_row + 8 * h2;
      float* wo = a.ws_o + (((size_t)part * a.Hkv + kvh) * QR + r) * ATT_HD;
#pragma unroll
      for (int j = 0; j < 16; j++) {
        *reinterpret_cast<float2*>(wo + j * 8 + t4 * 2) =
            make_float2(oacc[j][2 * h2], oacc[j][2 * h2 + 1]);
      }
      if (t4 == 0) {
        float* wm = a.ws_ml + (((size_t)part * a.Hkv + kvh) * QR + r) * 2;
        wm[0] = mrow[h2];
        wm[1] = lrow[h2];
      }
    }
  }
}

// merge the split partials: o = sum_c O_c 2^(m_c - M) / sum_c l_c 2^(m_c - M)
// grid (npad, H), block 128 (one thread per head-dim element)
__global__ void attn_combine_kernel(AttnArgs a, bf16* out, int ks, int n_parts_fixed = 0) {
  const int m = blockIdx.x, h = blockIdx.y;
  pdl_trigger();   // the next kernel streams its weights meanwhile
  if (m >= a.rows->n_rows) return;
  const int n_parts = n_parts_fixed > 0 ? n_parts_fixed : (a.rows->n_keys + ATT_KC - 1) / ATT_KC * ks;
  const int G = a.H / a.Hkv;
  const int kvh = h / G, g = h % G;
  const int QR = G * a.npad;
  const int r = g * a.npad + m;
  const int j = threadIdx.x;
  pdl_wait();      // the split partials come from the attention kernel
  // loads of 8 splits in flight together; accumulation in split order (deterministic)
  constexpr int B = 8;
  float M = -INFINITY;
  for (int c0 = 0; c0 < n_parts; c0 += B) {
    float mm[B];
#pragma unroll
    for (int i = 0; i < B; i++)
      mm[i] = (c0 + i < n_parts) ? a.ws_ml[(((size_t)(c0 + i) * a.Hkv + kvh) * QR + r) * 2] : -INFINITY;
#pragma unroll
    for (int i = 0; i < B; i++) M = fmaxf(M, mm[i]);
  }
  float L = 0.f, acc = 0.f;
  for (int c0 = 0; c0 < n_parts; c0 += B) {
    float mm[B], ll[B], oo[B];
#pragma unroll
    for (int i = 0; i < B; i++) {
      mm[i] = -INFINITY;
      if (c0 + i < n_parts) {
        const size_t base = ((size_t)(c0 + i) * a.Hkv + kvh) * QR + r;
        mm[i] = a.ws_ml[base * 2];
        ll[i] = a.ws_ml[base * 2 + 1];
        oo[i] = a.ws_o[base * ATT_HD + j];
      }
    }
#pragma unroll
    for (int i = 0; i < B; i++) {
      if (mm[i] == -INFINITY) continue;
      const float w = exp2f(mm[i] - M);
      L += ll[i] * w;
      acc += oo[i] * w;
    }
  }
  const float o = acc / L;
  const bf16 hi = __float2bfloat16_rn(o);
  out[((size_t)m * a.H + h) * ATT_HD + j] = hi;  // hi/lo activation pair
  out[((size_t)(a.npad + m) * a.H + h) * ATT_HD + j] = __float2bfloat16_rn(o - __bfloat162float(hi));
}

// The same merge with one warp per (row, head): lane i reads split i's (m, l)
// (one coalesced load for up to 32 splits), the maximum and the weighted sum
// come from warp shuffles, and every lane accumulates its float4 of the 128
// dims over the splits in split order with all O loads of a batch in flight.
// Deterministic (fixed shuffle tree, fixed split order).  CTA = 4 heads of one
// row; grid (npad, H / 4).
__global__ void __launch_bounds__(128) attn_combine_warp_kernel(AttnArgs a, bf16* out, int n_parts) {
  const int m = blockIdx.x, h = blockIdx.y * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  pdl_trigger();   // the next kernel streams its weights meanwhile
  if (m >= a.rows->n_rows || h >= a.H) return;
  const int G = a.H / a.Hkv;
  const int kvh = h / G, g = h % G;
  const int QR = G * a.npad;
  const int r = g * a.npad + m;
  pdl_wait();      // the split partials come from the attention kernel
  auto base_of = [&](int i) { return ((size_t)i * a.Hkv + kvh) * QR + r; };
  // maximum over the splits (log2 units; -inf marks an empty split)
  float M = -INFINITY;
  for (int i0 = 0; i0 < n_parts; i0 += 32) {
    const float mi = (i0 + lane < n_parts) ? a.ws_ml[base_of(i0 + lane) * 2] : -INFINITY;
    M = fmaxf(M, mi);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i0 = 0; i0 < n_parts; i0 += 32) {
    float w = 0.f;
    if (i0 + lane < n_parts) {
      const float mi = a.ws_ml[base_of(i0 + lane) * 2];
      if (mi != -INFINITY) {
        w = exp2f(mi - M);
        L += a.ws_ml[base_of(i0 + lane) * 2 + 1] * w;
      }
    }
    const int nb = min(32, n_parts - i0);
    constexpr int B = 8;
    for (int b0 = 0; b0 < nb; b0 += B) {
      float4 o[B];
      float wi[B];
#pragma unroll
      for (int k = 0; k < B; k++) {
        wi[k] = __shfl_sync(0xffffffffu, w, (b0 + k) & 31);
        o[k] = (b0 + k < nb && wi[k] != 0.f)
                   ? *reinterpret_cast<const float4*>(a.ws_o + base_of(i0 + b0 + k) * ATT_HD + lane * 4)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < B; k++) {
        if (b0 + k >= nb || wi[k] == 0.f) continue;
        acc.x += o[k].x * wi[k];
        acc.y += o[k].y * wi[k];
        acc.z += o[k].z * wi[k];
        acc.w += o[k].w * wi[k];
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  const float inv = 1.f / L;
  const float v[4] = {acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv};
  uint32_t hi2[2], lo2[2];
#pragma unroll
  for (int k = 0; k < 2; k++) {
    const __nv_bfloat162 hb = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
    hi2[k] = *reinterpret_cast<const uint32_t*>(&hb);
    lo2[k] = pack_bf16(v[2 * k] - __bfloat162float(hb.x), v[2 * k + 1] - __bfloat162float(hb.y));
  }
  *reinterpret_cast<uint2*>(out + ((size_t)m * a.H + h) * ATT_HD + lane * 4) = make_uint2(hi2[0], hi2[1]);
  *reinterpret_cast<uint2*>(out + ((size_t)(a.npad + m) * a.H + h) * ATT_HD + lane * 4) =
      make_uint2(lo2[0], lo2[1]);
}

// ---------------------------------------------------------------- MHA attention
// Segment rows x heads with G*npad <= 32 query rows per kv head (MHA configs).
// CTA = (key split, kv head); the nsplit (<= 8) splits of one kv head form a
// thread-block cluster.  Each CTA streams its keys through a ring of ATT_NBUF
// 64-key cp.async sub-chunk buffers (all issued up front when they fit); each
// m16 query tile is shared by KS = 4/MT warps taking KPW = 64/KS keys of every
// sub-chunk with a running (m, l, O).  The KS warp states merge in shared
// memory into one CTA partial; after a cluster barrier, CTA rank r merges rows
// r, r+nsplit, ... of all splits through distributed shared memory (split
// order: deterministic) and writes the bf16 hi/lo attention output pair.
constexpr int ATT_SUB = 64;   // keys per sub-chunk
#ifndef FS_ATT_NBUF
#define FS_ATT_NBUF 3
#endif
constexpr int ATT_NBUF = FS_ATT_NBUF;   // sub-chunk ring depth
constexpr int ATT_MAXQR = 32;
constexpr int ATT_SO_LD = ATT_HD + 8;   // padded row of the key-warp state scratch (float2
                                        // stores of a half-warp: 4 rows x 8 banks, conflict-free)

struct AttnMhaArgs {
  AttnArgs a;
  bf16* out;            // [2*npad][H*128] hi rows then lo rows
};

FS_DEV float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- MHA attention building blocks, shared by attn_mha_kernel and the fused
// QKV + attention kernel (k_qkv_attn.cuh).  tid / warp / lane are the indices
// within the 4 attention warps; bar_id names the barrier of those 128 threads.

// per-warp running state of one m16 query tile over its key slice
template <int KPW>
struct MhaWarp {
  float oacc[16][4];
  float mrow[2], lrow[2];
  uint32_t qf[ATT_HD / 16][4];
  int qm[2], ctx[2], sl[2];
  int mt, ks;
};

template <int KPW>
FS_DEV void mha_warp_init(MhaWarp<KPW>& w, const AttnArgs& a, int warp, int lane, int n_rows) {
  const int QR = (a.H / a.Hkv) * a.npad, MT = QR / 16;
  w.mt = warp % MT;
  w.ks = warp / MT;
  const int g_row = lane >> 2;
  for (int h2 = 0; h2 < 2; h2++) {
    const int r = w.mt * 16 + g_row + 8 * h2;
    w.qm[h2] = r % a.npad;
    w.ctx[h2] = (w.qm[h2] < n_rows) ? a.rows->ctx_lim[w.qm[h2]] : 0;
    w.sl[h2] = (w.qm[h2] < n_rows) ? a.rows->sidx[w.qm[h2]] : -1;
  }
#pragma unroll
  for (int j = 0; j < 16; j++) w.oacc[j][0] = w.oacc[j][1] = w.oacc[j][2] = w.oacc[j][3] = 0.f;
  w.mrow[0] = w.mrow[1] = -INFINITY;
  w.lrow[0] = w.lrow[1] = 0.f;
}
// after the key loop: a V outside fp16's range became inf in the fp16 P.V
// (inf, or NaN where P = 0) and stays non-finite in the fp32 accumulator, so
// one check of the accumulators flags it (fails the call loudly) without a
// per-fragment test in the inner loop
template <int KPW>
FS_DEV void mha_flag_range(const MhaWarp<KPW>& w, const AttnArgs& a) {
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 16; j++)
#pragma unroll
    for (int e = 0; e < 4; e++) bad |= !isfinite(w.oacc[j][e]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && a.num_err) *a.num_err = 1;
}

// Q fragments of the warp's m-tile into registers (once)
template <int KPW>
FS_DEV void mha_load_q(MhaWarp<KPW>& w, const bf16* sQ, int lane) {
#pragma unroll
  for (int kk = 0; kk < ATT_HD / 16; kk++)
    ldsm_x4(w.qf[kk][0], w.qf[kk][1], w.qf[kk][2], w.qf[kk][3],
            sQ + (size_t)(w.mt * 16 + (lane & 15)) * ATT_LD + kk * 16 + (lane >> 4) * 8);
}

// address of the 8-element (16-byte) chunk at (row, col) of a K or V tile:
// padded rows (cp.async staging) or the TMA SWIZZLE_128B layout of two
// [rows][64] boxes (hd 0-63, 64-127; box stride rows * 128 B), where the
// 16-byte chunk index is XORed with the row's index mod 8
template <bool SW, int ROWS>
FS_DEV const bf16* kv_chunk(const bf16* base, int row, int col) {
  if constexpr (SW) {
    const int off = (col >> 6) * ROWS * 128 + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4);
    return reinterpret_cast<const bf16*>(reinterpret_cast<const char*>(base) + off);
  } else {
    return base + (size_t)row * ATT_LD + col;
  }
}

// one 64-key sub-chunk (keys kbase..kbase+63 in sK / sV): the warp's KPW keys,
// tree mask unless every key is context of every live row, online softmax, P V
// with P as a bf16 hi/lo pair (R18).  SW: sK / sV in the TMA swizzled layout
template <int KPW, bool SW = false>
FS_DEV void mha_subchunk(MhaWarp<KPW>& w, const AttnArgs& a, const bf16* sK, const bf16* sV, int kbase,
                         int kend, int ctx_min, int l_glo, int n_rows, const uint32_t* sAnc, int lane) {
  constexpr int NT8 = KPW / 8;
  const int t4 = lane & 3;
  const int kb = w.ks * KPW;
  const int key0 = kbase + kb;
  float sacc[NT8][4];
#pragma unroll
  for (int j = 0; j < NT8; j++) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < ATT_HD / 16; kk++) {
#pragma unroll
    for (int j = 0; j < NT8; j++) {
      uint32_t b0, b1;
      ldsm_x2(b0, b1, kv_chunk<SW, ATT_SUB>(sK, kb + j * 8 + (lane & 7), kk * 16 + ((lane >> 3) & 1) * 8));
      mma_bf16_16816(sacc[j], w.qf[kk][0], w.qf[kk][1], w.qf[kk][2], w.qf[kk][3], b0, b1);
    }
  }
  float mnew[2] = {w.mrow[0], w.mrow[1]};
  if (key0 + KPW <= min(kend, ctx_min)) {
    // every key of this warp is context of every live row: no tree mask
    // (padding rows produce finite values that are never written)
#pragma unroll
    for (int j = 0; j < NT8; j++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const float v = sacc[j][e] * a.scale_log2;
        sacc[j][e] = v;
        mnew[e >> 1] = fmaxf(mnew[e >> 1], v);
      }
  } else {
#pragma unroll
    for (int j = 0; j < NT8; j++)
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const int h2 = e >> 1;
        const int key = key0 + j * 8 + t4 * 2 + (e & 1);
        bool vis = key < kend && w.qm[h2] < n_rows;
        if (vis && key >= w.ctx[h2]) {
          const int aa = key - l_glo;
          vis = w.sl[h2] >= 0 && aa >= 0 && aa < a.max_live &&
                ((sAnc[w.qm[h2] * a.ancw + (aa >> 5)] >> (aa & 31)) & 1u);
        }
        const float v = vis ? sacc[j][e] * a.scale_log2 : -INFINITY;
        sacc[j][e] = v;
        mnew[h2] = fmaxf(mnew[h2], v);
      }
  }
#pragma unroll
  for (int h2 = 0; h2 < 2; h2++) {
    mnew[h2] = fmaxf(mnew[h2], __shfl_xor_sync(0xffffffffu, mnew[h2], 1));
    mnew[h2] = fmaxf(mnew[h2], __shfl_xor_sync(0xffffffffu, mnew[h2], 2));
  }
  float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
  for (int h2 = 0; h2 < 2; h2++) {
    corr[h2] = (mnew[h2] == -INFINITY) ? 1.f : ex2_approx(w.mrow[h2] - mnew[h2]);
    w.mrow[h2] = mnew[h2];
  }
#pragma unroll
  for (int j = 0; j < NT8; j++)
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const int h2 = e >> 1;
      const float p = (sacc[j][e] == -INFINITY) ? 0.f : ex2_approx(sacc[j][e] - w.mrow[h2]);
      sacc[j][e] = p;
      rs[h2] += p;
    }
#pragma unroll
  for (int h2 = 0; h2 < 2; h2++) w.lrow[h2] = w.lrow[h2] * corr[h2] + rs[h2];
#pragma unroll
  for (int j = 0; j < 16; j++) {
    w.oacc[j][0] *= corr[0];
    w.oacc[j][1] *= corr[0];
    w.oacc[j][2] *= corr[1];
    w.oacc[j][3] *= corr[1];
  }
#if FS_MHA_P16
  // O += P V in fp16: P rounded to fp16 (R18 allows rounding P for P.V; 2^-12
  // relative, finer than bf16) and the V fragments converted bf16 -> fp16 in
  // registers (exact in fp16's normal range): one MMA per fragment instead of
  // the hi/lo pair's two
#pragma unroll
  for (int kk = 0; kk < KPW / 16; kk++) {
    uint32_t pf[4];
#pragma unroll
    for (int f = 0; f < 4; f++) {
      const int jt = 2 * kk + (f >> 1), e0 = (f & 1) * 2;
      const __half2 h = __floats2half2_rn(sacc[jt][e0], sacc[jt][e0 + 1]);
      pf[f] = *reinterpret_cast<const uint32_t*>(&h);
    }
#pragma unroll
    for (int j = 0; j < 16; j++) {
      uint32_t b0, b1;
      ldsm_x2_t(b0, b1, kv_chunk<SW, ATT_SUB>(sV, kb + kk * 16 + (lane & 15), j * 8));
      mma_f16_16816(w.oacc[j], pf[0], pf[1], pf[2], pf[3], bf16x2_to_f16x2(b0), bf16x2_to_f16x2(b1));
    }
  }
#else
  // O += P V with P as a bf16 hi + lo pair (R18: fp32 softmax/accumulation)
#pragma unroll
  for (int kk = 0; kk < KPW / 16; kk++) {
    uint32_t ph[4], pl[4];
#pragma unroll
    for (int f = 0; f < 4; f++) {
      const int jt = 2 * kk + (f >> 1), e0 = (f & 1) * 2;
      const float x0 = sacc[jt][e0], x1 = sacc[jt][e0 + 1];
      const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
      ph[f] = *reinterpret_cast<const uint32_t*>(&h);
      pl[f] = pack_bf16(x0 - __bfloat162float(h.x), x1 - __bfloat162float(h.y));
    }
#pragma unroll
    for (int j = 0; j < 16; j++) {
      uint32_t b0, b1;
      ldsm_x2_t(b0, b1, kv_chunk<SW, ATT_SUB>(sV, kb + kk * 16 + (lane & 15), j * 8));
      mma_bf16_16816(w.oacc[j], ph[0], ph[1], ph[2], ph[3], b0, b1);
      mma_bf16_16816(w.oacc[j], pl[0], pl[1], pl[2], pl[3], b0, b1);
    }
  }
#endif
}

// merge the KS key-warps of each m-tile into the CTA partial sPart [QR][HD] +
// sPml [QR][2] (scratch: `so` [4][16][SO_LD] + [4][16][2], which may alias the
// K/V ring: every warp is past its last sub-chunk at the first barrier)
template <int KPW>
FS_DEV void mha_ks_merge(MhaWarp<KPW>& w, const AttnArgs& a, float* so, float* sPart, float* sPml, int tid,
                         int warp, int lane, int bar_id) {
  constexpr int KS = ATT_SUB / KPW;
  const int QR = (a.H / a.Hkv) * a.npad, MT = QR / 16;
  const int g_row = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int h2 = 0; h2 < 2; h2++) {
    w.lrow[h2] += __shfl_xor_sync(0xffffffffu, w.lrow[h2], 1);
    w.lrow[h2] += __shfl_xor_sync(0xffffffffu, w.lrow[h2], 2);
  }
  float* sml = so + 4 * 16 * ATT_SO_LD;                       // [4][16][2]
  named_bar_sync(bar_id, 128);
  for (int h2 = 0; h2 < 2; h2++) {
    const int r16 = g_row + 8 * h2;
#pragma unroll
    for (int j = 0; j < 16; j++)
      *reinterpret_cast<float2*>(so + ((size_t)warp * 16 + r16) * ATT_SO_LD + j * 8 + t4 * 2) =
          make_float2(w.oacc[j][2 * h2], w.oacc[j][2 * h2 + 1]);
    if (t4 == 0) {
      sml[(warp * 16 + r16) * 2] = w.mrow[h2];
      sml[(warp * 16 + r16) * 2 + 1] = w.lrow[h2];
    }
  }
  named_bar_sync(bar_id, 128);
  // 8 threads per row, 16 head dims each as 4 float4 interleaved at a 32-float
  // stride (a quarter-warp's 8 float4 cover 32 consecutive banks: no conflicts);
  // KS <= 4 unrolled
  for (int r = tid >> 3; r < QR; r += 16) {
    const int m2 = r / 16, r16 = r % 16, d0 = (tid & 7) * 4;
    float mm[KS], M = -INFINITY;
#pragma unroll
    for (int k2 = 0; k2 < KS; k2++) {
      mm[k2] = sml[((m2 + MT * k2) * 16 + r16) * 2];
      M = fmaxf(M, mm[k2]);
    }
    float L = 0.f;
    float4 acc[4];
#pragma unroll
    for (int u = 0; u < 4; u++) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k2 = 0; k2 < KS; k2++) {
      const int ww = m2 + MT * k2;
      const float wt = (mm[k2] == -INFINITY) ? 0.f : exp2f(mm[k2] - M);
      L += sml[(ww * 16 + r16) * 2 + 1] * wt;
      const float* src = so + ((size_t)ww * 16 + r16) * ATT_SO_LD + d0;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const float4 o = *reinterpret_cast<const float4*>(src + 32 * u);
        acc[u].x += o.x * wt;
        acc[u].y += o.y * wt;
        acc[u].z += o.z * wt;
        acc[u].w += o.w * wt;
      }
    }
    float* dst = sPart + r * ATT_HD + d0;
#pragma unroll
    for (int u = 0; u < 4; u++) *reinterpret_cast<float4*>(dst + 32 * u) = acc[u];
    if ((tid & 7) == 0) {
      sPml[r * 2] = M;
      sPml[r * 2 + 1] = L;
    }
  }
}

// after a cluster barrier: CTA rank crank merges rows crank, crank + nsplit, ...
// of all splits through distributed shared memory (split order: deterministic)
// and writes the bf16 hi/lo attention output pair
FS_DEV void mha_cluster_merge(const AttnArgs& a, bf16* out, const float* sPart, const float* sPml, int crank,
                              int nsplit, int kvh, int n_rows, int tid) {
  const int G = a.H / a.Hkv, QR = G * a.npad;
  for (int rr = crank + nsplit * (tid >> 5); rr < QR; rr += nsplit * 4) {
    const int m = rr % a.npad, g = rr / a.npad;
    if (m >= n_rows) continue;
    const int q4 = (tid & 31) * 4;
    float mm[8], ll[8], M = -INFINITY;
    float4 oo[8];
#pragma unroll
    for (int c = 0; c < 8; c++) {   // all ranks' loads in flight together
      mm[c] = -INFINITY;
      ll[c] = 0.f;
      oo[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < nsplit) {
        const uint32_t pm = dsmem_addr(sPml + rr * 2, (uint32_t)c);
        mm[c] = ld_dsmem_f32(pm);
        ll[c] = ld_dsmem_f32(pm + 4);
        oo[c] = ld_dsmem_f32x4(dsmem_addr(sPart + rr * ATT_HD + q4, (uint32_t)c));
      }
      M = fmaxf(M, mm[c]);
    }
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c = 0; c < 8; c++) {
      if (c < nsplit && mm[c] != -INFINITY) {
        const float wt = exp2f(mm[c] - M);
        L += ll[c] * wt;
        acc.x += oo[c].x * wt;
        acc.y += oo[c].y * wt;
        acc.z += oo[c].z * wt;
        acc.w += oo[c].w * wt;
      }
    }
    const float v[4] = {acc.x / L, acc.y / L, acc.z / L, acc.w / L};
    const size_t base = ((size_t)m * a.H + kvh * G + g) * ATT_HD + q4;
    const size_t lob = ((size_t)(a.npad + m) * a.H + kvh * G + g) * ATT_HD + q4;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const bf16 hi = __float2bfloat16_rn(v[u]);
      out[base + u] = hi;
      out[lob + u] = __float2bfloat16_rn(v[u] - __bfloat162float(hi));
    }
  }
}

template <int KPW>
__global__ void __launch_bounds__(128) attn_mha_kernel(AttnMhaArgs args) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const AttnArgs& a = args.a;
  extern __shared__ __align__(16) uint8_t att_smem[];
  const int split = blockIdx.x, kvh = blockIdx.y, nsplit = gridDim.x;
  const TickRows* rows = a.rows;
  const int G = a.H / a.Hkv;
  const int QR = G * a.npad;
  // smem: Q [QR][LD] | K/V ring [NBUF][K|V][SUB][LD] | ancestor rows [npad][ancw]
  // after the key loop the ring is reused: key-warp states [4][16][HD] + [4][16][2],
  // then the CTA partial [QR][HD] + [QR][2] read by the cluster peers
  bf16* sQ = reinterpret_cast<bf16*>(att_smem);
  bf16* sKV = sQ + (size_t)QR * ATT_LD;
  uint32_t* sAnc = reinterpret_cast<uint32_t*>(sKV + (size_t)ATT_NBUF * 2 * ATT_SUB * ATT_LD);
  int* sCtxMin = reinterpret_cast<int*>(sAnc + (size_t)a.npad * a.ancw);   // context floor of the live rows
  float* sPart = reinterpret_cast<float*>(sKV) + 4 * 16 * ATT_SO_LD + 4 * 16 * 2;
  float* sPml = sPart + ATT_MAXQR * ATT_HD;
  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  // keys of this split; rows/sizes are written before the tick's first kernel
  const int nk = rows->n_keys;
  // keys per split from the device-side sizes (graph-replayable launch)
  const int per = (nk + nsplit * ATT_SUB - 1) / (nsplit * ATT_SUB) * ATT_SUB;
  const int kbeg = min(nk, split * per);
  const int kend = min(nk, kbeg + per);
  const int nsc = kend > kbeg ? (kend - kbeg + ATT_SUB - 1) / ATT_SUB : 0;
  const bf16* kbase = a.kc + ((size_t)kvh * a.max_ctx) * ATT_HD;
  const bf16* vbase = a.vc + ((size_t)kvh * a.max_ctx) * ATT_HD;
  auto load_sub = [&](int sc) {
    bf16* dK = sKV + (size_t)(sc % ATT_NBUF) * 2 * ATT_SUB * ATT_LD;
    bf16* dV = dK + ATT_SUB * ATT_LD;
    const int k0 = kbeg + sc * ATT_SUB;
    for (int idx = tid; idx < ATT_SUB * (ATT_HD / 8); idx += 128) {
      const int r = idx / (ATT_HD / 8), c = idx % (ATT_HD / 8);
      const int slot = min(k0 + r, a.max_ctx - 1);
      cp_async16(dK + (size_t)r * ATT_LD + c * 8, kbase + (size_t)slot * ATT_HD + c * 8);
      cp_async16(dV + (size_t)r * ATT_LD + c * 8, vbase + (size_t)slot * ATT_HD + c * 8);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // context K/V below the first slot written this tick do not depend on the
  // previous kernel (PDL): stream them before the grid dependency resolves
  ATT_PROBE(0);
  const long long clk0 = clock64();
  const int first_written = rows->slot[0];
  const int npre = min(nsc, ATT_NBUF);
  int issued = 0;
  while (issued < npre && kbeg + (issued + 1) * ATT_SUB <= first_written) load_sub(issued++);
  const int n_early = issued;   // sub-chunk groups committed before the Q group
  // row descriptor and ancestor bitsets are written before the tick's first
  // kernel (tick setup / submit / prune): stage them before the dependency too
  const int n_rows = rows->n_rows;
  for (int idx = tid; idx < a.npad * a.ancw; idx += 128) {
    const int m = idx / a.ancw, w = idx % a.ancw;
    const int s = (m < n_rows) ? rows->sidx[m] : -1;
    sAnc[idx] = (s >= 0) ? a.anc[(size_t)s * a.ancw + w] : 0u;
  }
  if (warp == 0) {  // keys below every live row's context limit need no tree mask
    int cm = 0x7fffffff;
    for (int m = lane; m < n_rows; m += 32) cm = min(cm, rows->ctx_lim[m]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cm = min(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    if (lane == 0) *sCtxMin = cm;
  }
  pdl_wait();
  // Q (GQA-packed rows): one cp.async group
  for (int idx = tid; idx < QR * (ATT_HD / 8); idx += 128) {
    const int r = idx / (ATT_HD / 8), c = idx % (ATT_HD / 8);
    const int g = r / a.npad, m = r % a.npad;
    cp_async16(sQ + (size_t)r * ATT_LD + c * 8, a.q + ((size_t)m * a.H + kvh * G + g) * ATT_HD + c * 8);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  while (issued < npre) load_sub(issued++);
  pdl_trigger();
  ATT_PROBE(1);
  MhaWarp<KPW> w;
  mha_warp_init<KPW>(w, a, warp, lane, n_rows);
  const int l_glo = rows->l_glo;
  int ctx_min = 0;
  for (int sc = 0; sc < nsc; sc++) {
    // cp.async groups in commit order: early sub-chunks, Q, later sub-chunks.
    // Both sub-chunk sc and Q must have landed: allow only the groups younger
    // than the younger of the two to stay pending.
    const int need = (sc < n_early) ? n_early : sc + 1;   // group index
    const int allowed = issued - need;                     // groups committed = issued + 1
    if (allowed >= 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else if (allowed == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    ATT_PROBE(2 + min(sc, 7));
    const bf16* sK = sKV + (size_t)(sc % ATT_NBUF) * 2 * ATT_SUB * ATT_LD;
    const bf16* sV = sK + ATT_SUB * ATT_LD;
    if (sc == 0) {  // Q fragments of this m-tile stay in registers for every sub-chunk
      mha_load_q<KPW>(w, sQ, lane);
      ctx_min = *sCtxMin;
    }
    mha_subchunk<KPW>(w, a, sK, sV, kbeg + sc * ATT_SUB, kend, ctx_min, l_glo, n_rows, sAnc, lane);
    __syncthreads();                                    // ring slot sc free
    if (issued < nsc) load_sub(issued++);
  }
  ATT_PROBE(10);
  mha_flag_range<KPW>(w, a);
  // ---- merge the KS key-warps of each m-tile (shared memory)
  mha_ks_merge<KPW>(w, a, reinterpret_cast<float*>(sKV), sPart, sPml, tid, warp, lane, 0);
  // ---- cluster merge of the splits through distributed shared memory:
  // CTA rank r owns rows r, r+nsplit, ...; 32 threads (float4 each) per row
  ATT_PROBE(11);
  cluster.sync();
  ATT_PROBE(12);
  mha_cluster_merge(a, args.out, sPart, sPml, (int)cluster.block_rank(), nsplit, kvh, n_rows, tid);
  ATT_PROBE(13);
  // keep every CTA's shared memory alive until all DSMEM reads are done (they
  // were consumed before arriving): relaxed, the output stores need not drain
  cluster_sync_relaxed();
  ATT_PROBE(14);
  if (a.dbg && threadIdx.x == 0)   // diagnostics: SM cycles between probes 0 and 14
    a.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + 15] = (unsigned long long)(clock64() - clk0);
}

// ---------------------------------------------------------------- argmax
// Final argmax / top-2 over the per-tile partials of the head GEMM.
__global__ void argmax_final_kernel(const Top2* part, int n_tiles, int nt_cols,
                                    const TickRows* rows, RowResult* res) {
  const int m = blockIdx.x;
  if (m >= rows->n_rows) return;
  Top2 t;
  t.v1 = -INFINITY;
  t.i1 = 0x7fffffff;
  t.v2 = -INFINITY;
  for (int i = threadIdx.x; i < n_tiles; i += 32) t = top2_merge(t, part[(size_t)i * nt_cols + m]);
  t = top2_warp(t);
  if (threadIdx.x == 0) {
    res[m].am = t.i1;
    res[m].margin = t.v1 - t.v2;
  }
}

// ---------------------------------------------------------------- fp32 GEMM path
// Y[m][n] = sum_k W[n][k] X[m][k]   (CUDA cores, fp32, no TF32) — fp32 config only
__global__ void gemm_f32_kernel(const float* __restrict__ W, const float* __restrict__ X,
                                float* Y, int N, int K, const TickRows* rows) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int nr = rows->n_rows;
  for (int m = 0; m < nr; m++) {
    float acc = 0.f;
    for (int k = 0; k < K; k++) acc += W[(size_t)n * K + k] * X[(size_t)m * K + k];
    Y[(size_t)m * N + n] = acc;
  }
}

// bias + rotate-half RoPE + store q / K cache / V cache (fp32 config)
__global__ void epi_qkv_f32_kernel(const float* Y, const float* bias, const float2* rope,
                                   float* q_out, float* kc, float* vc, int H, int Hkv, int hd,
                                   int max_ctx, const TickRows* rows) {
  const int m = blockIdx.y;
  if (m >= rows->n_rows) return;
  const int half = hd / 2;
  const int nheads = H + 2 * Hkv;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nheads * half) return;
  const int hh = idx / half, i = idx % half;
  const int N = nheads * hd;
  float a = Y[(size_t)m * N + hh * hd + i];
  float b = Y[(size_t)m * N + hh * hd + i + half];
  if (bias) {
    a += bias[hh * hd + i];
    b += bias[hh * hd + i + half];
  }
  float oa = a, ob = b;
  if (hh < H + Hkv) {
    const float2 cs = rope[(size_t)rows->pos[m] * half + i];
    oa = a * cs.x - b * cs.y;
    ob = b * cs.x + a * cs.y;
  }
  if (hh < H) {
    q_out[((size_t)m * H + hh) * hd + i] = oa;
    q_out[((size_t)m * H + hh) * hd + i + half] = ob;
  } else {
    float* dst = (hh < H + Hkv) ? kc + ((size_t)(hh - H) * max_ctx + rows->slot[m]) * hd
                                : vc + ((size_t)(hh - H - Hkv) * max_ctx + rows->slot[m]) * hd;
    dst[i] = oa;
    dst[i + half] = ob;
  }
}

// silu(gate) * up with the 64-row interleaved gate/up layout (fp32 config)
__global__ void epi_glu_f32_kernel(const float* Y, float* act, int ffn, const TickRows* rows) {
  const int m = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= rows->n_rows || j >= ffn) return;
  const size_t base = (size_t)m * 2 * ffn + (size_t)(j / 64) * 128 + (j % 64);
  const float g = Y[base], u = Y[base + 64];
  act[(size_t)m * ffn + j] = g / (1.0f + expf(-g)) * u;
}

__global__ void epi_resid_f32_kernel(const float* Y, float* x, int N, const TickRows* rows) {
  const int m = blockIdx.y;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= rows->n_rows || n >= N) return;
  x[(size_t)m * N + n] += Y[(size_t)m * N + n];
}

// argmax/top-2 of fp32 logits rows; optional copy to the parity buffer
__global__ void argmax_rows_kernel(const float* Y, int V, const TickRows* rows, RowResult* res,
                                   float* logits_out, int logits_by_s) {
  const int m = blockIdx.x;
  if (m >= rows->n_rows) return;
  if (logits_out && logits_by_s) logits_out += (size_t)rows->s_begin * V;
  Top2 t;
  t.v1 = -INFINITY;
  t.i1 = 0x7fffffff;
  t.v2 = -INFINITY;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float y = Y[(size_t)m * V + v];
    if (logits_out) logits_out[(size_t)m * V + v] = y;
    Top2 u;
    u.v1 = y;
    u.i1 = v;
    u.v2 = -INFINITY;
    t = top2_merge(t, u);
  }
  t = top2_warp(t);
  __shared__ Top2 sm[32];
  if (lane_id() == 0) sm[warp_id()] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    Top2 r = sm[0];
    for (int w = 1; w < (int)blockDim.x / 32; w++) r = top2_merge(r, sm[w]);
    res[m].am = r.i1;
    res[m].margin = r.v1 - r.v2;
  }
}

}  // namespace fs
