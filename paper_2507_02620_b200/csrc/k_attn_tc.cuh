// k_attn_tc.cuh — GQA tree attention on 5th-gen tensor cores (tcgen05 + TMEM).
//
// For grouped-query configs (72B: G = 8 query heads per kv head) the G * npad
// query rows of one kv head share every K/V row, so attention sits at the
// ridge (256 flop/B at configs[4]) and belongs on the tensor
// cores.  CTA = (key split, kv head), one CTA per SM:
//   warp 0     TMA producer: K and V tiles of 128 keys, SWIZZLE_128B, 2 stages
//   warp 1     MMA issuer (one thread): S = Q K^T into TMEM; O += P V from TMEM
//   warps 2..  softmax: 4 warps per 128-row M-tile, one query row per thread
// TMEM per M-tile: 128 columns S (fp32; P aliases it as bf16 hi | lo halves)
// and 128 columns O.  One pass with an online softmax: P = 2^(s - M) against
// a running row maximum M that is raised lazily -- only when a tile's maximum
// exceeds it by more than 2^8, in which case the thread rescales its O row
// in TMEM (after the previous P V completed) and its running sum; otherwise
// P may reach 2^8, exact in fp32 and in the bf16 hi/lo pair (PLO; precision
// contract R18, as the MHA kernel) or bf16.  The split's unnormalised O and
// (M, l) go to a workspace that attn_combine_kernel merges in split order
// (deterministic).
// Tree visibility (§8(a) a6): context keys [0, ctx_lim[m]) plus
// ancestors-or-self of the row's node; key tiles below every live row's
// context limit skip the mask.
#pragma once
#include "k_fwd.cuh"

// softmax warps per M-tile: 8 (two threads per query row, one per 64-key half)
// or 4 (FS_TCA_SPLITROW=0: one thread per row)
#ifndef FS_TCA_SPLITROW
#define FS_TCA_SPLITROW 1
#endif
// 1: the split-row softmax computes its scaled scores, row sums and hi/lo
// residuals with Blackwell's packed FP32 instructions (FFMA2 / FADD2: two lanes
// per instruction, each lane an IEEE fma / add with round-to-nearest)
#ifndef FS_TCA_F32X2
#define FS_TCA_F32X2 1
#endif
// 1: QK^T(j+1) of an M-tile is issued right after P.V(j), relying on the
// in-order execution of one thread's tcgen05.mma for the P (read by P.V) that
// QK^T overwrites; 0: wait for P.V(j) to complete first
#ifndef FS_TCA_ORDERED
#define FS_TCA_ORDERED 0
#endif

namespace fs {

constexpr int TCA_KT = 128;              // keys per tile
constexpr int TCA_BOX = 128 * 128;       // one SW128 box: 128 rows x 64 bf16 = 16 KB

template <int MT2>
struct TcAttnCfg {
  // producer, MMA, softmax warps: 8 per M-tile (two threads per query row, one
  // per 64-key half; FS_TCA_SPLITROW=0: 4 per M-tile, one thread per row)
  static constexpr int SMW = FS_TCA_SPLITROW ? 8 : 4;
  static constexpr int ROLE_WARPS = 2;   // TMA producer, MMA issuer
  static constexpr int THREADS = 32 * ROLE_WARPS + 32 * SMW * MT2;
  static constexpr int Q_BYTES = MT2 * 2 * TCA_BOX;   // M-tiles x 2 head-dim boxes
  static constexpr int STAGE_BYTES = 4 * TCA_BOX;     // K (2 boxes) | V (2 boxes)
  static constexpr int NST = 2;
  static constexpr int SMEM = 1024 + Q_BYTES + NST * STAGE_BYTES + 256 + 2048 + 4 * 128 * MT2 +
                              (FS_TCA_SPLITROW ? 6 * 128 * 4 * MT2 + 2048 : 0);   // row-half exchange
  static constexpr int TMEM_COLS = 256 * MT2;         // 256 or 512
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

struct TcAttnArgs {
  AttnArgs a;
};

FS_DEV void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
FS_DEV void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// TMEM -> registers without the wait (the caller waits once for a batch)
FS_DEV void tmem_ld16_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
FS_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
FS_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]
FS_DEV void umma_bf16_tmemA(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// shared-memory descriptor of an MN-major SWIZZLE_128B operand made of 64-wide
// TMA boxes: LBO = distance between the boxes along MN, SBO = 8 rows along K
// (validated by tools/micro/umma_mn_test.cu)
FS_DEV uint64_t umma_sdesc_sw128_mn(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
FS_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// P formats of the P.V MMA: bf16, bf16 hi + lo pair (two MMAs), fp16 (A f16
// from TMEM with B = V bf16 in the same kind::f16 instruction)
constexpr int TCA_P_BF16 = 0, TCA_P_HILO = 1, TCA_P_F16 = 2;

// packed FP32 pairs (sm_100a): {lo lane, hi lane} in one 64-bit register pair
FS_DEV uint64_t f2_pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
FS_DEV void f2_unpack(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
FS_DEV uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
FS_DEV uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int MT2, int PF>
__global__ void __launch_bounds__(TcAttnCfg<MT2>::THREADS, 1)
    attn_gqa_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       TcAttnArgs args) {
  using C = TcAttnCfg<MT2>;
  constexpr bool PLO = PF == TCA_P_HILO;
  const AttnArgs& a = args.a;
  extern __shared__ uint8_t tsm_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + C::Q_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sKV + C::NST * C::STAGE_BYTES);
  uint64_t* empty = full + C::NST;
  uint64_t* s_full = empty + C::NST;     // [MT2]
  uint64_t* p_full = s_full + 2;         // [MT2]
  uint64_t* pv_done = p_full + 2;        // [MT2]: P V of the step complete (S/P columns free)
  uint64_t* o_full = pv_done + 2;        // [MT2]: the M-tile's last P V complete
  uint64_t* v_ready = o_full + 2;        // [NST] (f16 P): the stage's V converted to fp16
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(v_ready + 2);
  int* sCtxMin = reinterpret_cast<int*>(tmem_holder + 1);
  uint32_t* sAnc = reinterpret_cast<uint32_t*>(smem + C::Q_BYTES + C::NST * C::STAGE_BYTES + 256);

  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  const int split = blockIdx.x, kvh = blockIdx.y, nsplit = gridDim.x;
#ifdef FS_DIAG  // timeline probes (diagnostic builds only)
#define TCA_PROBE(k)                                                                       \
  do {                                                                                     \
    if (a.dbg && threadIdx.x == 64)                                                        \
      a.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (k)] = gtimer();          \
  } while (0)
// accumulated durations: slot k = this CTA's start + the sum (the host prints
// offsets from the earliest CTA start)
#define TCA_T() gtimer()
#define TCA_ACC(cond, k, v)                                                                 \
  do {                                                                                     \
    if (a.dbg && (cond)) a.dbg[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + (k)] = t_cta0 + (v); \
  } while (0)
  const unsigned long long t_cta0 = gtimer();
#else
#define TCA_PROBE(k) do {} while (0)
#define TCA_T() 0ull
#define TCA_ACC(cond, k, v) do {} while (0)
#endif
  TCA_PROBE(0);
  const TickRows* rows = a.rows;
  const int G = a.H / a.Hkv;
  const int QR = G * a.npad;             // == 128 * MT2 (host-checked)
  const int nk = rows->n_keys;
  const int per = (nk + nsplit * TCA_KT - 1) / (nsplit * TCA_KT) * TCA_KT;
  const int kbeg = min(nk, split * per);
  const int kend = min(nk, kbeg + per);
  const int T = (kend - kbeg + TCA_KT - 1) / TCA_KT;
  float* ws_o = a.ws_o + ((size_t)split * a.Hkv + kvh) * QR * ATT_HD;
  float* ws_ml = a.ws_ml + ((size_t)split * a.Hkv + kvh) * QR * 2;
  if (T == 0) {   // empty split: a neutral partial (the combine skips M = -inf)
    for (int r = tid; r < QR; r += C::THREADS) {
      ws_ml[r * 2] = -INFINITY;
      ws_ml[r * 2 + 1] = 0.f;
    }
    return;
  }
  if (tid == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < C::NST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int mi = 0; mi < MT2; mi++) {
      mbar_init(&s_full[mi], 1);
      mbar_init(&p_full[mi], 32 * C::SMW);
      mbar_init(&pv_done[mi], 1);
    }
    mbar_init(&o_full[0], 1);
    mbar_init(&o_full[1], 1);
    for (int st = 0; st < C::NST; st++) mbar_init(&v_ready[st], FS_TCA_SPLITROW ? 32 * C::SMW * MT2 : 62);
    fence_barrier_init();
  }
  const int n_rows = rows->n_rows;
  for (int idx = tid; idx < a.npad * a.ancw; idx += C::THREADS) {
    const int m = idx / a.ancw, w = idx % a.ancw;
    const int s = (m < n_rows) ? rows->sidx[m] : -1;
    sAnc[idx] = (s >= 0) ? a.anc[(size_t)s * a.ancw + w] : 0u;
  }
  if (warp == 1) {   // keys below every live row's context limit need no tree mask
    int cm = 0x7fffffff;
    for (int m = lane; m < n_rows; m += 32) cm = min(cm, rows->ctx_lim[m]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cm = min(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    if (lane == 0) *sCtxMin = cm;
  }
  __syncwarp();
  if (warp == 0) tmem_alloc(tmem_holder, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // context K/V tiles (below the first slot this tick writes) do not depend on
  // the QKV GEMM: the producer streams the first stages before the dependency
  int npre = 0;
  __shared__ int s_npre;
  if (tid == 0) {
    const int first_written = rows->slot[0];
    const uint64_t pol = l2_evict_first_policy();
    while (npre < min(T, C::NST) && kbeg + (npre + 1) * TCA_KT <= first_written) {
      const int y = kvh * a.max_ctx + kbeg + npre * TCA_KT;
      mbar_arrive_expect_tx(&full[npre], 4 * TCA_BOX);
      uint8_t* sK = sKV + npre * C::STAGE_BYTES;
      tma_load_2d(sK, &tmK, &full[npre], 0, y, pol);
      tma_load_2d(sK + TCA_BOX, &tmK, &full[npre], 64, y, pol);
      tma_load_2d(sK + 2 * TCA_BOX, &tmV, &full[npre], 0, y, pol);
      tma_load_2d(sK + 3 * TCA_BOX, &tmV, &full[npre], 64, y, pol);
      npre++;
    }
    s_npre = npre;
  }
  // dependents may launch only now: this CTA already holds its TMEM columns
  pdl_trigger();
  pdl_wait();   // Q and this tick's K/V rows come from the QKV GEMM
  // Q tile (GQA-packed rows r = g * npad + m) into the K-major SW128 layout
  for (int idx = tid; idx < QR * 16; idx += C::THREADS) {
    const int r = idx >> 4, c16 = idx & 15;
    const int g = r / a.npad, m = r % a.npad;
    const int mi = r >> 7, rr = r & 127, b = c16 >> 3, c = c16 & 7;
    uint8_t* dst = sQ + mi * 2 * TCA_BOX + b * TCA_BOX + rr * 128 + ((c ^ (rr & 7)) << 4);
    cp_async16(dst, a.q + ((size_t)m * a.H + kvh * G + g) * ATT_HD + c16 * 8);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  fence_proxy_async_smem();
  __syncthreads();
  TCA_PROBE(1);

  if constexpr (PF == TCA_P_F16 && !FS_TCA_SPLITROW) {
    if (warp <= 1 && lane > 0) {
      // ---------------- V bf16 -> fp16 in place (62 lanes of the producer and MMA
      // warps): element-wise, so the SW128 layout the MMA reads is unchanged;
      // exact for |v| in [2^-14, 65504] (fp16 normal range; smaller values keep
      // their fp16-subnormal part, an absolute error below 2^-25)
      const int cid = warp * 31 + (lane - 1);
      for (int j = 0; j < T; j++) {
        const int st = j % C::NST;
        mbar_wait(&full[st], (uint32_t)((j / C::NST) & 1));
        uint4* v = reinterpret_cast<uint4*>(sKV + st * C::STAGE_BYTES + 2 * TCA_BOX);
        for (int i = cid; i < 2 * TCA_BOX / 16; i += 62) {
          uint4 x = v[i];
          uint32_t* w = reinterpret_cast<uint32_t*>(&x);
#pragma unroll
          for (int k = 0; k < 4; k++) {
            const __half2 h = __floats2half2_rn(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xFFFF0000u));
            w[k] = *reinterpret_cast<const uint32_t*>(&h);
          }
          v[i] = x;
        }
        fence_proxy_async_smem();   // the MMA reads V through the async proxy
        mbar_arrive(&v_ready[st]);
      }
    }
  }
  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer: K + V tiles
      const uint64_t pol = l2_evict_first_policy();
      const int np0 = s_npre;
      for (int j = np0; j < T; j++) {
        const int st = j % C::NST;
        const int y = kvh * a.max_ctx + kbeg + j * TCA_KT;
        mbar_wait(&empty[st], (uint32_t)(((j / C::NST) & 1) ^ 1));
        mbar_arrive_expect_tx(&full[st], 4 * TCA_BOX);
        uint8_t* sK = sKV + st * C::STAGE_BYTES;
        tma_load_2d(sK, &tmK, &full[st], 0, y, pol);
        tma_load_2d(sK + TCA_BOX, &tmK, &full[st], 64, y, pol);
        tma_load_2d(sK + 2 * TCA_BOX, &tmV, &full[st], 0, y, pol);
        tma_load_2d(sK + 3 * TCA_BOX, &tmV, &full[st], 64, y, pol);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      // Ping-pong over the two M-tiles: after P V of (tile j, M-tile mi) comes
      // Q K^T of (j+1, mi), so one M-tile's softmax overlaps the other's MMAs.
      constexpr uint32_t idesc_qk = umma_idesc_bf16(128, 128);
      constexpr uint32_t idesc_pv = (umma_idesc_bf16(128, 128) | (1u << 16))     // B (V) MN-major
                                    & (PF == TCA_P_F16 ? ~((7u << 7) | (7u << 10)) : ~0u);   // A, B f16
      const uint32_t q0 = smem_u32(sQ);
      const uint32_t kv0 = smem_u32(sKV);
      auto stage_of = [&](int j) { return j % C::NST; };
      unsigned long long w_p = 0, w_full = 0, w_pv = 0;
      auto issue_qk = [&](int j, int mi) {
        unsigned long long t0 = TCA_T();
        if (mi == 0) mbar_wait(&full[stage_of(j)], (uint32_t)((j / C::NST) & 1));
        unsigned long long t1 = TCA_T();
        w_full += t1 - t0;
        // the S / P columns of M-tile mi are free once P V of tile j-1 read P
#if !FS_TCA_ORDERED
        if (j > 0) mbar_wait(&pv_done[mi], (uint32_t)((j - 1) & 1));
#endif
        w_pv += TCA_T() - t1;
        tc_fence_after();
        const uint32_t k0 = kv0 + (uint32_t)(stage_of(j) * C::STAGE_BYTES);
        const uint32_t tS = tmem + (uint32_t)(mi * 256);
#pragma unroll
        for (int kk = 0; kk < 8; kk++) {
          const uint32_t off = (uint32_t)((kk >> 2) * TCA_BOX + (kk & 3) * 32);
          umma_bf16(tS, umma_sdesc_sw128(q0 + mi * 2 * TCA_BOX + off), umma_sdesc_sw128(k0 + off), idesc_qk,
                    kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[mi]);
      };
      auto issue_pv = [&](int j, int mi) {
        unsigned long long t0 = TCA_T();
        mbar_wait(&p_full[mi], (uint32_t)(j & 1));   // P of this tile written (and O rescaled)
        w_p += TCA_T() - t0;
        if constexpr (PF == TCA_P_F16)
          if (mi == 0) mbar_wait(&v_ready[stage_of(j)], (uint32_t)((j / C::NST) & 1));
        tc_fence_after();
        const uint32_t v0 = kv0 + (uint32_t)(stage_of(j) * C::STAGE_BYTES) + 2 * TCA_BOX;
        const uint32_t tS = tmem + (uint32_t)(mi * 256), tO = tS + 128;
#pragma unroll
        for (int ks = 0; ks < 8; ks++) {
          const uint64_t bd = umma_sdesc_sw128_mn(v0 + ks * 2048, TCA_BOX, 1024);
          // keys 16ks.. live in the column half ks / 4: P_hi at +0, P_lo at +32
          const uint32_t pa = tS + (uint32_t)((ks >> 2) * 64 + (ks & 3) * 8);
          umma_bf16_tmemA(tO, pa, bd, idesc_pv, (j > 0 || ks > 0) ? 1u : 0u);
          if constexpr (PLO) umma_bf16_tmemA(tO, pa + 32, bd, idesc_pv, 1u);
        }
        umma_commit(&pv_done[mi]);
      };
      for (int mi = 0; mi < MT2; mi++) issue_qk(0, mi);
      for (int j = 0; j < T; j++) {
        for (int mi = 0; mi < MT2; mi++) {
          issue_pv(j, mi);
          if (j + 1 == T) umma_commit(&o_full[mi]);   // M-tile mi's O is final: its epilogue may start
          if (j + 1 < T) issue_qk(j + 1, mi);
        }
        umma_commit(&empty[stage_of(j)]);   // stage j's K / V reads are all issued
      }
      TCA_ACC(true, 3, w_p);
      TCA_ACC(true, 4, w_full);
      TCA_ACC(true, 5, w_pv);
    }
    __syncwarp();
  } else {
#if FS_TCA_SPLITROW
    // ---------------- softmax: two threads per query row, one per 64-key half
    // (warps 8*mi + 4*hf + q): each reads only its half of S and writes only its
    // half of P; the row maximum (and, at the end, the row sum) is exchanged
    // through shared memory at one named barrier per tile and M-tile.  The
    // running maximum M is in raw-score units.
    const int wi = warp - C::ROLE_WARPS, mi = wi >> 3, hf = (wi >> 2) & 1, q = warp & 3;
    const int rr = q * 32 + lane, r = mi * 128 + rr;
    const int m = r % a.npad;
    const bool live = m < n_rows;
    const int ctxr = live ? rows->ctx_lim[m] : 0;
    const int slr = live ? rows->sidx[m] : -1;
    const int l_glo = rows->l_glo;
    const int ctx_min = *sCtxMin;
    const float sc = a.scale_log2;
    // after the ancestor rows (npad x ancw words, <= 4 KB)
    float* xmax = reinterpret_cast<float*>(sAnc + a.npad * a.ancw) + (size_t)mi * 6 * 128;   // [2 parity][2 half][128]
    float* xsum = xmax + 4 * 128;                                                // [2 half][128]
    const uint32_t lq = ((uint32_t)(q * 32) << 16);
    const uint32_t tS = tmem + (uint32_t)(mi * 256) + lq + (uint32_t)(hf * 64), tO = tmem + (uint32_t)(mi * 256) + 128 + lq;
    float M = -INFINITY, L = 0.f;
    unsigned long long w_s = 0, b_s = 0, t_arr = 0;
    for (int j = 0; j < T; j++) {
      const unsigned long long tw0 = TCA_T();
      if constexpr (PF == TCA_P_F16) {
        // V(j) bf16 -> fp16 in place while S(j) is computed: this M-tile's
        // threads convert their half of the stage's V boxes (element-wise, the
        // SW128 layout the MMA reads is unchanged; exact for |v| in fp16's
        // normal range [2^-14, 65504], smaller values keep their fp16-subnormal
        // part, an absolute error below 2^-25)
        const int st = j % C::NST;
        mbar_wait(&full[st], (uint32_t)((j / C::NST) & 1));
        uint4* v = reinterpret_cast<uint4*>(sKV + st * C::STAGE_BYTES + 2 * TCA_BOX) + mi * (2 * TCA_BOX / 16 / MT2);
        const int ti = wi % 8 * 32 + lane;
        uint32_t ovf = 0;
#pragma unroll
        for (int i = ti; i < 2 * TCA_BOX / 16 / MT2; i += 32 * C::SMW) {
          uint4 x = v[i];
          ovf |= f16_range_check(x.x) | f16_range_check(x.y) | f16_range_check(x.z) | f16_range_check(x.w);
          x.x = bf16x2_to_f16x2(x.x);
          x.y = bf16x2_to_f16x2(x.y);
          x.z = bf16x2_to_f16x2(x.z);
          x.w = bf16x2_to_f16x2(x.w);
          v[i] = x;
        }
        fence_proxy_async_smem();   // the MMA reads V through the async proxy
        mbar_arrive(&v_ready[st]);
        if (ovf) *a.num_err = 1;   // fails the call loudly (FS_ERANGE), no silent inf
      }
      mbar_wait(&s_full[mi], j & 1);
      tc_fence_after();
      const unsigned long long tw1 = TCA_T();
      w_s += tw1 - tw0;
      if (j == 0) TCA_PROBE(2);
      if (j == T - 1) TCA_PROBE(6);
      const int key0 = kbeg + j * TCA_KT + hf * 64;
      const bool need_mask = !(kbeg + j * TCA_KT + TCA_KT <= min(kend, ctx_min));
      auto mask16 = [&](float* t, int kb) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
          const int key = kb + i;
          bool vis = live && key < kend;
          if (vis && key >= ctxr) {
            const int aa = key - l_glo;
            vis = slr >= 0 && aa >= 0 && aa < a.max_live &&
                  ((sAnc[m * a.ancw + (aa >> 5)] >> (aa & 31)) & 1u);
          }
          if (!vis) t[i] = -INFINITY;
        }
      };
      // pass A: the maximum of this half, exchanged with the other half
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 4; c += 2) {
        float t[32];
        tmem_ld16_nw(tS + c * 16, reinterpret_cast<uint32_t*>(t));
        tmem_ld16_nw(tS + c * 16 + 16, reinterpret_cast<uint32_t*>(t + 16));
        tmem_ld_wait();
        if (need_mask) {
          mask16(t, key0 + c * 16);
          mask16(t + 16, key0 + c * 16 + 16);
        }
#pragma unroll
        for (int i = 0; i < 32; i++) mx[i & 3] = fmaxf(mx[i & 3], t[i]);
      }
      const float mh = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      float* xm = xmax + (j & 1) * 256;
      xm[hf * 128 + rr] = mh;
      named_bar_sync(1 + mi, 32 * C::SMW);
      const float Mn = fmaxf(M, fmaxf(xm[rr], xm[128 + rr]));   // same value in both halves
      if (j == 0) {
        M = Mn;
      } else {
        const bool resc = Mn != -INFINITY && (M == -INFINITY || (Mn - M) * sc > a.resc_log2);
        if (__any_sync(0xffffffffu, resc)) {
          mbar_wait(&pv_done[mi], (uint32_t)((j - 1) & 1));   // O holds tiles < j
          tc_fence_after();
          const float f = resc ? ((M == -INFINITY) ? 0.f : ex2_approx((M - Mn) * sc)) : 1.f;
#pragma unroll 1
          for (int c = 0; c < 4; c++) {   // this thread's 64 of the row's 128 O columns
            uint32_t o[16];
            const uint32_t to = tO + (uint32_t)(hf * 64 + c * 16);
            tmem_ld16_nw(to, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; i++) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            tmem_st8(to, o);
            tmem_st8(to + 8, o + 8);
          }
          tmem_st_wait();
          if (resc) {
            L *= f;
            M = Mn;
          }
        }
      }
      // pass B: P of this half into its own S columns (bf16 hi at +0, lo at +32)
      const float nm = (M == -INFINITY) ? 0.f : -M * sc;
      float ls[4] = {0.f, 0.f, 0.f, 0.f};
      float sv[64];
#pragma unroll
      for (int c = 0; c < 4; c++) tmem_ld16_nw(tS + c * 16, reinterpret_cast<uint32_t*>(sv + c * 16));
      tmem_ld_wait();
      if (need_mask)
#pragma unroll
        for (int c = 0; c < 4; c++) mask16(sv + c * 16, key0 + c * 16);
#if FS_TCA_F32X2
      if constexpr (PF != TCA_P_F16) {
        // p = 2^(s*c - M*c) two scores per FFMA2, row sums in two packed
        // accumulators, P_lo = p - float(P_hi) two per FFMA2 (h * -1 + p: exact product)
        const uint64_t sc2 = f2_pack(sc, sc), nm2 = f2_pack(nm, nm), m12 = f2_pack(-1.f, -1.f);
        uint64_t acc2[2] = {f2_pack(0.f, 0.f), f2_pack(0.f, 0.f)};
#pragma unroll
        for (int c16 = 0; c16 < 4; c16++) {
          uint32_t pk[8], pl[8];
#pragma unroll
          for (int i = 0; i < 8; i++) {
            const int k0 = c16 * 16 + 2 * i;
            float t0, t1;
            f2_unpack(f2_fma(f2_pack(sv[k0], sv[k0 + 1]), sc2, nm2), t0, t1);
            const float x0 = ex2_approx(t0), x1 = ex2_approx(t1);
            const uint64_t x2 = f2_pack(x0, x1);
            acc2[i & 1] = f2_add(acc2[i & 1], x2);
            const __nv_bfloat162 hb = __floats2bfloat162_rn(x0, x1);
            const uint32_t u = *reinterpret_cast<const uint32_t*>(&hb);
            pk[i] = u;
            if constexpr (PLO) {
              float l0, l1;
              f2_unpack(f2_fma(f2_pack(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u)), m12, x2), l0, l1);
              pl[i] = pack_bf16(l0, l1);
            }
          }
          tmem_st8(tS + c16 * 8, pk);
          if constexpr (PLO) tmem_st8(tS + 32 + c16 * 8, pl);
        }
        f2_unpack(f2_add(acc2[0], acc2[1]), ls[0], ls[1]);
      } else
#endif
#pragma unroll
      for (int c16 = 0; c16 < 4; c16++) {
        uint32_t pk[8], pl[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const int k0 = c16 * 16 + 2 * i;
          const float x0 = ex2_approx(fmaf(sv[k0], sc, nm)), x1 = ex2_approx(fmaf(sv[k0 + 1], sc, nm));
          uint32_t u;
          if constexpr (PF == TCA_P_F16) {
            // the row sum takes the fp16-rounded weights the P.V MMA uses, so O / l
            // is an exact weighted mean of V (consistent normalisation)
            const __half2 hv = __floats2half2_rn(x0, x1);
            const float2 hr = __half22float2(hv);
            ls[i & 3] += hr.x + hr.y;
            u = *reinterpret_cast<const uint32_t*>(&hv);
          } else {
            ls[i & 3] += x0 + x1;
            const __nv_bfloat162 hb = __floats2bfloat162_rn(x0, x1);
            u = *reinterpret_cast<const uint32_t*>(&hb);
          }
          pk[i] = u;
          if constexpr (PLO)
            pl[i] = pack_bf16(x0 - __uint_as_float(u << 16), x1 - __uint_as_float(u & 0xFFFF0000u));
        }
        tmem_st8(tS + c16 * 8, pk);
        if constexpr (PLO) tmem_st8(tS + 32 + c16 * 8, pl);
      }
      L += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[mi]);
      t_arr = TCA_T();
      b_s += t_arr - tw1;
    }
    TCA_ACC(wi % 8 == 0 && lane == 0, 10 + 2 * mi, w_s);
    TCA_ACC(wi % 8 == 0 && lane == 0, 11 + 2 * mi, b_s);
    // ---------------- unnormalised O (this thread's 64 columns) and (M, l)
    TCA_PROBE(7);
    mbar_wait(&o_full[mi], 0);
    tc_fence_after();
    TCA_PROBE(8);
    // this M-tile's MMAs have completed; the other M-tile's last P.V may still
    // read V of the final stage.  M-tile 0 stages in [0, 8*32*68*4) = Q plus K
    // of stage 0 (last read by the final Q.K^T, issued before any final P.V);
    // M-tile 1 after it (its o_full follows the kernel's last MMA).
    constexpr int SLD = 64 + 4;
    static_assert(MT2 == 1 || 8 * 32 * SLD * 4 <= C::Q_BYTES + 2 * TCA_BOX,
                  "M-tile 0's output staging would overlap V of stage 0");
    float* stg = reinterpret_cast<float*>(smem) + (size_t)(wi) * 32 * SLD;
#pragma unroll
    for (int c = 0; c < 2; c++) {
      float o[32];
      const uint32_t to = tO + (uint32_t)(hf * 64 + c * 32);
      tmem_ld16_nw(to, reinterpret_cast<uint32_t*>(o));
      tmem_ld16_nw(to + 16, reinterpret_cast<uint32_t*>(o + 16));
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 8; i++)
        *reinterpret_cast<float4*>(stg + lane * SLD + c * 32 + 4 * i) =
            make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
    }
    xsum[hf * 128 + rr] = L;
    __syncwarp();
    // 16 lanes x float4 = one 256-byte half row; two rows per instruction
    float* dst = ws_o + (size_t)(r - lane) * ATT_HD + hf * 64;
#pragma unroll 4
    for (int row = 0; row < 32; row += 2) {
      const int rw = row + (lane >> 4), c4 = (lane & 15) * 4;
      *reinterpret_cast<float4*>(dst + (size_t)rw * ATT_HD + c4) =
          *reinterpret_cast<const float4*>(stg + rw * SLD + c4);
    }
    named_bar_sync(1 + mi, 32 * C::SMW);
    if (hf == 0) {
      ws_ml[r * 2] = (M == -INFINITY) ? -INFINITY : M * sc;   // log2 units, as the combine expects
      ws_ml[r * 2 + 1] = xsum[rr] + xsum[128 + rr];           // half 0 + half 1 (fixed order)
    }
    TCA_PROBE(9);
  }
#else
    // ---------------- softmax: one thread per query row (TMEM lane quarter
    // warp % 4); the running maximum M is in raw-score units
    const int wi = warp - C::ROLE_WARPS, mi = wi >> 2, q = warp & 3;
    const int rr = q * 32 + lane, r = mi * 128 + rr;
    const int m = r % a.npad;
    const bool live = m < n_rows;
    const int ctxr = live ? rows->ctx_lim[m] : 0;
    const int slr = live ? rows->sidx[m] : -1;
    const int l_glo = rows->l_glo;
    const int ctx_min = *sCtxMin;
    const float sc = a.scale_log2;
    const uint32_t tS = tmem + (uint32_t)(mi * 256) + ((uint32_t)(q * 32) << 16), tO = tS + 128;
    float M = -INFINITY, L = 0.f;
    for (int j = 0; j < T; j++) {
      mbar_wait(&s_full[mi], j & 1);
      tc_fence_after();
      if (j == 0) TCA_PROBE(2);
      if (j == T - 1) TCA_PROBE(6);
      const int key0 = kbeg + j * TCA_KT;
      // raw scores; invisible keys -> -inf (ex2 maps them to 0 below)
      const bool need_mask = !(key0 + TCA_KT <= min(kend, ctx_min));
      auto mask16 = [&](float* t, int kb) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
          const int key = kb + i;
          bool vis = live && key < kend;
          if (vis && key >= ctxr) {
            const int aa = key - l_glo;
            vis = slr >= 0 && aa >= 0 && aa < a.max_live &&
                  ((sAnc[m * a.ancw + (aa >> 5)] >> (aa & 31)) & 1u);
          }
          if (!vis) t[i] = -INFINITY;
        }
      };
      // pass A: the tile's row maximum (S re-read from TMEM in pass B, which
      // keeps the register footprint at one 64-key half)
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};   // independent chains
#pragma unroll
      for (int c = 0; c < 8; c += 2) {
        float t[32];
        tmem_ld16_nw(tS + c * 16, reinterpret_cast<uint32_t*>(t));
        tmem_ld16_nw(tS + c * 16 + 16, reinterpret_cast<uint32_t*>(t + 16));
        tmem_ld_wait();
        if (need_mask) {
          mask16(t, key0 + c * 16);
          mask16(t + 16, key0 + c * 16 + 16);
        }
#pragma unroll
        for (int i = 0; i < 32; i++) mx[i & 3] = fmaxf(mx[i & 3], t[i]);
      }
      const float Mn = fmaxf(M, fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])));
      if (j == 0) {
        M = Mn;
      } else {
        // lazy rescale: only when the tile maximum exceeds M by more than 2^resc_log2 (8)
        const bool resc = Mn != -INFINITY && (M == -INFINITY || (Mn - M) * sc > a.resc_log2);
        if (__any_sync(0xffffffffu, resc)) {   // tcgen05.ld / st are warp-collective
          mbar_wait(&pv_done[mi], (uint32_t)((j - 1) & 1));   // O holds tiles < j
          tc_fence_after();
          const float f = resc ? ((M == -INFINITY) ? 0.f : ex2_approx((M - Mn) * sc)) : 1.f;
#pragma unroll
          for (int c = 0; c < 4; c++) {
            uint32_t o[32];
            tmem_ld16_nw(tO + c * 32, o);
            tmem_ld16_nw(tO + c * 32 + 16, o + 16);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i++) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
            tmem_st32(tO + c * 32, o);
          }
          tmem_st_wait();
          if (resc) {
            L *= f;
            M = Mn;
          }
        }
      }
      // p = 2^(s * scale - M * scale): one FFMA + ex2 per element (the scale
      // is positive); a row with no visible key so far has M = -inf, p = 0
      const float nm = (M == -INFINITY) ? 0.f : -M * sc;
      float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int hh = 0; hh < 2; hh++) {
        // pass B, one 64-key half at a time: its P columns alias only its own S
        // columns, so the half is fully read before any of them is written
        float s[64];
#pragma unroll
        for (int c = 0; c < 4; c++) tmem_ld16_nw(tS + hh * 64 + c * 16, reinterpret_cast<uint32_t*>(s + c * 16));
        tmem_ld_wait();
        if (need_mask)
#pragma unroll
          for (int c = 0; c < 4; c++) mask16(s + c * 16, key0 + hh * 64 + c * 16);
#pragma unroll
        for (int c16 = 0; c16 < 4; c16++) {   // 16 keys: 8 packed hi columns (+ 8 lo columns)
          uint32_t pk[8], pl[8];
#pragma unroll
          for (int i = 0; i < 8; i++) {
            const int k0 = c16 * 16 + 2 * i;
            const float x0 = ex2_approx(fmaf(s[k0], sc, nm)), x1 = ex2_approx(fmaf(s[k0 + 1], sc, nm));
            ls[i & 3] += x0 + x1;
            // P_hi -> columns [0, 32) of the half; P_lo = p - float(P_hi) -> [32, 64)
            // (hi halves unpacked with integer ops, no second rounding)
            uint32_t u;
            if constexpr (PF == TCA_P_F16) {
              const __half2 hf = __floats2half2_rn(x0, x1);
              u = *reinterpret_cast<const uint32_t*>(&hf);
            } else {
              const __nv_bfloat162 hb = __floats2bfloat162_rn(x0, x1);
              u = *reinterpret_cast<const uint32_t*>(&hb);
            }
            pk[i] = u;
            if constexpr (PLO)
              pl[i] = pack_bf16(x0 - __uint_as_float(u << 16), x1 - __uint_as_float(u & 0xFFFF0000u));
          }
          tmem_st8(tS + hh * 64 + c16 * 8, pk);
          if constexpr (PLO) tmem_st8(tS + hh * 64 + 32 + c16 * 8, pl);
        }
      }
      L += (ls[0] + ls[1]) + (ls[2] + ls[3]);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&p_full[mi]);
    }
    // ---------------- unnormalised O row and (M, l) of this split
    TCA_PROBE(7);
    mbar_wait(&o_full[mi], 0);
    tc_fence_after();
    TCA_PROBE(8);
    // this M-tile's MMAs have completed (o_full[mi]); the other M-tile's last
    // P.V may still be reading V of the final stage.  M-tile 0's staging rows
    // cover [0, 4*32*132*4) = Q plus K of stage 0, whose last reader (the
    // final Q.K^T of both M-tiles) finished before any P.V was issued; they
    // never reach V (static_assert below).  Staging makes the workspace write
    // coalesced (a warp's rows r are consecutive); rows padded to 132 floats
    // keep the 16-byte stores at 4 wavefronts.
    constexpr int SLD = 128 + 4;
    static_assert(MT2 == 1 || 4 * 32 * SLD * 4 <= C::Q_BYTES + 2 * TCA_BOX,
                  "M-tile 0's output staging would overlap V of stage 0");
    float* stg = reinterpret_cast<float*>(smem) + (size_t)wi * 32 * SLD;
#pragma unroll
    for (int c = 0; c < 4; c++) {
      float o[32];
      tmem_ld16_nw(tO + c * 32, reinterpret_cast<uint32_t*>(o));
      tmem_ld16_nw(tO + c * 32 + 16, reinterpret_cast<uint32_t*>(o + 16));
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 8; i++)
        *reinterpret_cast<float4*>(stg + lane * SLD + c * 32 + 4 * i) =
            make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
    }
    __syncwarp();
    float* dst = ws_o + (size_t)(r - lane) * ATT_HD;
#pragma unroll 8
    for (int row = 0; row < 32; row++)   // one 512-byte row per instruction
      *reinterpret_cast<float4*>(dst + (size_t)row * ATT_HD + 4 * lane) =
          *reinterpret_cast<const float4*>(stg + row * SLD + 4 * lane);
    ws_ml[r * 2] = (M == -INFINITY) ? -INFINITY : M * sc;   // log2 units, as the combine expects
    ws_ml[r * 2 + 1] = L;
    TCA_PROBE(9);
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

}  // namespace fs
