// k_attn_mha.cuh — tree-masked MHA attention with TMA-staged K/V (SURVEY §8(a)
// a6; PAPER.md:248 tree attention mask over the prefix KV plus the in-flight
// drafts; decode attention is I/O-bound).
//
// CTA = (key split, kv head), 4 consumer warps + 1 producer warp.  The
// producer streams 64-key sub-chunks of this head's K and V planes with
// cp.async.bulk.tensor (SWIZZLE_128B boxes of 64 keys x 64 dims, four per
// sub-chunk) into an NST-deep mbarrier ring; context sub-chunks below the
// first slot this tick writes are issued before griddepcontrol.wait (they do
// not depend on the QKV GEMM).  The consumers run the mma.sync QK^T / online
// softmax / P V of mha_subchunk on the swizzled tiles (ldmatrix addresses XOR
// the 16-byte chunk with the row), merge their key slices in shared memory and
// write the split's unnormalised partial (O, m, l) to the workspace;
// attn_combine_kernel (programmatic launch: resident while the splits run)
// merges the splits in split order.  The split count is sized to the SM count
// (key ranges of whole sub-chunks, balanced to +-1), not to cluster
// co-residency.  (A last-arriving-CTA merge through bulk copies into the free
// ring was measured slower: 7B 12.4 vs 10.0 us, 13B 18.4 vs 16.4 us per layer.)
#pragma once
#include "common.cuh"
#include "k_fwd.cuh"

namespace fs {

#ifndef FS_MHA_NST
#define FS_MHA_NST 3
#endif
constexpr int MHA_NST = FS_MHA_NST;                 // ring depth (sub-chunks)
constexpr int MHA_BOX = ATT_SUB * 128;             // one [64 keys][64 dims] bf16 box = 8 KB
constexpr int MHA_STAGE = 4 * MHA_BOX;             // K (2 boxes) | V (2 boxes) = 32 KB
constexpr int MHA_THREADS = 160;                   // 4 consumer warps + 1 TMA warp
constexpr int MHA_TMA_MIN_KEYS = 2048;             // shorter contexts: the cluster kernel
// dynamic smem: ring | Q [QR][LD] | anc [npad][ancw] | barriers  (QR = G * npad
// query rows: 16 / 32 for tree segments, 64 for prefill chunks)
__host__ __device__ constexpr size_t mha_tma_smem(int npad, int ancw, int qr) {
  return 1024 + (size_t)MHA_NST * MHA_STAGE + (size_t)qr * ATT_LD * 2 + (size_t)npad * ancw * 4 + 256;
}


template <int KPW>
__global__ void __launch_bounds__(MHA_THREADS) attn_mha_tma_kernel(const __grid_constant__ CUtensorMap tmK,
                                                                    const __grid_constant__ CUtensorMap tmV,
                                                                    AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t att_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(att_smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRing = smem;
  bf16* sQ = reinterpret_cast<bf16*>(sRing + (size_t)MHA_NST * MHA_STAGE);
  const int QRs = (a.H / a.Hkv) * a.npad;
  uint32_t* sAnc = reinterpret_cast<uint32_t*>(sQ + (size_t)QRs * ATT_LD);
  uint64_t* full = reinterpret_cast<uint64_t*>(sAnc + (size_t)a.npad * a.ancw);
  uint64_t* empty = full + MHA_NST;
  int* sCtxMin = reinterpret_cast<int*>(empty + MHA_NST);
  const int split = blockIdx.x, kvh = blockIdx.y, nsplit = gridDim.x;
  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  const TickRows* rows = a.rows;
  const int G = a.H / a.Hkv, QR = G * a.npad;
  // whole 64-key sub-chunks of this split (balanced to +-1 over the splits)
  const int nk = rows->n_keys;
  const int n_sub = (nk + ATT_SUB - 1) / ATT_SUB;
  const int sc0 = (int)((long long)split * n_sub / nsplit);
  const int sc1 = (int)((long long)(split + 1) * n_sub / nsplit);
  const int nsc = sc1 - sc0;
  const int kbeg = sc0 * ATT_SUB;
  const int kend = min(nk, sc1 * ATT_SUB);
  if (tid == 0) {
    for (int s = 0; s < MHA_NST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 4) {
    // ---------------- TMA producer (one elected lane)
    if (lane == 0) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      const uint64_t pol = l2_evict_first_policy();
      const int row0 = kvh * a.max_ctx;
      const int first_written = rows->slot[0];
      auto issue = [&](int sc) {
        const int s = sc % MHA_NST;
        uint8_t* st = sRing + (size_t)s * MHA_STAGE;
        const int y = row0 + (sc0 + sc) * ATT_SUB;
        mbar_arrive_expect_tx(&full[s], MHA_STAGE);
        tma_load_2d(st, &tmK, &full[s], 0, y, pol);
        tma_load_2d(st + MHA_BOX, &tmK, &full[s], 64, y, pol);
        tma_load_2d(st + 2 * MHA_BOX, &tmV, &full[s], 0, y, pol);
        tma_load_2d(st + 3 * MHA_BOX, &tmV, &full[s], 64, y, pol);
      };
      int issued = 0;
      // context sub-chunks do not depend on the previous kernel (PDL)
      while (issued < nsc && issued < MHA_NST && kbeg + (issued + 1) * ATT_SUB <= first_written) issue(issued++);
      pdl_wait();
      for (; issued < nsc; issued++) {
        if (issued >= MHA_NST) mbar_wait(&empty[issued % MHA_NST], ((issued / MHA_NST) - 1) & 1);
        issue(issued);
      }
    }
    return;
  }
  // ---------------- consumers: row descriptors before the dependency
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
  for (int idx = tid; idx < QR * (ATT_HD / 8); idx += 128) {
    const int r = idx / (ATT_HD / 8), c = idx % (ATT_HD / 8);
    const int g = r / a.npad, m = r % a.npad;
    *reinterpret_cast<uint4*>(sQ + (size_t)r * ATT_LD + c * 8) =
        *reinterpret_cast<const uint4*>(a.q + ((size_t)m * a.H + kvh * G + g) * ATT_HD + c * 8);
  }
  named_bar_sync(1, 128);
  pdl_trigger();
  MhaWarp<KPW> w;
  mha_warp_init<KPW>(w, a, warp, lane, n_rows);
  mha_load_q<KPW>(w, sQ, lane);
  const int ctx_min = *sCtxMin;
  const int l_glo = rows->l_glo;
  for (int sc = 0; sc < nsc; sc++) {
    const int s = sc % MHA_NST;
    mbar_wait(&full[s], (sc / MHA_NST) & 1);
    const bf16* sK = reinterpret_cast<const bf16*>(sRing + (size_t)s * MHA_STAGE);
    const bf16* sV = reinterpret_cast<const bf16*>(sRing + (size_t)s * MHA_STAGE + 2 * MHA_BOX);
    mha_subchunk<KPW, true>(w, a, sK, sV, kbeg + sc * ATT_SUB, kend, ctx_min, l_glo, n_rows, sAnc, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  mha_flag_range<KPW>(w, a);
  // ---- merge the key-warps of each m-tile (the ring is free: every stage consumed)
  float* so = reinterpret_cast<float*>(sRing);
  float* sPart = so + 4 * 16 * ATT_SO_LD + 4 * 16 * 2;
  float* sPml = sPart + QRs * ATT_HD;   // so | sml | sPart | sPml fit the free ring (<= 68 KB at QR 64)
  mha_ks_merge<KPW>(w, a, so, sPart, sPml, tid, warp, lane, 1);
  named_bar_sync(1, 128);
  // ---- this split's partial -> workspace [split][Hkv][QR][HD] (+ [..][2]), coalesced
  const size_t pbase = ((size_t)split * a.Hkv + kvh) * QR;
  for (int idx = tid; idx < QR * (ATT_HD / 4); idx += 128) {
    const int r = idx / (ATT_HD / 4), c = idx % (ATT_HD / 4);
    *reinterpret_cast<float4*>(a.ws_o + (pbase + r) * ATT_HD + c * 4) =
        *reinterpret_cast<const float4*>(sPart + r * ATT_HD + c * 4);
  }
  for (int r = tid; r < QR; r += 128) {
    a.ws_ml[(pbase + r) * 2] = nsc > 0 ? sPml[r * 2] : -INFINITY;
    a.ws_ml[(pbase + r) * 2 + 1] = nsc > 0 ? sPml[r * 2 + 1] : 0.f;
  }
}

}  // namespace fs
