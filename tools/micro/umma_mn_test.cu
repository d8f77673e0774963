// Microtest: tcgen05.mma kind::f16 with A from TMEM (tcgen05.st) and B
// MN-major (N contiguous) from a TMA SWIZZLE_128B tile, D = A * B in TMEM.
// Shapes of the GQA attention P*V step: A = P [128 rows x 128 keys] bf16,
// B = V [128 keys x 128 d] (d contiguous), D = O [128 x 128] fp32.
// Tries candidate (LBO, SBO) encodings and reports the max error of each.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2507_02620_b200/csrc/common.cuh"
using namespace fs;

__device__ __forceinline__ void tmem_st64(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,"
      "%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]), "r"(r[36]),
      "r"(r[37]), "r"(r[38]), "r"(r[39]), "r"(r[40]), "r"(r[41]), "r"(r[42]), "r"(r[43]), "r"(r[44]), "r"(r[45]),
      "r"(r[46]), "r"(r[47]), "r"(r[48]), "r"(r[49]), "r"(r[50]), "r"(r[51]), "r"(r[52]), "r"(r[53]), "r"(r[54]),
      "r"(r[55]), "r"(r[56]), "r"(r[57]), "r"(r[58]), "r"(r[59]), "r"(r[60]), "r"(r[61]), "r"(r[62]), "r"(r[63])
      : "memory");
}

__device__ __forceinline__ void umma_tmemA(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(128) k_test(const __grid_constant__ CUtensorMap tmV, const __nv_bfloat16* P,
                                              float* O, uint32_t lbo, uint32_t sbo, int kstep_bytes) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sV = sm;                       // 2 boxes x 16 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768);
  uint64_t* mbar = bar + 1;
  uint32_t* holder = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(mbar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) tmem_alloc(holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, 32768);
    tma_load_2d(sV, &tmV, bar, 0, 0, l2_evict_last_policy());
    tma_load_2d(sV + 16384, &tmV, bar, 64, 0, l2_evict_last_policy());
  }
  // A = P row tid (128 bf16 = 64 x b32) into TMEM columns [0, 64)
  uint32_t r[64];
  for (int i = 0; i < 64; i++) {
    __nv_bfloat162 h;
    h.x = P[tid * 128 + 2 * i];
    h.y = P[tid * 128 + 2 * i + 1];
    r[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  tmem_st64(tmem + ((uint32_t)(warp * 32) << 16), r);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  mbar_wait(bar, 0);
  if (tid == 0) {
    // idesc: D f32, A/B bf16, B MN-major (bit 16), N = 128, M = 128
    const uint32_t idesc = umma_idesc_bf16(128, 128) | (1u << 16);
    const uint32_t base = smem_u32(sV);
    for (int ks = 0; ks < 8; ks++)
      umma_tmemA(tmem + 128, tmem + ks * 8, sdesc(base + ks * kstep_bytes, lbo, sbo), idesc, ks > 0 ? 1u : 0u);
    umma_commit(mbar);
  }
  mbar_wait(mbar, 0);
  tc_fence_after();
  float v[16];
  for (int c = 0; c < 128; c += 16) {
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + 128 + c, v);
    for (int i = 0; i < 16; i++) O[tid * 128 + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int K = 128, N = 128, M = 128;
  std::vector<__nv_bfloat16> hV(K * N), hP(M * K);
  std::vector<float> fV(K * N), fP(M * K);
  srand(1);
  for (int i = 0; i < K * N; i++) { float x = (rand() % 2001 - 1000) / 1000.f; hV[i] = __float2bfloat16(x); fV[i] = __bfloat162float(hV[i]); }
  for (int i = 0; i < M * K; i++) { float x = (rand() % 2001 - 1000) / 1000.f; hP[i] = __float2bfloat16(x); fP[i] = __bfloat162float(hP[i]); }
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; m++)
    for (int k = 0; k < K; k++)
      for (int n = 0; n < N; n++) ref[m * N + n] += (double)fP[m * K + k] * fV[k * N + n];
  __nv_bfloat16 *dV, *dP;
  float* dO;
  cudaMalloc(&dV, K * N * 2);
  cudaMalloc(&dP, M * K * 2);
  cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dV, hV.data(), K * N * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, hP.data(), M * K * 2, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};          // inner d, outer keys
  cuuint64_t strides[1] = {(cuuint64_t)N * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dV, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  struct Cand { uint32_t lbo, sbo; int kstep; } cands[] = {
      {16384, 1024, 2048}, {1024, 16384, 2048}, {16384, 2048, 2048}, {2048, 16384, 2048},
      {8192, 1024, 2048}, {1024, 8192, 2048}};
  std::vector<float> hO(M * N);
  for (auto& c : cands) {
    cudaMemset(dO, 0, M * N * 4);
    k_test<<<1, 128, 40 * 1024>>>(tm, dP, dO, c.lbo, c.sbo, c.kstep);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("LBO %u SBO %u: launch error %s\n", c.lbo, c.sbo, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(hO.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < M * N; i++) err = fmax(err, fabs(hO[i] - ref[i]));
    printf("LBO %5u SBO %5u kstep %d: max err %.3e  (O[0]=%f ref %f, O[130]=%f ref %f)\n", c.lbo, c.sbo, c.kstep, err,
           hO[0], ref[0], hO[130], ref[130]);
  }
  return 0;
}
