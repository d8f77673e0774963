// k_gen.cuh — on-device synthetic inputs: counter-based random-init weights,
// synthetic prefix KV, RoPE cos/sin table.  Input recipe of DESIGN.md
// (SURVEY §8(d) "Generators"); an independent implementation of the recipe
// the oracle also implements (no shared code).
#pragma once
#include "state.cuh"

namespace fs {

// value of element e of the tensor whose key is mix(seed ^ tid*C):
//   h = mix(key ^ e); u = h >> 40; i = 2u - (2^24 - 1); x = RN32(i * c)
//   gain tensors: 1 + x
FS_DEV float gen_value(uint64_t key, uint64_t e, float c, int gain) {
  const uint64_t h = mix64(key ^ e);
  const int32_t u = (int32_t)(h >> 40);
  const int32_t i = 2 * u - 16777215;
  float x = __fmul_rn((float)i, c);
  if (gain) x = __fadd_rn(1.0f, x);
  return x;
}

// row_mode: 0 identity (dst row = row_off + r); 1 / 2: gate / up rows of the
// 64-row interleaved gate|up matrix (dst row = (r/64)*128 + r%64 (+64 for up)).
// tiled: GEMM weight in the TMA-box-major layout [rows/128][cols/64][128][64]
// (one 16 KB contiguous block per 128 x 64 box; cols % 64 == 0)
template <typename T>
__global__ void gen_weight_kernel(T* dst, uint64_t key, float c, int gain, int64_t rows,
                                  int64_t cols, int row_mode, int64_t row_off, int tiled) {
  const int64_t n = rows * cols;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, k = idx - r * cols;
    int64_t dr = row_off + r;
    if (row_mode == 1) dr = (r / 64) * 128 + (r % 64);
    if (row_mode == 2) dr = (r / 64) * 128 + 64 + (r % 64);
    const int64_t o = tiled ? (((dr >> 7) * (cols >> 6) + (k >> 6)) << 13) + ((dr & 127) << 6) + (k & 63)
                            : dr * cols + k;
    dst[o] = from_f32<T>(gen_value(key, (uint64_t)idx, c, gain));
  }
}

// synthetic prefix K/V for slots [0, n): sigma 1,
// key = mix(kv_seed ^ (0x200000 + layer*2 + which) * C), e = (kvh*2^32 + slot)*hd + j
template <typename T>
__global__ void gen_kv_kernel(T* plane_base, uint64_t key, float c, int Hkv, int max_ctx,
                              int hd, int n) {
  const int64_t total = (int64_t)Hkv * n * hd;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx % hd;
    const int64_t s = (idx / hd) % n;
    const int64_t h = idx / ((int64_t)hd * n);
    const uint64_t e = (((uint64_t)h << 32) + (uint64_t)s) * (uint64_t)hd + (uint64_t)j;
    plane_base[((size_t)h * max_ctx + s) * hd + j] = from_f32<T>(gen_value(key, e, c, 0));
  }
}

// RoPE table (cos, sin) per (position, i < hd/2): angle in fp64, rounded to
// fp32 (precision contract R18)
__global__ void rope_table_kernel(float2* tab, int max_ctx, int half, double theta, int hd) {
  const int64_t n = (int64_t)max_ctx * half;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx / half, i = idx % half;
    const double ang = (double)p * pow(theta, -2.0 * (double)i / (double)hd);
    tab[idx] = make_float2((float)cos(ang), (float)sin(ang));
  }
}

}  // namespace fs
