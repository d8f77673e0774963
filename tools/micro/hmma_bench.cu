// Microbenchmark: mma.sync.m16n8k16 bf16 latency (dependent chain) and
// throughput (independent accumulators) per warp / per SM on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void mma(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int IND>
__global__ void k(float* out, long long* cyc, int iters) {
  float acc[IND][4];
  for (int i = 0; i < IND; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  uint32_t a = threadIdx.x * 0x10001u, b = 0x3f803f80u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < IND; i++) mma(acc[i], a, a + 1, a + 2, a + 3, b, b + 1);
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < IND; i++) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int IND>
void run(int warps, int blocks) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, blocks * warps * 32 * 4);
  cudaMalloc(&cyc, blocks * 8);
  const int iters = 256;
  k<IND><<<blocks, warps * 32>>>(out, cyc, iters);
  k<IND><<<blocks, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * IND);
  printf("IND=%2d warps/CTA=%2d blocks=%3d: %.2f cycles per mma per warp (chain=%s)\n", IND, warps, blocks, per,
         IND == 1 ? "dependent" : "independent");
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>(1, 1);
  run<2>(1, 1);
  run<4>(1, 1);
  run<8>(1, 1);
  run<8>(4, 1);
  run<8>(8, 1);
  run<8>(16, 1);
  run<4>(4, 148);
  return 0;
}
