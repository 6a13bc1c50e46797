// Microbenchmark: does a predicated-off quarter-warp skip its shared-memory
// wavefront on a 16-B gather?  Each lane reads float4 rows of a table held as
// 8 interleaved copies (lane l reads copy l & 7, conflict-free, as k_gravity),
// with the load predicated by a lane mask.  Time per load vs mask pattern.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_quarter tools/lds_quarter.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const float4* __restrict__ g, float* out, unsigned mask, int iters, int rows) {
  extern __shared__ float4 tab[];
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) tab[i] = g[i / 8];
  __syncthreads();
  int lane = threadIdx.x & 31;
  bool on = (mask >> lane) & 1u;
  float4 acc = make_float4(0, 0, 0, 0);
  unsigned r = (threadIdx.x * 2654435761u) ^ blockIdx.x;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      r = r * 1664525u + 1013904223u;
      int row = (r >> 8) & (rows - 1);
      float4 c = make_float4(0, 0, 0, 0);
      if (on) c = tab[row * 8 + (lane & 7)];
      acc.x += c.x; acc.y += c.y; acc.z += c.z; acc.w += c.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

int main() {
  const int rows = 512, iters = 4096, blocks = 148 * 2, threads = 512;
  float4* g;
  float* out;
  cudaMalloc(&g, rows * sizeof(float4));
  cudaMemset(g, 0, rows * sizeof(float4));
  cudaMalloc(&out, blocks * threads * sizeof(float));
  size_t sm = rows * 8 * sizeof(float4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  struct P { const char* name; unsigned mask; } pats[] = {
      {"all 32 lanes", 0xffffffffu},
      {"lanes 0-15 (2 quarters)", 0x0000ffffu},
      {"lanes 0-7 (1 quarter)", 0x000000ffu},
      {"1 lane per quarter (4 quarters)", 0x01010101u},
      {"13 lanes spread over 4 quarters", 0x11224489u},
      {"13 lanes in quarters 0-1", 0x00001fffu},
      {"no lane", 0u},
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& p : pats) {
    k<<<blocks, threads, sm>>>(g, out, p.mask, iters, rows);
    cudaEventRecord(a);
    k<<<blocks, threads, sm>>>(g, out, p.mask, iters, rows);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double loads = (double)blocks * threads / 32 * iters * 8;
    printf("%-36s %8.3f ms  %.3f ns per warp-load per SM\n", p.name, ms, ms * 1e6 / loads * 148);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
