// imma_latency.cu — cycles for n dependent / independent IMMA.16832 in a fresh
// kernel (first-use cost), and for LDS->IMMA chains.  One warp per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a, uint32_t b) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};\n"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a), "r"(b));
}

template <int N, bool DEP>
__global__ void k_lat(long long* out, int* sink) {
  int acc[8][4] = {};
  uint32_t a = threadIdx.x * 7 + 1, b = threadIdx.x ^ 5;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    if (DEP) imma(acc[0], a, b);
    else imma(acc[i & 7], a, b);
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][3];
  __syncwarp();
  asm volatile("" ::"r"(s));
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (s == 0x7fffffff) sink[0] = s;
}

template <int N, bool DEP>
void run(const char* name) {
  long long* d;
  int* sink;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&sink, 4);
  long long h[148];
  for (int rep = 0; rep < 2; ++rep) {
    k_lat<N, DEP><<<148, 32>>>(d, sink);
    cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    long long mn = h[0], mx = h[0], sm = 0;
    for (int i = 0; i < 148; ++i) { mn = h[i] < mn ? h[i] : mn; mx = h[i] > mx ? h[i] : mx; sm += h[i]; }
    printf("%-28s N=%3d rep%d: cycles min %lld avg %lld max %lld\n", name, N, rep, mn, sm / 148, mx);
  }
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<1, true>("dependent");
  run<2, true>("dependent");
  run<8, true>("dependent");
  run<64, true>("dependent");
  run<8, false>("8 independent chains");
  run<64, false>("8 independent chains");
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
