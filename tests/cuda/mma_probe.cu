// mma_probe.cu — measures legacy mma.sync throughput on the B200 (IMMA u8.s8
// m16n8k32, HMMA f16 m16n8k16 and BMMA b1 m16n8k256 .and.popc), independent chains, all SMs busy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_imma(int iters, int* out) {
  int acc[CH][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 0x12345) out[0] = s;
}

template <int CH>
__global__ void k_hmma(int iters, float* out) {
  float acc[CH][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1234.5f) out[0] = s;
}

template <int CH>
__global__ void k_bmma(int iters, int* out) {
  int acc[CH][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 0x12345) out[0] = s;
}

template <typename K> struct ArgOf;
template <typename T> struct ArgOf<void (*)(int, T)> { using type = T; };

template <typename K>
void run(const char* name, K kern, int warps, int chains, int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* out;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  using Arg = typename ArgOf<K>::type;
  kern<<<sms, warps * 32>>>(iters, (Arg)out);
  cudaEventRecord(e0);
  kern<<<sms, warps * 32>>>(iters, (Arg)out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)sms * warps * chains * iters;
  const double per_sm_per_us = mmas / sms / (ms * 1e3);
  printf("%s warps/SM=%2d chains=%d: %.3f ms, %.1f warp-MMA/us/SM = %.3f per cycle at %.0f MHz max\n", name,
         warps, chains, ms, per_sm_per_us, per_sm_per_us / (clk / 1e3), clk / 1e3);
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {
    run("IMMA.16832.u8s8", (void (*)(int, int*))k_imma<8>, w, 8, 20000);
    run("HMMA.16816.f16 ", (void (*)(int, float*))k_hmma<8>, w, 8, 20000);
    run("BMMA.168256.and", (void (*)(int, int*))k_bmma<8>, w, 8, 20000);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
