// fullrun_probe.cu — IMMA issue rate of the decode kernels' inner loop (full_run,
// decode_dev.cuh) with W warps per SM all busy on resident shared-memory slabs.
// Reports IMMA per clock per SM (the legacy-IMMA peak measured by mma_probe.cu
// is ~0.48).  Build from the repo root:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2602_06694_b200/csrc -o fullrun_probe tests/cuda/fullrun_probe.cu
#include <cstdio>

#include "decode_dev.cuh"

using namespace nqb::dec;

template <int NT>
__global__ void k_probe(int slabs, int reps, long long* cyc, int* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  // A units: slabs x NT x 512 B; B fragments: slabs x 256 x kBytesPerK
  uint8_t* A = smem;
  uint8_t* B = smem + slabs * NT * 512;
  for (int i = threadIdx.x; i < slabs * NT * 512 / 4; i += blockDim.x)
    ((uint32_t*)A)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < slabs * 256 * kBytesPerK / 4; i += blockDim.x)
    ((uint32_t*)B)[i] = i * 40503u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t gq = lane >> 2, c = lane & 3;
  int acc[2][4][4] = {};
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    full_run<NT>(A, 512u * NT, B + (gq * 4 + c) * 16, slabs, lane, gq < (uint32_t)kLimbs, acc);
  __syncthreads();
  const long long t1 = clock64();
  int s = 0;
  for (int j = 0; j < 2; ++j)
    for (int q = 0; q < 4; ++q) s += acc[j][q][0] + acc[j][q][3];
  if (s == 0x12345) sink[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int* sink;
  long long* cyc;
  cudaMalloc(&sink, 4);
  cudaMalloc(&cyc, 8 * 148);
  for (int warps : {4, 8, 12, 16})
    for (int slabs : {1, 2, 4, 8, 16}) {
      const int reps = 256 / slabs;
      const size_t sm = slabs * 2 * 512 + slabs * 256 * kBytesPerK;
      cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_probe<2><<<148, 32 * warps, sm>>>(slabs, reps, cyc, sink);
      k_probe<2><<<148, 32 * warps, sm>>>(slabs, reps, cyc, sink);
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (long long v : h) mx = v > mx ? v : mx;
      const double imma = (double)warps * reps * slabs * 16;  // NT=2: 16 IMMA per slab
      printf("warps %2d run of %2d slabs: %6.3f IMMA/clk/SM  (%.1f cycles per IMMA per warp)\n", warps,
             slabs, imma / mx, (double)mx / (imma / warps));
    }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
