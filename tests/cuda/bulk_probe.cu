// bulk_probe.cu — per-SM streaming rate of 1-D TMA bulk copies (cp.async.bulk
// global->shared, mbarrier complete_tx) on the B200, as a function of chunk size
// and chunks in flight.  One CTA per SM; a producer thread keeps `depth` chunks
// of `chunk` bytes in flight through a ring; one consumer warp waits for each
// chunk and releases it (no compute).  Each CTA streams its own contiguous
// region of a buffer larger than L2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_probe bulk_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

constexpr int kMaxDepth = 32;

__global__ void __launch_bounds__(64, 1) k_stream(const uint8_t* buf, size_t per_cta, uint32_t chunk,
                                                  uint32_t depth, unsigned long long* cyc) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + kMaxDepth;
  uint8_t* ring = smem + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxDepth; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const uint8_t* src = buf + per_cta * blockIdx.x;
  const uint32_t n = (uint32_t)(per_cta / chunk);
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {  // producer
    for (uint32_t c = 0; c < n; ++c) {
      const uint32_t s = c % depth;
      if (c >= depth) mbar_wait(&empty[s], ((c / depth) - 1) & 1);
      expect_tx(&full[s], chunk);
      bulk(ring + (size_t)s * chunk, src + (size_t)c * chunk, chunk, &full[s]);
    }
  } else if (threadIdx.x == 32) {  // consumer
    for (uint32_t c = 0; c < n; ++c) {
      const uint32_t s = c % depth;
      mbar_wait(&full[s], (c / depth) & 1);
      mbar_arrive(&empty[s]);
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t per_cta = 8u << 20;  // 8 MB per CTA -> 1.18 GB total (> L2)
  uint8_t* buf;
  cudaMalloc(&buf, per_cta * sms);
  cudaMemset(buf, 1, per_cta * sms);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8 * sms);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const uint32_t chunks[] = {4096, 8192, 16384, 32768, 65536};
  const uint32_t depths[] = {2, 4, 8, 16, 32};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (uint32_t ch : chunks)
    for (uint32_t d : depths) {
      if ((size_t)ch * d + 1024 > 227 * 1024) continue;
      for (int grid : {sms, 1}) {
        k_stream<<<grid, 64, 227 * 1024>>>(buf, per_cta, ch, d, cyc);
        cudaEventRecord(e0);
        k_stream<<<grid, 64, 227 * 1024>>>(buf, per_cta, ch, d, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = (double)per_cta * grid / (ms * 1e-3) / 1e9;
        printf("chunk %6u depth %2u in-flight %7u B grid %3d: %8.1f GB/s total, %6.2f GB/s per SM\n", ch,
               d, ch * d, grid, gbs, gbs / grid);
      }
    }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
