// tc_probe.cu — validates the tcgen05 encodings used by libnqb on a real B200:
// TMEM alloc/st/ld, the K-major SWIZZLE_NONE smem descriptor, the kind::i8 and
// kind::f16 instruction descriptors, A-from-TMEM (TS) and A-from-smem (SS)
// MMAs and commit->mbarrier.  Prints one PASS/FAIL line per probe; exit code
// is the number of failures.  Built by tests/test_gpu_tc_probe.py.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../paper_2602_06694_b200/csrc/tc_common.cuh"

using namespace nqb::tc;

constexpr int M = 128;

// B (N x K bytes, K-major) -> smem canonical layout:
//   [kstep(32B)][khalf(16B)][ngroup(8 rows)][row][16B]
__device__ void stage_kmajor(uint8_t* s, const uint8_t* g, int rows, int kbytes) {
  const int ksteps = kbytes / 32, groups = rows / 8;
  for (int e = threadIdx.x; e < rows * kbytes; e += blockDim.x) {
    const int row = e / kbytes, kb = e % kbytes;
    const int ks = kb / 32, kh = (kb / 16) % 2, byte = kb % 16;
    const int off = ((ks * 2 + kh) * groups + row / 8) * 128 + (row % 8) * 16 + byte;
    s[off] = g[e];
  }
}

template <int N, int KBYTES, bool TS, bool F16>
__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* sa = smem;                 // M x KBYTES
  uint8_t* sb = smem + M * KBYTES;    // N x KBYTES
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    tmem_alloc(&tmem_base, 128);
    tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  stage_kmajor(sb, B, N, KBYTES);
  if (!TS) stage_kmajor(sa, A, M, KBYTES);
  fence_proxy_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base;
  const uint32_t a_tmem = tbase + 32;  // A columns [32, 32 + KBYTES/4)
  const uint32_t d_tmem = tbase;       // D columns [0, N)
  if (TS) {
    // thread (warp w, lane t) owns TMEM lane 32w + t = row of A
    const int row = warp * 32 + lane;
    for (int c = 0; c < KBYTES / 4; c += 8) {
      uint32_t v[8];
      for (int q = 0; q < 8; ++q) v[q] = *(const uint32_t*)(A + row * KBYTES + (c + q) * 4);
      tmem_st_x8(a_tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    }
    wait_st();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (threadIdx.x == 0) {
    const uint32_t idesc = F16 ? idesc_f16(M, N) : idesc_i8(M, N, true, true);
    for (int ks = 0; ks < KBYTES / 32; ++ks) {
      const uint64_t bd = smem_desc_kmajor(smem_u32(sb) + ks * 2 * (N / 8) * 128,
                                           (N / 8) * 128, 128);
      if (TS) {
        mma_i8_ts(d_tmem, a_tmem + ks * 8, bd, idesc, ks > 0);
      } else {
        const uint64_t ad = smem_desc_kmajor(smem_u32(sa) + ks * 2 * (M / 8) * 128,
                                             (M / 8) * 128, 128);
        if (F16) mma_f16_ss(d_tmem, ad, bd, idesc, ks > 0);
        else mma_i8_ss(d_tmem, ad, bd, idesc, ks > 0);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  uint32_t v[16];
  for (int c = 0; c < N; c += 16) {
    tmem_ld_x16(d_tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    wait_ld();
    const int row = warp * 32 + lane;
    for (int q = 0; q < 16 && c + q < N; ++q) D[row * N + c + q] = (int32_t)v[q];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 128);
}

static uint32_t lcg = 12345;
static uint32_t rnd() { return lcg = lcg * 1664525u + 1013904223u; }

template <int N, int KBYTES, bool TS, bool F16>
int run(const char* name) {
  const int K = F16 ? KBYTES / 2 : KBYTES;
  uint8_t *hA = (uint8_t*)malloc(M * KBYTES), *hB = (uint8_t*)malloc(N * KBYTES);
  for (int i = 0; i < M * KBYTES; ++i) hA[i] = (uint8_t)(rnd() >> 24);
  for (int i = 0; i < N * KBYTES; ++i) hB[i] = (uint8_t)(rnd() >> 24);
  if (F16) {  // small exact integers as fp16
    for (int i = 0; i < M * K; ++i) ((__half*)hA)[i] = __float2half((float)((int)(rnd() >> 28) - 8));
    for (int i = 0; i < N * K; ++i) ((__half*)hB)[i] = __float2half((float)((int)(rnd() >> 28) - 8));
  }
  uint8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, M * KBYTES);
  cudaMalloc(&dB, N * KBYTES);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * KBYTES, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * KBYTES, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  const int smem = (M + N) * KBYTES + 1024;
  cudaFuncSetAttribute(probe<N, KBYTES, TS, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, KBYTES, TS, F16><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  int32_t* hD = (int32_t*)malloc(M * N * 4);
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M && e == cudaSuccess; ++i)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) {
        if (F16) ref += (double)__half2float(((__half*)hA)[i * K + k]) * __half2float(((__half*)hB)[n * K + k]);
        else ref += (double)(int8_t)hA[i * K + k] * (int8_t)hB[n * K + k];
      }
      float fv;
      memcpy(&fv, &hD[i * N + n], 4);
      const double got = F16 ? (double)fv : (double)hD[i * N + n];
      if (got != ref) {
        if (bad < 5) printf("  %s mismatch D[%d][%d] got %g want %g\n", name, i, n, got, ref);
        ++bad;
      }
    }
  printf("%s %s (cuda=%s, mismatches=%d)\n", (e == cudaSuccess && bad == 0) ? "PASS" : "FAIL", name,
         cudaGetErrorString(e), bad);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return (e == cudaSuccess && bad == 0) ? 0 : 1;
}

int main() {
  int fails = 0;
  fails += run<16, 32, false, false>("i8_SS_M128_N16_K32");
  fails += run<16, 128, false, false>("i8_SS_M128_N16_K128");
  fails += run<16, 32, true, false>("i8_TS_M128_N16_K32");
  fails += run<16, 128, true, false>("i8_TS_M128_N16_K128");
  fails += run<32, 256, true, false>("i8_TS_M128_N32_K256");
  fails += run<16, 64, false, true>("f16_SS_M128_N16_K32");
  fails += run<64, 128, false, true>("f16_SS_M128_N64_K64");
  printf("failures=%d\n", fails);
  return fails;
}
