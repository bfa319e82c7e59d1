// op_probe.cu -- issue cost (cycles, one thread, back to back) of the producer-side
// operations: 1-D bulk copy, mbarrier arrive.expect_tx, try_wait on a completed phase,
// and the same bulk copies issued from 1, 2 or 4 warps of the CTA concurrently.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_17435_b200/csrc -o scripts/op_probe scripts/op_probe.cu
#include <cstdio>
#include <cstdint>
#include "zs_device.cuh"

using namespace zs;

__global__ void probe(const uint8_t* src, int mode, int n, int bytes, int warps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  if (w < warps && lane == 0) {
    uint8_t* dst = sm + (w % 4) * 16384;
    const uint8_t* s = src + (size_t)((blockIdx.x * 8 + w) % 1024) * (1 << 20);
    unsigned long long c0 = clock64();
    if (mode == 0) {        // bulk copies, one barrier with the total tx
      mbar_arrive_expect_tx(&bar[w], (uint32_t)(n * bytes));
      for (int i = 0; i < n; ++i) bulk_g2s(dst + (i % 2) * bytes, s + (size_t)i * bytes, bytes, &bar[w], pol);
    } else if (mode == 1) {  // expect_tx arrivals only (phase never completes: count 1 per call)
      for (int i = 0; i < n; ++i) {
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[w])), "r"(16u));
      }
    } else if (mode == 2) {  // test_wait on a completed phase (parity 1 of a fresh barrier)
      uint32_t acc = 0;
      for (int i = 0; i < n; ++i) acc += mbar_test_wait(&bar[w], 1u);
      if (acc == 12345) out[2] = acc;
    }
    unsigned long long c1 = clock64();
    if (mode == 0) mbar_wait(&bar[w], 0);
    unsigned long long c2 = clock64();
    out[w * 2] = c1 - c0;
    out[w * 2 + 1] = c2 - c0;
  }
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, (size_t)1 << 30);
  cudaMemset(src, 1, (size_t)1 << 30);
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  unsigned long long h[16];
  const int n = 64;
  for (int warps : {1, 2, 4, 8})
    for (int bytes : {512, 2048, 8192}) {
      probe<<<148, 256, 140 * 1024>>>(src, 0, n, bytes, warps, d);
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("bulk  warps=%d bytes=%5d  issue %.1f cyc/copy (warp0)  issue+land %.1f cyc/copy\n", warps, bytes,
             (double)h[0] / n, (double)h[1] / n);
    }
  probe<<<148, 256, 140 * 1024>>>(src, 1, n, 0, 1, d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("expect_tx  %.1f cyc/op\n", (double)h[0] / n);
  probe<<<148, 256, 140 * 1024>>>(src, 2, n, 0, 1, d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("test_wait(done)  %.1f cyc/op\n", (double)h[0] / n);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
