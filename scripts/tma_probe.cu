// tma_probe.cu -- microbenchmark: HBM read bandwidth of 1-D bulk copies (cp.async.bulk)
// as a function of the copy size and the number of copies in flight per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe scripts/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint8_t* src, size_t total, uint32_t chunk, int slots, int per_copy_ops,
                      unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  uint8_t* buf = sm + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = total / chunk;
  const uint32_t sub = chunk / per_copy_ops;
  unsigned long long acc = 0;
  int it = 0;
  size_t c = blockIdx.x;
  size_t issued = 0;
  // prologue: fill all slots
  size_t cc = c;
  for (int s = 0; s < slots && cc < nchunks; ++s, cc += gridDim.x) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(chunk));
    for (int q = 0; q < per_copy_ops; ++q)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(buf + (size_t)s * chunk + q * sub)),
                   "l"(src + cc * chunk + q * sub), "r"(sub), "r"(su32(&bars[s]))
                   : "memory");
    ++issued;
  }
  for (; c < nchunks; c += gridDim.x, ++it) {
    const int s = it % slots;
    const uint32_t par = (it / slots) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok)
                   : "r"(su32(&bars[s])), "r"(par)
                   : "memory");
    acc += buf[(size_t)s * chunk];
    if (cc < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bars[s])), "r"(chunk));
      for (int q = 0; q < per_copy_ops; ++q)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(buf + (size_t)s * chunk + q * sub)),
                     "l"(src + cc * chunk + q * sub), "r"(sub), "r"(su32(&bars[s]))
                     : "memory");
      cc += gridDim.x;
    }
  }
  sink[blockIdx.x] = acc;
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  uint32_t chunks[] = {512, 2048, 8192, 16384, 32768};
  int opss[] = {1, 4, 16};
  for (uint32_t ch : chunks)
    for (int ops : opss) {
      if (ch / ops < 128) continue;
      int slots = (int)std::min<size_t>(16, (200 * 1024) / ch);
      size_t smem = 1024 + (size_t)slots * ch;
      for (int ctas_per_sm : {1, 2}) {
        if (smem * ctas_per_sm > 220 * 1024) continue;
        int grid = sms * ctas_per_sm;
        probe<<<grid, 32, smem>>>(src, total, ch, slots, ops, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) probe<<<grid, 32, smem>>>(src, total, ch, slots, ops, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("chunk %6u B  copies/chunk %2d (%6u B each)  slots %2d  ctas/SM %d  ->  %7.1f GB/s  (%.0f copies/us)\n",
               ch, ops, ch / ops, slots, ctas_per_sm, 5.0 * total / (ms * 1e-3) / 1e9,
               5.0 * total / ch * ops / (ms * 1e3));
      }
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
