// umma_probe2.cu -- tensor-pipe cost of tcgen05.mma.cta_group::1.kind::f16 (SS form) per
// instruction, as a function of M (64 / 128), N, the number of independent accumulators, and
// background traffic from other warps (none / STS.128 storm / tcgen05.st storm).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_17435_b200/csrc -o scripts/umma_probe2 scripts/umma_probe2.cu
#include <cstdio>
#include <cstdint>
#include "zs_device.cuh"

// probe-only helpers (not used by the library kernels)
namespace zs {
__device__ __forceinline__ void umma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint4 a, uint4 b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(a.x),
               "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
}  // namespace zs

using namespace zs;

__global__ void probe(int n_mma, uint32_t M, uint32_t N, int nacc, int bg, int bg_warps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3F803F80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    stop = 0;
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t0 = tbase;
  const int w = threadIdx.x >> 5;
  if (w >= 1 && w <= bg_warps) {
    if (bg == 1) {   // STS.128 storm into smem [64 KB, 96 KB)
      uint4* dst = reinterpret_cast<uint4*>(base + 65536);
      uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
      while (!stop) {
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[((threadIdx.x & 255) + r * 256) & 2047] = v;
        v.x += 1;
      }
    } else if (bg == 2) {   // tcgen05.st storm into TMEM columns 384..511
      const uint32_t ta = t0 + ((uint32_t)(32 * (w & 3)) << 16) + 384u + 8u * ((w >> 2) & 15);
      uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
      while (!stop) {
        for (int r = 0; r < 16; ++r) tmem_st8(ta, v, v);
        tmem_wait_st();
        v.x += 1;
      }
    }
  }
  if (w == 0) {
    const uint32_t idesc = umma_idesc_bf16(M, N);
    const uint32_t a_s = smem_u32(base), b_s = smem_u32(base + 16384);
    const uint64_t a0 = umma_desc_sw128(a_s), b0 = umma_desc_sw128(b_s);
    unsigned long long c0 = clock64();
    for (int i = 0; i < n_mma; i += 4) {
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t d = t0 + (uint32_t)((i + j) % nacc) * N;
          umma_bf16_ss(d, a0 + 2 * j, b0 + 2 * j, idesc, 1u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long c2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = c2 - c0;
      stop = 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(t0, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int n = 1024;
  for (int bg : {1, 2})
    for (uint32_t M : {64u, 128u})
      for (uint32_t N : {64u, 128u, 256u})
        for (int nacc : {1, 2}) {
          if (N * nacc > 384) continue;
          probe<<<1, 32 * 25, 99 * 1024>>>(n, M, N, nacc, bg, bg ? 24 : 0, d);
          unsigned long long h = 0;
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("bg=%d M=%3u N=%3u nacc=%d  %.1f cyc/mma  (%.0f weight-rows*K16 per 100 cyc if W=N side)\n", bg, M, N,
                 nacc, (double)h / n, 100.0 * N / ((double)h / n));
        }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
