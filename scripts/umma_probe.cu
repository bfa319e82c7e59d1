// umma_probe.cu -- cycles per tcgen05.mma (kind::f16, M=128, K=16) for A in TMEM (TS) vs
// A in shared memory (SS), N = 16..256, measured by one elected thread issuing a
// dependent chain into one accumulator and waiting on a final commit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_17435_b200/csrc -o /tmp/umma_probe scripts/umma_probe.cu
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

__device__ volatile int g_stop;

__global__ void probe(int n_mma, uint32_t N, int ts, int nacc, unsigned long long* out, int st_warps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3F803F80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t0 = tbase;
  unsigned long long c0 = 0, c1 = 0, c2 = 0;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w >= 4 && w < 4 + st_warps) {   // background tcgen05.st traffic into columns 384..511
    const uint32_t ta = t0 + ((uint32_t)(32 * (w & 3)) << 16) + 384u + 8u * ((w >> 2) & 15);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    while (!stop) {
      for (int r = 0; r < 16; ++r) tmem_st8(ta, v, v);
      tmem_wait_st();
      v.x += 1;
    }
  }
  if (threadIdx.x < 32) {   // whole warp runs the loop; one elected lane issues
    const uint32_t idesc = umma_idesc_bf16(128, N);
    const uint32_t a_s = smem_u32(base), b_s = smem_u32(base + 32768);
    c0 = clock64();
    if (nacc == 8) {   // fully unrolled, operands precomputed (4 distinct descriptors)
      const uint64_t b0 = umma_desc_sw128(b_s), b1 = umma_desc_sw128(b_s + 32), b2 = umma_desc_sw128(b_s + 64),
                     b3 = umma_desc_sw128(b_s + 96);
      for (int i = 0; i < n_mma; i += 4) {
        if (elect_one()) {
          umma_bf16_ts(t0, t0 + 256, b0, idesc, 1);
          umma_bf16_ts(t0, t0 + 264, b1, idesc, 1);
          umma_bf16_ts(t0, t0 + 272, b2, idesc, 1);
          umma_bf16_ts(t0, t0 + 280, b3, idesc, 1);
        }
        __syncwarp();
      }
    } else
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t d = t0 + (uint32_t)(i & (nacc - 1)) * N;
      const uint64_t bd = umma_desc_sw128(b_s + 32 * (i & 3));
      const uint32_t acc = i >= nacc;
      if (ts) {
        const uint32_t at = t0 + 256 + 8 * (i & 3);
        if (elect_one()) umma_bf16_ts(d, at, bd, idesc, acc);
      } else {
        const uint64_t ad = umma_desc_sw128(a_s + 32 * (i & 3));
        if (elect_one()) umma_bf16_ss(d, ad, bd, idesc, acc);
      }
      __syncwarp();
    }
    c1 = clock64();
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    c2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = c1 - c0;
      out[1] = c2 - c0;
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
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int stw : {0, 24})
  for (int ts = 0; ts < 2; ++ts)
    for (uint32_t N : {16u, 32u, 64u, 256u})
      for (int nacc : {1})
      for (int n : {512}) {
        printf("st_warps=%d ", stw);
        probe<<<1, 128 + 32 * (stw + 4), 70 * 1024>>>(n, N, ts, nacc, d, stw);
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("nacc=%d ", nacc);
        printf("%s N=%3u n_mma=%4d  issue %7llu cyc  (%.1f/mma)  issue+complete %7llu cyc  (%.1f/mma)\n",
               ts ? "TS" : "SS", N, n, h[0], (double)h[0] / n, h[1], (double)h[1] / n);
      }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
