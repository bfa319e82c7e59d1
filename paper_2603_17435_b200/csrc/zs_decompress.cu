// zs_decompress.cu -- ZipServ-Decomp on sm_100a.
//
// Persistent CTAs walk BlockTiles (64x64).  Per BlockTile the compressed bytes (three
// 512-B plane slices, the H and L segments) arrive by 1-D TMA bulk copies into a
// double-buffered smem stage; warp 0 scans the 64 FragTile popcounts (the paper's
// __popc/__shfl_sync addressing); every thread then decodes two FragTile rows
// with the shared branch-free row decoder and writes 16 B of BF16 to global memory
// (8 consecutive threads = one 128-B row segment, fully coalesced).
#include "zs_device.cuh"
#include "zs_kernels.h"

namespace zs {

constexpr int kDecompThreads = 256;

__global__ void __launch_bounds__(kDecompThreads) decompress_kernel(DecompParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint4* lut = reinterpret_cast<uint4*>(smem);                        // 4 KB
  uint32_t* ftpref = reinterpret_cast<uint32_t*>(smem + 4096);        // 64 x u32
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4096 + 256);    // 2 mbarriers
  uint8_t* stage_base = smem + 4096 + 256 + 64;
  const uint32_t stage_bytes = p.stage_bytes;

  const int tid = threadIdx.x;
  lut[tid] = build_lut_entry((uint32_t)tid);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t nbt = p.n_blocktiles;
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t bt, int s) {
    uint8_t* st = stage_base + (size_t)s * stage_bytes;
    const uint64_t h0 = p.offsets[2 * bt], h1 = p.offsets[2 * bt + 2];
    const uint64_t l0 = p.offsets[2 * bt + 1], l1 = p.offsets[2 * bt + 3];
    const uint32_t hb = (uint32_t)(h1 - h0), lb = (uint32_t)(l1 - l0);
    mbar_arrive_expect_tx(&bars[s], 1536u + hb + lb);
    bulk_g2s(st, p.b1 + bt * 64, 512, &bars[s], pol);
    bulk_g2s(st + 512, p.b2 + bt * 64, 512, &bars[s], pol);
    bulk_g2s(st + 1024, p.b3 + bt * 64, 512, &bars[s], pol);
    if (hb) bulk_g2s(st + 1536, p.h + h0, hb, &bars[s], pol);
    if (lb) bulk_g2s(st + 1536 + p.hcap, reinterpret_cast<const uint8_t*>(p.l) + l0, lb, &bars[s], pol);
  };

  int64_t bt = blockIdx.x;
  if (tid == 0 && bt < nbt) issue(bt, 0);
  uint32_t it = 0;
  for (; bt < nbt; bt += gridDim.x, ++it) {
    const int s = it & 1;
    const int64_t nxt = bt + gridDim.x;
    if (tid == 0 && nxt < nbt) issue(nxt, s ^ 1);  // stage s^1 was released by the last barrier
    mbar_wait(&bars[s], (it >> 1) & 1);

    const uint8_t* st = stage_base + (size_t)s * stage_bytes;
    const uint64_t* P1 = reinterpret_cast<const uint64_t*>(st);
    const uint64_t* P2 = P1 + 64;
    const uint64_t* P3 = P1 + 128;
    const uint8_t* H = st + 1536;
    const uint16_t* L = reinterpret_cast<const uint16_t*>(st + 1536 + p.hcap);

    // FragTile prefix popcounts in canonical order (warp 0, two FragTiles per lane)
    if (tid < 32) {
      const uint32_t c0 = __popcll(P1[2 * tid] | P2[2 * tid] | P3[2 * tid]);
      const uint32_t c1 = __popcll(P1[2 * tid + 1] | P2[2 * tid + 1] | P3[2 * tid + 1]);
      uint32_t incl = c0 + c1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (tid >= d) incl += v;
      }
      const uint32_t excl = incl - c0 - c1;
      ftpref[2 * tid] = excl;
      ftpref[2 * tid + 1] = excl + c0;
    }
    __syncthreads();

    const int64_t br = bt / p.nbc, bc = bt % p.nbc;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int q = tid + kDecompThreads * i;
      const int lr = q >> 3, fc = q & 7;        // row in BlockTile, FragTile column
      const int fr = lr >> 3, r8 = lr & 7;
      const int o = ((fr >> 1) * 4 + (fc >> 1)) * 4 + (fc & 1) * 2 + (fr & 1);  // canonical FT index
      const uint64_t q1 = P1[o], q2 = P2[o], q3 = P3[o];
      const uint64_t M = q1 | q2 | q3;
      const uint32_t hs = ftpref[o] + (uint32_t)__popcll(M & ((1ull << (8 * r8)) - 1ull));
      const uint32_t ls = (uint32_t)(o * 8 + r8) * 8u - hs;
      const uint4 v = decode_row(q1, q2, q3, (uint32_t)r8, H, hs, L, ls, lut, p.eb7x2);
      const int64_t row = br * 64 + lr;
      const int64_t col = bc * 64 + fc * 8;
      if (row < p.rows) {
        uint16_t* dst = p.out + row * p.ld_out + col;
        if (p.vec_ok && col + 8 <= p.cols) {
          *reinterpret_cast<uint4*>(dst) = v;
        } else {
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (col + e < p.cols) dst[e] = (uint16_t)(w[e >> 1] >> (16 * (e & 1)));
        }
      }
    }
    __syncthreads();  // stage s and ftpref are free again
  }
}

cudaError_t launch_decompress(const DecompParams& p, int grid, size_t smem, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(decompress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  decompress_kernel<<<grid, kDecompThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

size_t decompress_smem_bytes(uint32_t stage_bytes) { return 4096 + 256 + 64 + 2 * (size_t)stage_bytes; }

int decompress_threads() { return kDecompThreads; }

}  // namespace zs
