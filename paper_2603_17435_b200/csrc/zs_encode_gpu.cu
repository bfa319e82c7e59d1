// zs_encode_gpu.cu -- GPU-side TCA-TBE encoder: the same bytes as the host
// zs_encode (Alg. 1, canonical order S:277), computed on the device.
//
//   zs_hist_kernel     exponent histogram of the logical elements (Alg. 1 line 2): per-CTA
//                      shared-memory bins, one global atomic per bin and CTA.
//   (host)             max-coverage window of 7 exponents (line 3, ties -> smallest start),
//                      the same function the host encoder uses.
//   zs_count_kernel    per BlockTile, the number of in-window elements (padding counts as
//                      in-window: pad_word = (0, e_base + 1, 0)) -> segment sizes.
//   (host)             exclusive prefix of the 16-B padded segment sizes -> offsets.
//   zs_pack_kernel     one warp per BlockTile: lane l packs FragTiles 2l, 2l+1 (canonical
//                      order): codeword bit-planes, then an exclusive prefix of the in-window
//                      counts over the warp gives each FragTile's H / L start; the lane writes
//                      its H bytes (s<<7 | m) and fallback words, and the warp zero-fills the
//                      16-B segment padding.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "zs_kernels.h"

namespace zs {

__global__ void zs_hist_kernel(const uint16_t* __restrict__ w, int64_t rows, int64_t cols, int64_t ld,
                               unsigned long long* __restrict__ hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint16_t* row = w + r * ld;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) atomicAdd(&h[(row[c] >> 7) & 0xFF], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

// one warp per BlockTile: lane handles columns 2*lane, 2*lane+1 of the 64 rows
__global__ void zs_count_kernel(const uint16_t* __restrict__ w, int64_t rows, int64_t cols, int64_t ld,
                                int64_t nbc, int64_t nbt, int lo, int hi, uint32_t* __restrict__ hcnt) {
  const int64_t bt = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bt >= nbt) return;
  const int64_t r0 = (bt / nbc) * 64, c0 = (bt % nbc) * 64;
  uint32_t n = 0;
  for (int r = 0; r < 64; ++r) {
    const int64_t gr = r0 + r;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int64_t gc = c0 + 2 * lane + k;
      if (gr < rows && gc < cols) {
        const int e = (w[gr * ld + gc] >> 7) & 0xFF;
        n += (e >= lo && e <= hi);
      } else {
        n += 1;   // padding: pad_word is in-window (code 1)
      }
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) n += __shfl_xor_sync(0xFFFFFFFFu, n, d);
  if (lane == 0) hcnt[bt] = n;
}

__global__ void zs_pack_kernel(const uint16_t* __restrict__ w, int64_t rows, int64_t cols, int64_t ld, int64_t nbc,
                               int64_t nbt, int32_t base_exp, const uint64_t* __restrict__ offsets,
                               uint64_t* __restrict__ b1, uint64_t* __restrict__ b2, uint64_t* __restrict__ b3,
                               uint8_t* __restrict__ h, uint16_t* __restrict__ l) {
  const int64_t bt = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bt >= nbt) return;
  const int lo = base_exp + 1, hi = base_exp + 7;   // window [e_base + 1, e_base + 7]
  const uint16_t pad = (uint16_t)((base_exp + 1) << 7);
  const int64_t br = bt / nbc, bc = bt % nbc;
  uint64_t mk[2];
  uint32_t cnt[2];
  // element (pos = rr * 8 + cc) of the lane's FragTile k, the padding word outside the matrix
  auto elem = [&](int k, int pos) -> uint16_t {
    const int o = 2 * lane + k, tct = o >> 2, f = o & 3;
    const int64_t gr = br * 64 + (tct >> 2) * 16 + (f & 1) * 8 + (pos >> 3);
    const int64_t gc = bc * 64 + (tct & 3) * 16 + (f >> 1) * 8 + (pos & 7);
    return (gr < rows && gc < cols) ? w[gr * ld + gc] : pad;
  };
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int o = 2 * lane + k;                       // canonical FragTile index
    const int tct = o >> 2, f = o & 3;
    const int r0 = (tct >> 2) * 16 + (f & 1) * 8;     // FragTile column-major in its TCT
    const int c0 = (tct & 3) * 16 + (f >> 1) * 8;
    uint64_t q1 = 0, q2 = 0, q3 = 0;
    uint32_t n = 0;
    for (int rr = 0; rr < 8; ++rr) {
      const int64_t gr = br * 64 + r0 + rr;
      for (int cc = 0; cc < 8; ++cc) {
        const int64_t gc = bc * 64 + c0 + cc;
        const uint16_t x = (gr < rows && gc < cols) ? w[gr * ld + gc] : pad;
        const int e = (x >> 7) & 0xFF;
        if (e >= lo && e <= hi) {
          const uint64_t code = (uint64_t)(e - base_exp);
          const int pos = rr * 8 + cc;
          q1 |= (code & 1u) << pos;
          q2 |= ((code >> 1) & 1u) << pos;
          q3 |= ((code >> 2) & 1u) << pos;
          ++n;
        }
      }
    }
    mk[k] = q1 | q2 | q3;
    cnt[k] = n;
    b1[bt * 64 + o] = q1;
    b2[bt * 64 + o] = q2;
    b3[bt * 64 + o] = q3;
  }
  // exclusive prefix of the in-window counts over the BlockTile's FragTiles
  const uint32_t mine = cnt[0] + cnt[1];
  uint32_t incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += t;
  }
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  const uint64_t hoff = offsets[2 * bt], loff = offsets[2 * bt + 1];
  uint32_t hs = incl - mine;                       // H index of FragTile 2*lane
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int o = 2 * lane + k;
    uint32_t ls = (uint32_t)o * 64u - hs;          // L index of FragTile o
    const uint64_t m = mk[k];
    for (int pos = 0; pos < 64; ++pos) {
      const uint16_t x = elem(k, pos);
      if ((m >> pos) & 1u)
        h[hoff + hs++] = (uint8_t)(((x >> 8) & 0x80) | (x & 0x7F));
      else
        l[loff / 2 + ls++] = x;
    }
  }
  // zero padding up to the 16-byte segment boundaries
  const uint64_t hend = offsets[2 * bt + 2], lend = offsets[2 * bt + 3];
  for (uint64_t i = hoff + total + lane; i < hend; i += 32) h[i] = 0;
  for (uint64_t i = loff / 2 + (4096u - total) + lane; i < lend / 2; i += 32) l[i] = 0;
}

cudaError_t launch_encode_hist(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, unsigned long long* hist,
                               int sms, cudaStream_t s) {
  const int grid = (int)std::min<int64_t>(rows, (int64_t)sms * 8);
  zs_hist_kernel<<<grid, 256, 0, s>>>(w, rows, cols, ld, hist);
  return cudaGetLastError();
}

cudaError_t launch_encode_count(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int64_t nbc, int64_t nbt,
                                int lo, int hi, uint32_t* hcnt, cudaStream_t s) {
  const int64_t grid = (nbt + 7) / 8;
  zs_count_kernel<<<(unsigned)grid, 256, 0, s>>>(w, rows, cols, ld, nbc, nbt, lo, hi, hcnt);
  return cudaGetLastError();
}

cudaError_t launch_encode_pack(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int64_t nbc, int64_t nbt,
                               int32_t base_exp, const uint64_t* offsets, uint64_t* b1, uint64_t* b2, uint64_t* b3,
                               uint8_t* h, uint16_t* l, cudaStream_t s) {
  const int64_t grid = (nbt + 3) / 4;
  zs_pack_kernel<<<(unsigned)grid, 128, 0, s>>>(w, rows, cols, ld, nbc, nbt, base_exp, offsets, b1, b2, b3, h, l);
  return cudaGetLastError();
}

}  // namespace zs
