// zs_decompress.cu -- ZipServ-Decomp on sm_100a.
//
// HBM-bound: reads 1.40 B and writes 2 B per weight element (8B GateUp: 165 MB in, 235 MB
// out).  Design: one persistent CTA per SM, every WARP is an independent decoder with its
// own double-buffered smem stage and mbarriers, so there is no CTA-wide barrier anywhere.
//
//   warp g (of G = grid x warps) decodes BlockTiles g, g + G, ...  Per BlockTile:
//   1. lane 0 issues the 1-D TMA bulk copies of the NEXT BlockTile (3 plane slices, the H
//      and L segments) into the other stage: one load in flight per warp while it decodes.
//   2. scan: lane l owns FragTiles 2l, 2l+1; popcounts of M = B1|B2|B3, a warp
//      prefix scan over the 64 FragTiles, and per-row byte prefixes -> the H start of every
//      FragTile row, stored as u16 in a bank-spread table [r8][o].
//   3. 16 passes of 32 rows: lane -> (row lr = 4 pass + lane/8, FragTile column lane%8),
//      the branch-free row decoder of zs_device.cuh, and one 16-B store per lane (8 lanes =
//      one 128-B row segment, fully coalesced); passes run in groups of 4 so the rank >= 2
//      patch is one warp-uniform branch per group.
#include "zs_device.cuh"
#include "zs_kernels.h"
#include "zs_lut.h"

namespace zs {

#ifndef ZS_DECOMP_WARPS
#define ZS_DECOMP_WARPS 16
#endif
constexpr int kDecompMaxWarps = ZS_DECOMP_WARPS;   // independent decoder warps per CTA (one CTA per SM)
#ifndef ZS_DECOMP_STAGES
#define ZS_DECOMP_STAGES 2
#endif
constexpr int kDecompStages = ZS_DECOMP_STAGES;   // smem stages per warp (BlockTiles in flight)
constexpr uint32_t kHsRow = 80;                  // u16 per r8 row of the H-start table
constexpr uint32_t kHsTabBytes = 8 * kHsRow * 2;  // 1280 B per warp

__global__ void __launch_bounds__(32 * kDecompMaxWarps, 1) decompress_kernel(DecompParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint4* lut = reinterpret_cast<uint4*>(smem);   // 4 KB selector table
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kBarBytes = 8 * kDecompStages * kDecompMaxWarps;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4096) + kDecompStages * warp;
  uint16_t* hst = reinterpret_cast<uint16_t*>(smem + 4096 + kBarBytes + warp * kHsTabBytes);
  uint8_t* stage0 = smem + 4096 + kBarBytes + kDecompMaxWarps * kHsTabBytes +
                    (size_t)warp * kDecompStages * p.stage_bytes;
  const uint32_t stage_bytes = p.stage_bytes;

  for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = __ldg(&c_lut[i]);
  if (lane == 0) {
    for (int i = 0; i < kDecompStages; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();   // lut visible (the only CTA-wide barrier)

  const int64_t nbt = p.n_blocktiles;
  const int64_t G = (int64_t)gridDim.x * nw;
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t bt, int s) {
    uint8_t* st = stage0 + (size_t)s * stage_bytes;
    const ulonglong2 a = reinterpret_cast<const ulonglong2*>(p.offsets)[bt];
    const ulonglong2 b = reinterpret_cast<const ulonglong2*>(p.offsets)[bt + 1];
    const uint32_t hb = (uint32_t)(b.x - a.x), lb = (uint32_t)(b.y - a.y);
    mbar_arrive_expect_tx(&bars[s], 1536u + hb + lb);
    bulk_g2s(st, p.b1 + bt * 64, 512, &bars[s], pol);
    bulk_g2s(st + 512, p.b2 + bt * 64, 512, &bars[s], pol);
    bulk_g2s(st + 1024, p.b3 + bt * 64, 512, &bars[s], pol);
    if (hb) bulk_g2s(st + 1536, p.h + a.x, hb, &bars[s], pol);
    if (lb) bulk_g2s(st + 1536 + p.hcap, reinterpret_cast<const uint8_t*>(p.l) + a.y, lb, &bars[s], pol);
  };

  // warp-major order: BlockTile g goes to SM g % grid, so the partial last round is spread
  // over all SMs (at most one extra tile per SM) instead of filling the first SMs' warps
  int64_t bt = (int64_t)warp * gridDim.x + blockIdx.x;
  if (lane == 0)
    for (int i = 0; i < kDecompStages - 1; ++i)
      if (bt + i * G < nbt) issue(bt + i * G, i);
  __syncwarp();

  // per-lane constants of the row passes
  const int fc = lane & 7;                                  // FragTile column (K / 8)
  const uint32_t ofc = (uint32_t)((fc >> 1) * 4 + (fc & 1) * 2);
  DecConst dk;
  load_dec_const(dk, p.eb7x2);
  const uint32_t lut_b = smem_u32(lut);

  for (uint32_t it = 0; bt < nbt; bt += G, ++it) {
    const int s = (int)(it % kDecompStages);
    const int64_t nxt = bt + (kDecompStages - 1) * G;
    // the stage consumed last iteration takes the BlockTile kDecompStages - 1 ahead
    if (lane == 0 && nxt < nbt) issue(nxt, (int)((it + kDecompStages - 1) % kDecompStages));
    mbar_wait(&bars[s], (it / kDecompStages) & 1);

    const uint8_t* st = stage0 + (size_t)s * stage_bytes;
    const uint32_t Hs = smem_u32(st + 1536);             // H segment (16-B aligned)
    const uint32_t Ls = smem_u32(st + 1536 + p.hcap);    // L segment

    // ---- scan: FragTiles 2*lane, 2*lane+1 (canonical order)
    {
      const uint4 a1 = *reinterpret_cast<const uint4*>(st + 16 * lane);
      const uint4 a2 = *reinterpret_cast<const uint4*>(st + 512 + 16 * lane);
      const uint4 a3 = *reinterpret_cast<const uint4*>(st + 1024 + 16 * lane);
      const uint32_t m0l = a1.x | a2.x | a3.x, m0h = a1.y | a2.y | a3.y;
      const uint32_t m1l = a1.z | a2.z | a3.z, m1h = a1.w | a2.w | a3.w;
      const uint32_t c0 = __popc(m0l) + __popc(m0h), c1 = __popc(m1l) + __popc(m1h);
      uint32_t incl = c0 + c1;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += v;
      }
      const uint32_t s0 = incl - c0 - c1, s1 = s0 + c0;
      // row prefix bytes of one FragTile -> H start of each of its 8 rows in [r8][o]
      auto put = [&](uint32_t ml, uint32_t mh, uint32_t start, uint32_t o) {
        uint32_t bl = ml - ((ml >> 1) & 0x55555555u);
        bl = (bl & 0x33333333u) + ((bl >> 2) & 0x33333333u);
        bl = (bl + (bl >> 4)) & 0x0F0F0F0Fu;
        uint32_t bh = mh - ((mh >> 1) & 0x55555555u);
        bh = (bh & 0x33333333u) + ((bh >> 2) & 0x33333333u);
        bh = (bh + (bh >> 4)) & 0x0F0F0F0Fu;
        const uint32_t pl = bl * 0x01010100u;                                   // rows 0..3
        const uint32_t ph = bh * 0x01010100u + ((bl * 0x01010101u) >> 24) * 0x01010101u;  // rows 4..7
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          hst[r * kHsRow + o] = (uint16_t)(start + ((pl >> (8 * r)) & 0xFFu));
          hst[(r + 4) * kHsRow + o] = (uint16_t)(start + ((ph >> (8 * r)) & 0xFFu));
        }
      };
      put(m0l, m0h, s0, 2u * lane);
      put(m1l, m1h, s1, 2u * lane + 1u);
    }
    __syncwarp();

    // ---- rows: 4 groups of 4 passes; the rank >= 2 patch is a warp-uniform branch per group
    const int64_t br = bt / p.nbc, bc = bt - br * p.nbc;
    const int64_t col = bc * 64 + fc * 8;
    // interior BlockTile with 16-B aligned rows: no bounds checks, one streaming STG.128 per row
    const bool interior = p.vec_ok && (bc * 64 + 64 <= p.cols) && (br * 64 + 64 <= p.rows);
#pragma unroll 1
    for (int g = 0; g < 4; ++g) {
      uint4 v[4];
      uint32_t rare = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int lr = 16 * g + 4 * i + (lane >> 3);          // row inside the BlockTile
        const int fr = lr >> 3, r8 = lr & 7;
        const uint32_t o = (uint32_t)((fr >> 1) * 16 + (fr & 1)) + ofc;   // canonical FragTile
        const uint32_t b1 = st[o * 8 + r8];
        const uint32_t b2 = st[512 + o * 8 + r8];
        const uint32_t b3 = st[1024 + o * 8 + r8];
        const uint32_t m = b1 | b2 | b3;
        const uint32_t hs = hst[r8 * kHsRow + o];
        const uint32_t ls = (o * 8 + (uint32_t)r8) * 8u - hs;
        const uint4 ent = ld_shared_v4(lut_b + 16u * m);
        rare |= ent.x;
        v[i] = decode_row_v3(b1, b2, b3, ent, Hs + (hs & ~3u), hs * 8u, Ls + 2u * ls, dk);
      }
      if (__any_sync(0xFFFFFFFFu, rare & 0x80u)) {
        // >= 3 fallbacks in some row of the group (rank >= 2): patch those rows
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int lr = 16 * g + 4 * i + (lane >> 3);
          const int fr = lr >> 3, r8 = lr & 7;
          const uint32_t o = (uint32_t)((fr >> 1) * 16 + (fr & 1)) + ofc;
          const uint32_t m = st[o * 8 + r8] | st[512 + o * 8 + r8] | st[1024 + o * 8 + r8];
          if (lut[m].x & 0x80u) {
            const uint32_t ls = (o * 8 + (uint32_t)r8) * 8u - hst[r8 * kHsRow + o];
            patch_rank2(m, reinterpret_cast<const uint16_t*>(st + 1536 + p.hcap) + ls, v[i].x, v[i].y, v[i].z,
                        v[i].w);
          }
        }
      }
      const int64_t row0 = br * 64 + 16 * g + (lane >> 3);
      if (interior) {
        uint16_t* dst = p.out + row0 * p.ld_out + col;
#pragma unroll
        for (int i = 0; i < 4; ++i)   // streaming stores: the output is not re-read here
          __stcs(reinterpret_cast<uint4*>(dst + (int64_t)(4 * i) * p.ld_out), v[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t row = row0 + 4 * i;
          if (row >= p.rows) continue;
          uint16_t* dst = p.out + row * p.ld_out + col;
          if (p.vec_ok && col + 8 <= p.cols) {
            __stcs(reinterpret_cast<uint4*>(dst), v[i]);
          } else {
            const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (col + e < p.cols) dst[e] = (uint16_t)(w[e >> 1] >> (16 * (e & 1)));
          }
        }
      }
    }
    __syncwarp();   // stage s and the H-start table are free again
  }
}

cudaError_t launch_decompress(const DecompParams& p, int grid, int warps, size_t smem, cudaStream_t stream) {
  static std::atomic<uint64_t> attr_done{0};
  cudaError_t e = once_per_device(attr_done, [] {
    return cudaFuncSetAttribute(decompress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e != cudaSuccess) return e;
  decompress_kernel<<<grid, 32 * warps, smem, stream>>>(p);
  return cudaGetLastError();
}

size_t decompress_smem_bytes(uint32_t stage_bytes, int warps) {
  return 4096 + 8 * kDecompStages * kDecompMaxWarps + kDecompMaxWarps * kHsTabBytes +
         (size_t)warps * kDecompStages * stage_bytes;
}

int decompress_max_warps() { return kDecompMaxWarps; }

}  // namespace zs
