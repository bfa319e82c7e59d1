// zs_gemm.cu -- ZipGEMM on sm_100a: Y[M][N] = X[M][K] * W[N][K]^T, W in TCA-TBE.
//
// The paper's Ada kernel decodes into mma.sync registers.  On sm_100a the
// tensor core reads operands from shared memory, so the kernel is re-designed around
// tcgen05 + TMEM + TMA, warp-specialised, persistent, stream-K:
//
//   work unit = (band of 128 weight rows = 2 BlockTile rows) x (one 64-wide K step).
//   The (band, k) iteration space is split evenly over the CTAs (stream-K), so no SM
//   idles on a partial wave (the O_proj "split-K tuning" issue of P:497).
//
//   warp 20      compressed producer: 1-D TMA bulk copies of the two BlockTiles' planes,
//                H and L segments into an S_c-slot ring (full_c / empty_c mbarriers);
//                offsets are prefetched 32 units ahead in registers.
//   warp 21      activation producer: 2-D TMA of the X tile [n_umma tokens][64 K],
//                SWIZZLE_128B, zero-filled out of bounds (token tail and K padding).
//   warps 4..19  4 decoder groups x 4 warps; thread = weight row.  Group g owns units
//                g, g+4, ...: FragTile popcount scan (warp shuffles), then the
//                branch-free row decoder writes 16-B chunks straight into the UMMA
//                canonical K-major SW128 layout (A operand, 128 x 64 bf16 = 16 KB).
//   warp 22      MMA issuer: 4 x tcgen05.mma (M=128, N=n_umma, K=16) per unit into a
//                double-buffered fp32 TMEM accumulator; tcgen05.commit frees the A/X slot.
//                Decode of unit k+1 (other groups) overlaps the MMA of unit k.
//   warps 0..3   epilogue: tcgen05.ld the accumulator (thread = TMEM lane = weight row),
//                BF16 store when the CTA owns the whole band, else fp32 atomics into the
//                workspace; the last-arriving CTA of a band converts it to BF16 and
//                zeroes the workspace again (self-cleaning split-K fixup).
#include "zs_device.cuh"
#include "zs_kernels.h"

#include <cuda_bf16.h>

namespace zs {

constexpr int kGroups = 4;                 // decoder warp groups
constexpr int kASlots = kGroups;           // one A/X slot per group
constexpr int kEpiWarps = 4;
constexpr int kDecWarps = 4 * kGroups;
constexpr int kWarpProdC = kEpiWarps + kDecWarps;  // 20
constexpr int kWarpProdX = kWarpProdC + 1;         // 21
constexpr int kWarpMma = kWarpProdX + 1;           // 22
constexpr int kGemmThreads = 32 * (kWarpMma + 1);  // 736
constexpr int kMaxCSlots = 16;

struct __align__(8) Bars {
  uint64_t full_c[kMaxCSlots];
  uint64_t empty_c[kMaxCSlots];
  uint64_t xfull[kASlots];
  uint64_t decoded[kASlots];
  uint64_t aempty[kASlots];
  uint64_t accfull[2];
  uint64_t accempty[2];
  uint32_t tmem_base;
  uint32_t last_flag;
};

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    zipgemm_kernel(const GemmParams p, const __grid_constant__ CUtensorMap xmap) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the SW128 operand tiles
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint4* lut = reinterpret_cast<uint4*>(smem);
  Bars* bars = reinterpret_cast<Bars*>(smem + 4096);
  uint8_t* aslots = smem + 4096 + 1024;
  uint8_t* cslots = aslots + (size_t)kASlots * p.aslot_bytes;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t S_c = p.n_cslots;

  // ---- stream-K range of this CTA
  const int64_t T = p.total_units;
  const int64_t u0 = (int64_t)blockIdx.x * T / gridDim.x;
  const int64_t u1 = (int64_t)(blockIdx.x + 1) * T / gridDim.x;
  const int nunits = (int)(u1 - u0);
  const int64_t nbc = p.nbc;

  // ---- setup
  if (tid < 256) lut[tid] = build_lut_entry((uint32_t)tid);
  if (tid == 32) {
    for (uint32_t i = 0; i < S_c; ++i) {
      mbar_init(&bars->full_c[i], 1);
      mbar_init(&bars->empty_c[i], 128);
    }
    for (int i = 0; i < kASlots; ++i) {
      mbar_init(&bars->xfull[i], 1);
      mbar_init(&bars->decoded[i], 128);
      mbar_init(&bars->aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->accfull[i], 1);
      mbar_init(&bars->accempty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc_dyn(&bars->tmem_base, p.tmem_cols);
  if (warp == kWarpProdX && lane == 0) prefetch_tmap(&xmap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = bars->tmem_base;

  if (warp == kWarpProdC) {
    // ================================================================ compressed producer
    const uint64_t pol = policy_evict_first();
    const ulonglong2* off2 = reinterpret_cast<const ulonglong2*>(p.offsets);
    // lane i holds {h,l} offsets for unit (batch + i): BlockTile a start/end, b start/end
    auto load_batch = [&](int b, ulonglong2 (&o)[4]) {
      const int it = b + lane;
      if (it < nunits) {
        const int64_t u = u0 + it;
        const int64_t band = u / nbc, kc = u % nbc;
        const int64_t bta = 2 * band * nbc + kc;
        o[0] = off2[bta];
        o[1] = off2[bta + 1];
        if (2 * band + 1 < p.nbr) {
          o[2] = off2[bta + nbc];
          o[3] = off2[bta + nbc + 1];
        } else {
          o[2] = make_ulonglong2(0, 0);
          o[3] = make_ulonglong2(0, 0);
        }
      }
    };
    ulonglong2 cur[4], nxt[4];
    load_batch(0, cur);
    for (int b = 0; b < nunits; b += 32) {
      if (b + 32 < nunits) load_batch(b + 32, nxt);
      const int cnt = min(32, nunits - b);
      for (int j = 0; j < cnt; ++j) {
        uint64_t v[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[2 * q] = __shfl_sync(0xFFFFFFFFu, cur[q].x, j);
          v[2 * q + 1] = __shfl_sync(0xFFFFFFFFu, cur[q].y, j);
        }
        if (lane == 0) {
          const int it = b + j;
          const int64_t u = u0 + it;
          const int64_t band = u / nbc, kc = u % nbc;
          const int64_t bta = 2 * band * nbc + kc;
          const bool has_b = (2 * band + 1 < p.nbr);
          const uint32_t c = (uint32_t)it % S_c;
          mbar_wait(&bars->empty_c[c], (((uint32_t)it / S_c) & 1u) ^ 1u);
          uint8_t* cs = cslots + (size_t)c * p.cslot_bytes;
          const uint32_t ha = (uint32_t)(v[2] - v[0]), la = (uint32_t)(v[3] - v[1]);
          const uint32_t hb = has_b ? (uint32_t)(v[6] - v[4]) : 0u, lb = has_b ? (uint32_t)(v[7] - v[5]) : 0u;
          const uint32_t bytes = 1536u + ha + la + (has_b ? 1536u + hb + lb : 0u);
          uint64_t* fb = &bars->full_c[c];
          mbar_arrive_expect_tx(fb, bytes);
          bulk_g2s(cs, p.b1 + bta * 64, 512, fb, pol);
          bulk_g2s(cs + 512, p.b2 + bta * 64, 512, fb, pol);
          bulk_g2s(cs + 1024, p.b3 + bta * 64, 512, fb, pol);
          if (ha) bulk_g2s(cs + 3072, p.h + v[0], ha, fb, pol);
          if (la) bulk_g2s(cs + 3072 + 2 * p.hcap, reinterpret_cast<const uint8_t*>(p.l) + v[1], la, fb, pol);
          if (has_b) {
            const int64_t btb = bta + nbc;
            bulk_g2s(cs + 1536, p.b1 + btb * 64, 512, fb, pol);
            bulk_g2s(cs + 2048, p.b2 + btb * 64, 512, fb, pol);
            bulk_g2s(cs + 2560, p.b3 + btb * 64, 512, fb, pol);
            if (hb) bulk_g2s(cs + 3072 + p.hcap, p.h + v[4], hb, fb, pol);
            if (lb)
              bulk_g2s(cs + 3072 + 2 * p.hcap + p.lcap, reinterpret_cast<const uint8_t*>(p.l) + v[5], lb, fb, pol);
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
    }
  } else if (warp == kWarpProdX) {
    // ================================================================ activation producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      const uint32_t xbytes = p.n_umma * 128u;
      for (int it = 0; it < nunits; ++it) {
        const uint32_t a = (uint32_t)it % kASlots;
        mbar_wait(&bars->aempty[a], (((uint32_t)it / kASlots) & 1u) ^ 1u);
        const int64_t kc = (u0 + it) % nbc;
        uint8_t* xs = aslots + (size_t)a * p.aslot_bytes + 16384;
        mbar_arrive_expect_tx(&bars->xfull[a], xbytes);
        tma_load_2d(xs, &xmap, (int32_t)(kc * 64), p.m0, &bars->xfull[a], pol);
      }
    }
  } else if (warp == kWarpMma) {
    // ================================================================ MMA issuer
    const uint32_t idesc = umma_idesc_bf16(128, p.n_umma);
    int seg = -1;
    for (int it = 0; it < nunits; ++it) {
      const int64_t u = u0 + it;
      const bool first = (it == 0) || (u % nbc == 0);
      const bool last = (it == nunits - 1) || ((u + 1) % nbc == 0);
      if (first) {
        ++seg;
        mbar_wait(&bars->accempty[seg & 1], (((uint32_t)seg >> 1) & 1u) ^ 1u);
        tc_fence_after();
      }
      const uint32_t a = (uint32_t)it % kASlots;
      mbar_wait(&bars->decoded[a], ((uint32_t)it / kASlots) & 1u);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t d = tmem_base + (uint32_t)(seg & 1) * p.n_umma;
        const uint32_t a_addr = smem_u32(aslots + (size_t)a * p.aslot_bytes);
        const uint32_t x_addr = a_addr + 16384;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16_ss(d, umma_desc_sw128(a_addr + 32 * k), umma_desc_sw128(x_addr + 32 * k), idesc,
                       (first && k == 0) ? 0u : 1u);
        umma_commit(&bars->aempty[a]);
        if (last) umma_commit(&bars->accfull[seg & 1]);
      }
      __syncwarp();
    }
  } else if (warp >= kEpiWarps) {
    // ================================================================ decoders
    const int g = (warp - kEpiWarps) >> 2;
    const int wg = (warp - kEpiWarps) & 3;
    const int bt_sel = wg >> 1, hh = wg & 1;
    const int lr = lane + 32 * hh;      // row inside the BlockTile
    const int fr = lr >> 3, r8 = lr & 7;
    const int R = 64 * bt_sel + lr;     // row inside the 128-row A tile
    const uint64_t rowmask = (1ull << (8 * r8)) - 1ull;
    const uint32_t a = (uint32_t)g;     // this group's A/X slot
    uint8_t* A = aslots + (size_t)a * p.aslot_bytes;
    for (int it = g; it < nunits; it += kGroups) {
      const uint32_t c = (uint32_t)it % S_c;
      mbar_wait(&bars->full_c[c], ((uint32_t)it / S_c) & 1u);
      mbar_wait(&bars->xfull[a], ((uint32_t)it / kASlots) & 1u);
      const int64_t band = (u0 + it) / nbc;
      const bool present = (2 * band + bt_sel) < p.nbr;
      if (present) {
        const uint8_t* cs = cslots + (size_t)c * p.cslot_bytes;
        const uint64_t* P1 = reinterpret_cast<const uint64_t*>(cs + bt_sel * 1536);
        const uint64_t* P2 = P1 + 64;
        const uint64_t* P3 = P1 + 128;
        const uint8_t* H = cs + 3072 + bt_sel * p.hcap;
        const uint16_t* L = reinterpret_cast<const uint16_t*>(cs + 3072 + 2 * p.hcap + bt_sel * p.lcap);
        // FragTile prefix: this warp's FragTiles are canonical 32*hh .. 32*hh+31
        const int fo = 32 * hh + lane;
        const uint32_t cnt = __popcll(P1[fo] | P2[fo] | P3[fo]);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
          if (lane >= d) incl += t;
        }
        const uint32_t excl = incl - cnt;
        uint32_t base = 0;
        if (hh) base = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)__popcll(P1[lane] | P2[lane] | P3[lane]));
#pragma unroll 2
        for (int fc = 0; fc < 8; ++fc) {
          const int o = ((fr >> 1) * 4 + (fc >> 1)) * 4 + (fc & 1) * 2 + (fr & 1);
          const uint32_t pref = __shfl_sync(0xFFFFFFFFu, excl, o - 32 * hh) + base;
          const uint64_t q1 = P1[o], q2 = P2[o], q3 = P3[o];
          const uint32_t hs = pref + (uint32_t)__popcll((q1 | q2 | q3) & rowmask);
          const uint32_t ls = (uint32_t)(o * 8 + r8) * 8u - hs;
          const uint4 v = decode_row(q1, q2, q3, (uint32_t)r8, H, hs, L, ls, lut, p.eb7x2);
          *reinterpret_cast<uint4*>(A + R * 128 + ((fc ^ (R & 7)) << 4)) = v;
        }
      }
      fence_proxy_async_smem();
      mbar_arrive(&bars->decoded[a]);
      mbar_arrive(&bars->empty_c[c]);
    }
  } else {
    // ================================================================ epilogue (warps 0..3)
    const int et = tid;  // 0..127 = TMEM lane = row inside the band
    const int64_t b_first = u0 / nbc, b_last = (u1 - 1) / nbc;
    int seg = 0;
    for (int64_t band = b_first; band <= b_last; ++band, ++seg) {
      const int64_t s0 = max(u0, band * nbc), s1 = min(u1, (band + 1) * nbc);
      const bool full = (s1 - s0) == nbc;
      mbar_wait(&bars->accfull[seg & 1], ((uint32_t)seg >> 1) & 1u);
      tc_fence_after();
      const int64_t n = band * 128 + et;
      const bool nvalid = n < p.N;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * warp) << 16) + (uint32_t)(seg & 1) * p.n_umma;
      for (uint32_t cb = 0; cb < p.n_umma; cb += 16) {
        uint32_t v[16];
        tmem_ld16(taddr + cb, v);
        if (nvalid) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = (int)cb + j;
            if (m < p.mc) {
              const float f = __uint_as_float(v[j]);
              if (full)
                p.y[(int64_t)(p.m0 + m) * p.ldy + n] = __bfloat16_as_ushort(__float2bfloat16_rn(f));
              else
                atomicAdd(p.ws + (int64_t)m * p.N + n, f);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->accempty[seg & 1]);
      if (!full) {
        __threadfence();
        named_bar_sync(1, 128);
        if (et == 0) {
          const uint32_t old = atomicAdd(&p.counters[band], (uint32_t)(s1 - s0));
          bars->last_flag = (old + (uint32_t)(s1 - s0) == (uint32_t)nbc) ? 1u : 0u;
        }
        named_bar_sync(1, 128);
        if (bars->last_flag) {
          __threadfence();
          if (nvalid) {
            for (int m = 0; m < p.mc; ++m) {
              float* wp = p.ws + (int64_t)m * p.N + n;
              const float f = __ldcg(wp);
              p.y[(int64_t)(p.m0 + m) * p.ldy + n] = __bfloat16_as_ushort(__float2bfloat16_rn(f));
              __stcg(wp, 0.0f);
            }
          }
          if (et == 0) p.counters[band] = 0u;
        }
        named_bar_sync(1, 128);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

cudaError_t launch_gemm(const GemmParams& p, const CUtensorMap& xmap, int grid, size_t smem, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(zipgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  zipgemm_kernel<<<grid, kGemmThreads, smem, stream>>>(p, xmap);
  return cudaGetLastError();
}

size_t gemm_smem_bytes(const GemmParams& p) {
  return 1024 /*align slack*/ + 4096 + 1024 + (size_t)kASlots * p.aslot_bytes + (size_t)p.n_cslots * p.cslot_bytes;
}

int gemm_threads() { return kGemmThreads; }
int gemm_groups() { return kGroups; }
int gemm_aslots() { return kASlots; }

}  // namespace zs
