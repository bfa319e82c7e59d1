// zs_gemm.cu -- ZipGEMM on sm_100a: Y[M][N] = X[M][K] * W[N][K]^T, W in TCA-TBE.
//
// The paper's Ada kernel decodes into mma.sync registers.  On sm_100a the
// tensor core reads A from shared or tensor memory, so the kernel is re-designed around
// tcgen05 + TMEM + TMA, warp-specialised, persistent, stream-K:
//
//   work unit = (band of 128 weight rows = 2 BlockTile rows) x (one 64-wide K step).
//   The (band, k) iteration space is split evenly over the CTAs (stream-K), so no SM
//   idles on a partial wave (the O_proj "split-K tuning" issue of P:497).  A ring stage
//   holds 4 consecutive units of a CTA.
//
//   warp 1    compressed producer.  Units of one band are contiguous along K in every
//             array, so a stage is fetched with one 1-D TMA bulk copy per array and run
//             of same-band units (B1/B2/B3 x 2 BlockTile rows, H x 2, L x 2: 10 copies
//             per 4 units).  Per-unit segment offsets and flags go into the stage header.
//   warp 2    activation producer: 2-D TMA of X tiles [n_umma tokens][64 K], SWIZZLE_128B,
//             zero-filled out of bounds (token tail and K padding), S_x-deep ring.
//   warps 8.. decoders, 4 per TMEM lane quarter q = warp % 4 (rows 32q..32q+31 of the
//             128-row A tile).  Every decoder warp visits every stage; inside a stage the
//             4 warps of a quarter take that quarter of the stage's units dynamically.
//             Per unit: FragTile popcount scan (warp shuffles), the branch-free row
//             decoder, and tcgen05.st of the decoded BF16 rows into a TMEM A slot.
//   warp 0    MMA issuer (one elected lane, warp-uniform operands): per stage, 4 x
//             tcgen05.mma (A from TMEM, B = X from smem, M=128, N=n_umma, K=16) per unit
//             into a double-buffered fp32 TMEM accumulator; decode of later units
//             overlaps the MMA of earlier ones (the two-level pipeline of P:442-448).
//             Completion is published as mma_done (monotonic unit count) which frees A
//             slots for the decoders and X slots for warp 2.
//   warps 4-7 epilogue: tcgen05.ld the accumulator (thread = TMEM lane = weight row), BF16
//             store when the CTA owns the whole band, else fp32 atomics into the
//             workspace; the last-arriving CTA of a band converts it to BF16 and zeroes the
//             workspace again (self-cleaning split-K fixup).
//
// The single-warp roles share SM sub-partitions with 4 busy decoder warps each, so they
// are written to issue few instructions per stage (no 64-bit division, batched waits).
#include "zs_device.cuh"
#include "zs_kernels.h"
#include "zs_lut.h"

#include <cuda_bf16.h>

namespace zs {

// The SMSP arbiter issues from the highest eligible warp id first, so the latency-critical
// single-warp roles take the TOP ids (a low-id producer / MMA warp starves behind six busy
// decoder warps on its SMSP and the whole pipeline idles): decoders 0..23, epilogue 24..27.
#ifndef ZS_BACKOFF_CTRL
#define ZS_BACKOFF_CTRL 256   // ns between barrier probes of the producer / MMA warps
#endif
#ifndef ZS_BACKOFF_DEC
#define ZS_BACKOFF_DEC 32     // ns between barrier probes of a decoder warp
#endif
constexpr uint32_t kLutBytes = 4096u;   // selector table (a second table of fallback selectors measured 4% slower)
#ifndef ZS_UPS
#define ZS_UPS 4   // units per ring stage = decoder warps per TMEM lane quarter
#endif
#ifndef ZS_DEC_PER_Q
#define ZS_DEC_PER_Q ZS_UPS   // decoder warps per TMEM lane quarter (static unit assignment, see below)
#endif
constexpr int kDecPerQuarter = ZS_DEC_PER_Q;
// one decoder warp per unit of a stage: with more warps than units per stage a warp's next unit
// can sit two stages ahead of its current one (measured: D = 5 deadlocks on the 3-slot
// compressed ring at M = 200 and is 25% slower where it completes, r02 it6)
static_assert(kDecPerQuarter == ZS_UPS, "the static unit assignment assumes one decoder warp per unit of a stage");
constexpr int kWarpDec0 = 0;                       // warps 0..4D-1: decoders (lane quarter = warp % 4)
constexpr int kWarpEpi0 = 4 * kDecPerQuarter;      // 4 epilogue warps (TMEM lane quarters)
constexpr int kWarpAlloc = kWarpEpi0 + 4;
constexpr int kWarpProdX = kWarpEpi0 + 5;
constexpr int kWarpProdC = kWarpEpi0 + 6;
constexpr int kWarpMma = kWarpEpi0 + 7;            // highest id: first pick of its SMSP's arbiter
constexpr int kGemmThreads = 32 * (kWarpEpi0 + 8);  // 768 at D = 4 (80 registers per thread)
constexpr int kUPS = ZS_UPS;                       // units per ring stage
constexpr int kMaxCSlots = 8;
constexpr int kMaxXSlots = 16;
constexpr int kMaxASlots = 3 * kUPS;
constexpr uint32_t kStageMeta = 128;               // see the stage header layout below
// planes of a stage: [BlockTile row a | b][B1 | B2 | B3][unit][512 B]; row b's planes start
// 32 B past a multiple of 128 B, so the two halves of a decoder warp (rows of BlockTile a and b
// at the same FragTile position) read their plane bytes from different banks
constexpr uint32_t kBtPlaneStride = 3 * kUPS * 512 + 32;
constexpr uint32_t kStagePlanes = 2 * kBtPlaneStride;
constexpr uint32_t kTmemCols = 512;
// row table: 32 FragTiles x 8 rows x u16 (+ pad)
constexpr uint32_t kRpBuf = 32 * 16 + 64;
constexpr uint32_t kRpWarp = 2 * kRpBuf;             // per decoder warp: double-buffered (software pipeline)
constexpr uint32_t kRpTabBytes = 4 * kDecPerQuarter * kRpWarp;

// stage header (u32 words): [4i+0..3] unit i {H a, H b, L a, L b} offsets inside the
// stage regions; [20+i] unit i has BlockTile row b; [24] stage index the slot holds.

struct __align__(16) Bars {
  uint64_t full_c[kMaxCSlots];
  uint64_t empty_c[kMaxCSlots];
  uint64_t xfull[kMaxXSlots];            // per X tile slot (one unit's [n_umma tokens][64 K])
  uint64_t xempty[kMaxXSlots];           // X tile consumed (tcgen05.commit after its unit's MMAs)
  uint64_t afree[kMaxASlots / kUPS];    // TMEM A stage free (tcgen05.commit after its MMAs)
  uint64_t afull[kMaxASlots / kUPS];    // TMEM A stage decoded: one arrival per (unit, lane quarter)
  uint64_t accfull[2];
  uint64_t accempty[2];
  uint32_t tmem_base;
  uint32_t last_flag;
};

#ifndef ZS_TRACE
#define ZS_TRACE 0   // build with -DZS_TRACE=1 for scripts/trace_gemm.py (costs issue slots)
#endif
__device__ __forceinline__ void trace_ev(unsigned long long* tr, int unit, int ev) {
#if ZS_TRACE
  // debug trace: trace[(cta * kTraceUnits + unit) * 16 + event] = clock64, first kTraceCtas CTAs
  constexpr int kTraceCtas = 4, kTraceUnits = 128;
  if (ZS_TRACE == 2 && ev >= 7 && ev < 16 && ev != 6 && (ev < 16) && (threadIdx.x >> 5) < kWarpEpi0) return;
  if (tr != nullptr && blockIdx.x < kTraceCtas && unit < kTraceUnits)
    tr[((size_t)blockIdx.x * kTraceUnits + unit) * 16 + ev] = clock64();
#else
  (void)tr; (void)unit; (void)ev;
#endif
}

__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// x / d for the small ring sizes d (magic = floor(2^32 / d) + 1, exact for x < 2^31 / d)
__device__ __forceinline__ uint32_t fastdiv(uint32_t x, uint32_t d, uint32_t magic) {
  return d == 1u ? x : __umulhi(x, magic);
}

__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint32_t bytepop(uint32_t x) {  // popcount of every byte
  x = x - ((x >> 1) & 0x55555555u);
  x = (x & 0x33333333u) + ((x >> 2) & 0x33333333u);
  return (x + (x >> 4)) & 0x0F0F0F0Fu;
}

// fused exchange (f2): copy the mc outputs of one weight row n (column of Y), just stored
// to the local Y by this thread, into every peer's Y.  Out of line, so the exchange adds no
// register pressure to the rest of the kernel (it shares one 64-register allocation).
// Loads go out 16 at a time (independent L2 round trips), then every peer gets the batch.
__device__ __noinline__ void copy_to_peers(uint16_t* const* ypeer, int npeer, const uint16_t* y, int64_t ldy,
                                           int64_t off, int mc) {
  for (int m0 = 0; m0 < mc; m0 += 16, off += 16 * ldy) {
    uint16_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (m0 + j < mc) v[j] = y[off + j * ldy];
    for (int i = 0; i < npeer; ++i) {
      uint16_t* d = ypeer[i];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (m0 + j < mc) d[off + j * ldy] = v[j];
    }
  }
}

// kPeer: the fused output exchange (peer stores + completion signal) is compiled in; the
// plain instance is the single-GPU kernel with no extra registers or branches
template <bool kPeer>
__global__ void __launch_bounds__(kGemmThreads, 1)
    zipgemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap xmap) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the SW128 X tiles
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Bars* bars = reinterpret_cast<Bars*>(smem);
  uint8_t* rptab = smem + 1024;                        // decoder row-prefix tables
  uint4* slut = reinterpret_cast<uint4*>(smem + 1024 + kRpTabBytes);   // PRMT selectors, 16 B per m
  uint8_t* xslots = smem + 1024 + kRpTabBytes + kLutBytes;
  uint8_t* cslots = xslots + (size_t)p.n_xslots * p.aslot_bytes;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t S_c = p.n_cslots;
  const uint32_t S_x = p.n_xslots;             // multiple of kUPS
  const uint32_t S_a = p.n_aslots;             // multiple of kUPS
  const uint32_t SXS = S_x / kUPS;             // X ring in stages
  const uint32_t capH = p.hcap, capL = p.lcap;

  // ---- stream-K range of this CTA (32-bit unit indices; the host checks the range)
  const uint32_t T = (uint32_t)p.total_units;
  const uint32_t u0 = (uint32_t)((uint64_t)blockIdx.x * T / gridDim.x);
  const uint32_t u1 = (uint32_t)((uint64_t)(blockIdx.x + 1) * T / gridDim.x);
  const int nunits = (int)(u1 - u0);
  const int nstages = (nunits + kUPS - 1) / kUPS;
  const uint32_t nbc = (uint32_t)p.nbc;
  const uint32_t nbr = (uint32_t)p.nbr;
  const uint32_t band0 = u0 / nbc, kc0 = u0 % nbc;

  // ---- setup
  // barrier init spread over the lanes of warp 1 (the selector table is loaded by the decoder
  // warps after the CTA barrier, off the producers' critical path)
  if (warp == 1) {
    for (uint32_t i = lane; i < S_c; i += 32) {
      mbar_init(&bars->full_c[i], 1);
      mbar_init(&bars->empty_c[i], 4 * kUPS);   // one arrival per (unit, lane quarter)
    }
    for (uint32_t i = lane; i < S_x; i += 32) {
      mbar_init(&bars->xfull[i], 1);
      mbar_init(&bars->xempty[i], 1);
    }
    if (lane < S_a / kUPS) {
      mbar_init(&bars->afree[lane], 1);
      mbar_init(&bars->afull[lane], 4 * kUPS);
    }
    if (lane < 2) {
      mbar_init(&bars->accfull[lane], 1);
      mbar_init(&bars->accempty[lane], 128);
    }
    fence_mbar_init();
  }
  if (warp == kWarpAlloc) tmem_alloc<kTmemCols>(&bars->tmem_base);
  if (warp == kWarpProdX && lane == 0) prefetch_tmap(&xmap);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Programmatic dependent launch: the next kernel on the stream may be scheduled now; its
  // CTAs become resident as ours exit, and it reads nothing of ours before its own
  // griddepcontrol.wait.  Weights and offsets are immutable, so the prologue and the
  // compressed stream of this kernel start before the previous kernel has finished.
  grid_launch_dependents();
  const uint32_t tmem_base = bars->tmem_base;
  // register budget: 24 decoder warps x 72 + 8 control / epilogue warps x 40 = the 64 K
  // register file (the decoders rematerialise addresses at the 64-register default)
  const uint32_t dcols = p.acc_cols;                   // accumulator buffer stride (columns)
  const uint32_t tmem_a = tmem_base + p.n_acc * dcols; // first A slot column
  // accumulator buffer of segment s and the parity of its use (n_acc = 2: double buffered;
  // n_acc = 1: a 256-token accumulator leaves room for one buffer next to the A ring)
  const uint32_t nacc1 = p.n_acc - 1u;
  // X ring in stage mode (>= 2 stages of 4 tiles: one barrier per stage, contiguous tiles) or
  // tile mode (one barrier per tile; the 256-token chunks' 32-KB tiles)
  const bool xstage = (S_x % kUPS) == 0 && S_x >= 2 * kUPS;
  auto abuf = [&](int s) { return (uint32_t)s & nacc1; };
  auto apar = [&](int s) { return ((uint32_t)s >> nacc1) & 1u; };

  if (warp == kWarpProdC) {
    // ================================================================ compressed producer
    // Batches of 32 units (8 stages): lane l owns unit b0 + l, loads its offsets, and
    // the quad of lanes of a stage computes the stage header with shuffles.
    const uint64_t pol = policy_evict_first();
    const ulonglong2* off2 = reinterpret_cast<const ulonglong2*>(p.offsets);
    const int quad = lane / kUPS, qi = lane % kUPS;   // lane group of a stage / unit in it
    uint32_t slot = 0, eph = 1;   // ring slot / empty-barrier parity of the next stage
    constexpr int kBatch = (32 / kUPS) * kUPS;   // units per batch: whole stages
    for (int b0 = 0; b0 < nunits; b0 += kBatch) {
      const int it = b0 + lane;
      const bool valid = it < nunits && lane < kBatch;
      const uint32_t kk = kc0 + (uint32_t)it;
      const uint32_t band = band0 + kk / nbc, kc = kk % nbc;
      const uint32_t bta = 2u * band * nbc + kc;
      const bool has_b = valid && (2u * band + 1u < nbr);
      uint32_t h0a = 0, h1a = 0, l0a = 0, l1a = 0, h0b = 0, h1b = 0, l0b = 0, l1b = 0;
      if (valid) {
        const ulonglong2 a0 = off2[bta], a1 = off2[bta + 1];
        h0a = (uint32_t)a0.x; l0a = (uint32_t)a0.y; h1a = (uint32_t)a1.x; l1a = (uint32_t)a1.y;
        if (has_b) {
          const ulonglong2 c0 = off2[bta + nbc], c1 = off2[bta + nbc + 1];
          h0b = (uint32_t)c0.x; l0b = (uint32_t)c0.y; h1b = (uint32_t)c1.x; l1b = (uint32_t)c1.y;
        }
      }
      // exclusive prefix of the segment sizes inside the quad (= stage)
      uint32_t pha = h1a - h0a, phb = h1b - h0b, pla = l1a - l0a, plb = l1b - l0b;
      const uint32_t tot_self = pha + phb + pla + plb + (valid ? (has_b ? 3072u : 1536u) : 0u);
#pragma unroll
      for (int d = 1; d < kUPS; d <<= 1) {
        const uint32_t a = __shfl_up_sync(0xFFFFFFFFu, pha, d), b = __shfl_up_sync(0xFFFFFFFFu, phb, d);
        const uint32_t c = __shfl_up_sync(0xFFFFFFFFu, pla, d), e = __shfl_up_sync(0xFFFFFFFFu, plb, d);
        if (qi >= d) { pha += a; phb += b; pla += c; plb += e; }
      }
      // pha.. are now inclusive; exclusive = inclusive - own size
      const uint32_t oha = pha - (h1a - h0a), ohb = phb - (h1b - h0b), ola = pla - (l1a - l0a), olb = plb - (l1b - l0b);
#if ZS_UPS == 4
      uint32_t stage_bytes = tot_self;
#pragma unroll
      for (int d = 1; d < kUPS; d <<= 1) stage_bytes += __shfl_xor_sync(0xFFFFFFFFu, stage_bytes, d);
#else
      // (not a power of two: inclusive scan inside the group, total from its last lane)
      uint32_t stage_bytes = tot_self;
#pragma unroll
      for (int d = 1; d < kUPS; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, stage_bytes, d);
        if (qi >= d) stage_bytes += t;
      }
      stage_bytes = __shfl_sync(0xFFFFFFFFu, stage_bytes, (quad * kUPS + kUPS - 1) & 31);
#endif
      // runs of same-band units inside the quad: a run starts at qi == 0 or on a band change
      const uint32_t band_prev = __shfl_up_sync(0xFFFFFFFFu, band, 1);
      const bool run_start = valid && (qi == 0 || band_prev != band);
      const uint32_t starts = __ballot_sync(0xFFFFFFFFu, run_start);
      const uint32_t validm = __ballot_sync(0xFFFFFFFFu, valid);
      // last lane of my run: next start in my quad minus one (or the quad's last valid lane)
      const uint32_t quad_mask = ((1u << kUPS) - 1u) << (kUPS * quad);
      const uint32_t later = starts & quad_mask & ~((2u << lane) - 1u);
      const uint32_t qvalid = validm & quad_mask;
      const int qlast = qvalid ? 31 - __clz(qvalid) : lane;
      const int rend = later ? (__ffs(later) - 2) : qlast;
      const uint32_t e_h1a = __shfl_sync(0xFFFFFFFFu, h1a, rend), e_l1a = __shfl_sync(0xFFFFFFFFu, l1a, rend);
      const uint32_t e_h1b = __shfl_sync(0xFFFFFFFFu, h1b, rend), e_l1b = __shfl_sync(0xFFFFFFFFu, l1b, rend);
      const uint32_t nrun = (uint32_t)(rend - lane + 1);
      const int st_hi = min(nstages, (b0 + kBatch) / kUPS);
      for (int st = b0 / kUPS; st < st_hi; ++st, slot = (slot + 1 == S_c) ? 0u : slot + 1u, eph ^= (slot == 0)) {
        mbar_wait(&bars->empty_c[slot], eph, ZS_BACKOFF_CTRL);
        uint8_t* cs = cslots + (size_t)slot * p.cslot_bytes;
        const bool mine = (quad == st - b0 / kUPS);
        // dbg & 8 (timing experiment): after the first ring fill the stages are not refilled;
        // decoders re-decode the stale (self-consistent) slot contents -> decode without HBM
        const bool stale = (p.dbg & 8) && st >= (int)S_c;
        if (mine && valid && !stale) {
          uint32_t* meta = reinterpret_cast<uint32_t*>(cs);
          *reinterpret_cast<uint4*>(meta + 4 * qi) = make_uint4(oha, ohb, ola, olb);
          meta[20 + qi] = has_b ? 1u : 0u;
        }
        __syncwarp();
        if (mine && qi == 0 && stale) mbar_arrive(&bars->full_c[slot]);
        if (mine && qi == 0 && !stale) {
          mbar_arrive_expect_tx(&bars->full_c[slot], stage_bytes);  // release: header visible
          trace_ev(p.trace, it, 0);
        }
        __syncwarp();
        if (mine && run_start && !stale) {
          uint64_t* fb = &bars->full_c[slot];
          uint8_t* planes = cs + kStageMeta;
          uint8_t* Hr = planes + kStagePlanes;   // [H a | H b | L a | L b]
          const uint32_t pb = nrun * 512u;
          const uint32_t po = (uint32_t)qi * 512u;
          bulk_g2s(planes + 0 * (kUPS * 512) + po, p.b1 + (size_t)bta * 64, pb, fb, pol);
          bulk_g2s(planes + 1 * (kUPS * 512) + po, p.b2 + (size_t)bta * 64, pb, fb, pol);
          bulk_g2s(planes + 2 * (kUPS * 512) + po, p.b3 + (size_t)bta * 64, pb, fb, pol);
          if (e_h1a > h0a) bulk_g2s(Hr + oha, p.h + h0a, e_h1a - h0a, fb, pol);
          if (e_l1a > l0a)
            bulk_g2s(Hr + 2 * capH + ola, reinterpret_cast<const uint8_t*>(p.l) + l0a, e_l1a - l0a, fb, pol);
          if (has_b) {
            const size_t btb = (size_t)bta + nbc;
            bulk_g2s(planes + kBtPlaneStride + 0 * (kUPS * 512) + po, p.b1 + btb * 64, pb, fb, pol);
            bulk_g2s(planes + kBtPlaneStride + 1 * (kUPS * 512) + po, p.b2 + btb * 64, pb, fb, pol);
            bulk_g2s(planes + kBtPlaneStride + 2 * (kUPS * 512) + po, p.b3 + btb * 64, pb, fb, pol);
            if (e_h1b > h0b) bulk_g2s(Hr + capH + ohb, p.h + h0b, e_h1b - h0b, fb, pol);
            if (e_l1b > l0b)
              bulk_g2s(Hr + 2 * capH + capL + olb, reinterpret_cast<const uint8_t*>(p.l) + l0b, e_l1b - l0b, fb,
                       pol);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == kWarpProdX) {
    // ================================================================ activation producer
    // one X tile [n_umma tokens][64 K] per unit into an S_x-slot ring; a slot is refilled once
    // the MMA warp's commit after its unit's MMAs has arrived
    const uint64_t pol = policy_evict_last();
    const uint32_t xbytes = p.n_umma * 128u;
    uint32_t k = kc0;
    uint32_t xs = 0, xuse = 0;   // tile slot / how often the ring has wrapped
    grid_dependency_wait();      // X may be the previous kernel's output (PDL)
    if (xstage) {
      // stage mode (the ring holds >= 2 stages of 4 tiles): one barrier per stage of 4 tiles
      uint32_t xr = 0;
      for (int st = 0; st < nstages; ++st) {
        if (xuse > 0) mbar_wait(&bars->xempty[xr], (xuse - 1u) & 1u, ZS_BACKOFF_CTRL);
        const int nu = min(kUPS, nunits - st * kUPS);
        if (elect_one()) {
          mbar_arrive_expect_tx(&bars->xfull[xr], xbytes * (uint32_t)nu);
          uint32_t k2 = k;
          for (int i = 0; i < nu; ++i) {
            tma_load_2d(xslots + (size_t)(xr * kUPS + i) * p.aslot_bytes, &xmap, (int32_t)(k2 * 64), p.m0,
                        &bars->xfull[xr], pol);
            if (++k2 == nbc) k2 = 0;
          }
        }
        __syncwarp();
        k += (uint32_t)nu;
        if (k >= nbc) k -= nbc;
        if (++xr == S_x / kUPS) { xr = 0; ++xuse; }
      }
    } else {
      // tile mode (256-token chunks: fewer tiles than 2 stages fit): one barrier per tile
      for (int it = 0; it < nunits; ++it) {
        if (xuse > 0) mbar_wait(&bars->xempty[xs], (xuse - 1u) & 1u, ZS_BACKOFF_CTRL);
        if (elect_one()) {
          mbar_arrive_expect_tx(&bars->xfull[xs], xbytes);
          tma_load_2d(xslots + (size_t)xs * p.aslot_bytes, &xmap, (int32_t)(k * 64), p.m0, &bars->xfull[xs], pol);
        }
        __syncwarp();
        if (++k == nbc) k = 0;
        if (++xs == S_x) { xs = 0; ++xuse; }
      }
    }
  } else if (warp == kWarpMma) {
    // ================================================================ MMA issuer
    // Stage-batched (4 units per iteration): this single warp shares its SMSP with six busy
    // decoder warps and is issued round-robin with them, so every instruction of its loop
    // costs ~7 cycles; a per-unit loop of waits / fences / commits took ~1000 cycles per
    // unit.  Readiness is a plain smem counter per A slot (decoded lane quarters); one
    // commit per stage frees the stage's TMEM A slots and X tiles.
    const uint32_t idesc = umma_idesc_bf16(128, p.n_umma);
    const uint32_t xbase = smem_u32(xslots);
    const uint32_t SAS = S_a / kUPS;
    const uint32_t nacc = p.n_acc;
    uint32_t kc = kc0;
    int seg = -1;
    // Accumulator hand-off to the epilogue on hardware named barriers 2/3 (sleeping warps
    // cost no issue slots; a polled mbarrier cost ~17% of all issued instructions).
    int sig = 0;                                                // segments signalled
    // segments < seg are fully issued: wake the epilogue for those whose accumulator is done
    auto try_signal = [&]() {
      while (sig < seg && mbar_test_wait(&bars->accfull[abuf(sig)], apar(sig))) {
        named_bar_arrive(2 + (sig & 1), 160);
        ++sig;
      }
    };
    uint32_t xs = 0, xph = 0;                     // X slot (stage mode: stage slot) / parity of its fill
    uint32_t as_ = 0, aph = 0;                    // A stage ring slot / parity of its afull phase
    uint32_t ta = tmem_a;                         // A slot column of the stage
    const uint32_t ta_end = tmem_a + 32u * S_a;
    const uint32_t SXS = S_x / kUPS;
    for (int st = 0; st < nstages; ++st) {
      const int i0 = st * kUPS, nu = min(kUPS, nunits - i0);
      // X tile of unit j of the stage: slot / fill parity (tile mode), or the stage's slot
      uint32_t xsl[kUPS], xpl[kUPS];
      if (xstage) {
#pragma unroll
        for (int j = 0; j < kUPS; ++j) { xsl[j] = xs * kUPS + (uint32_t)j; xpl[j] = xph; }
        mbar_wait(&bars->xfull[xs], xph, ZS_BACKOFF_CTRL);
      } else {
#pragma unroll
        for (int j = 0; j < kUPS; ++j) {
          xsl[j] = xs;
          xpl[j] = xph;
          if (j < nu && ++xs == S_x) { xs = 0; xph ^= 1u; }
        }
      }
      try_signal();
      mbar_wait(&bars->afull[as_], aph, ZS_BACKOFF_CTRL);   // all 4 x 4 unit-quarters of the stage decoded
      tc_fence_after();
      if (nu == kUPS && i0 != 0 && i0 + kUPS < nunits && kc != 0 && kc + kUPS < nbc) {
        // fast path: a full stage strictly inside one accumulation segment -> 16 MMAs
        const uint32_t d = tmem_base + abuf(seg) * dcols;
        if (xstage) {
          // the stage's 4 tiles are contiguous: one descriptor base, 16 back-to-back MMAs
          const uint64_t bdesc = umma_desc_sw128(xbase + xsl[0] * p.aslot_bytes);
          const uint32_t bstep = p.aslot_bytes >> 4;   // descriptor address units per X tile
          if (elect_one()) {
            if (!(p.dbg & 4)) {
#pragma unroll
              for (int i = 0; i < kUPS; ++i) {
                const uint64_t bd = bdesc + (uint64_t)(bstep * (uint32_t)i);
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_bf16_ts(d, ta + 32u * i + 8u * k, bd + 2 * k, idesc, 1u);
              }
            }
            umma_commit(&bars->afree[as_]);
            umma_commit(&bars->xempty[xs]);
          }
          __syncwarp();
        } else {
          // each unit's tile is awaited right before its MMAs and released right after them
#pragma unroll
          for (int i = 0; i < kUPS; ++i) {
            mbar_wait(&bars->xfull[xsl[i]], xpl[i], ZS_BACKOFF_CTRL);
            tc_fence_after();
            if (elect_one()) {
              if (!(p.dbg & 4)) {
                const uint64_t bd = umma_desc_sw128(xbase + xsl[i] * p.aslot_bytes);
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_bf16_ts(d, ta + 32u * i + 8u * k, bd + 2 * k, idesc, 1u);
              }
              umma_commit(&bars->xempty[xsl[i]]);
            }
            __syncwarp();
          }
          if (elect_one()) umma_commit(&bars->afree[as_]);
          __syncwarp();
        }
        ta += 32u * kUPS; if (ta == ta_end) ta = tmem_a;
        kc += kUPS;
      } else {
        for (int j = 0; j < nu; ++j) {
          const int it = i0 + j;
          const bool first = (it == 0) || (kc == 0);
          const bool last = (it == nunits - 1) || (kc + 1 == nbc);
          if (first) {
            ++seg;
            // the epilogue must have been woken for segment seg - n_acc (the previous user of
            // this accumulator buffer) before the buffer is reused
            while (sig + (int)nacc <= seg) {
              mbar_wait(&bars->accfull[abuf(sig)], apar(sig));
              named_bar_arrive(2 + (sig & 1), 160);
              ++sig;
            }
            mbar_wait(&bars->accempty[abuf(seg)], apar(seg) ^ 1u);
            tc_fence_after();
          }
          const uint32_t d = tmem_base + abuf(seg) * dcols;
          const uint64_t bdesc = umma_desc_sw128(xbase + xsl[j] * p.aslot_bytes);
          if (!xstage) {
            mbar_wait(&bars->xfull[xsl[j]], xpl[j], ZS_BACKOFF_CTRL);
            tc_fence_after();
          }
          if (elect_one()) {
            if (!(p.dbg & 4)) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                umma_bf16_ts(d, ta + 8u * k, bdesc + 2 * k, idesc, (first && k == 0) ? 0u : 1u);
            }
            trace_ev(p.trace, it, 6);
            if (last) umma_commit(&bars->accfull[abuf(seg)]);
            if (!xstage) umma_commit(&bars->xempty[xsl[j]]);
            if (j == nu - 1) {
              umma_commit(&bars->afree[as_]);
              if (xstage) umma_commit(&bars->xempty[xs]);
            }
          }
          __syncwarp();
          ta += 32u; if (ta == ta_end) ta = tmem_a;
          if (++kc == nbc) kc = 0;
        }
        // a partial last stage leaves its remaining A slots unused: skip them
        if (nu < kUPS) {
          ta += 32u * (uint32_t)(kUPS - nu); if (ta >= ta_end) ta -= ta_end - tmem_a;
        }
      }
      if (xstage && ++xs == SXS) { xs = 0; xph ^= 1u; }
      if (++as_ == SAS) { as_ = 0; aph ^= 1u; }
    }
    // the last segment(s): wait for their accumulators, then wake the epilogue
    while (sig <= seg) {
      mbar_wait(&bars->accfull[abuf(sig)], apar(sig));
      named_bar_arrive(2 + (sig & 1), 160);
      ++sig;
    }
  } else if (warp < kWarpEpi0) {
    // ================================================================ decoders
    // Static assignment: decoder warp jd (0..D-1) of TMEM lane quarter q decodes quarter q
    // of the CTA's units jd, jd + D, jd + 2D, ... in order.  The D warps of a quarter issue at
    // the same rate on one SMSP (no tickets), and a warp that visits its stages in order cannot
    // see a stale ring phase (its previous unit's stage was filled after the slot's older fill).
    //
    // Lane -> weight row: quarter q = half hh = q & 1 of BlockTile row bt = q >> 1; lane t holds
    // row 32 hh + t of that BlockTile, so the warp's 32 FragTiles (TCT rows 2hh, 2hh + 1) are
    // contiguous in canonical order and its scan needs only the first half's total.
    const int q = warp & 3;                       // TMEM lane quarter (== warp % 4)
    const int jd = (warp - kWarpDec0) >> 2;       // decoder index inside the quarter
    const int bt = q >> 1, hh = q & 1;
    const uint32_t tq = tmem_a + ((uint32_t)(32 * q) << 16);
    const int fo = 32 * hh + lane;                // scan lane's FragTile
    uint8_t* rpt = rptab + (warp - kWarpDec0) * kRpWarp;
    // Row passes (16x32bx2 TMEM stores): pass p covers rows 32 hh + 16 p + (lane & 15) of the
    // BlockTile; lanes 0..15 decode FragTile columns 0..3 of those rows and lanes 16..31
    // columns 4..7 of the SAME rows, so at every step the two half-warps read plane bytes
    // 8 FragTiles (64 B) apart -- different banks -- instead of 16 FragTiles (128 B, the
    // same banks) apart.
    const int kh = lane >> 4;                     // column half: FragTile columns 4 kh .. 4 kh + 3
    const int rl = lane & 15;
    // row table: FragTile o (local 0..31) at o*16 + (o >> 3)*16 bytes, row r8 at + 2*r8 (the
    // pad puts FragTiles o and o + 8 -- the two half-warps -- on different banks)
    const uint32_t rp_wr = (uint32_t)lane * 16u + ((uint32_t)lane >> 3) * 16u;
    const uint32_t SAS = S_a / kUPS;
    DecConst dk;
    load_dec_const(dk, p.eb7x2);
    const uint32_t slut_b = smem_u32(slut);
    const uint32_t sbase = smem_u32(smem);
    if (tid < 256) {
      const uint4 e = __ldg(&c_lut[tid]);
      slut[tid] = e;
    }
    named_bar_sync(4, 32 * 4 * kDecPerQuarter);   // the decoder warps: selector table in smem
    // Per-unit stage pointers (smem offsets) of unit u; waits for the unit's stage data.
    struct UnitPtr {
      uint32_t p1;     // BlockTile row's plane B1 slice of this unit (B2, B3 at + kUPS*512, 2*kUPS*512)
      uint32_t hb;     // H segment base (16-B aligned)
      uint32_t lb;     // L segment base
      uint32_t slot;   // compressed ring slot
    };
    auto unit_ptr = [&](int u) {
      const uint32_t st = (uint32_t)u / kUPS, j = (uint32_t)u % kUPS;
      const uint32_t stc = fastdiv(st, S_c, p.cdiv_magic);
      const uint32_t slot = st - stc * S_c;
      const uint8_t* cs = cslots + (size_t)slot * p.cslot_bytes;
      const uint32_t* meta = reinterpret_cast<const uint32_t*>(cs);
      mbar_wait(&bars->full_c[slot], stc & 1u, ZS_BACKOFF_DEC);
      if (lane == 0) trace_ev(p.trace, u, 7 + q);
      // an absent BlockTile row b (odd row count) is aliased to row a: its rows decode valid
      // bytes into TMEM lanes whose outputs (rows >= N) the epilogue never stores
      const int btx = (bt == 1 && meta[20 + j] != 0u) ? 1 : 0;
      const uint4 mt = *reinterpret_cast<const uint4*>(meta + 4 * j);  // {H a, H b, L a, L b}
      const uint8_t* Hr = cs + kStageMeta + kStagePlanes;
      UnitPtr r;
      r.p1 = (uint32_t)(cs + kStageMeta + btx * kBtPlaneStride + j * 512 - smem);
      r.hb = (uint32_t)(Hr + btx * capH + (btx ? mt.y : mt.x) - smem);
      r.lb = (uint32_t)(Hr + 2 * capH + btx * capL + (btx ? mt.w : mt.z) - smem);
      r.slot = slot;
      return r;
    };
    // Scan of unit u: lane = FragTile 32 hh + lane (canonical order); writes the H
    // offset (from the BlockTile's H base) of each of its FragTile's 8 rows into row table buf.
    auto scan_unit = [&](const UnitPtr& up, uint8_t* tab) {
      const uint8_t* P1 = smem + up.p1;
      const uint8_t* P2 = P1 + kUPS * 512;
      const uint8_t* P3 = P2 + kUPS * 512;
      const uint2 s1 = *reinterpret_cast<const uint2*>(P1 + fo * 8);
      const uint2 s2 = *reinterpret_cast<const uint2*>(P2 + fo * 8);
      const uint2 s3 = *reinterpret_cast<const uint2*>(P3 + fo * 8);
      const uint32_t mlo = s1.x | s2.x | s3.x, mhi = s1.y | s2.y | s3.y;
      const uint32_t cnt = __popc(mlo) + __popc(mhi);
      // straight-line (no branch on hh) so that ptxas schedules the scan's loads and popcounts
      // among the row decode it is placed next to: the first-half total is computed by every
      // warp and weighted by hh (measured ~1% over the branchy form, r02 A/B)
      uint32_t incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t t;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "shfl.sync.up.b32 %0|p, %1, %2, 0, -1;\n\t"
            "@!p mov.b32 %0, 0;\n\t}"
            : "=r"(t)
            : "r"(incl), "r"(d));
        incl += t;
      }
      uint32_t excl = incl - cnt;
      {
        const uint2 t1 = *reinterpret_cast<const uint2*>(P1 + lane * 8);
        const uint2 t2 = *reinterpret_cast<const uint2*>(P2 + lane * 8);
        const uint2 t3 = *reinterpret_cast<const uint2*>(P3 + lane * 8);
        uint32_t first;
        asm volatile("redux.sync.add.u32 %0, %1, -1;"
                     : "=r"(first)
                     : "r"(__popc(t1.x | t2.x | t3.x) + __popc(t1.y | t2.y | t3.y)));
        excl += first & (0u - (uint32_t)hh);
      }
      const uint32_t bl = bytepop(mlo), bh = bytepop(mhi);
      const uint32_t rp_lo = bl * 0x01010100u;
      const uint32_t rp_hi = bh * 0x01010100u + ((bl * 0x01010101u) >> 24) * 0x01010101u;
      const uint32_t ex2 = excl * 0x10001u;
      *reinterpret_cast<uint4*>(tab + rp_wr) =
          make_uint4(prmt(rp_lo, 0u, 0x4140u) + ex2, prmt(rp_lo, 0u, 0x4342u) + ex2, prmt(rp_hi, 0u, 0x4140u) + ex2,
                     prmt(rp_hi, 0u, 0x4342u) + ex2);
    };
    // Software pipeline: the scan of the warp's NEXT unit is issued with the second row pass of
    // the current one (same basic block), so its latency chain (loads -> popcounts -> 5
    // dependent shuffles -> table) overlaps row-decode work of the same warp instead of idling
    // all four phase-aligned decoder warps of the SMSP at every stage boundary.
    UnitPtr cur{};
    if (jd < nunits) {
      cur = unit_ptr(jd);
      scan_unit(cur, rpt);
    }
    uint32_t tb = 0;                              // row table buffer of the current unit
    for (int u = jd; u < nunits; u += kDecPerQuarter, tb ^= 1u) {
      const int un = u + kDecPerQuarter;
      const uint32_t st = (uint32_t)u / kUPS, j = (uint32_t)u % kUPS;
      const uint32_t ag = fastdiv(st, SAS, p.adiv_magic);  // use count of the A stage
      const uint32_t astg = st - ag * SAS;                 // TMEM A stage of this unit
      const uint32_t a = astg * kUPS + j;                  // TMEM A slot of this unit
      const uint8_t* tab = rpt + tb * kRpBuf;
      __syncwarp();                                        // this unit's row table is written
      // the slot is free once the MMAs of stage st - SAS have completed (their commit)
      if (ag > 0) mbar_wait(&bars->afree[astg], (ag - 1u) & 1u);
      tc_fence_after();
      if (lane == 0) trace_ev(p.trace, u, 11 + q);
      UnitPtr nxt = cur;
      const uint32_t taddr0 = tq + 32u * a;
      const uint32_t hb = cur.hb;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        // next unit: wait for its data here; its scan is issued with this pass's rows (one
        // basic block).  Past the last unit the current one is re-scanned into the unused buffer.
        if (pass == 1) nxt = unit_ptr(un < nunits ? un : u);
        if (p.dbg & 1) {   // timing experiment: no row decode (the scan and the pipeline stay)
          if (pass == 1) scan_unit(nxt, rpt + (tb ^ 1u) * kRpBuf);
          continue;
        }
        const int lr = 32 * hh + 16 * pass + rl;                    // row inside the BlockTile
        const int fr = lr >> 3, r8 = lr & 7;
        // FragTile of (row, column f): (lr >> 4) * 16 + cf(f) + (fr & 1), cf(f) = (f>>1)*4 + (f&1)*2;
        // this lane's columns f = 4 kh + qq give cf = 8 kh + cf(qq)
        const uint32_t ob = (uint32_t)((lr >> 4) * 16 + (fr & 1) + 8 * kh);   // FragTile for qq = 0
        const uint32_t ol = ob - 32u * hh;                                    // local FragTile
        const uint8_t* pb = smem + cur.p1 + ob * 8u + (uint32_t)r8;           // plane byte, qq = 0
        const uint8_t* rb = tab + ol * 16u + (ol >> 3) * 16u + 2u * (uint32_t)r8;
        // fallback values of the row start at element 8*(o*8 + r8) - (its H offset) of the L segment
        const uint32_t la0 = cur.lb + 2u * hb + 16u * (ob * 8u + (uint32_t)r8);
        uint4 v[4];
        uint32_t rare = 0;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const uint32_t cf = (uint32_t)((qq >> 1) * 4 + (qq & 1) * 2);
          // table offset of FragTile ol + cf: cf in {0,2,4,6} never crosses an 8-FragTile pad
          const uint32_t hs_abs = hb + *reinterpret_cast<const uint16_t*>(rb + cf * 16u);
          const uint32_t b1 = pb[cf * 8u];
          const uint32_t b2 = pb[cf * 8u + kUPS * 512];
          const uint32_t b3 = pb[cf * 8u + 2 * kUPS * 512];
          const uint32_t m = b1 | b2 | b3;
          const uint4 ent = ld_shared_v4(slut_b + m * 16u);
          rare |= ent.x;
          const uint32_t haddr = sbase + (hs_abs & ~3u), hsh8 = hs_abs * 8u, laddr = sbase + la0 + 128u * cf - 2u * hs_abs;
          v[qq] = decode_row_v3(b1, b2, b3, ent, haddr, hsh8, laddr, dk);
        }
        if (pass == 1) scan_unit(nxt, rpt + (tb ^ 1u) * kRpBuf);   // (the other table buffer)
        if (p.dbg & 2) {
          uint32_t x = 0;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) x ^= v[qq].x ^ v[qq].y ^ v[qq].z ^ v[qq].w;
          if (x == 0x9E3779B9u) p.counters[0] = x;   // keeps the decode live
        } else {
          // TMEM lanes 32q + 16 pass + (0..15); half-warp kh writes columns 16 kh .. 16 kh + 15
          tmem_st16x2(taddr0 + ((uint32_t)(16 * pass) << 16), v[0], v[1], v[2], v[3]);
        }
        if (__any_sync(0xFFFFFFFFu, rare & 0x80u)) {
          // rare: a row of this pass has >= 3 fallbacks (rank >= 2); warp-uniform branch.  The
          // fast-path rows are already in TMEM (storing them before this check lets ptxas
          // decode straight into the store's registers); the patched rows are stored again
          // once the first stores have completed.
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const uint32_t cf = (uint32_t)((qq >> 1) * 4 + (qq & 1) * 2);
            const uint32_t hs_abs = hb + *reinterpret_cast<const uint16_t*>(rb + cf * 16u);
            const uint32_t m = pb[cf * 8u] | pb[cf * 8u + kUPS * 512] | pb[cf * 8u + 2 * kUPS * 512];
            if (slut[m].x & 0x80u)
              patch_rank2(m, reinterpret_cast<const uint16_t*>(smem + la0 + 128u * cf - 2u * hs_abs), v[qq].x,
                          v[qq].y, v[qq].z, v[qq].w);
          }
          tmem_wait_st();
          tmem_st16x2(taddr0 + ((uint32_t)(16 * pass) << 16), v[0], v[1], v[2], v[3]);
        }
      }
      // publish the unit-quarter (release: the MMA warp's acquire on afull orders its MMAs
      // after these TMEM stores)
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->afull[astg]);
      if (lane == 0) trace_ev(p.trace, u, 2 + q);
      if (lane == 0) mbar_arrive(&bars->empty_c[cur.slot]);   // all lanes are done with the stage
      cur = nxt;
    }
    // A partial last stage still needs its 16 afull arrivals: this warp's units past the end
    // that fall in that stage arrive without decoding (after the slot's previous use is
    // retired, so the arrival lands in the right phase).
    for (int u = jd + ((nunits - jd + kDecPerQuarter - 1) / kDecPerQuarter) * kDecPerQuarter;
         u < nstages * kUPS; u += kDecPerQuarter) {
      const uint32_t st = (uint32_t)u / kUPS;
      const uint32_t ag = fastdiv(st, SAS, p.adiv_magic), astg = st - ag * SAS;
      if (ag > 0) mbar_wait(&bars->afree[astg], (ag - 1u) & 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->afull[astg]);
    }
  } else if (warp < kWarpEpi0 + 4) {
    // ================================================================ epilogue (warps 4..7)
    const int et = tid - 32 * kWarpEpi0;  // 0..127 = TMEM lane = row inside the band
    const int eq = warp & 3;              // TMEM lane quarter
    const uint32_t b_last = (u1 - 1) / nbc;
    int seg = 0;
    for (uint32_t band = band0; band <= b_last; ++band, ++seg) {
      const uint32_t s0 = max(u0, band * nbc), s1 = min(u1, (band + 1) * nbc);
      const bool full = (s1 - s0) == nbc;
      // sleep on the named barrier the MMA warp arrives at once the segment's MMAs are
      // complete; the mbarrier wait after it then passes at once (and orders the TMEM reads)
      named_bar_sync(2 + (seg & 1), 160);
      if (seg == 0) grid_dependency_wait();   // Y / workspace / counters: previous kernel done (PDL)
      mbar_wait(&bars->accfull[abuf(seg)], apar(seg));
      tc_fence_after();
      const int64_t n = (int64_t)band * 128 + et;
      const bool nvalid = n < p.N;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * eq) << 16) + abuf(seg) * dcols;
      for (uint32_t cb = 0; cb < p.n_umma; cb += 16) {
        uint32_t v[16];
        tmem_ld16(taddr + cb, v);
        if (nvalid) {
          if (full) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int m = (int)cb + j;
              if (m < p.mc)
                p.y[(int64_t)(p.m0 + m) * p.ldy + n] = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(v[j])));
            }
          } else {
            // partial band: the thread's 16 token sums go to its workspace row [n][cb, cb+16)
            // as four 16-B vector reductions (columns >= mc hold zeros: X is zero-filled)
            float* wrow = p.ws + (int64_t)n * p.ldws + cb;
#pragma unroll
            for (int j = 0; j < 16; j += 4) red_add_v4(wrow + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->accempty[abuf(seg)]);
      if (kPeer && full && nvalid && p.npeer > 0)
        copy_to_peers(p.ypeer, p.npeer, p.y, p.ldy, (int64_t)p.m0 * p.ldy + n, p.mc);
      if (!full) {
        __threadfence();
        named_bar_sync(1, 128);
        if (et == 0) {
          const uint32_t old = atomicAdd(&p.counters[band], s1 - s0);
          bars->last_flag = (old + (s1 - s0) == nbc) ? 1u : 0u;
        }
        named_bar_sync(1, 128);
        if (bars->last_flag) {
          __threadfence();
          if (nvalid) {
            // the thread's workspace row: 16-B loads, 4 in flight per batch of 16 tokens, then
            // zeroed again with 16-B stores (self-cleaning)
            float4* wrow = reinterpret_cast<float4*>(p.ws + (int64_t)n * p.ldws);
            for (int m0 = 0; m0 < (int)p.n_umma; m0 += 16) {
              float4 f[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) f[j] = __ldcg(wrow + m0 / 4 + j);
              const float* g = reinterpret_cast<const float*>(f);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (m0 + j < p.mc)
                  p.y[(int64_t)(p.m0 + m0 + j) * p.ldy + n] = __bfloat16_as_ushort(__float2bfloat16_rn(g[j]));
#pragma unroll
              for (int j = 0; j < 4; ++j) __stcg(wrow + m0 / 4 + j, make_float4(0.f, 0.f, 0.f, 0.f));
            }
          }
          if (kPeer && nvalid && p.npeer > 0)
            copy_to_peers(p.ypeer, p.npeer, p.y, p.ldy, (int64_t)p.m0 * p.ldy + n, p.mc);
          if (et == 0) p.counters[band] = 0u;
        }
        named_bar_sync(1, 128);
      }
    }
    if (kPeer && p.done) {
      // fused exchange (f2): this CTA's Y stores (local and peer) happen before its
      // arrival; the CTA that arrives last then releases the flags, so a peer that
      // acquires flag == epoch sees every tile of this rank's slice
      named_bar_sync(1, 128);   // the 128 epilogue threads' stores happen before et 0's release
      if (et < 32) signal_peers(p.done, p.flag, p.nflag, p.epoch, lane);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpAlloc) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

int g_pdl = 1;   // programmatic dependent launch on (zs_debug_set_pdl)

cudaError_t launch_gemm(const GemmParams& p, const CUtensorMap& xmap, int grid, size_t smem, cudaStream_t stream) {
  static std::atomic<uint64_t> attr_done{0};
  cudaError_t e = once_per_device(attr_done, [] {
    cudaError_t r = cudaFuncSetAttribute(zipgemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(zipgemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    return r;
  });
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (p.npeer > 0 || p.nflag > 0 || (p.dbg & 0x100u)) return cudaLaunchKernelEx(&cfg, zipgemm_kernel<true>, p, xmap);
  return cudaLaunchKernelEx(&cfg, zipgemm_kernel<false>, p, xmap);
}

size_t gemm_smem_bytes(const GemmParams& p) {
  return 1024 /*align slack*/ + 1024 + kRpTabBytes + kLutBytes + (size_t)p.n_xslots * p.aslot_bytes +
         (size_t)p.n_cslots * p.cslot_bytes;
}

int gemm_threads() { return kGemmThreads; }
int gemm_max_xslots() { return kMaxXSlots; }
int gemm_max_cslots() { return kMaxCSlots; }
int gemm_max_aslots() { return kMaxASlots; }
uint32_t gemm_stage_fixed_bytes() { return kStageMeta + kStagePlanes; }
int gemm_units_per_stage() { return kUPS; }
int gemm_max_chunk() { return 256; }
uint32_t gemm_fixed_smem() { return 1024 + 1024 + kRpTabBytes + kLutBytes; }

}  // namespace zs
