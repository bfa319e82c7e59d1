// zs_device.cuh -- sm_100a device primitives shared by zs_decompress and zs_gemm.
//
// PTX wrappers (mbarrier, cp.async.bulk / TMA, tcgen05) and the branch-free TCA-TBE row
// decoder.  Citations: P:<line> = PAPER.md, S:<line> = SPEC.md.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace zs {

// one lane of the (converged) warp returns true
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "elect.sync _|P1, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "+r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------------ smem / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// try_wait without a suspend hint: the hardware blocks for a short, system-defined time
// and returns as soon as the phase completes -- used on the critical path.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// non-blocking probe
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Watchdog: a wait that spins ~2^28 times (seconds) reports the barrier and traps, so a
// pipeline bug surfaces as a CUDA error instead of a hung GPU.
static __device__ __noinline__ void zs_watchdog_fire(const void* what, uint32_t parity) {
  printf("zs watchdog: block %d thread %d stuck on smem %#x parity %u\n", blockIdx.x, threadIdx.x,
         (unsigned)__cvta_generic_to_shared(what), parity);
  __trap();
}

__device__ __forceinline__ uint64_t globaltimer_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Wait for the phase with the given parity.  After one probe the waiting warp suspends inside
// mbarrier.try_wait (suspend-time hint ZS_WAIT_SUSPEND ns; it resumes as soon as the phase
// completes): a waiting warp shares its SMSP with decoder warps, and a nanosleep polling loop
// (ZS_WAIT_SUSPEND=0) issued 18% of all the fused kernel's instructions (ncu r02b: 726 K
// probe iterations per launch).  The watchdog is time based (every 256 probes): > 10 s traps.
static __device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity, uint32_t backoff_ns);

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, uint32_t backoff_ns = 64) {
  if (!mbar_try_wait(bar, parity)) mbar_wait_slow(bar, parity, backoff_ns);
}

__device__ __forceinline__ bool mbar_try_wait_suspend(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

#ifndef ZS_WAIT_SUSPEND
#define ZS_WAIT_SUSPEND 1000   // > 0: slow waits suspend in mbarrier.try_wait (hint, ns); 0: nanosleep polling
#endif
static __device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity, uint32_t backoff_ns) {
  uint64_t t0 = 0;
#if ZS_WAIT_SUSPEND == 2
  // hybrid: long back-offs (the control warps, which mostly wait for the decoders) sleep between
  // probes; short ones (decoders) suspend in try_wait
  for (uint32_t n = 1; !(backoff_ns >= 128u ? mbar_try_wait(bar, parity) : mbar_try_wait_suspend(bar, parity, 1000u));
       ++n) {
    if (backoff_ns >= 128u) __nanosleep(backoff_ns);
#elif ZS_WAIT_SUSPEND
  (void)backoff_ns;
  for (uint32_t n = 1; !mbar_try_wait_suspend(bar, parity, ZS_WAIT_SUSPEND); ++n) {
#else
  for (uint32_t n = 1; !mbar_try_wait(bar, parity); ++n) {
    __nanosleep(backoff_ns);
#endif
    if ((n & 255u) == 0u) {
      const uint64_t t = globaltimer_now();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 10000000000ull) zs_watchdog_fire(bar, parity);
    }
  }
}

__device__ __forceinline__ uint32_t ld_acquire_shared(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// system-scope flag hand-off between GPUs (peer memory over NVLink, or CUDA-IPC-mapped
// memory of another process): release store / acquire load of a global u32
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Completion signal of the fused exchange, called by one full warp of every CTA after a
// CTA barrier that follows all of the CTA's output stores.  Lane 0 counts the CTA in with
// a GPU-scope release (cumulative over the CTA's stores; every CTA is on this GPU, so the
// counter needs no system scope); the warp of the CTA that arrives last (its acquire
// sees every CTA's release) resets the counter and stores `epoch` to the nflag flags,
// lane i -> flag[i], as ONE warp-wide system-scope release: causality order is
// transitive, so a peer that acquires a flag sees every CTA's stores (one system fence
// per launch instead of one per CTA and flag).
__device__ __forceinline__ void signal_peers(uint32_t* done, uint32_t* const* flag, int nflag, uint32_t epoch,
                                             int lane) {
  uint32_t old = 0;
  if (lane == 0) old = atom_add_acq_rel_gpu(done, 1u);
  old = __shfl_sync(0xFFFFFFFFu, old, 0);
  if (old != gridDim.x - 1) return;
  if (lane == 0) *done = 0u;   // self-cleaning for the next call
  __syncwarp();                // lane 0's acquire happens before the other lanes' releases
  uint32_t* f = nullptr;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i == lane && i < nflag) f = flag[i];
  if (f) st_release_sys(f, epoch);
}

// fire-and-forget fp32 vector reduction into global memory (16-B aligned)
__device__ __forceinline__ void red_add_v4(float* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(__uint_as_float(a)),
               "f"(__uint_as_float(b)), "f"(__uint_as_float(c)), "f"(__uint_as_float(d))
               : "memory");
}


// ------------------------------------------------------------------ bulk copies (TMA)
// 1-D bulk copy global -> shared, completion counted in bytes on `bar` (UBLKCP in SASS).
// Requires 16-byte aligned addresses and a size that is a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 2-D tiled TMA load (UTMALDG): box of the tensor map at coordinates (c0 inner, c1 outer).
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int32_t c0, int32_t c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// ------------------------------------------------------------------ tcgen05 / TMEM
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]^T (A operand resident in tensor memory, K-major).
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 16 TMEM lanes (base lane + t, t = lane & 15), two column blocks: threads 0..15 write columns
// [c, c+16) of their lane, threads 16..31 columns [c+16, c+32) of the SAME lanes
__device__ __forceinline__ void tmem_st16x2(uint32_t taddr, uint4 a, uint4 b, uint4 c, uint4 d) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], 16, {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::
          "r"(taddr),
      "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "r"(c.x), "r"(c.y), "r"(c.z),
      "r"(c.w), "r"(d.x), "r"(d.y), "r"(d.z), "r"(d.w)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread (thread i <-> TMEM lane base+i)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B canonical layout (8-row x 128-B
// atoms stacked every 1024 B).  start must be inside a 1024-B aligned atom column.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);  // start address, 16-B units
  d |= (uint64_t)1 << 16;                      // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;            // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                      // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                      // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, shape M x N.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4)            // D format: f32
         | (1u << 7)          // A format: bf16
         | (1u << 10)         // B format: bf16
         | ((N >> 3) << 17)   // N >> 3
         | ((M >> 4) << 24);  // M >> 4
}

// ------------------------------------------------------------------ TCA-TBE row decoder
//
// The decode unit on sm_100a is one FragTile ROW: 8 consecutive K-elements of one weight
// row = one byte of each bit-plane = one 16-byte chunk of the UMMA SW128 row.  It computes
// exactly Alg. 2 for those 8 positions, amortised per row instead of per
// element:
//   M       = B1 | B2 | B3 restricted to the row's byte                   (Alg. 2 l.2)
//   idx_H   = hs + popc(m & ((1<<i)-1))  -> PRMT byte selectors from a 256-entry table
//   idx_L   = ls + i - popc(...)         -> PRMT selectors for the fallback merge
//   e       = e_base + c, c = B3[p]B2[p]B1[p]                             (Alg. 2 l.15-16)
//   word    = MakeBF16(sign, e, mantissa) or L[idx_L]                      (l.17 / l.21)
// Both arms are computed for every element and merged by a byte permute: there is no
// data-dependent branch on the common path.  Rows with >= 3 fallback
// elements (rank >= 2) take a short patch loop (~0.05% of rows at r = 0.98).
//
// Selector table entry lut[m] (csrc/zs_lut.h, generated by scripts/gen_lut.py), m = the
// row's spatial-indicator byte; for output word j (elements 2j, 2j+1):
//   bits  0..15  PRMT selector that pulls the H byte of element 2j into byte 0 and its
//                sign-replicated copy into byte 1, likewise element 2j+1 into bytes 2, 3
//   bits 16..31  PRMT selector over {Lpair, assembled word}: fallback elements of rank 0/1
//                take L bytes (0,1)/(2,3), in-window elements keep their assembled half.
// Bit 7 of word 0 (a sign-replicate bit whose two modes give the same result) flags rows
// with >= 3 fallbacks, which take the rare patch path.

// Exponent assembly by multiply-spread (FMA pipe): (b & 0xF) * K, K = 1 + 2^6 + 2^15 + 2^21,
// drops plane-byte bits 0..3 on the LSBs of bytes 0, 2, 1, 3 with no overlapping partial
// products (no carries), so WA = [c0, c2, c1, c3] and WB = [c4<<4, c6<<4, c5<<4, c7<<4]
// bytewise, and E0 = WA*128 + EB, E1 = umulhi(WA, 2^31) + EB, E2 = WB*8 + EB,
// E3 = umulhi(WB, 2^27) + EB put (e_base + c) of elements (2j, 2j+1) on bits 7..14 / 23..30
// of word j exactly; the garbage they also produce stays outside those bits (checked
// exhaustively by the GPU parity tests on all 65,536 patterns).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {  // all 4 selector bits
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// (a & mask) | (b & ~mask) in one LOP3
template <uint32_t kMask>
__device__ __forceinline__ uint32_t bitsel(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "n"(kMask));
  return d;
}

// Multipliers of the row decoder, read from constant memory so that ptxas keeps the
// multiply-adds on the FMA pipe (with immediates it strength-reduces them to LEA / SHF,
// which issue on the ALU pipe -- the decoder's bottleneck).
#define ZS_KSPREAD (1u | (1u << 6) | (1u << 15) | (1u << 21))
__constant__ uint32_t c_mul[8] = {1u << 28, 128u, 1u << 31, 8u, 1u << 27, 1u << 16, 0u, 0u};
enum : int { kM28 = 0, kM7 = 1, kM31 = 2, kM3 = 3, kM27 = 4, kM16 = 5 };

__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {  // a*b + c (FMA pipe)
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint32_t mul_hi(uint32_t a, uint32_t b) {  // hi(a*b) (FMA pipe, quarter rate)
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {  // hi(a*b) + c (FMA pipe)
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Row decoder on absolute smem pointers (the GEMM precomputes them):
//   H32 : 4-byte aligned word containing the row's first H byte, hsh8 = 8 * (that byte's
//         offset) -- only its low 5 bits are used (funnel shift wraps mod 32)
//   Lrow: the row's first fallback value
// Rows with >= 3 fallbacks (rank >= 2) are flagged by bit 7 of ent.x (the sign-replicate
// bit of a selector nibble whose two modes give the same result) and patched on a rare path.
// Fallback words of rank >= 2 in a row (the fast path merges ranks 0 and 1): one iteration
// per such position -- the positions are the zero bits of m after its two lowest ones.
__device__ __forceinline__ void patch_rank2(uint32_t m, const uint16_t* __restrict__ Lrow, uint32_t& o0,
                                            uint32_t& o1, uint32_t& o2, uint32_t& o3) {
  uint32_t z = ~m & 0xFFu;
  z &= z - 1u;
  z &= z - 1u;
  while (z) {
    const uint32_t i = __ffs(z) - 1u;
    z &= z - 1u;
    const uint32_t v = Lrow[i - __popc(m & ((1u << i) - 1u))];
    const uint32_t sh = 16u * (i & 1u), keep = 0xFFFF0000u >> sh, ins = v << sh, j = i >> 1;
    // named words, not an indexed array (an indexed array is demoted to local memory)
    o0 = j == 0u ? ((o0 & keep) | ins) : o0;
    o1 = j == 1u ? ((o1 & keep) | ins) : o1;
    o2 = j == 2u ? ((o2 & keep) | ins) : o2;
    o3 = j == 3u ? ((o3 & keep) | ins) : o3;
  }
}

// ------------------------------------------------------------------ row decoder, v3 (GEMM)
// decode_row_abs with every operand in registers: smem addresses as 32-bit shared-window
// addresses (ld.shared with immediate offsets), the power-of-two multipliers of the
// multiply-spread held in registers (loaded once per warp from c_mul, so ptxas cannot
// strength-reduce the FMA-pipe multiplies into ALU shifts), the fallback-merge selector
// taken from the high half of the table word with one IMAD.HI.
struct DecConst {
  uint32_t k28, k7, k31, k3, k27, k16, eb7x2;
};

__device__ __forceinline__ void load_dec_const(DecConst& d, uint32_t eb7x2) {
  d.k28 = c_mul[kM28];
  d.k7 = c_mul[kM7];
  d.k31 = c_mul[kM31];
  d.k3 = c_mul[kM3];
  d.k27 = c_mul[kM27];
  d.k16 = c_mul[kM16];
  d.eb7x2 = eb7x2;
}

__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t ld_shared_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

// Spread of one plane byte b (bit i = element i) into WA / WB positions:
//   lo = (b & 0xF) * K  and  hi = (b & 0xF0) * K = b * K - lo   (K shifted by the plane's weight)
// one LOP3 + two full-rate IMADs; no IMAD.HI (a quarter-rate instruction on sm_100a:
// 0.24 vs 0.5 warp-instructions / cycle / SMSP, scripts/pipe_probe.cu)
#ifndef ZS_DEC_BAL
// Pipe balance of the row decoder (sm_100a: LOP3 / PRMT / SHF and IMAD issue at 0.5 warp-instr
// per cycle per SMSP, IMAD.HI at 0.24; scripts/pipe_probe.cu).  2: shifts split between the
// FMA pipe (IMAD.HI) and the ALU pipe (SHF) so both pipes carry about the same cycles per row;
// 1: all shifts on the FMA pipe; 0: all shifts on the ALU pipe; 3 (default): as 2 but the odd
// exponent words by LEA.HI (ALU) instead of IMAD.HI (8B GateUp M = 32: 69.2 -> 67.5 us, r02 it4);
// 4: as 3 and the plane spread masks with LOP3; 5: as 4 and every selector shift on SHF.
#define ZS_DEC_BAL 3
#endif
template <int kShift>
__device__ __forceinline__ void spread_plane_k(uint32_t b, const DecConst& d, uint32_t& lo, uint32_t& hi) {
#if ZS_DEC_BAL && ZS_DEC_BAL != 4 && ZS_DEC_BAL != 5
  hi = mul_hi(b, d.k28) * (ZS_KSPREAD << (4 + kShift));   // (b >> 4) on the FMA pipe
  lo = b * (ZS_KSPREAD << kShift) - hi;
#else
  lo = (b & 0xFu) * (ZS_KSPREAD << kShift);
  hi = b * (ZS_KSPREAD << kShift) - lo;
#endif
}

// haddr: shared address of the aligned word holding the row's first H byte; hsh8: 8 x that
// byte's offset (low 5 bits used); laddr: shared address of the row's first fallback value.
__device__ __forceinline__ uint4 decode_row_v3(uint32_t b1, uint32_t b2, uint32_t b3, uint4 ent, uint32_t haddr,
                                               uint32_t hsh8, uint32_t laddr, const DecConst& d) {
  const uint32_t h0 = ld_shared_u32(haddr), h1 = ld_shared_u32(haddr + 4), h2 = ld_shared_u32(haddr + 8);
  const uint32_t hlo = __funnelshift_r(h0, h1, hsh8);
  const uint32_t hhi = __funnelshift_r(h1, h2, hsh8);
#if ZS_DEC_BAL
  const uint32_t lpair = mad_lo(ld_shared_u16(laddr + 2), d.k16, ld_shared_u16(laddr));
#else
  const uint32_t lpair = prmt(ld_shared_u16(laddr), ld_shared_u16(laddr + 2), 0x5410u);
#endif
  uint32_t l1, u1, l2, u2, l3, u3;
  spread_plane_k<0>(b1, d, l1, u1);
  spread_plane_k<1>(b2, d, l2, u2);
  spread_plane_k<2>(b3, d, l3, u3);
  // WA = [c0, c2, c1, c3], WB = [c4<<4, c6<<4, c5<<4, c7<<4] bytewise
  const uint32_t WA = (l1 & 0x01010101u) | (l2 & 0x02020202u) | (l3 & 0x04040404u);
  const uint32_t WB = (u1 & 0x10101010u) | (u2 & 0x20202020u) | (u3 & 0x40404040u);
  // (e_base + c) of elements (2j, 2j+1) on bits 7..14 / 23..30 of word j
#if ZS_DEC_BAL >= 3
  // odd words as (W >> s) + EB: one LEA.HI each on the ALU pipe (no quarter-rate IMAD.HI)
  const uint32_t E[4] = {mad_lo(WA, d.k7, d.eb7x2), (WA >> 1) + d.eb7x2, mad_lo(WB, d.k3, d.eb7x2),
                         (WB >> 5) + d.eb7x2};
#elif ZS_DEC_BAL
  // (IMAD.HI with an addend needs a 64-bit addend register pair: the add goes to IADD3)
  const uint32_t E[4] = {mad_lo(WA, d.k7, d.eb7x2), mul_hi(WA, d.k31) + d.eb7x2, mad_lo(WB, d.k3, d.eb7x2),
                         mul_hi(WB, d.k27) + d.eb7x2};
#else
  const uint32_t E[4] = {mad_lo(WA, d.k7, d.eb7x2), (WA >> 1) + d.eb7x2, mad_lo(WB, d.k3, d.eb7x2),
                         (WB >> 5) + d.eb7x2};
#endif
  const uint32_t sel[4] = {ent.x, ent.y, ent.z, ent.w};
  uint32_t out[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t P = prmt(hlo, hhi, sel[j]);
    const uint32_t w = bitsel<0x807F807Fu>(P, E[j]);
#if ZS_DEC_BAL == 1
    out[j] = prmt(lpair, w, mul_hi(sel[j], d.k16));
#elif ZS_DEC_BAL >= 5
    out[j] = prmt(lpair, w, sel[j] >> 16);
#elif ZS_DEC_BAL >= 2
    out[j] = prmt(lpair, w, j < 2 ? mul_hi(sel[j], d.k16) : (sel[j] >> 16));
#else
    out[j] = prmt(lpair, w, sel[j] >> 16);
#endif
  }
  return make_uint4(out[0], out[1], out[2], out[3]);
}


}  // namespace zs
