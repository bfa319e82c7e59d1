// zs_kernels.h -- host-side launch interface of the sm_100a kernels (internal to libzs.so).
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace zs {

struct DecompParams {
  const uint64_t* b1;
  const uint64_t* b2;
  const uint64_t* b3;
  const uint8_t* h;
  const uint16_t* l;
  const uint64_t* offsets;  // n_blocktiles + 1 pairs
  uint16_t* out;
  int64_t ld_out;
  int64_t rows, cols;
  int64_t nbc;              // BlockTile columns
  int64_t n_blocktiles;
  uint32_t hcap, stage_bytes;
  uint32_t eb7x2;
  int vec_ok;
};

cudaError_t launch_decompress(const DecompParams& p, int grid, int warps, size_t smem, cudaStream_t stream);
size_t decompress_smem_bytes(uint32_t stage_bytes, int warps);
int decompress_max_warps();

constexpr int kMaxPeers = 8;   // ZS_MAX_PEERS

// Run a kernel-attribute setter once per device (the attribute lives in the current
// device's context).  Concurrent first calls may both run f, which is idempotent.
template <typename F>
inline cudaError_t once_per_device(std::atomic<uint64_t>& done, F&& f) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = f();
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

struct GemmParams {
  const uint64_t* b1;
  const uint64_t* b2;
  const uint64_t* b3;
  const uint8_t* h;
  const uint16_t* l;
  const uint64_t* offsets;
  uint16_t* y;
  int64_t ldy;
  float* ws;                // [N][ldws] fp32 split-K partials, row n = weight row (zero between calls)
  int64_t ldws;             // workspace row stride (floats): roundup(min(M, 256), 16) >= n_umma
  uint32_t* counters;       // [nbands] arrival counters (zero between calls)
  int64_t N;                // logical output features
  int64_t nbr, nbc;         // BlockTile grid
  int64_t nbands;           // ceil(nbr / 2): 128-row bands
  int64_t total_units;      // nbands * nbc
  int32_t m0, mc;           // token chunk [m0, m0 + mc)
  uint32_t n_umma;          // mc rounded up to 16
  uint32_t hcap, lcap;      // per-stage H / L capacity of one BlockTile row (4 units)
  uint32_t cslot_bytes;     // compressed ring stage (4 units)
  uint32_t aslot_bytes;     // X (B operand) slot; the decoded A operand lives in TMEM
  uint32_t n_cslots;        // ring stages
  uint32_t n_xslots;        // X tile ring (one tile = one unit's [n_umma][64] X slice)
  uint32_t n_aslots;        // TMEM A-operand ring (32 columns each, multiple of 4)
  uint32_t acc_cols;        // TMEM columns per accumulator buffer (>= n_umma, multiple of 32)
  uint32_t n_acc;           // accumulator buffers: 2 (double buffered), 1 when 2 x acc_cols leaves no A ring
  uint32_t eb7x2;
  uint32_t cdiv_magic, adiv_magic;  // fastdiv multipliers of n_cslots / n_aslots
  unsigned long long* trace;  // optional per-unit event timestamps (debug; nullptr = off)
  uint32_t dbg;               // debug experiment flags (0 in production; zs_debug_set_flags)
  // fused output exchange: every Y element is also stored to ypeer[i]
  // (same [m][n] addressing and ldy as y), and once all CTAs' stores are visible the last
  // CTA writes `epoch` to flag[0..nflag) (system scope).  npeer = nflag = 0: plain GEMM.
  uint16_t* ypeer[kMaxPeers];
  uint32_t* flag[kMaxPeers];
  uint32_t* done;             // CTA completion counter (zero between calls), nullptr = no signal
  int32_t npeer, nflag;
  uint32_t epoch;
};

// Copy a [rows][cols] BF16 slice (leading dimension ld) from src to each of npeer
// destinations (same addressing), then -- after every CTA's stores are visible at system
// scope -- write `epoch` to flag[0..nflag).  `done`: zeroed counter, left zeroed.
struct PeerCopyParams {
  const uint16_t* src;
  uint16_t* dst[kMaxPeers];
  uint32_t* flag[kMaxPeers];
  uint32_t* done;
  int64_t rows, cols, ld;
  int32_t npeer, nflag;
  uint32_t epoch;
};
cudaError_t launch_peer_copy(const PeerCopyParams& p, int sms, cudaStream_t s);
// Spin (one thread per flag, ld.acquire.sys) until flags[0..n) have all reached `epoch`
// (wrap-safe comparison); traps after timeout_ns so a missing peer cannot hang the GPU.
cudaError_t launch_peer_wait(const uint32_t* flags, int n, uint32_t epoch, uint64_t timeout_ns, cudaStream_t s);

cudaError_t launch_gemm(const GemmParams& p, const CUtensorMap& xmap, int grid, size_t smem, cudaStream_t stream);
extern int g_pdl;   // launch_gemm uses programmatic dependent launch when nonzero
size_t gemm_smem_bytes(const GemmParams& p);
int gemm_threads();
int gemm_groups();
int gemm_aslots();
int gemm_max_xslots();
int gemm_max_cslots();
int gemm_max_aslots();
uint32_t gemm_stage_fixed_bytes();
int gemm_units_per_stage();
int gemm_max_chunk();
uint32_t gemm_fixed_smem();

// GPU encoder (zs_encode_gpu.cu)
cudaError_t launch_encode_hist(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, unsigned long long* hist,
                               int sms, cudaStream_t s);
cudaError_t launch_encode_count(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int64_t nbc, int64_t nbt,
                                int lo, int hi, uint32_t* hcnt, cudaStream_t s);
cudaError_t launch_encode_pack(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int64_t nbc, int64_t nbt,
                               int32_t base_exp, const uint64_t* offsets, uint64_t* b1, uint64_t* b2, uint64_t* b3,
                               uint8_t* h, uint16_t* l, cudaStream_t s);

}  // namespace zs
