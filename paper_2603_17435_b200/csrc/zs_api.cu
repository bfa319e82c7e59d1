// zs_api.cu -- C ABI entry points of libzs.so (declared in include/zs.h).
//
// Validation happens synchronously before any launch; errors map to zs_status codes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "../../include/zs.h"
#include "zs_host.h"
#include "zs_kernels.h"

#include <vector>

namespace {

thread_local int g_last_launches = 0;
unsigned long long* g_trace = nullptr;  // debug: set by zs_debug_set_trace
uint32_t g_dbg = 0;                     // debug: experiment flags (zs_debug_set_flags)
#ifndef ZS_RING_CAP
#define ZS_RING_CAP 16
#endif
uint32_t g_max_cslots = ZS_RING_CAP;    // ring depth cap (tunable via zs_debug_set_ring)
int64_t g_large_m = -1;                 // forced decoupled-path threshold (zs_debug_set_large_m), -1 = per shape

// cuBLAS handle of the decoupled prefill path: one per (host thread, device), created on
// first use.  cuBLAS only runs the plain dense GEMM on the already-decoded weights.
cublasHandle_t blas_handle(int dev) {
  thread_local cublasHandle_t h[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  if (!h[dev] && cublasCreate(&h[dev]) != CUBLAS_STATUS_SUCCESS) h[dev] = nullptr;
  return h[dev];
}

// Fused for small M, decoupled above a per-shape threshold (measured on the 8B layers,
// DESIGN.md 7.3): ZS_GEMM_LARGE_M for large matrices; for matrices of at most
// ZS_GEMM_SMALL_NK elements the decompression is cheap and the fused kernel's fixed cost
// dominates, so the crossover is ZS_GEMM_LARGE_M_SMALL_NK.
bool use_decoupled(int64_t M, int64_t N, int64_t K) {
  if (g_large_m >= 0) return M > g_large_m;
  const int64_t thr = (N * K <= ZS_GEMM_SMALL_NK) ? ZS_GEMM_LARGE_M_SMALL_NK : ZS_GEMM_LARGE_M;
  return M > thr;
}

inline int64_t up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct DevInfo {
  int ok = 0;
  int sms = 0;
};

zs_status device_check(int* sms) {
  // per-device cache: the attribute queries cost several microseconds per call
  static int cached_sms[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return ZS_ERR_UNSUPPORTED;
  if (dev >= 0 && dev < 64 && cached_sms[dev] > 0) {
    *sms = cached_sms[dev];
    return ZS_OK;
  }
  int major = 0, minor = 0, n = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return ZS_ERR_CUDA;
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (major != 10 || minor != 0) return ZS_ERR_UNSUPPORTED;  // built for sm_100a only
  if (dev >= 0 && dev < 64) cached_sms[dev] = n;
  *sms = n;
  return ZS_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

zs_status validate_tensor(const zs_tensor* w) {
  if (!w || !w->b1 || !w->b2 || !w->b3 || !w->offsets) return ZS_ERR_INVALID_ARG;
  const zs_sizes& s = w->sz;
  if (s.rows < 1 || s.cols < 1 || s.padded_rows != up(s.rows, 64) || s.padded_cols != up(s.cols, 64))
    return ZS_ERR_SHAPE;
  if (s.n_blocktiles != (s.padded_rows / 64) * (s.padded_cols / 64) || s.n_fragtiles != s.n_blocktiles * 64)
    return ZS_ERR_CORRUPT;
  if (s.max_h_seg_bytes < 0 || s.max_h_seg_bytes > 4096 || s.max_l_seg_bytes < 0 || s.max_l_seg_bytes > 8192 ||
      (s.max_h_seg_bytes & 15) || (s.max_l_seg_bytes & 15))
    return ZS_ERR_CORRUPT;
  if ((s.h_bytes && !w->h) || (s.l_words && !w->l)) return ZS_ERR_INVALID_ARG;
  if (w->base_exp < -1 || w->base_exp > 248) return ZS_ERR_INVALID_ARG;
  if (!aligned16(w->b1) || !aligned16(w->b2) || !aligned16(w->b3) || !aligned16(w->offsets) ||
      (w->h && !aligned16(w->h)) || (w->l && !aligned16(w->l)))
    return ZS_ERR_ALIGNMENT;
  return ZS_OK;
}

uint32_t eb7x2_of(int32_t base_exp) {
  const uint32_t eb = (uint32_t)base_exp & 0xFFu;
  return (eb << 7) | (eb << 23);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

PFN_cuMemGetAddressRange_v3020 get_addr_range() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

}  // namespace

extern "C" const char* zs_status_string(zs_status s) {
  switch (s) {
    case ZS_OK: return "ZS_OK";
    case ZS_ERR_INVALID_ARG: return "ZS_ERR_INVALID_ARG";
    case ZS_ERR_SHAPE: return "ZS_ERR_SHAPE";
    case ZS_ERR_ALIGNMENT: return "ZS_ERR_ALIGNMENT";
    case ZS_ERR_UNSUPPORTED: return "ZS_ERR_UNSUPPORTED";
    case ZS_ERR_CORRUPT: return "ZS_ERR_CORRUPT";
    case ZS_ERR_CUDA: return "ZS_ERR_CUDA";
    case ZS_ERR_CAPACITY: return "ZS_ERR_CAPACITY";
  }
  return "ZS_ERR_UNKNOWN";
}

extern "C" int zs_last_launch_count(void) { return g_last_launches; }

// Debug hook (not part of include/zs.h): device buffer of 4*128*16 u64 for per-unit
// pipeline timestamps of the first 4 CTAs of subsequent zs_gemm launches; NULL disables.
extern "C" void zs_debug_set_trace(unsigned long long* dev_buf) { g_trace = dev_buf; }
// Debug hook: 1 = decoders skip the row decode, 2 = skip tcgen05.st, 4 = no tcgen05.mma
// (timing experiments only: results are wrong with any flag set).
extern "C" void zs_debug_set_flags(int flags) { g_dbg = (uint32_t)flags; }
extern "C" void zs_debug_set_ring(int max_cslots) { g_max_cslots = (uint32_t)std::max(1, max_cslots); }
// Debug hook: programmatic dependent launch of the fused kernel on (1, default) / off (0).
extern "C" void zs_debug_set_pdl(int on) { zs::g_pdl = on ? 1 : 0; }
// Debug hook: move the fused / decoupled threshold (crossover measurement); < 0 restores it.
extern "C" void zs_debug_set_large_m(long long m) { g_large_m = m < 0 ? -1 : (int64_t)m; }

extern "C" zs_status zs_decompress(const zs_tensor* w, uint16_t* out, int64_t ld_out, void* stream) {
  g_last_launches = 0;
  zs_status st = validate_tensor(w);
  if (st != ZS_OK) return st;
  if (!out || ld_out < w->sz.cols) return ZS_ERR_INVALID_ARG;
  int sms = 0;
  if ((st = device_check(&sms)) != ZS_OK) return st;

  zs::DecompParams p{};
  p.b1 = w->b1;
  p.b2 = w->b2;
  p.b3 = w->b3;
  p.h = w->h;
  p.l = w->l;
  p.offsets = w->offsets;
  p.out = out;
  p.ld_out = ld_out;
  p.rows = w->sz.rows;
  p.cols = w->sz.cols;
  p.nbc = w->sz.padded_cols / 64;
  p.n_blocktiles = w->sz.n_blocktiles;
  p.hcap = (uint32_t)w->sz.max_h_seg_bytes + 16;
  const uint32_t lcap = (uint32_t)w->sz.max_l_seg_bytes + 16;
  p.stage_bytes = (uint32_t)up(1536 + p.hcap + lcap, 128);
  p.eb7x2 = eb7x2_of(w->base_exp);
  p.vec_ok = aligned16(out) && (ld_out % 8 == 0);
  // one CTA per SM; as many independent decoder warps (2 stages each) as fit in smem
  int warps = zs::decompress_max_warps();
  while (warps > 1 && zs::decompress_smem_bytes(p.stage_bytes, warps) > 227 * 1024) --warps;
  if (zs::decompress_smem_bytes(p.stage_bytes, warps) > 227 * 1024) return ZS_ERR_UNSUPPORTED;
  const size_t smem = zs::decompress_smem_bytes(p.stage_bytes, warps);
  const int64_t grid = std::min<int64_t>((p.n_blocktiles + warps - 1) / warps, (int64_t)sms);
  cudaError_t e = zs::launch_decompress(p, (int)grid, warps, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return ZS_ERR_CUDA;
  g_last_launches = 1;
  return ZS_OK;
}

#ifndef ZS_UPS
#define ZS_UPS 4   // must match zs_gemm.cu (units per ring stage)
#endif
#ifndef ZS_SPLIT3
#define ZS_SPLIT3 2   // > 0: prefer 3 compressed stages with that many X tiles over 2 stages with 4
                      // (2: M = 129..256 run 3 stages + 2 X tiles; 8B GateUp M = 144 / 256: 108.5 / 122.3 -> 93.0 / 111.5 us)
#endif
#ifndef ZS_XTILES_MAX
#define ZS_XTILES_MAX (ZS_UPS == 4 ? 12 : 15)   // X tiles in the ring at most (L2-sourced; 3 stages)
#endif

// split-K region: fp32 partials [min(M,256)][N] + per-band counters (zero between calls)
static size_t splitk_bytes(int64_t M, int64_t N) {
  const int64_t mc = up(std::min<int64_t>(M, 256), 16);   // row stride of the [N][mc] partials
  const int64_t nbands = (up(N, 64) / 64 + 1) / 2;
  return (size_t)up(mc * N * 4 + up(nbands * 4, 256), 256);
}

extern "C" size_t zs_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  if (M < 1 || N < 1 || K < 1) return 0;
  // decoupled path: scratch for the decoded W [N][roundup(K,8)] bf16
  if (use_decoupled(M, N, K)) return (size_t)up(N * up(K, 8) * 2, 256);
  return splitk_bytes(M, N);
}

extern "C" int zs_gemm_is_decoupled(int64_t M, int64_t N, int64_t K) { return use_decoupled(M, N, K) ? 1 : 0; }

// fused output exchange (f2) of zs_gemm_peer: extra output copies and the flags to signal
struct PeerSetup {
  uint16_t* ypeer[zs::kMaxPeers];
  uint32_t* flag[zs::kMaxPeers];
  uint32_t* done;
  int npeer, nflag;
  uint32_t epoch;
};

static zs_status gemm_core(const uint16_t* x, int64_t ldx, const zs_tensor* w, uint16_t* y, int64_t ldy, int64_t M,
                           int64_t N, int64_t K, void* workspace, size_t workspace_bytes, void* stream,
                           const PeerSetup* ps) {
  g_last_launches = 0;
  zs_status st = validate_tensor(w);
  if (st != ZS_OK) return st;
  if (!x || !y || M < 1 || N < 1 || K < 1) return ZS_ERR_INVALID_ARG;
  if (N != w->sz.rows || K != w->sz.cols) return ZS_ERR_SHAPE;
  if (ldx < K || ldy < N) return ZS_ERR_SHAPE;
  if (!aligned16(x) || (ldx * 2) % 16 != 0) return ZS_ERR_ALIGNMENT;
  if (!workspace || workspace_bytes < zs_gemm_workspace_bytes(M, N, K)) return ZS_ERR_CAPACITY;
  if (!aligned16(workspace)) return ZS_ERR_ALIGNMENT;
  int sms = 0;
  if ((st = device_check(&sms)) != ZS_OK) return st;

  if (use_decoupled(M, N, K)) {
    // Large M (prefill): ZipServ-Decomp into the workspace, then a dense BF16 GEMM
    // on the tensor cores (cuBLAS).  The decode runs once per call instead of once per
    // 128-token chunk.
    const int64_t ldw = up(K, 8);
    uint16_t* wdense = reinterpret_cast<uint16_t*>(workspace);
    if ((st = zs_decompress(w, wdense, ldw, stream)) != ZS_OK) return st;
    int dev = 0;
    cudaGetDevice(&dev);
    cublasHandle_t h = blas_handle(dev);
    if (!h || cublasSetStream(h, (cudaStream_t)stream) != CUBLAS_STATUS_SUCCESS) return ZS_ERR_CUDA;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return ZS_ERR_UNSUPPORTED;
    const float one = 1.0f, zero = 0.0f;
    // column-major view: Y^T[N][M] = W[N][K] (op T of the K x N col-major W) * X^T[K][M]
    cublasStatus_t bs = cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)N, (int)M, (int)K, &one, wdense,
                                     CUDA_R_16BF, (int)ldw, x, CUDA_R_16BF, (int)ldx, &zero, y, CUDA_R_16BF,
                                     (int)ldy, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (bs != CUBLAS_STATUS_SUCCESS) return ZS_ERR_CUDA;
    g_last_launches = 1;   // our kernels only (the cuBLAS GEMM is library code)
    if (ps) {
      // broadcast the slice cuBLAS wrote to the peers' Y, then signal (one launch)
      zs::PeerCopyParams cp{};
      cp.src = y;
      for (int i = 0; i < ps->npeer; ++i) cp.dst[i] = ps->ypeer[i];
      for (int i = 0; i < ps->nflag; ++i) cp.flag[i] = ps->flag[i];
      cp.done = ps->done;
      cp.rows = M;
      cp.cols = N;
      cp.ld = ldy;
      cp.npeer = ps->npeer;
      cp.nflag = ps->nflag;
      cp.epoch = ps->epoch;
      if (zs::launch_peer_copy(cp, sms, (cudaStream_t)stream) != cudaSuccess) return ZS_ERR_CUDA;
      g_last_launches = 2;
    }
    return ZS_OK;
  }

  auto enc = get_encode_tiled();
  if (!enc) return ZS_ERR_UNSUPPORTED;

  const int64_t mc_max = std::min<int64_t>(M, 256);  // workspace rows (>= any chunk)
  zs::GemmParams p{};
  p.b1 = w->b1;
  p.b2 = w->b2;
  p.b3 = w->b3;
  p.h = w->h;
  p.l = w->l;
  p.offsets = w->offsets;
  p.y = y;
  p.ldy = ldy;
  p.ws = reinterpret_cast<float*>(workspace);
  p.ldws = up(mc_max, 16);
  p.counters = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(workspace) + p.ldws * N * 4);
  p.N = N;
  p.nbr = w->sz.padded_rows / 64;
  p.nbc = w->sz.padded_cols / 64;
  p.nbands = (p.nbr + 1) / 2;
  p.total_units = p.nbands * p.nbc;
  if (p.total_units >= (int64_t(1) << 31)) return ZS_ERR_UNSUPPORTED;
  {
    const int64_t ups = zs::gemm_units_per_stage();
    if (w->sz.h_bytes >= (int64_t(1) << 32) || 2 * w->sz.l_words >= (int64_t(1) << 32)) return ZS_ERR_UNSUPPORTED;
    p.hcap = (uint32_t)(ups * w->sz.max_h_seg_bytes + 16);
    p.lcap = (uint32_t)(ups * w->sz.max_l_seg_bytes + 16);
    p.cslot_bytes = (uint32_t)up(zs::gemm_stage_fixed_bytes() + 2 * (int64_t)p.hcap + 2 * (int64_t)p.lcap, 1024);
  }
  p.eb7x2 = eb7x2_of(w->base_exp);
  p.trace = g_trace;
  p.dbg = g_dbg;

  // X tensor map: dims {K, M}, row stride ldx*2 bytes, box {64, n_umma}, SWIZZLE_128B;
  // out-of-bounds rows/columns are zero-filled by the TMA unit.
  const size_t budget = 227 * 1024;
  const size_t base = zs::gemm_fixed_smem();
  // smem split for a token chunk of nu rows: X tiles (one per unit, [nu][64] bf16) and
  // compressed stages (4 units each): at least 2 of each, so both streams stay double
  // buffered; prefer up to 16 X tiles (L2-sourced, cheap) and then as many compressed stages
  // as fit (the HBM stream is the one whose latency must be hidden)
  auto split = [&](int64_t nu, uint32_t* nx, uint32_t* nc) {
    const size_t xs = (size_t)up(nu * 128, 1024);
    const size_t cs = p.cslot_bytes;
    const uint32_t cmax = std::min<uint32_t>((uint32_t)zs::gemm_max_cslots(), g_max_cslots);
    // preference: 3 compressed stages with >= 4 X tiles (measured best at small M; a 4th
    // stage measured no change), then 3 stages with >= ZS_SPLIT3 tiles (the 129..256-token
    // chunks: a 2-stage ring does not hide HBM there), then 2 stages with >= 4 / >= 2 tiles
#if ZS_SPLIT3
    static const uint32_t pref[][2] = {{3, 4}, {3, ZS_SPLIT3}, {2, 4}, {2, 2}, {1, 2}};
#else
    static const uint32_t pref[][2] = {{3, 4}, {2, 4}, {2, 2}, {1, 2}};
#endif
    for (const auto& pr : pref) {
      const uint32_t c = std::min(pr[0], cmax);
      if (base + c * cs + pr[1] * xs > budget) continue;
      *nc = c;
      *nx = (uint32_t)std::min<size_t>({(size_t)zs::gemm_max_xslots(), (size_t)ZS_XTILES_MAX, (budget - base - c * cs) / xs});
      // whole stages of X tiles when the ring holds at least two (stage mode)
      const uint32_t ups = (uint32_t)zs::gemm_units_per_stage();
      if (ups != 4 && *nx >= 2 * ups) *nx -= *nx % ups;
      return true;
    }
    return false;
  };
  // token chunk: the largest power of two <= 256 whose smem split fits (a chunk re-decodes W)
  int64_t chunk = zs::gemm_max_chunk();
  for (; chunk >= 16; chunk /= 2) {
    uint32_t nx, nc;
    if (split(up(std::min<int64_t>(chunk, M), 16), &nx, &nc)) break;
  }
  if (chunk < 16) return ZS_ERR_UNSUPPORTED;
  int launches = 0;
  CUtensorMap xmap;
  uint32_t cur_box = 0;
  for (int64_t m0 = 0; m0 < M; m0 += chunk) {
    const int64_t mc = std::min<int64_t>(chunk, M - m0);
    p.m0 = (int32_t)m0;
    p.mc = (int32_t)mc;
    p.n_umma = (uint32_t)up(mc, 16);
    p.aslot_bytes = (uint32_t)up((int64_t)p.n_umma * 128, 1024);
    uint32_t nx = 0, nc = 0;
    if (!split(p.n_umma, &nx, &nc)) return ZS_ERR_UNSUPPORTED;
    p.n_cslots = nc;
    p.n_xslots = nx;
    // TMEM (512 columns): accumulator buffer(s) + an A-operand ring of 32-column slots in
    // whole stages of 4; two accumulator buffers when that leaves at least one A stage
    p.acc_cols = (uint32_t)up(p.n_umma, 32);
    // two buffers only while they leave a 2-stage A ring (8 slots): with a 1-stage ring the
    // decoders and the MMA warp serialise per stage (measured: 8B GateUp M = 129, acc 160,
    // 4 A slots: 123 us; one buffer + 8 slots is the better trade above 128 tokens)
    p.n_acc = (2u * p.acc_cols + 2u * 32u * (uint32_t)zs::gemm_units_per_stage() <= 512u) ? 2u : 1u;
    uint32_t na = (512u - p.n_acc * p.acc_cols) / 32u;
    na = std::min<uint32_t>(na, (uint32_t)zs::gemm_max_aslots());
    p.n_aslots = na - na % (uint32_t)zs::gemm_units_per_stage();
    auto magic = [](uint32_t d) { return d <= 1u ? 0u : (uint32_t)((1ull << 32) / d + 1ull); };
    p.cdiv_magic = magic(p.n_cslots);
    p.adiv_magic = magic(p.n_aslots / (uint32_t)zs::gemm_units_per_stage());
    // one-entry cache per host thread: repeated calls on the same activation buffer (the
    // usual serving loop) skip the tensor-map encode
    thread_local struct { const void* x; int64_t K, M, ldx; uint32_t box; CUtensorMap map; } xcache = {};
    if (p.n_umma != cur_box && xcache.x == x && xcache.K == K && xcache.M == M && xcache.ldx == ldx &&
        xcache.box == p.n_umma) {
      xmap = xcache.map;
      cur_box = p.n_umma;
    }
    if (p.n_umma != cur_box) {
      cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
      cuuint64_t strides[1] = {(cuuint64_t)(ldx * 2)};
      cuuint32_t box[2] = {64, p.n_umma};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(x), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return ZS_ERR_CUDA;
      cur_box = p.n_umma;
      xcache.x = x; xcache.K = K; xcache.M = M; xcache.ldx = ldx; xcache.box = p.n_umma; xcache.map = xmap;
    }
    if (ps) {
      // every chunk stores to the peers; only the last one signals (chunks are stream-ordered)
      for (int i = 0; i < ps->npeer; ++i) p.ypeer[i] = ps->ypeer[i];
      for (int i = 0; i < ps->nflag; ++i) p.flag[i] = ps->flag[i];
      p.npeer = ps->npeer;
      p.nflag = ps->nflag;
      p.epoch = ps->epoch;
      p.done = (m0 + chunk >= M) ? ps->done : nullptr;
    }
    const int64_t grid = std::min<int64_t>(p.total_units, sms);
    cudaError_t e = zs::launch_gemm(p, xmap, (int)grid, zs::gemm_smem_bytes(p), (cudaStream_t)stream);
    if (e != cudaSuccess) return ZS_ERR_CUDA;
    ++launches;
  }
  g_last_launches = launches;
  return ZS_OK;
}

extern "C" zs_status zs_gemm(const uint16_t* x, int64_t ldx, const zs_tensor* w, uint16_t* y, int64_t ldy, int64_t M,
                             int64_t N, int64_t K, void* workspace, size_t workspace_bytes, void* stream) {
  return gemm_core(x, ldx, w, y, ldy, M, N, K, workspace, workspace_bytes, stream, nullptr);
}

// ------------------------------------------------------------------ output exchange (f2)
extern "C" size_t zs_gemm_peer_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const size_t b = zs_gemm_workspace_bytes(M, N, K);
  return b ? b + 256 : 0;   // + the CTA completion counter of the signalling launch (first 256 B)
}

extern "C" zs_status zs_gemm_peer(const uint16_t* x, int64_t ldx, const zs_tensor* w, const zs_peer_out* out,
                                  int64_t M, int64_t N, int64_t K, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  g_last_launches = 0;
  if (!out) return ZS_ERR_INVALID_ARG;
  const int world = out->world, rank = out->rank;
  if (world < 1 || world > ZS_MAX_PEERS || rank < 0 || rank >= world) return ZS_ERR_INVALID_ARG;
  for (int r = 0; r < world; ++r)
    if (!out->y[r] || !out->flags[r]) return ZS_ERR_INVALID_ARG;
  if (out->col0 < 0 || N < 1 || out->ldy < out->col0 + N) return ZS_ERR_SHAPE;
  if (!workspace || workspace_bytes < zs_gemm_peer_workspace_bytes(M, N, K)) return ZS_ERR_CAPACITY;
  const size_t base = zs_gemm_workspace_bytes(M, N, K);
  PeerSetup ps{};
  for (int r = 0; r < world; ++r) {
    if (r != rank) ps.ypeer[ps.npeer++] = out->y[r] + out->col0;
    ps.flag[ps.nflag++] = out->flags[r] + rank;
  }
  // the counter leads the workspace, so the decoupled path's (dirty) scratch never covers it
  ps.done = reinterpret_cast<uint32_t*>(workspace);
  ps.epoch = out->epoch;
  return gemm_core(x, ldx, w, out->y[rank] + out->col0, out->ldy, M, N, K,
                   reinterpret_cast<uint8_t*>(workspace) + 256, base, stream, &ps);
}

extern "C" zs_status zs_peer_wait(const uint32_t* flags, int32_t world, uint32_t epoch, void* stream) {
  g_last_launches = 0;
  if (!flags || world < 1 || world > ZS_MAX_PEERS) return ZS_ERR_INVALID_ARG;
  int sms = 0;
  zs_status st = device_check(&sms);
  if (st != ZS_OK) return st;
  if (zs::launch_peer_wait(flags, world, epoch, ZS_PEER_WAIT_TIMEOUT_NS, (cudaStream_t)stream) != cudaSuccess)
    return ZS_ERR_CUDA;
  g_last_launches = 1;
  return ZS_OK;
}

extern "C" zs_status zs_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset) {
  if (!dev_ptr || !handle || !offset) return ZS_ERR_INVALID_ARG;
  auto range = get_addr_range();
  if (!range) return ZS_ERR_UNSUPPORTED;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return ZS_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return ZS_ERR_CUDA;
  static_assert(sizeof(h) == ZS_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)((CUdeviceptr)dev_ptr - base);
  return ZS_OK;
}

extern "C" zs_status zs_ipc_open(const void* handle, void** base) {
  if (!handle || !base) return ZS_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return ZS_ERR_CUDA;
  }
  return ZS_OK;
}

extern "C" zs_status zs_ipc_close(void* base) {
  if (!base) return ZS_ERR_INVALID_ARG;
  if (cudaIpcCloseMemHandle(base) != cudaSuccess) {
    cudaGetLastError();
    return ZS_ERR_CUDA;
  }
  return ZS_OK;
}

// ------------------------------------------------------------------ GPU encoder (f3)
extern "C" size_t zs_encode_device_workspace_bytes(int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) return 0;
  const int64_t nbt = (up(rows, 64) / 64) * (up(cols, 64) / 64);
  return (size_t)(256 * 8 + up(nbt * 4, 256));
}

namespace {
zs_status encode_counts(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int lo, int hi, void* ws,
                        cudaStream_t s, std::vector<uint32_t>& hcnt) {
  const int64_t nbc = up(cols, 64) / 64, nbt = (up(rows, 64) / 64) * nbc;
  uint32_t* dcnt = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ws) + 256 * 8);
  if (zs::launch_encode_count(w, rows, cols, ld, nbc, nbt, lo, hi, dcnt, s) != cudaSuccess) return ZS_ERR_CUDA;
  hcnt.resize(nbt);
  if (cudaMemcpyAsync(hcnt.data(), dcnt, nbt * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return ZS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ZS_ERR_CUDA;
  return ZS_OK;
}
}  // namespace

extern "C" zs_status zs_encode_measure_device(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, void* ws,
                                              size_t ws_bytes, void* stream, int32_t* base_exp, int64_t* covered,
                                              zs_sizes* exact) {
  g_last_launches = 0;
  if (!w || rows < 1 || cols < 1 || ld < cols || !base_exp || !exact || !ws) return ZS_ERR_INVALID_ARG;
  if (ws_bytes < zs_encode_device_workspace_bytes(rows, cols)) return ZS_ERR_CAPACITY;
  int sms = 0;
  zs_status st = device_check(&sms);
  if (st != ZS_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* dh = reinterpret_cast<unsigned long long*>(ws);
  if (cudaMemsetAsync(dh, 0, 256 * 8, s) != cudaSuccess) return ZS_ERR_CUDA;
  if (zs::launch_encode_hist(w, rows, cols, ld, dh, sms, s) != cudaSuccess) return ZS_ERR_CUDA;
  unsigned long long hh[256];
  if (cudaMemcpyAsync(hh, dh, sizeof(hh), cudaMemcpyDeviceToHost, s) != cudaSuccess) return ZS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ZS_ERR_CUDA;
  int64_t hist[256];
  for (int i = 0; i < 256; ++i) hist[i] = (int64_t)hh[i];
  int64_t best = 0;
  const int s0 = zs::window_start(hist, &best);
  *base_exp = s0 - 1;
  if (covered) *covered = best;
  std::vector<uint32_t> hcnt;
  if ((st = encode_counts(w, rows, cols, ld, s0, s0 + 6, ws, s, hcnt)) != ZS_OK) return st;
  zs::sizes_and_offsets(rows, cols, hcnt.data(), exact, nullptr);
  g_last_launches = 2;
  return ZS_OK;
}

extern "C" zs_status zs_encode_device(const uint16_t* w, int64_t rows, int64_t cols, int64_t ld, int32_t base_exp,
                                      const zs_sizes* cap, uint64_t* b1, uint64_t* b2, uint64_t* b3, uint8_t* h,
                                      uint16_t* l, uint64_t* offsets, zs_sizes* actual, uint16_t* pad_word, void* ws,
                                      size_t ws_bytes, void* stream) {
  g_last_launches = 0;
  if (!w || rows < 1 || cols < 1 || ld < cols || !cap || !b1 || !b2 || !b3 || !offsets || !actual || !ws)
    return ZS_ERR_INVALID_ARG;
  if (base_exp < -1 || base_exp > 248) return ZS_ERR_INVALID_ARG;
  if (ws_bytes < zs_encode_device_workspace_bytes(rows, cols)) return ZS_ERR_CAPACITY;
  int sms = 0;
  zs_status st = device_check(&sms);
  if (st != ZS_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<uint32_t> hcnt;
  if ((st = encode_counts(w, rows, cols, ld, base_exp + 1, base_exp + 7, ws, s, hcnt)) != ZS_OK) return st;
  const int64_t nbc = up(cols, 64) / 64, nbt = (up(rows, 64) / 64) * nbc;
  zs_sizes sz;
  std::vector<uint64_t> off(2 * (nbt + 1));
  zs::sizes_and_offsets(rows, cols, hcnt.data(), &sz, off.data());
  if (cap->n_fragtiles < sz.n_fragtiles || cap->n_blocktiles < sz.n_blocktiles || cap->h_bytes < sz.h_bytes ||
      cap->l_words < sz.l_words)
    return ZS_ERR_CAPACITY;
  if ((sz.h_bytes && !h) || (sz.l_words && !l)) return ZS_ERR_INVALID_ARG;
  if (cudaMemcpyAsync(offsets, off.data(), off.size() * 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return ZS_ERR_CUDA;
  if (zs::launch_encode_pack(w, rows, cols, ld, nbc, nbt, base_exp, offsets, b1, b2, b3, h, l, s) != cudaSuccess)
    return ZS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return ZS_ERR_CUDA;   // `off` must outlive the copy
  *actual = sz;
  if (pad_word) *pad_word = (uint16_t)((base_exp + 1) << 7);
  g_last_launches = 2;
  return ZS_OK;
}
