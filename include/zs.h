/*
 * zs.h -- C ABI of the B200-native ZipGEMM library (libzs.so).
 *
 * Method: ZipServ / TCA-TBE (arxiv 2603.17435).  Citations: P:<line> = PAPER.md,
 * S:<line> = SPEC.md (read while writing; nothing reads them at run time).
 *
 *   zs_encode        offline compressor, Alg. 1 with the layout of P:355-361
 *                    and SPEC's ledger                              [host]
 *   zs_decompress    ZipServ-Decomp: TCA-TBE -> BF16 in global memory
 *                    using the decode of Alg. 2                     [device]
 *   zs_gemm          ZipGEMM: Y = X * W^T with W streamed compressed and decoded per
 *                    tile inside the kernel (north star)             [device]
 *   zs_gemm_peer     column-sharded ZipGEMM whose epilogue also stores into every
 *                    rank's Y over NVLink and signals flags    [device]
 *   zs_peer_wait     stream wait for those flags                                [device]
 *
 * Notation: the paper writes Y = W X with W (M out x K) and X (K x N tokens).
 * This ABI uses the F.linear convention: X is [M tokens][K], W is [N out][K], Y is [M][N].
 *
 * Conventions for every call
 *   - Ownership: the caller owns every buffer.  The library allocates no device memory
 *     for data; the only library-held state is (a) one cuBLAS handle per (host thread,
 *     device), created by the first zs_gemm call that takes the decoupled large-M path
 *     (cublasCreate allocates a small device workspace -- make that first call outside
 *     CUDA-graph capture), (b) a per-thread launch count (zs_last_launch_count) and a
 *     per-thread X tensor-map cache, (c) the zs_debug_* experiment knobs of zs_api.cu,
 *     which are NOT part of this ABI: process-global, not synchronised, for the repo's
 *     own timing scripts only (they change kernel behaviour and, for
 *     zs_debug_set_large_m, what zs_gemm_workspace_bytes returns).  With the knobs left
 *     alone every entry point is thread-safe for concurrent callers.
 *   - Launch mode: zs_gemm / zs_gemm_peer launch with programmatic dependent launch
 *     (PDL).  Their compressed-weight producer reads W and its offsets BEFORE
 *     griddepcontrol.wait, so the kernel launched immediately before them on the same
 *     stream must not write the encoded W (X, Y and the workspace are read/written only
 *     after the wait).  Encoded weights are immutable by contract, so this only matters
 *     to a caller that re-encodes into the same buffers on the GEMM's stream: put an
 *     event or any non-PDL launch between the two.
 *   - Device calls are asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  Validation is synchronous and happens before
 *     launch; no exceptions cross the ABI.  Launch failures return ZS_ERR_CUDA.
 *   - Encoded data is immutable after zs_encode and safe for concurrent readers.
 *   - There is no CPU fallback: device entry points need an sm_100a GPU and return
 *     ZS_ERR_UNSUPPORTED otherwise.
 */
#ifndef ZS_H_
#define ZS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ZS_OK = 0,
    ZS_ERR_INVALID_ARG = 1,   /* null pointer, non-positive dimension, bad base_exp */
    ZS_ERR_SHAPE = 2,         /* M/N/K inconsistent with the encoded tensor        */
    ZS_ERR_ALIGNMENT = 3,     /* pointer/stride violates the 16-byte TMA rule      */
    ZS_ERR_UNSUPPORTED = 4,   /* no sm_100a device, or a size beyond the kernels   */
    ZS_ERR_CORRUPT = 5,       /* offsets / segment sizes inconsistent       */
    ZS_ERR_CUDA = 6,          /* a CUDA runtime call or kernel launch failed       */
    ZS_ERR_CAPACITY = 7       /* caller buffer smaller than required               */
} zs_status;

/* Sizes of one encoded matrix.  Element counts unless suffixed _bytes / _words. */
typedef struct {
    int64_t rows, cols;                  /* logical N (out features), K (in features)      */
    int64_t padded_rows, padded_cols;    /* multiples of 64 (BlockTile)      */
    int64_t n_fragtiles;                 /* (padded_rows/8) * (padded_cols/8)             */
    int64_t n_blocktiles;                /* (padded_rows/64) * (padded_cols/64)           */
    int64_t h_bytes;                     /* PackedSignMantissa array, incl. 16-B padding   */
    int64_t l_words;                     /* FullValue array (u16), incl. 16-B padding      */
    int64_t max_h_seg_bytes;             /* largest per-BlockTile H segment (padded)       */
    int64_t max_l_seg_bytes;             /* largest per-BlockTile L segment (padded)       */
} zs_sizes;

/*
 * Non-owning view of an encoded matrix (all pointers host OR all device).
 * Layout:
 *   b1, b2, b3  one uint64 per 8x8 FragTile, bit p = codeword bit of the element at
 *               position p = row*8 + col inside the FragTile (LSB first); b1 holds the
 *               codeword LSB (Alg. 1 line 12).  FragTile order is canonical: BlockTile
 *               (64x64) row-major -> TensorCoreTile (16x16) row-major -> FragTile
 *               column-major in its 2x2 grid -> position ascending.
 *   h           one byte (sign<<7 | mantissa) per in-window element, canonical order;
 *               each BlockTile's segment starts 16-byte aligned and is zero padded.
 *   l           one raw BF16 word per fallback element (codeword 000), same segmentation.
 *   offsets     n_blocktiles + 1 pairs {h_start_bytes, l_start_bytes}; the last pair is a
 *               sentinel = {h_bytes, 2*l_words}.  Both 16-byte aligned, non-decreasing.
 *   base_exp    e_base = min(window) - 1 in [-1, 248], one per matrix.
 *   pad_word    (0, base_exp+1, 0): the value stored in padded rows/columns.
 * Decoding element p: if (b1|b2|b3) bit p is set, exponent = base_exp + codeword and
 * sign/mantissa come from h[h_start + popc(M & ((1<<p)-1))]; else the word is
 * l[l_start + p - popc(...)] (Alg. 2).
 */
typedef struct {
    zs_sizes sz;
    int32_t base_exp;
    uint16_t pad_word;
    uint16_t reserved;
    const uint64_t *b1, *b2, *b3;
    const uint8_t *h;
    const uint16_t *l;
    const uint64_t *offsets;
} zs_tensor;

/* Worst-case sizes for a rows x cols matrix (every element in H and in L). Host, O(1).
 * Errors: ZS_ERR_INVALID_ARG if rows < 1, cols < 1 or upper == NULL. */
zs_status zs_encode_bound(int64_t rows, int64_t cols, zs_sizes *upper);

/* Phase I of Alg. 1: exponent histogram over the rows x cols LOGICAL
 * elements of w (host, row-major, leading dimension ld >= cols), max-coverage window of
 * 7 consecutive exponents (ties -> smallest start), base_exp = start - 1, and
 * the exact sizes the encoding will need.  covered (may be NULL) = #elements in window.
 * Errors: ZS_ERR_INVALID_ARG. */
zs_status zs_encode_measure(const uint16_t *w, int64_t rows, int64_t cols, int64_t ld,
                            int32_t *base_exp, int64_t *covered, zs_sizes *exact);

/* Phase II of Alg. 1: encode w with the given base_exp (normally the one
 * zs_encode_measure returned; a caller-forced base_exp is allowed, e.g. one window for a
 * whole model).  Host buffers, caller-allocated with at least cap->... entries:
 *   b1/b2/b3: cap->n_fragtiles, h: cap->h_bytes, l: cap->l_words,
 *   offsets: 2 * (cap->n_blocktiles + 1).
 * actual receives the sizes written.  Errors: ZS_ERR_INVALID_ARG (null, base_exp outside
 * [-1, 248]), ZS_ERR_CAPACITY (a buffer too small; nothing beyond capacity is written). */
zs_status zs_encode(const uint16_t *w, int64_t rows, int64_t cols, int64_t ld, int32_t base_exp,
                    const zs_sizes *cap, uint64_t *b1, uint64_t *b2, uint64_t *b3,
                    uint8_t *h, uint16_t *l, uint64_t *offsets,
                    zs_sizes *actual, uint16_t *pad_word);

/* ZipServ-Decomp: decode the DEVICE tensor w into out (device, row-major
 * [w->sz.rows][ld_out] BF16, only the logical rows x cols are written), bit-exact.
 * Errors: ZS_ERR_INVALID_ARG (null, ld_out < cols), ZS_ERR_UNSUPPORTED (no sm_100a),
 * ZS_ERR_CUDA. */
zs_status zs_decompress(const zs_tensor *w, uint16_t *out, int64_t ld_out, void *stream);

/* Token count above which zs_gemm takes the decoupled prefill path ("decoupled
 * decompression + dense GEMM for the compute-bound prefill stage"): zs_decompress of W
 * into the workspace, then one dense BF16 tensor-core GEMM (cuBLAS, fp32 accumulate).
 * At or below it the fused ZipGEMM kernel runs (decode stage).  Values measured on B200,
 * see DESIGN.md 7.3 (crossover of the two paths over LLaMA-3.1-8B layer shapes): matrices
 * of at most ZS_GEMM_SMALL_NK elements switch at ZS_GEMM_LARGE_M_SMALL_NK tokens. */
#define ZS_GEMM_LARGE_M 256
#define ZS_GEMM_SMALL_NK (32ll * 1024 * 1024)
#define ZS_GEMM_LARGE_M_SMALL_NK 48

/* Workspace (device bytes) zs_gemm needs for an M x N x K problem.
 *   fused path (zs_gemm_is_decoupled == 0): fp32 split-K partial sums [M][N] plus per-band arrival
 *     counters.  It must be zero-filled once before its first use; zs_gemm leaves it
 *     zero-filled again when it completes, so one workspace can be reused by every later
 *     call on the same stream.
 *   decoupled path: scratch for the decoded weight, N x roundup(K, 8) BF16.  Any
 *     contents on entry; NOT zero on exit, so do not hand the same buffer to a fused
 *     call afterwards without zero-filling it (zs_gemm_is_decoupled tells the paths apart).
 * Returns 0 for non-positive sizes. */
size_t zs_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K);

/* 1 if zs_gemm takes the decoupled path for this problem (M above the shape's threshold, see
 * ZS_GEMM_LARGE_M), else 0.  Host, O(1), no errors. */
int zs_gemm_is_decoupled(int64_t M, int64_t N, int64_t K);

/* ZipGEMM: Y[M][N] = X[M][K] * W[N][K]^T with fp32 accumulation in tensor
 * memory and BF16 output (RNE).  x: device BF16, row-major, leading dimension ldx
 * (elements), base 16-byte aligned and ldx*2 % 16 == 0 (TMA rule).  w: DEVICE tensor with
 * w->sz.rows == N, w->sz.cols == K.  y: device BF16 [M][ldy], ldy >= N.  Outputs of
 * padded rows are not written.  M >= 1: small M runs the fused kernel (one launch); M above
 * the shape's threshold (ZS_GEMM_LARGE_M) runs zs_decompress + a cuBLAS BF16 GEMM on the same stream (the
 * library keeps one cuBLAS handle per host thread and device, created on first use).
 * workspace: see zs_gemm_workspace_bytes.
 * Errors: ZS_ERR_INVALID_ARG, ZS_ERR_SHAPE, ZS_ERR_ALIGNMENT, ZS_ERR_CAPACITY
 * (workspace too small), ZS_ERR_UNSUPPORTED, ZS_ERR_CUDA. */
zs_status zs_gemm(const uint16_t *x, int64_t ldx, const zs_tensor *w, uint16_t *y, int64_t ldy,
                  int64_t M, int64_t N, int64_t K, void *workspace, size_t workspace_bytes,
                  void *stream);

/* ---------------------------------------------------------------- output exchange (f2)
 * Column-sharded ZipGEMM (north star) with the all-gather of the Y slices fused
 * into the GEMM (the paper leaves multi-GPU to the serving layer).
 * Rank r of `world` holds the W rows [col0, col0 + N) (a contiguous byte range of the
 * encoding, dist.shard_rows) and a full output Y_r [M][ldy].  zs_gemm_peer computes its
 * slice and STORES EVERY ELEMENT INTO ALL RANKS' Y (the epilogue writes the local copy and
 * the peers' copies through peer pointers over NVLink), then, once the whole grid's stores
 * are visible at system scope, writes `epoch` to flags[r][rank] for every r.  zs_peer_wait
 * on rank r then blocks its stream until flags[r][0..world) all reached `epoch`, after
 * which Y_r holds the full product.  No collective library call, no permute.
 *
 *   y[r], flags[r]: device pointers valid in the calling process -- the caller's own
 *     buffers for r == rank, CUDA-IPC-mapped (zs_ipc_open) or same-device buffers otherwise.
 *     flags[r] has `world` u32 words.  Caller-owned; the library keeps no state.
 *   epoch: a value the flags have not held since the previous wait (e.g. a step counter;
 *     the wait compares wrap-safely, flag - epoch >= 0 as int32).
 *   Reuse: the caller must not start a step that writes Y_r while rank r may still read
 *     the previous contents (double-buffer Y by epoch parity, or a barrier).
 * Large M (zs_gemm_is_decoupled): cuBLAS writes the local slice, then one copy kernel
 * broadcasts it and signals.  workspace: zs_gemm_peer_workspace_bytes = 256 B holding the
 * signalling launch's CTA counter, then zs_gemm's workspace; zero-filled once before first
 * use (the counter is self-cleaning; the rest follows zs_gemm_workspace_bytes). */
#define ZS_MAX_PEERS 8
#define ZS_IPC_HANDLE_BYTES 64
#define ZS_PEER_WAIT_TIMEOUT_NS 20000000000ull   /* zs_peer_wait traps after 20 s */

typedef struct {
    int32_t world;                    /* 1..ZS_MAX_PEERS                                  */
    int32_t rank;                     /* 0..world-1                                       */
    uint16_t *y[ZS_MAX_PEERS];        /* rank r's full Y [M][ldy] BF16 (device pointers)  */
    int64_t ldy;                      /* elements, >= col0 + N, the same on every rank    */
    int64_t col0;                     /* first Y column of this rank's slice              */
    uint32_t *flags[ZS_MAX_PEERS];    /* rank r's flag array, `world` u32 words           */
    uint32_t epoch;                   /* written to flags[r][rank] when the slice landed  */
} zs_peer_out;

size_t zs_gemm_peer_workspace_bytes(int64_t M, int64_t N, int64_t K);

/* Y_r[:, col0:col0+N] = X W^T for every rank r (see above).  x, w, M, N, K as zs_gemm (N =
 * this rank's shard rows).  Errors: as zs_gemm, plus ZS_ERR_INVALID_ARG (world / rank out
 * of range, null y[r] or flags[r]) and ZS_ERR_SHAPE (ldy < col0 + N). */
zs_status zs_gemm_peer(const uint16_t *x, int64_t ldx, const zs_tensor *w, const zs_peer_out *out,
                       int64_t M, int64_t N, int64_t K, void *workspace, size_t workspace_bytes,
                       void *stream);

/* Blocks `stream` until flags[0..world) (this rank's flag array, device memory) all reached
 * epoch (one 32-thread launch, acquire loads at system scope).  A flag that does not arrive
 * within ZS_PEER_WAIT_TIMEOUT_NS traps the kernel (the stream reports a launch failure)
 * instead of hanging.  Errors: ZS_ERR_INVALID_ARG, ZS_ERR_UNSUPPORTED, ZS_ERR_CUDA. */
zs_status zs_peer_wait(const uint32_t *flags, int32_t world, uint32_t epoch, void *stream);

/* CUDA IPC plumbing for zs_peer_out (host calls).  zs_ipc_get_handle: the handle
 * (ZS_IPC_HANDLE_BYTES opaque bytes) of the allocation holding dev_ptr and dev_ptr's byte
 * offset inside it.  zs_ipc_open (in ANOTHER process): map it; *base + offset is the peer's
 * dev_ptr.  zs_ipc_close: unmap.  Errors: ZS_ERR_INVALID_ARG, ZS_ERR_UNSUPPORTED, ZS_ERR_CUDA
 * (including opening a handle in the process that created it). */
zs_status zs_ipc_get_handle(const void *dev_ptr, void *handle, int64_t *offset);
zs_status zs_ipc_open(const void *handle, void **base);
zs_status zs_ipc_close(void *base);

/* GPU-side encoder: the same bytes as zs_encode_measure / zs_encode (Alg. 1,
 * P:306-333; canonical order S:277), computed on the device from a DEVICE matrix w (row-major,
 * leading dimension ld >= cols, BF16 bit patterns).  Kernels: exponent histogram, per-BlockTile
 * in-window counts, and one warp per BlockTile packing the bit-planes and the H / L segments;
 * the window choice and the offsets prefix run on the host over the copied-back counts.
 * Both calls are SYNCHRONOUS on `stream` (they return host-side sizes).  All output pointers
 * of zs_encode_device are device buffers with the capacities of `cap` (zs_encode_bound or the
 * exact sizes from zs_encode_measure_device); offsets receives n_blocktiles + 1 pairs.
 * ws: device scratch of zs_encode_device_workspace_bytes(rows, cols) bytes.
 * Errors: as zs_encode, plus ZS_ERR_CAPACITY (workspace), ZS_ERR_UNSUPPORTED, ZS_ERR_CUDA. */
size_t zs_encode_device_workspace_bytes(int64_t rows, int64_t cols);
zs_status zs_encode_measure_device(const uint16_t *w, int64_t rows, int64_t cols, int64_t ld, void *ws,
                                   size_t ws_bytes, void *stream, int32_t *base_exp, int64_t *covered,
                                   zs_sizes *exact);
zs_status zs_encode_device(const uint16_t *w, int64_t rows, int64_t cols, int64_t ld, int32_t base_exp,
                           const zs_sizes *cap, uint64_t *b1, uint64_t *b2, uint64_t *b3, uint8_t *h,
                           uint16_t *l, uint64_t *offsets, zs_sizes *actual, uint16_t *pad_word, void *ws,
                           size_t ws_bytes, void *stream);

/* Number of kernel launches the most recent successful zs_gemm / zs_decompress call on
 * this thread issued (for the bench's gpu_launches count). */
int zs_last_launch_count(void);

/* Human-readable name of a status code (static storage). */
const char *zs_status_string(zs_status s);

#ifdef __cplusplus
}
#endif
#endif /* ZS_H_ */
