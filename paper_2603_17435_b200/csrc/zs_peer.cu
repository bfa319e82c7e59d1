// zs_peer.cu -- output exchange for column-sharded ZipGEMM.
//
// Each rank owns the full output Y [M][N_total] and computes the column slice
// [col0, col0 + N_shard).  The fused path (zipgemm_kernel with npeer > 0) stores every
// BF16 element of the slice into all ranks' Y (peer memory over NVLink: CUDA-IPC-mapped or
// same-device pointers) from the epilogue and signals the ranks' flag arrays once the whole
// grid's stores are visible; no all-gather launch and no permute.  This file holds the two
// pieces outside the GEMM kernel:
//
//   peer_copy_kernel  the decoupled (large-M) path: cuBLAS writes the local slice, then this
//                     kernel broadcasts it to the peers (16-B vector copies when aligned)
//                     and signals, with the same last-CTA protocol as the fused epilogue.
//   peer_wait_kernel  one thread per rank: acquire-spin until that rank's flag reached the
//                     epoch, then the stream may read Y.  A watchdog traps after timeout_ns
//                     (a peer that never signals is an error, not a hang).
#include <cstdint>
#include <cuda_runtime.h>

#include "zs_device.cuh"
#include "zs_kernels.h"

namespace zs {

__global__ void __launch_bounds__(256) peer_copy_kernel(const PeerCopyParams p) {
  const int64_t rows = p.rows, cols = p.cols, ld = p.ld;
  const bool vec = ((reinterpret_cast<uintptr_t>(p.src) & 15u) == 0) && (ld % 8 == 0) && (cols % 8 == 0);
  bool dvec = vec;
#pragma unroll
  for (int i = 0; i < kMaxPeers; ++i)
    if (i < p.npeer) dvec = dvec && ((reinterpret_cast<uintptr_t>(p.dst[i]) & 15u) == 0);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  if (dvec) {
    const int64_t cv = cols / 8, total = rows * cv;
    for (int64_t i = tid; i < total; i += nthr) {
      const int64_t r = i / cv, c = (i - r * cv) * 8;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.src + r * ld + c));
#pragma unroll
      for (int k = 0; k < kMaxPeers; ++k)
        if (k < p.npeer) *reinterpret_cast<uint4*>(p.dst[k] + r * ld + c) = v;
    }
  } else {
    const int64_t total = rows * cols;
    for (int64_t i = tid; i < total; i += nthr) {
      const int64_t r = i / cols, c = i - r * cols;
      const uint16_t v = p.src[r * ld + c];
#pragma unroll
      for (int k = 0; k < kMaxPeers; ++k)
        if (k < p.npeer) p.dst[k][r * ld + c] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) signal_peers(p.done, p.flag, p.nflag, p.epoch, threadIdx.x);
}

__global__ void peer_wait_kernel(const uint32_t* flags, int n, uint32_t epoch, uint64_t timeout_ns) {
  // launched with programmatic stream serialization: the next kernel (the next layer's
  // ZipGEMM) may start its prologue and weight stream now; it reads outputs only after its
  // own griddepcontrol.wait, i.e. after this kernel -- and so every peer's slice -- is done
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int i = threadIdx.x;
  if (i < n) {
    const uint64_t t0 = globaltimer_now();
    while ((int32_t)(ld_acquire_sys(flags + i) - epoch) < 0) {
      __nanosleep(256);
      if (globaltimer_now() - t0 > timeout_ns) {
        printf("zs_peer_wait: flag %d = %u never reached epoch %u\n", i, ld_acquire_sys(flags + i), epoch);
        __trap();
      }
    }
  }
  __syncthreads();
  // this kernel may have started during the preceding GEMM's tail (PDL): complete only after
  // it (the flags already order its Y stores; this also covers the rest of the stream)
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

cudaError_t launch_peer_copy(const PeerCopyParams& p, int sms, cudaStream_t s) {
  const int64_t work = p.rows * p.cols / 8;
  int64_t grid = (work + 255) / 256;
  if (grid > 2LL * sms) grid = 2LL * sms;
  if (grid < 1) grid = 1;
  peer_copy_kernel<<<(unsigned)grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const uint32_t* flags, int n, uint32_t epoch, uint64_t timeout_ns, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, peer_wait_kernel, flags, n, epoch, timeout_ns);
}

}  // namespace zs
