"""B200-native ZipGEMM (arxiv 2603.17435): TCA-TBE weights decoded inside a tcgen05 GEMM.

Public API (all compute runs in libzs.so; see include/zs.h):
    encode(w_bf16_host)            -> ZsHost      Alg. 1 offline compressor (host C++)
    encode_device(w_bf16_cuda)     -> ZsDevice    the same bytes, computed on the GPU
    ZsHost.to(device)              -> ZsDevice
    decompress(ZsDevice)           -> bf16 [N][K]   ZipServ-Decomp (sm_100a)
    gemm(x, ZsDevice)              -> bf16 [M][N]   ZipGEMM, Y = X W^T (sm_100a, tcgen05)
    dist.ShardedZipLinear          column-sharded ZipGEMM + NCCL all-gather
"""
from .zs import (ZsDevice, ZsError, ZsHost, decompress, encode, encode_device, gemm, last_launch_count, lib,  # noqa: F401
                 workspace)

__all__ = ["encode", "encode_device", "decompress", "gemm", "ZsHost", "ZsDevice", "ZsError", "lib", "workspace",
           "last_launch_count"]
