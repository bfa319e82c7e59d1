"""B200-native ZipGEMM (arxiv 2603.17435): TCA-TBE weights decoded inside a tcgen05 GEMM.

Public API (all compute runs in libzs.so; see include/zs.h):
    encode(w_bf16_host)            -> ZsHost      Alg. 1 offline compressor (host C++)
    encode_device(w_bf16_cuda)     -> ZsDevice    the same bytes, computed on the GPU
    ZsHost.to(device)              -> ZsDevice
    decompress(ZsDevice)           -> bf16 [N][K]   ZipServ-Decomp (sm_100a)
    gemm(x, ZsDevice)              -> bf16 [M][N]   ZipGEMM, Y = X W^T (sm_100a, tcgen05)
    gemm_peer(x, shard, ys, flags, rank, col0, epoch)   column shard stored into every rank's Y
    peer_wait(flags, world, epoch)                        (fused output exchange, zs_gemm_peer)
    dist.ShardedZipLinear          column-sharded ZipGEMM + NCCL all-gather or the fused exchange
"""
from .zs import (ZsDevice, ZsError, ZsHost, decompress, encode, encode_device, gemm, gemm_peer,  # noqa: F401
                 ipc_close, ipc_handle, ipc_open, last_launch_count, lib, peer_wait, peer_workspace, workspace)

__all__ = ["encode", "encode_device", "decompress", "gemm", "gemm_peer", "peer_wait", "ZsHost", "ZsDevice", "ZsError",
           "lib", "workspace", "peer_workspace", "ipc_handle", "ipc_open", "ipc_close", "last_launch_count"]
