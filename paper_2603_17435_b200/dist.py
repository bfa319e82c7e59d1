"""Column sharding of a TCA-TBE weight + output all-gather (north star).

W [N][K] is split into contiguous row blocks (output features = columns of Y) at 128-row
band granularity.  Because BlockTiles are stored row-major (reading C6), a row block is a
contiguous byte range of B1/B2/B3/H/L; the shard keeps the full matrix's e_base (reading
C3), so 1-GPU and w-GPU runs decode identical bytes.  Each rank runs zs_gemm on its shard
with the replicated X and the slices Y_r [M][N/w] are all-gathered (NCCL over NVLink on
the GPU box; gloo in the CPU tests) and permuted to Y [M][N].

exchange="peer" replaces the all-gather: every rank maps every other
rank's Y buffers and flag array through CUDA IPC (handles exchanged over the process group),
zs_gemm_peer stores the slice into all ranks' Y from the GEMM epilogue and signals, and
zs_peer_wait blocks the stream until every rank's slice has landed.
"""
from __future__ import annotations

import numpy as np

from .zs import ZsHost

BAND = 128


def shard_bounds(rows: int, world: int, rank: int, granule: int = BAND):
    """[r0, r1) rows of `rank`: contiguous, `granule`-aligned, as even as possible."""
    ngr = (rows + granule - 1) // granule
    g0 = rank * ngr // world
    g1 = (rank + 1) * ngr // world
    return min(rows, g0 * granule), min(rows, g1 * granule)


def shard_rows(zh: ZsHost, r0: int, r1: int) -> ZsHost:
    """Slice rows [r0, r1) (r0 % 64 == 0; r1 % 64 == 0 or r1 == rows) out of an encoding."""
    assert r0 % 64 == 0 and (r1 % 64 == 0 or r1 == zh.rows) and 0 <= r0 < r1 <= zh.rows
    nbc = zh.sizes["padded_cols"] // 64
    br0, br1 = r0 // 64, (r1 + 63) // 64
    bt0, bt1 = br0 * nbc, br1 * nbc
    off = zh.offsets.astype(np.int64)
    h0, h1 = off[bt0, 0], off[bt1, 0]
    l0, l1 = off[bt0, 1] // 2, off[bt1, 1] // 2
    new_off = (off[bt0: bt1 + 1] - off[bt0]).astype(np.uint64)
    seg = np.diff(new_off.astype(np.int64), axis=0)
    rows = r1 - r0
    sizes = dict(zh.sizes)
    sizes.update(rows=rows, padded_rows=(br1 - br0) * 64, n_fragtiles=(bt1 - bt0) * 64, n_blocktiles=bt1 - bt0,
                 h_bytes=int(h1 - h0), l_words=int(l1 - l0),
                 max_h_seg_bytes=int(seg[:, 0].max()), max_l_seg_bytes=int(seg[:, 1].max()))
    return ZsHost(sizes, zh.base_exp, zh.pad_word, -1, zh.b1[bt0 * 64: bt1 * 64].copy(),
                  zh.b2[bt0 * 64: bt1 * 64].copy(), zh.b3[bt0 * 64: bt1 * 64].copy(), zh.h[h0:h1].copy(),
                  zh.l[l0:l1].copy(), new_off)


def gather_columns(y_local, world: int, group=None):
    """all-gather Y_r [M][N/w] from every rank -> Y [M][N] (equal shard widths)."""
    import torch
    import torch.distributed as dist
    M, nw = y_local.shape
    buf = torch.empty((world * M, nw), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather_into_tensor(buf, y_local.contiguous(), group=group)
    buf = buf.view(world, M, nw)
    if M == 1:
        return buf.view(1, world * nw)
    return buf.permute(1, 0, 2).reshape(M, world * nw)


def peer_tables(rank: int, world: int, local_addrs, all_handles, open_fn):
    """Address tables of the fused exchange from the all-gathered IPC handles (host logic).

    local_addrs: this rank's own buffer addresses (one per exchanged buffer).
    all_handles[r][j] = (handle bytes, byte offset) of rank r's buffer j.
    open_fn(handle) -> base address in this process; called once per distinct handle of
    another rank (buffers sharing an allocation share its mapping).
    Returns (tables[j][r] = address of rank r's buffer j in this process, opened bases).
    """
    assert len(all_handles) == world
    nbuf = len(local_addrs)
    opened = {}
    tables = [[0] * world for _ in range(nbuf)]
    for r in range(world):
        assert len(all_handles[r]) == nbuf
        for j, (h, off) in enumerate(all_handles[r]):
            if r == rank:
                tables[j][r] = local_addrs[j]
                continue
            if h not in opened:
                opened[h] = open_fn(h)
            tables[j][r] = opened[h] + off
    return tables, list(opened.values())


class PeerOutputs:
    """The symmetric output buffers of the fused exchange: on every rank, `nbuf` full outputs
    Y [M][N] (double-buffered by step parity, so a rank that runs ahead never overwrites an
    output a slower rank may still read) and one flag array [world] u32, mapped into every
    other rank's address space by CUDA IPC."""

    def __init__(self, M: int, N: int, rank: int, world: int, device, group=None, nbuf: int = 2):
        import torch
        import torch.distributed as dist
        from . import zs as Z
        self.rank, self.world, self.M, self.N = rank, world, M, N
        self.y = [torch.zeros((M, N), dtype=torch.bfloat16, device=device) for _ in range(nbuf)]
        self.flags = torch.zeros(world, dtype=torch.int32, device=device)
        mine = [Z.ipc_handle(t) for t in self.y + [self.flags]]
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        local = [t.data_ptr() for t in self.y + [self.flags]]
        tables, self._opened = peer_tables(rank, world, local, allh, Z.ipc_open)
        self.y_tables, self.flag_table = tables[:nbuf], tables[nbuf]
        dist.barrier(group=group)

    def close(self):
        from . import zs as Z
        for b in self._opened:
            Z.ipc_close(b)
        self._opened = []


class ShardedZipLinear:
    """Y = X W^T with W column-sharded over the ranks of the default process group.

    exchange="nccl": zs_gemm on the shard, all_gather_into_tensor + permute.
    exchange="peer": zs_gemm_peer (epilogue stores into every rank's Y over NVLink, flags)
    + zs_peer_wait; M is fixed at construction (the exchanged buffers are [M][N])."""

    def __init__(self, zh_full: ZsHost, rank: int, world: int, device, exchange: str = "nccl", M: int | None = None,
                 group=None):
        self.rank, self.world = rank, world
        self.r0, self.r1 = shard_bounds(zh_full.rows, world, rank)
        widths = {shard_bounds(zh_full.rows, world, r)[1] - shard_bounds(zh_full.rows, world, r)[0]
                  for r in range(world)}
        assert exchange == "peer" or len(widths) == 1, "the all-gather needs equal shard widths"
        self.host = shard_rows(zh_full, self.r0, self.r1)
        self.dev = self.host.to(device)
        self.N = zh_full.rows
        self.exchange = exchange
        self.step = 0
        if exchange == "peer":
            assert M is not None, "exchange='peer' needs M"
            self.peer = PeerOutputs(M, self.N, rank, world, device, group=group)
        else:
            assert exchange == "nccl", exchange

    def __call__(self, x):
        from .zs import gemm, gemm_peer, peer_wait
        if self.exchange == "peer":
            # the exchanged buffers are [M][N] on every rank: a larger x would make every
            # rank's epilogue store past the end of its peers' IPC-mapped outputs
            assert x.shape[0] == self.peer.M, f"exchange='peer' was built for M={self.peer.M}, got {x.shape[0]}"
            self.step += 1
            b = self.step % len(self.peer.y)
            gemm_peer(x, self.dev, self.peer.y_tables[b], self.peer.flag_table, self.rank, self.r0, self.step,
                      ldy=self.N)
            peer_wait(self.peer.flags, self.world, self.step)
            return self.peer.y[b]
        y_local = gemm(x, self.dev)
        if self.world == 1:
            return y_local
        return gather_columns(y_local, self.world)
