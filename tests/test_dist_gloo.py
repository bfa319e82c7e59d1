"""Multi-rank host logic of the column-sharded path on CPU (gloo, world_size 2).

Each rank slices its shard out of the full encoding (paper_2603_17435_b200.dist), the
oracle decodes the shard and computes its Y slice, and dist.gather_columns all-gathers
the slices; the result must equal the single-rank oracle product exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import zs_inputs as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_to_oracle(sh):
    return O.Encoded(sh.rows, sh.cols, sh.sizes["padded_rows"], sh.sizes["padded_cols"], sh.base_exp, sh.pad_word,
                     sh.b1, sh.b2, sh.b3, sh.h, sh.l, sh.offsets[:-1].copy())


def _worker(rank, world, port, N, K, M, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_17435_b200 as Z
        from paper_2603_17435_b200 import dist as D
        w = G.gaussian_bf16(N, K, 0.02, seed=42)
        x = G.activations_bf16(M, K, seed=43)
        full = Z.encode(w)
        r0, r1 = D.shard_bounds(N, world, rank)
        sh = D.shard_rows(full, r0, r1)
        assert sh.base_exp == full.base_exp
        wd = O.decode_sequential(_shard_to_oracle(sh))        # shard decodes to its rows
        assert np.array_equal(wd, w[r0:r1])
        y_local = torch.from_numpy(O.gemm_f64(x, wd))
        y = D.gather_columns(y_local, world)
        q.put((rank, bool(np.array_equal(y.numpy(), O.gemm_f64(x, w)))))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,K,M", [(512, 192, 3), (1024, 130, 1)])
def test_sharded_gemm_gloo_world2(N, K, M):
    from paper_2603_17435_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, K, M, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def test_shard_bounds_cover_and_align():
    from paper_2603_17435_b200 import dist as D
    for rows, world in [(28672, 8), (1280 * 8, 8), (4096, 4), (300, 2), (6144, 3)]:
        b = [D.shard_bounds(rows, world, r) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == rows
        for (a0, a1), (c0, _) in zip(b, b[1:]):
            assert a1 == c0 and a0 % 128 == 0


def _tables_worker(rank, world, port, q):
    # the fused exchange's host logic: IPC handles all-gathered over the group, one mapping
    # per distinct foreign allocation, own buffers by local address (fake handles on CPU)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_17435_b200 import dist as D
        # buffers 0 and 1 share an allocation (same handle, different offsets), 2 is its own
        mine = [(b"alloc%d-A" % rank, 0), (b"alloc%d-A" % rank, 4096), (b"alloc%d-B" % rank, 256)]
        local = [1000 * rank + 1, 1000 * rank + 2, 1000 * rank + 3]
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        calls = []

        def open_fn(h):
            calls.append(h)
            return 10 ** 6 * (1 + int(h[5:6])) + (0 if h.endswith(b"A") else 50000)

        tables, opened = D.peer_tables(rank, world, local, allh, open_fn)
        other = 1 - rank
        base = 10 ** 6 * (1 + other)
        ok = (tables[0] == [local[0] if r == rank else base for r in range(world)]
              and tables[1] == [local[1] if r == rank else base + 4096 for r in range(world)]
              and tables[2] == [local[2] if r == rank else base + 50256 for r in range(world)]
              and sorted(calls) == [b"alloc%d-A" % other, b"alloc%d-B" % other] and len(opened) == 2)
        q.put((rank, bool(ok)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_peer_tables_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tables_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res
