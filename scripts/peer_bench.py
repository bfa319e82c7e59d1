"""Cost of the fused output exchange (f2) on ONE GPU: per-rank column shard of a layer,
zs_gemm (slice only) vs zs_gemm_peer storing the slice into `world` output buffers (the
own one + world-1 "peer" copies, here on the same device) + zs_peer_wait, vs zs_gemm +
NCCL-style all-gather emulated by world-1 device copies of the slice + the permute.
CUDA graphs (10 steps per graph), rotated weight copies; prints one JSON line per case.

On one GPU the peer stores go to local HBM, so this measures the epilogue / signalling
overhead and the launch count, not NVLink transfer time.
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_17435_b200 as Z  # noqa: E402
from paper_2603_17435_b200 import dist as D  # noqa: E402
import zs_inputs as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="L70B.QKV,L70B.O,L70B.GateUp,L70B.Down")
ap.add_argument("--ms", default="1,8,32")
ap.add_argument("--worlds", default="2,8")
ap.add_argument("--iters", type=int, default=100)
a = ap.parse_args()
dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
S = 10


def timeit(fn, n_rot):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    gs = []
    with torch.cuda.stream(s):
        for i in range(n_rot):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for j in range(S):
                    fn(i * S + j)
            gs.append(g)
    torch.cuda.current_stream(dev).wait_stream(s)
    for i in range(5):
        gs[i % n_rot].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        gs[i % n_rot].replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (a.iters * S)


for layer in a.layers.split(","):
    K, N = G.LAYERS[layer]
    w = G.gaussian_bf16(N, K, 0.02, G.seed_of(layer))
    full = Z.encode(w)
    for world in [int(v) for v in a.worlds.split(",")]:
        r0, r1 = D.shard_bounds(N, world, 0)
        sh = D.shard_rows(full, r0, r1)
        R = max(2, math.ceil(3 * l2 / sh.nbytes()))
        comp = [sh.to(dev) for _ in range(R)]
        ns = r1 - r0
        for M in [int(m) for m in a.ms.split(",")]:
            x = torch.randn((M, K), device=dev).to(torch.bfloat16)
            ysl = torch.empty((M, ns), dtype=torch.bfloat16, device=dev)
            ys = [torch.zeros((M, N), dtype=torch.bfloat16, device=dev) for _ in range(world)]
            flags = torch.zeros(world, dtype=torch.int32, device=dev)
            # only rank 0 runs here: pre-set the other ranks' flags far ahead so the wait passes
            flags[1:] = 1 << 30
            gath = torch.empty((world, M, ns), dtype=torch.bfloat16, device=dev)
            ws = Z.workspace(M, ns, K, dev)
            pws = Z.peer_workspace(M, ns, K, dev)
            epoch = [0]

            def plain(i):
                Z.gemm(x, comp[i % R], out=ysl, ws=ws)

            def peer(i):
                epoch[0] += 1
                Z.gemm_peer(x, comp[i % R], ys, [flags] * world, 0, r0, epoch[0], ldy=N, ws=pws)
                Z.peer_wait(flags, world, epoch[0])

            def signal_only(i):      # world 1: flags + wait, no peer copies
                epoch[0] += 1
                Z.gemm_peer(x, comp[i % R], [ysl], [flags], 0, 0, epoch[0], ldy=ns, ws=pws)
                Z.peer_wait(flags, 1, epoch[0])

            def peer_nowait(i):      # peer copies + signal, no wait kernel
                epoch[0] += 1
                Z.gemm_peer(x, comp[i % R], ys, [flags] * world, 0, r0, epoch[0], ldy=N, ws=pws)

            def gather(i):
                Z.gemm(x, comp[i % R], out=ysl, ws=ws)
                gath.copy_(ysl.unsqueeze(0).expand(world, M, ns))           # world-1 slices "received"
                ys[0].view(M, world, ns).copy_(gath.permute(1, 0, 2))        # permute to [M][N]

            t_plain = timeit(plain, R)
            t_peer = timeit(peer, R)
            t_gather = timeit(gather, R)
            t_sig = timeit(signal_only, R)
            t_nowait = timeit(peer_nowait, R)
            print(json.dumps({"layer": layer, "world": world, "M": M, "N_shard": ns, "K": K,
                              "us_gemm_slice": round(t_plain, 2), "us_gemm_peer_wait": round(t_peer, 2),
                              "us_gemm_copy_permute": round(t_gather, 2),
                              "us_signal_wait_w1": round(t_sig, 2), "us_peer_nowait": round(t_nowait, 2),
                              "peer_overhead_us": round(t_peer - t_plain, 2)}), flush=True)
