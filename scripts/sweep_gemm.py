"""Quick timing sweep of zs_gemm (CUDA graphs, rotated weights) over layers / M / ring depth."""
import argparse
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_17435_b200 as Z  # noqa: E402
import zs_inputs as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="L8B.GateUp")
ap.add_argument("--ms", default="32")
ap.add_argument("--rings", default="")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--cublas", action="store_true")
ap.add_argument("--modes", default="auto", help="comma list of auto,fused,decoupled (forces the zs_gemm path)")
ap.add_argument("--flags", default="0", help="comma list of zs_debug_set_flags values (timing experiments)")
ap.add_argument("--graph-steps", type=int, default=1, help="GEMMs per captured graph (PDL needs >1)")
ap.add_argument("--pdl", default="1", help="comma list of 0/1: programmatic dependent launch")
ap.add_argument("--dist", default="gaussian", choices=["gaussian", "realistic"],
                help="weights: N(0, 0.02^2), or per-row sigma 0.02*2^U(-1,1) + 0.1%% outliers at 20 sigma")
a = ap.parse_args()
dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
L = Z.lib()
L.zs_debug_set_ring.argtypes = [ctypes.c_int]
L.zs_debug_set_large_m.argtypes = [ctypes.c_longlong]
L.zs_debug_set_flags.argtypes = [ctypes.c_int]
L.zs_debug_set_pdl.argtypes = [ctypes.c_int]
MODE_THR = {"auto": -1, "fused": 1 << 40, "decoupled": 0}


def timeit(fn, n_rot):
    for i in range(5):
        fn(i)
    gs = []
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.current_stream(dev).wait_stream(s)
    S = a.graph_steps
    for i in range(n_rot):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for j in range(S):
                fn(i + j)
        gs.append(g)
    for i in range(10):
        gs[i % n_rot].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        gs[i % n_rot].replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (a.iters * a.graph_steps)


for layer in a.layers.split(","):
    K, N = G.LAYERS[layer]
    w = (G.gaussian_bf16(N, K, 0.02, G.seed_of(layer)) if a.dist == "gaussian"
         else G.realistic_bf16(N, K, seed=G.seed_of(layer)))
    zh = Z.encode(w)
    R = max(2, math.ceil(3 * l2 / zh.nbytes()))
    comp = [zh.to(dev) for _ in range(R)]
    dense = None
    if a.cublas:
        wdd = torch.from_numpy(w.view(np.int16)).view(torch.bfloat16).to(dev)
        Rd = max(2, math.ceil(3 * l2 / (w.size * 2)))
        dense = [wdd.clone() for _ in range(Rd)]
    for M in [int(m) for m in a.ms.split(",")]:
        x = torch.randn((M, K), device=dev).to(torch.bfloat16)
        y = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        for mode, ring, fl, pdl in [(md, r, f, pd) for md in a.modes.split(",")
                                    for r in ([int(r) for r in a.rings.split(",")] if a.rings else [0])
                                    for f in [int(f) for f in a.flags.split(",")]
                                    for pd in [int(x) for x in a.pdl.split(",")]]:
            L.zs_debug_set_large_m(MODE_THR[mode])
            L.zs_debug_set_flags(fl)
            L.zs_debug_set_pdl(pdl)
            ws = Z.workspace(M, N, K, dev)
            if ring:
                L.zs_debug_set_ring(ring)
            us = timeit(lambda i: Z.gemm(x, comp[i % R], out=y, ws=ws), R)
            rec = {"layer": layer, "dist": a.dist, "M": M, "mode": mode, "ring": ring, "flags": fl, "pdl": pdl,
                   "graph_steps": a.graph_steps, "us": round(us, 2),
                   "bits_per_el": round(zh.bits_per_element(), 3), "coverage": round(zh.covered / w.size, 4),
                   "tflops": round(2 * M * N * K / us / 1e6, 1),
                   "gbs": round((zh.nbytes() + 2 * M * K + 2 * M * N) / us / 1e3, 1)}
            if dense is not None:
                cu = timeit(lambda i: torch.mm(x, dense[i % len(dense)].t(), out=y), len(dense))
                rec["cublas_us"] = round(cu, 2)
                rec["speedup"] = round(cu / us, 3)
            print(json.dumps(rec), flush=True)
            L.zs_debug_set_large_m(-1)
            L.zs_debug_set_flags(0)
