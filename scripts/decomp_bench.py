"""zs_decompress throughput on LLaMA-3.1-8B layer shapes (GB/s of compressed-in + bf16-out bytes)."""
import argparse
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
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--layers", default="L8B.QKV,L8B.O,L8B.GateUp,L8B.Down")
ap.add_argument("--dist", default="gaussian", choices=["gaussian", "realistic"])
a = ap.parse_args()
dev = torch.device("cuda:0")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
for layer in a.layers.split(","):
    K, N = G.LAYERS[layer]
    gen = G.realistic_bf16 if a.dist == "realistic" else G.gaussian_bf16
    w = gen(N, K, 0.02, seed=G.seed_of(layer))
    zh = Z.encode(w)
    R = max(2, math.ceil(3 * l2 / zh.nbytes()))
    ws = [zh.to(dev) for _ in range(R)]
    out = torch.empty((N, K), dtype=torch.bfloat16, device=dev)
    for i in range(3):
        Z.decompress(ws[i % R], out=out)
    torch.cuda.synchronize()
    ok = np.array_equal(out.cpu().view(torch.int16).numpy().view(np.uint16), w)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        Z.decompress(ws[i % R], out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    byts = zh.nbytes() + 2 * N * K
    print(json.dumps({"layer": layer, "dist": a.dist, "us": us, "gbs": byts / us / 1e3, "bit_exact": ok,
                      "compressed_mb": zh.nbytes() / 1e6}))
