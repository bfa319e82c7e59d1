"""PCIe copy rates on the box: D2H / H2D of the bench's Y / X sizes (pinned), alone and
concurrently with ZipGEMM on another stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_17435_b200 as Z  # noqa: E402
import zs_inputs as G  # noqa: E402

dev = torch.device("cuda:0")
for nbytes in (262144, 1835008, 8 << 20):
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 50
        print(f"{name} {nbytes} B: {us:.1f} us, {nbytes / us / 1e3:.1f} GB/s")

K, N = G.LAYERS["L8B.GateUp"]
w = Z.encode(G.gaussian_bf16(N, K, 0.02, 1)).to(dev)
x = torch.randn((32, K), device=dev).to(torch.bfloat16)
y = torch.empty((32, N), dtype=torch.bfloat16, device=dev)
yh = torch.empty((32, N), dtype=torch.bfloat16).pin_memory()
y2 = torch.empty_like(y)
cs = torch.cuda.Stream(dev)
for mode in ("gemm", "d2h", "both"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        if mode in ("gemm", "both"):
            Z.gemm(x, w, out=y)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(cs):
                yh.copy_(y2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(cs)
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode}: {e0.elapsed_time(e1) * 1e3 / 50:.1f} us per iteration")
