"""Per-unit pipeline timeline of zipgemm_kernel (debug hook zs_debug_set_trace)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_17435_b200 as Z  # noqa: E402
import zs_inputs as G  # noqa: E402

layer = sys.argv[1] if len(sys.argv) > 1 else "L8B.GateUp"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 32
K, N = G.LAYERS[layer]
dev = torch.device("cuda:0")
w = G.gaussian_bf16(N, K, 0.02, 1)
wd = Z.encode(w).to(dev)
x = torch.randn(M, K, device=dev).to(torch.bfloat16)
tr = torch.zeros(4 * 128 * 16, dtype=torch.int64, device=dev)
L = Z.lib()
L.zs_debug_set_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    Z.gemm(x, wd)
L.zs_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
Z.gemm(x, wd)
torch.cuda.synchronize()
L.zs_debug_set_trace(None)
t = tr.cpu().numpy().reshape(4, 128, 16).astype(np.int64)[:, :, :7]
names = ["prod", "-", "dq0", "dq1", "dq2", "dq3", "mma"]
for cta in range(1):
    base = t[cta][t[cta] > 0].min()
    print(f"CTA {cta}: times in cycles relative to first event")
    print("unit " + " ".join(f"{n:>8s}" for n in names))
    for u in range(0, 24):
        row = t[cta, u]
        if row.max() == 0:
            break
        print(f"{u:4d} " + " ".join(f"{(v - base) if v else -1:8d}" for v in row))
