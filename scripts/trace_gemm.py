"""Per-unit pipeline timeline of zipgemm_kernel (debug hook zs_debug_set_trace).

Needs the trace build:  python -m paper_2603_17435_b200.build --trace
                        ZS_LIB=paper_2603_17435_b200/libzs_trace.so python scripts/trace_gemm.py L M [flags]
Events: prod = stage issued, tick0/tick1 = ticket drawn (quarter 0/1), drN = stage data ready,
asN = A slot free, dqN = unit-quarter decoded, mma = MMAs issued.
"""
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
L.zs_debug_set_ring.argtypes = [ctypes.c_int]
if len(sys.argv) > 3:
    L.zs_debug_set_flags.argtypes = [ctypes.c_int]
    L.zs_debug_set_flags(int(sys.argv[3]))
for _ in range(3):
    Z.gemm(x, wd)
L.zs_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
Z.gemm(x, wd)
torch.cuda.synchronize()
L.zs_debug_set_trace(None)
t = tr.cpu().numpy().reshape(4, 128, 16).astype(np.int64)[:, :, :16]
names = ["prod", "tick0", "dq0", "dq1", "dq2", "dq3", "mma", "dr0", "dr1", "dr2", "dr3", "as0", "as1", "as2", "as3", "tick1"]
# summary over the first 4 CTAs: decode duration (slot-acquired -> done) and ticket->done
d1, d2 = [], []
for cta in range(4):
    for u in range(128):
        r = t[cta, u]
        for q in range(4):
            if r[2 + q] and r[11 + q]:
                d1.append(r[2 + q] - r[11 + q])
            if r[2 + q] and r[7 + q]:
                d2.append(r[2 + q] - r[7 + q])
if d1:
    print("decode (A slot ready -> done) cycles: mean %.0f  p10 %.0f  p90 %.0f" % (np.mean(d1), np.percentile(d1, 10), np.percentile(d1, 90)))
if d2:
    print("ticket -> done cycles: mean %.0f" % np.mean(d2))
for cta in range(4):
    r = t[cta]
    nz = r[r > 0]
    last_mma = r[:, 6].max()
    first = nz.min()
    n = int((r[:, 6] > 0).sum())
    print(f"CTA {cta}: units traced {n}, span first->last MMA {last_mma - first} cycles, per unit {(last_mma - first) / max(n, 1):.0f}")
for cta in range(1):
    base = t[cta][t[cta] > 0].min()
    print(f"CTA {cta}: times in cycles relative to first event")
    print("unit " + " ".join(f"{n:>8s}" for n in names))
    for u in range(0, 100):
        row = t[cta, u]
        if row.max() == 0:
            break
        print(f"{u:4d} " + " ".join(f"{(v - base) if v else -1:8d}" for v in row))
