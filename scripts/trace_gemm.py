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
names = ["prod", "-", "dq0", "dq1", "dq2", "dq3", "mma", "dr0", "dr1", "dr2", "dr3", "as0", "as1", "as2", "as3", "-"]
# per unit-quarter (static assignment: decoder warp jd of quarter q takes units jd, jd+4, ...):
#   dr = stage data ready (after the full-barrier wait), as = A slot free (scan + row table done,
#   afree waited), dq = decoded and published
scan, rows, gap = [], [], []
for cta in range(4):
    for u in range(128):
        r = t[cta, u]
        for q in range(4):
            if r[7 + q] and r[11 + q] and r[2 + q]:
                scan.append(r[11 + q] - r[7 + q])
                rows.append(r[2 + q] - r[11 + q])
            if u + 4 < 128 and r[2 + q] and t[cta, u + 4][7 + q]:
                gap.append(t[cta, u + 4][7 + q] - r[2 + q])
# (round 2 loop: the data wait of unit u + 4 happens between the two row passes of unit u, so
# dr(u + 4) < dq(u); the unit period per warp is as(u + 4) - as(u), the gap dq(u) -> as(u + 4)
# is the publish + afree wait)
period, gap2 = [], []
for cta in range(4):
    for u in range(124):
        r, n = t[cta, u], t[cta, u + 4]
        for q in range(4):
            if r[11 + q] and n[11 + q]:
                period.append(n[11 + q] - r[11 + q])
            if r[2 + q] and n[11 + q]:
                gap2.append(n[11 + q] - r[2 + q])
for name, d in (("scan+afree (dr->as)", scan), ("rows (as->dq)", rows), ("next unit wait (dq->dr')", gap),
                ("unit period (as->as')", period), ("publish+afree (dq->as')", gap2)):
    if d:
        print("%-26s cycles: mean %6.0f  p10 %6.0f  p50 %6.0f  p90 %6.0f" % (name, np.mean(d), np.percentile(d, 10),
                                                                            np.percentile(d, 50), np.percentile(d, 90)))
for cta in range(1):
    r = t[cta]
    t0 = r[r > 0].min()
    for u in range(0, 24):
        print("u%3d " % u + " ".join("%s=%7d" % (names[e], r[u, e] - t0) for e in (0, 6, 7, 11, 2) if r[u, e]))
