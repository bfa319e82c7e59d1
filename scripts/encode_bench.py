"""GPU encoder (zs_encode_device) vs host encoder (zs_encode, all host threads) on the 8B
layers: wall time per matrix (the device path includes its host syncs and the offsets scan)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_17435_b200 as Z  # noqa: E402
import zs_inputs as G  # noqa: E402

dev = torch.device("cuda:0")
for layer in (sys.argv[1] if len(sys.argv) > 1 else "L8B.QKV,L8B.O,L8B.GateUp,L8B.Down").split(","):
    K, N = G.LAYERS[layer]
    w = G.gaussian_bf16(N, K, 0.02, G.seed_of(layer))
    wd = torch.from_numpy(w.view(np.int16)).view(torch.bfloat16).to(dev)
    Z.encode_device(wd)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 5
    for _ in range(n):
        e = Z.encode_device(wd)
    torch.cuda.synchronize()
    gpu_ms = (time.perf_counter() - t0) * 1e3 / n
    t0 = time.perf_counter()
    hst = Z.encode(w)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    same = bool(np.array_equal(e.h.cpu().numpy().view(np.uint8)[: hst.h.size], hst.h))
    print(json.dumps({"layer": layer, "elements": int(w.size), "gpu_encode_ms": round(gpu_ms, 3),
                      "host_encode_ms": round(cpu_ms, 1), "host_threads": os.cpu_count(),
                      "gpu_gb_per_s_of_bf16_in": round(2 * w.size / gpu_ms / 1e6, 1), "h_equal": same}))
