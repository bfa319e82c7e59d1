"""Timing experiments with the zs_debug_set_flags knobs (results are wrong under flags)."""
import ctypes, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2603_17435_b200 as Z  # noqa: E402
import zs_inputs as G  # noqa: E402

dev = torch.device("cuda:0")
L = Z.lib()
L.zs_debug_set_flags.argtypes = [ctypes.c_int]
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
layers = (sys.argv[1] if len(sys.argv) > 1 else "L8B.GateUp").split(",")
FLAGS = [int(f) for f in (sys.argv[2] if len(sys.argv) > 2 else "0,4,2,6,1,5").split(",")]
MS = [int(m) for m in (sys.argv[3] if len(sys.argv) > 3 else "1,32").split(",")]
DIST = sys.argv[sys.argv.index("--dist") + 1] if "--dist" in sys.argv else "gaussian"
for layer in layers:
  K, N = G.LAYERS[layer]
  gen = G.realistic_bf16 if DIST == "realistic" else G.gaussian_bf16
  zh = Z.encode(gen(N, K, 0.02, seed=G.seed_of(layer)))
  R = max(2, math.ceil(3 * l2 / zh.nbytes()))
  comp = [zh.to(dev) for _ in range(R)]
  for M in MS:
    x = torch.randn((M, K), device=dev).to(torch.bfloat16)
    y = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    ws = Z.workspace(M, N, K, dev)
    for flags in FLAGS:
        L.zs_debug_set_flags(flags)
        for i in range(3):
            Z.gemm(x, comp[i % R], out=y, ws=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 100
        e0.record()
        for i in range(n):
            Z.gemm(x, comp[i % R], out=y, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"layer": layer, "mb": round(zh.nbytes() / 1e6, 1), "M": M, "flags": flags, "dist": DIST, "us": round(e0.elapsed_time(e1) * 1e3 / n, 2)}), flush=True)
    L.zs_debug_set_flags(0)
    ws.zero_()
