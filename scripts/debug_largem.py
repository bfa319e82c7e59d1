"""Fused ZipGEMM at M > 128 (token chunks up to 256, one accumulator buffer): exactness check
on small integer problems, one M per process so a launch failure names its M."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O, paper_2603_17435_b200 as Z, zs_inputs as G
M = int(sys.argv[1]); N = int(sys.argv[2]) if len(sys.argv) > 2 else 512; K = int(sys.argv[3]) if len(sys.argv) > 3 else 512
L = Z.lib(); L.zs_debug_set_large_m.argtypes = [ctypes.c_longlong]; L.zs_debug_set_large_m(1 << 40)
w = G.integer_weights(N, K, seed=3); x = G.integer_activations(M, K, seed=4)
dev = torch.device("cuda:0")
y = Z.gemm(torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev), Z.encode(w).to(dev))
torch.cuda.synchronize()
y = y.cpu().view(torch.int16).numpy().view(np.uint16)
ok = np.array_equal(y, O.round_bf16_array(O.gemm_f64(x, w)))
print(f"M={M} N={N} K={K} exact={ok}", flush=True)
