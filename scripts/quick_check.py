"""Fast exactness check of a libzs build (ZS_LIB=...) for A/B runs: integer weights and
activations (order-independent fp32 sums, so Y must equal RNE_bf16 of the exact integer
product bit for bit) on the fused path at the bench's launch shapes, plus one heavy-tailed
(realistic) case against a dense fp32 matmul.  Exact reference = numpy int64 matmul (no oracle)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2603_17435_b200 as Z  # noqa: E402
import zs_inputs as G  # noqa: E402

dev = torch.device("cuda:0")
ok = True
for (N, K, M) in [(1024, 4096, 32), (640, 1000, 17), (28672, 4096, 32), (4096, 14336, 1), (28672, 4096, 200),
                  (14336, 4096, 256), (6144, 4096, 8), (28672, 4096, 128), (14336, 4096, 96)]:
    w = G.integer_weights(N, K, seed=G.seed_of(f"qc.W{N}.{K}"))
    x = G.integer_activations(M, K, seed=G.seed_of(f"qc.X{M}.{K}"))
    wf = G.bf16_bits_to_fp32(w).astype(np.int64)
    xf = G.bf16_bits_to_fp32(x).astype(np.int64)
    exact = xf @ wf.T
    ref = torch.from_numpy(exact.astype(np.float64)).float().to(torch.bfloat16)
    xt = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev)
    y = Z.gemm(xt, Z.encode(w).to(dev))
    torch.cuda.synchronize()
    eq = torch.equal(y.cpu().view(torch.int16), ref.view(torch.int16))
    ok &= eq
    print(f"integer N={N} K={K} M={M}: {'exact' if eq else 'MISMATCH'}", flush=True)
w = G.realistic_bf16(4096, 4096, 0.02, seed=G.seed_of("qc.real"))
x = G.activations_bf16(32, 4096, seed=G.seed_of("qc.realx"))
xt = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev)
y = Z.gemm(xt, Z.encode(w).to(dev)).float().cpu().numpy()
wf, xf = G.bf16_bits_to_fp32(w).astype(np.float64), G.bf16_bits_to_fp32(x).astype(np.float64)
err = float(np.max(np.abs(y - xf @ wf.T) / np.maximum(np.abs(xf) @ np.abs(wf).T, 1e-30)))
ok &= err <= 1e-2
print(f"realistic 4096x4096 M=32: err {err:.2e}", flush=True)
print("QUICK_CHECK", "OK" if ok else "FAIL")
