"""One small zs_gemm (fused kernel, split-K fixup, M = 8 and M = 40) and one zs_decompress,
checked against the oracle: the target program of the compute-sanitizer tests
(tests/test_gpu_sanitizer.py).  Exits 0 on success."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2603_17435_b200 as Z  # noqa: E402
import zs_inputs as G  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    w = G.integer_weights(384, 640, seed=5)
    wd = Z.encode(w).to(dev)
    for M in (8, 40):
        x = G.integer_activations(M, 640, seed=M)
        xt = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev)
        y = Z.gemm(xt, wd).cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(y, O.round_bf16_array(O.gemm_f64(x, w))), f"gemm M={M}"
    d = Z.decompress(wd).cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(d, w), "decompress"
    torch.cuda.synchronize()
    print("sanitize target ok")


if __name__ == "__main__":
    main()
