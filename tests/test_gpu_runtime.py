"""GPU: the graphed serving executor (runtime.GraphedZipLinear) returns, for every step of a
replay, exactly the product of that step's host input -- integer inputs, so the expected
value is the fp64 oracle rounded to BF16 -- for the fused and the decoupled paths, over
repeated replays with new inputs written into the pinned slots."""
import numpy as np
import pytest

import oracle as O
import zs_inputs as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,K,M,S", [(1024, 512, 8, 4), (768, 320, 33, 3), (512, 256, 200, 5)])
def test_graphed_linear_steps_exact(N, K, M, S):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2603_17435_b200 as Z
    from paper_2603_17435_b200.runtime import GraphedZipLinear
    w = G.integer_weights(N, K, seed=61)
    lin = GraphedZipLinear(Z.encode(w).to("cuda:0"), M, steps=S)
    for rep in range(2):
        xs = [G.integer_activations(M, K, seed=100 * rep + j) for j in range(S)]
        for j, x in enumerate(xs):
            lin.x_host[j].copy_(torch.from_numpy(x.view(np.int16)).view(torch.bfloat16))
        lin.run()
        torch.cuda.synchronize()
        for j, x in enumerate(xs):
            got = lin.y_host[j].view(torch.int16).numpy().view(np.uint16)
            np.testing.assert_array_equal(got, O.round_bf16_array(O.gemm_f64(x, w)), err_msg=f"rep {rep} step {j}")
