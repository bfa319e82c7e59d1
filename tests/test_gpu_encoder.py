"""GPU parity of the device encoder against the CPU oracle encoder, byte by
byte (bit-planes, H, L, offsets incl. the sentinel, base_exp, pad_word), plus a round trip
through zs_decompress and the full-size 8B GateUp layer (sampled against the oracle's window
and sizes, and byte-equal to the host zs_encode)."""
import numpy as np
import pytest

import oracle as O
import zs_inputs as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def Z():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2603_17435_b200 as Zm
    Zm.lib()
    return Zm


def dev_bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(DEV)


def host(t, dtype):
    if t.dtype == torch.bfloat16:
        t = t.view(torch.int16)
    return t.cpu().numpy().view(dtype)


CASES = {
    "tiny_1x1": lambda: G.gaussian_bf16(1, 1, 0.02, 1),
    "odd_7x9": lambda: G.gaussian_bf16(7, 9, 0.005, 2),
    "specials_65x63": lambda: G.special_patterns(G.gaussian_bf16(65, 63, 0.1, 3)),
    "g300": lambda: G.gaussian_bf16(300, 300, 0.02, 4),
    "realistic_512x1024": lambda: G.realistic_bf16(512, 1024, seed=5),
    "all_patterns": G.all_patterns_256,
    "all_zero": lambda: np.zeros((64, 128), np.uint16),
    "integer_128x256": lambda: G.integer_weights(128, 256),
}


def check_equal(e, o):
    assert e.base_exp == o.base_exp and e.pad_word == o.pad_word
    np.testing.assert_array_equal(host(e.b1, np.uint64), o.B1)
    np.testing.assert_array_equal(host(e.b2, np.uint64), o.B2)
    np.testing.assert_array_equal(host(e.b3, np.uint64), o.B3)
    nh, nl = e.sizes["h_bytes"], e.sizes["l_words"]
    assert nh == o.H.size and nl == o.L.size
    np.testing.assert_array_equal(host(e.h, np.uint8)[:nh], o.H)
    np.testing.assert_array_equal(host(e.l, np.uint16)[:nl], o.L)
    off = host(e.offsets, np.uint64).reshape(-1, 2)
    np.testing.assert_array_equal(off[:-1], o.offsets)
    np.testing.assert_array_equal(off[-1], [o.H.size, 2 * o.L.size])


@pytest.mark.parametrize("case", sorted(CASES))
def test_device_encoder_byte_equal_to_oracle(Z, case):
    w = CASES[case]()
    e = Z.encode_device(dev_bf16(w))
    check_equal(e, O.encode(w))
    # and it decodes back to the input, bit for bit
    np.testing.assert_array_equal(host(Z.decompress(e), np.uint16), w)


def test_device_encoder_forced_base_exp(Z):
    w = G.gaussian_bf16(100, 130, 0.02, 7)
    for be in (-1, 0, 100, 248):
        check_equal(Z.encode_device(dev_bf16(w), base_exp=be), O.encode(w, base_exp=be))


def test_device_encoder_strided_input(Z):
    w = G.gaussian_bf16(96, 200, 0.02, 8)
    big = torch.zeros((96, 256), dtype=torch.bfloat16, device=DEV)
    big[:, :200] = dev_bf16(w)
    check_equal(Z.encode_device(big[:, :200]), O.encode(w))


def test_device_encoder_full_size_gateup(Z):
    K, N = G.LAYERS["L8B.GateUp"]
    w = G.gaussian_bf16(N, K, 0.02, G.seed_of("L8B.GateUp"))
    e = Z.encode_device(dev_bf16(w))
    hst = Z.encode(w)   # host encoder, itself byte-equal to the oracle (tests/test_abi_encode.py)
    assert e.base_exp == hst.base_exp == 115
    for a, b in ((e.b1, hst.b1), (e.b2, hst.b2), (e.b3, hst.b3)):
        np.testing.assert_array_equal(host(a, np.uint64), b)
    np.testing.assert_array_equal(host(e.h, np.uint8)[: hst.h.size], hst.h)
    np.testing.assert_array_equal(host(e.l, np.uint16)[: hst.l.size], hst.l)
    np.testing.assert_array_equal(host(e.offsets, np.uint64).reshape(-1, 2), hst.offsets)
    # the oracle's window on the same matrix (Alg. 1 line 3)
    start, cov = O.select_window(O.histogram(w))
    assert start - 1 == e.base_exp
