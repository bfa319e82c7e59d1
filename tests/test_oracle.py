"""Pins for the CPU oracle (oracle/), checked against what the paper and the mathematics fix.

Every expected value here comes from PAPER.md / SPEC.md text (cited), from a closed form,
from brute force on tiny inputs, from an independent library routine (numpy), or from an
invariant -- never from the oracle itself and never from the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import zs_inputs as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- bf16 fields
def test_split_fields_examples():
    assert O.split_fields(0x3F80) == (0, 127, 0)      # 1.0
    assert O.split_fields(0x8000) == (1, 0, 0)        # -0.0
    assert O.split_fields(0x7FC0) == (0, 255, 64)     # qNaN


def test_assemble_fields_examples():
    assert O.assemble_fields(0, 120, 0x40) == 0x3C40
    assert O.assemble_fields(1, 128, 0) == 0xC000     # -2.0
    with pytest.raises(ValueError):
        O.assemble_fields(0, 256, 0)


def test_fields_exhaustive_against_numpy():
    # every pattern: split -> value matches numpy's IEEE interpretation of the bits
    w = np.arange(65536, dtype=np.uint32)
    f32 = (w << 16).view(np.float32)
    for bits in range(0, 65536, 97):
        s, e, m = O.split_fields(bits)
        assert O.assemble_fields(s, e, m) == bits
        v = O.bf16_to_double(bits)
        ref = float(f32[bits])
        if math.isnan(ref):
            assert math.isnan(v)
        else:
            assert v == ref and math.copysign(1, v) == math.copysign(1, ref)


def test_pack_sm_bijection():
    seen = set()
    for s in (0, 1):
        for m in range(128):
            b = O.pack_sm(s, m)
            assert (b >> 7, b & 0x7F) == (s, m)
            seen.add(b)
    assert len(seen) == 256
    assert O.pack_sm(1, 0x7F) == 0xFF and O.pack_sm(0, 0) == 0x00


# ----------------------------------------------------------------- Phase I (Alg. 1)
def test_histogram_example():
    c = O.histogram(np.array([0x3F80, 0x3F80, 0xC000], np.uint16))
    assert c[127] == 2 and c[128] == 1 and c.sum() == 3


def test_window_examples():
    c = np.zeros(256, np.int64)
    c[127] = 10
    assert O.select_window(c) == (121, 10)                            # S:125, smallest start
    c = np.zeros(256, np.int64)
    c[10:17] = 5
    assert O.select_window(c) == (10, 35)
    with pytest.raises(ValueError):
        O.select_window(np.zeros(256, np.int64))


def test_window_brute_force_random():
    rng = np.random.default_rng(0)
    for _ in range(200):
        c = rng.integers(0, 50, 256) * (rng.random(256) < 0.3)
        if c.sum() == 0:
            continue
        sums = np.convolve(c, np.ones(7, np.int64), mode="valid")     # 250 windows
        start, cov = O.select_window(c)
        assert cov == sums.max() and start == int(np.argmax(sums))   # argmax = first max


def test_gaussian_sigma002_window_base115():
    # worked example base 115; sigma = 0.02 Gaussian gives window E = [116, 122]
    w = G.gaussian_bf16(256, 256, 0.02, seed=0)
    start, cov = O.select_window(O.histogram(w))
    assert start - 1 == gold("paper_numbers.json")["sigma002_base_exp"]
    assert cov / w.size > 0.95                                         # "top-7 > 95%"


# ----------------------------------------------------------------- tiling
def test_coords_examples():
    assert O.coords_of(0, 0, 0, 0, 0) == (0, 0)
    assert O.coords_of(0, 0, 0, 1, 0) == (8, 0)                       # frag 1 = row offset 8
    assert O.coords_of(0, 0, 0, 2, 0) == (0, 8)                       # column-major 2x2 grid
    assert O.coords_of(0, 0, 1, 0, 0) == (0, 16)                      # TCT row-major
    assert O.coords_of(0, 0, 4, 0, 0) == (16, 0)
    assert O.coords_of(0, 0, 0, 0, 9) == (1, 1)                       # pos = row*8 + col


def test_coords_bijection_128x192():
    seen = set()
    for br in range(2):
        for bc in range(3):
            for t in range(16):
                for f in range(4):
                    for p in range(64):
                        seen.add(O.coords_of(br, bc, t, f, p))
    assert seen == {(r, c) for r in range(128) for c in range(192)}


# ----------------------------------------------------------------- Phase II layout pins
def test_encode_all_ones_8x8():
    # 8x8 of 1.0 -> window [121,127], base 120, codes 7, H = 64 x 0x00, L empty.
    w = np.full((8, 8), 0x3F80, np.uint16)
    e = O.encode(w)
    assert e.base_exp == 120 and e.pad_word == (121 << 7)
    ones = np.uint64(0xFFFFFFFFFFFFFFFF)
    assert e.B1[0] == ones and e.B2[0] == ones and e.B3[0] == ones    # code 7 = 111
    # padding: pad_word exponent 121 -> code 1 in the 63 padded FragTiles
    assert np.all(e.B1[1:] == ones) and np.all(e.B2[1:] == 0) and np.all(e.B3[1:] == 0)
    assert np.all(e.H == 0) and e.H.size == 4096 and e.L.size == 0  # C11: padding wins
    assert e.n_fragtiles == 64 and e.n_blocktiles == 1


def test_encode_bit_order_and_planes():
    # all 1.0 except (0,1) = 2.0 -> window [122,128] (covers all), base 121:
    # 1.0 -> c = 6 (110), 2.0 -> c = 7 (111); B1 holds the codeword LSB (Alg. 1 l.12),
    # bit index = row*8 + col, LSB first -> B1[0] == 0b10.
    w = np.full((64, 64), 0x3F80, np.uint16)
    w[0, 1] = 0x4000
    e = O.encode(w)
    assert e.base_exp == 121
    assert e.B1[0] == 0b10 and e.B2[0] == 0xFFFFFFFFFFFFFFFF and e.B3[0] == 0xFFFFFFFFFFFFFFFF
    # -1.5 = 0xBFC0: sign 1, exponent 127, mantissa 0x40 -> H byte 0xC0
    w[0, 0] = 0xBFC0
    e = O.encode(w)
    assert e.H[0] == 0xC0 and e.H[1] == 0x00


def test_encode_fallback_goes_to_L_verbatim():
    w = np.full((64, 64), 0x3F80, np.uint16)
    w[9, 3] = 0x7FC0       # NaN, exponent 255 outside the window
    w[63, 63] = 0x0001     # subnormal
    e = O.encode(w)
    assert list(e.L[:2]) == [0x7FC0, 0x0001]
    # (9,3): TCT 0, FragTile 1 (rows 8-15, column-major), pos 1*8+3 = 11
    M1 = int(e.B1[1] | e.B2[1] | e.B3[1])
    assert M1 == (0xFFFFFFFFFFFFFFFF ^ (1 << 11))
    # per-FragTile invariant: popc(M) H bytes, 64 - popc(M) L words
    Ms = e.B1 | e.B2 | e.B3
    nh = sum(bin(int(m)).count("1") for m in Ms)
    assert nh == 4096 - 2 and e.H.size == 4096 and e.L.size == 8    # L padded to 16 B


def test_offsets_and_alignment():
    w = G.gaussian_bf16(130, 200, 0.02, seed=4)
    e = O.encode(w)
    assert e.padded_rows == 192 and e.padded_cols == 256
    off = e.offsets.astype(np.int64)
    assert np.all(off % 16 == 0)
    assert np.all(np.diff(off[:, 0]) >= 0) and np.all(np.diff(off[:, 1]) >= 0)
    # H segment length of each BlockTile = sum of popc over its 64 FragTiles, padded to 16
    Ms = (e.B1 | e.B2 | e.B3).reshape(-1, 64)
    ends = np.append(off[1:, 0], e.H.size)
    for bt in range(e.n_blocktiles):
        nh = sum(bin(int(m)).count("1") for m in Ms[bt])
        assert ends[bt] - off[bt, 0] == (nh + 15) // 16 * 16


# ----------------------------------------------------------------- round trips
ROUNDTRIP_DIMS = [(1, 1), (7, 9), (64, 64), (65, 63), (300, 300)]


@pytest.mark.parametrize("sigma", [0.005, 0.02, 0.1])
@pytest.mark.parametrize("dims", ROUNDTRIP_DIMS)
def test_roundtrip_gaussian_with_specials(sigma, dims):
    w = G.special_patterns(G.gaussian_bf16(*dims, sigma, seed=hash(dims) & 0xFFFF), 0.05)
    e = O.encode(w)
    np.testing.assert_array_equal(O.decode_sequential(e), w)
    np.testing.assert_array_equal(O.decode_lanes(e), w)


def test_roundtrip_all_65536_patterns():
    w = G.all_patterns_256()
    e = O.encode(w)
    assert e.base_exp == -1                 # all counts equal -> start 0 (C4)
    np.testing.assert_array_equal(O.decode_sequential(e), w)
    np.testing.assert_array_equal(O.decode_lanes(e), w)
    r = 7 * 256 / 65536
    assert abs(e.H.size - r * 65536) <= 16 * e.n_blocktiles


def test_roundtrip_all_zero_and_edge_windows():
    z = np.zeros((64, 64), np.uint16)
    e = O.encode(z)
    assert e.base_exp == -1 and np.all(e.B1 == 0xFFFFFFFFFFFFFFFF)   # code 1 -> exponent 0
    np.testing.assert_array_equal(O.decode_lanes(e), z)
    # window touching exponent 255 (base 248): Inf/NaN are then in-window
    w = np.full((64, 64), 0x7F80, np.uint16)
    w[::2] = 0x7FC0
    e = O.encode(w, base_exp=248)
    assert e.L.size == 0
    np.testing.assert_array_equal(O.decode_sequential(e), w)
    np.testing.assert_array_equal(O.decode_lanes(e), w)
    with pytest.raises(ValueError):
        O.encode(w, base_exp=249)


def test_all_fallback_matrix():
    w = G.gaussian_bf16(64, 128, 0.02, seed=9)
    e = O.encode(w, base_exp=-1)             # window [0, 6]: every weight misses
    assert e.H.size == 0 and e.L.size == w.size
    np.testing.assert_array_equal(O.decode_lanes(e), w)


# ----------------------------------------------------------------- Alg. 2 worked examples
def test_alg2_worked_example_compressed():
    g = gold("alg2_worked_example.json")
    bit, code, base = g["bit_compressed"], g["codeword"], g["base_exp"]
    # planes give 101 at bit 38; all other bits in-window with code 1
    B1 = 0xFFFFFFFFFFFFFFFF
    B2 = 0
    B3 = 1 << bit
    H = np.arange(64, dtype=np.uint8) | 0x80       # sign 1, mantissa = H index
    w0, _ = O.decode_lane(B1, B2, B3, H, 0, 64, [], 0, 0, base, g["thread_compressed"])
    s, e, m = O.split_fields(w0)
    assert e == g["exponent"] == base + code       # 115 + 5 = 120
    assert m == bit and s == 1                      # idx_H = #ones in bits [0, 37] = 38


def test_alg2_worked_example_fallback():
    g = gold("alg2_worked_example.json")
    rng = np.random.default_rng(7)
    for _ in range(50):
        M = int(rng.integers(0, 2 ** 63)) & ~(1 << g["bit_fallback"])
        zeros_before = sum(1 for b in range(g["bit_fallback"]) if not (M >> b) & 1)
        nh = bin(M).count("1")
        L = np.arange(64, dtype=np.uint16) + 0x1000
        H = np.zeros(64, np.uint8)
        w0, _ = O.decode_lane(M, 0, 0, H, 0, nh, L, 0, 64 - nh, 115, g["thread_fallback"])
        assert w0 == 0x1000 + zeros_before          # count of 0s in bits [0, 11]


def test_alg2_all_ones_lane19():
    # M = all ones, c = 3 everywhere: lane 19, k=0 -> idx_H = 38
    H = np.arange(64, dtype=np.uint8)
    w0, w1 = O.decode_lane(2 ** 64 - 1, 2 ** 64 - 1, 0, H, 0, 64, [], 0, 0, 100, 19)
    assert (w0 & 0x7F) == 38 and (w1 & 0x7F) == 39 and ((w0 >> 7) & 0xFF) == 103


def test_alg2_mask_zero_and_full():
    L = np.arange(64, dtype=np.uint16) * 3 + 1
    for lane in range(32):                      # M = 0 -> output = L verbatim
        assert O.decode_lane(0, 0, 0, [], 0, 0, L, 0, 64, 50, lane) == (L[2 * lane], L[2 * lane + 1])


def test_lane_equals_sequential_random_fragments():
    # SPEC acceptance #2, >= 1e4 random fragments: 160 BlockTiles x 64 FragTiles
    rng = np.random.default_rng(11)
    w = rng.integers(0, 65536, size=(640, 1024), dtype=np.uint64).astype(np.uint16)
    mask = rng.random(w.shape) < 0.7            # ~70% Gaussian (in-window), the rest raw patterns
    g = G.gaussian_bf16(640, 1024, 0.02, 2)
    w[mask] = g[mask]
    e = O.encode(w)
    assert e.n_fragtiles >= 10_000
    np.testing.assert_array_equal(O.decode_lanes(e), O.decode_sequential(e))


# ----------------------------------------------------------------- size accounting
def test_average_bits_paper_numbers():
    g = gold("paper_numbers.json")
    assert abs(O.average_bits(3, g["r3_llama"]) - g["avgbits_3"]) < 0.05
    assert abs(O.average_bits(2, 0.70) - g["avgbits_2"]) < 1e-9
    assert abs(O.average_bits(4, 0.9875) - g["avgbits_4"]) < 1e-9
    assert O.average_bits(3, 1.0) == 11.0


def test_payload_fragtile_counts():
    # one BlockTile, every element in-window -> 11.0 b/el + offsets
    e = O.encode(np.full((64, 64), 0x3F80, np.uint16))
    assert e.payload_bits() == 64 * (192 + 512) + 128
    # all fallback -> 19.0 b/el + offsets
    e = O.encode(np.full((64, 64), 0x3F80, np.uint16), base_exp=0)
    assert e.payload_bits() == 64 * (192 + 1024) + 128


def test_compression_accounting_4096():
    # SPEC acceptance #6: bits/el = AverageBits(3, r) + overhead, overhead <= 0.2; size <= 0.73x
    w = G.gaussian_bf16(4096, 4096, 0.02, seed=1234)
    e = O.encode(w)
    start, cov = O.select_window(O.histogram(w))
    r = cov / w.size
    overhead = e.bits_per_element() - O.average_bits(3, r)
    assert 0 <= overhead <= 0.2
    assert e.payload_bits() / (16 * w.size) <= 0.73


# ----------------------------------------------------------------- fp64 GEMM
def test_gemm_identity_zero_and_numpy():
    x = G.activations_bf16(8, 64, seed=3)
    eye = np.zeros((64, 64), np.uint16)
    np.fill_diagonal(eye, 0x3F80)
    np.testing.assert_array_equal(O.gemm_f64(x, eye), O.bf16_array_to_double(x))
    assert np.all(O.gemm_f64(x, np.zeros((32, 64), np.uint16)) == 0)
    w = G.gaussian_bf16(48, 64, 0.02, 5)
    ref = O.bf16_array_to_double(x) @ O.bf16_array_to_double(w).T                   # numpy BLAS
    np.testing.assert_allclose(O.gemm_f64(x, w), ref, rtol=1e-13, atol=1e-15)
    cols = np.array([0, 7, 47])
    np.testing.assert_allclose(O.gemm_f64_cols(x, w, cols), ref[:, cols], rtol=1e-13, atol=1e-15)


def test_gemm_integer_exact():
    x = G.integer_activations(4, 300, seed=1)
    w = G.integer_weights(20, 300, seed=2)
    xi = G.bf16_bits_to_fp32(x).astype(np.int64)
    wi = G.bf16_bits_to_fp32(w).astype(np.int64)
    assert np.array_equal(O.gemm_f64(x, w), (xi @ wi.T).astype(np.float64))


def test_round_bf16_against_numpy():
    rng = np.random.default_rng(0)
    v = (rng.standard_normal(3000) * 10.0 ** rng.integers(-40, 38, 3000)).astype(np.float32)
    v = np.concatenate([v, np.float32([0.0, -0.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1e-40, -3e38])])
    ref = G.fp32_to_bf16_bits(v)                      # fp32-exact inputs: no double rounding
    got = O.round_bf16_array(v.astype(np.float64))
    np.testing.assert_array_equal(got, ref)
    assert O.round_bf16(1.0 + 2 ** -8) == 0x3F80      # tie -> even
    assert O.round_bf16(1.0 + 3 * 2 ** -8) == 0x3F82


# ----------------------------------------------------------------- CI model
def test_ci_degradation_paper_numbers():
    g = gold("paper_numbers.json")
    MK, CR = g["ci_MK"], g["ci_cr"]
    for n, pct in g["ci_degradation_pct"].items():
        N = int(n)
        d = 100 * (1 - O.ci_decoupled(MK, N, MK, CR) / O.ci_gemm(MK, N, MK))
        assert math.floor(d * 10) / 10 == pytest.approx(pct, abs=1e-9)   # printed truncated (C19)
        assert abs(d - pct) < 0.1
        gain = O.ci_fused(MK, N, MK, CR) / O.ci_gemm(MK, N, MK) - 1
        assert abs(gain - g["fused_gain_approx"]) < 0.02
    assert O.ci_gemm(4096, 8, 4096) == pytest.approx(7.9688, abs=1e-4)
    assert O.ci_decoupled(4096, 8, 4096, 1.51) == pytest.approx(3.001, abs=1e-3)
    assert O.ci_gemm(1, 1, 1) == pytest.approx(1 / 3)
    assert O.ci_fused(64, 8, 64, 1.0) == pytest.approx(O.ci_gemm(64, 8, 64))


# ----------------------------------------------------------------- Appendix A (input sanity)
def test_gaussian_pmf_paper_values():
    g = gold("paper_numbers.json")
    assert O.gaussian_pmf(1.0, 0) == pytest.approx(g["pmf_sigma1_x0"], abs=1e-5)
    assert O.gaussian_pmf(1.0, -1) == pytest.approx(g["pmf_sigma1_xm1"], abs=1e-5)
    assert math.sqrt(math.log(2) / 3) == pytest.approx(g["u0"], abs=1e-6)
    # Monte-Carlo (library sampler) vs closed form
    s = np.abs(np.random.default_rng(0).standard_normal(2_000_000))
    assert np.mean((s >= 1) & (s < 2)) == pytest.approx(O.gaussian_pmf(1.0, 0), abs=1.5e-3)
    # scale shift: pmf(2 sigma, x+1) = pmf(sigma, x)
    for x in range(-10, 3):
        assert O.gaussian_pmf(2.0, x + 1) == pytest.approx(O.gaussian_pmf(1.0, x), abs=1e-12)


def test_theorems_unimodal_and_contiguous():
    for sigma in 2.0 ** np.linspace(-10, 2, 60):
        p = np.array([O.gaussian_pmf(sigma, x) for x in range(-60, 11)])
        k = int(np.argmax(p))
        assert np.all(np.diff(p[: k + 1]) >= -1e-12) and np.all(np.diff(p[k:]) <= 1e-12)
        order = np.argsort(-p, kind="stable")
        for K in range(1, 16):
            top = np.sort(order[:K])
            assert top[-1] - top[0] == K - 1


def test_gaussian_exponent_entropy_range():
    w = G.gaussian_bf16(1000, 1000, 0.02, 0)
    h = O.shannon_entropy(O.histogram(w))
    assert 2.3 <= h <= 2.8
    ps = np.array([O.gaussian_pmf(0.02, x) for x in range(-60, 11)])
    ps = ps[ps > 0]
    assert abs(h + float((ps * np.log2(ps)).sum())) < 0.05


def test_coverage_ratio_topk_pins():
    # r_n: fraction of elements covered by the 2^n - 1 most frequent exponents.
    # Closed forms: uniform histogram -> (2^n - 1) / 256; one spike -> 1.
    u = np.ones(256, np.int64)
    for n in range(1, 9):
        assert O.coverage_ratio_topk(u, n) == pytest.approx((2 ** n - 1) / 256, abs=1e-15)
    spike = np.zeros(256, np.int64)
    spike[120] = 99
    assert O.coverage_ratio_topk(spike, 1) == 1.0
    # Theorem 2 (contiguity): for a Gaussian the top 2^n - 1 exponents form one
    # contiguous window, so r_3 equals the coverage of the max-coverage 7-window (Alg. 1)
    w = G.gaussian_bf16(1024, 1024, 0.02, 7)
    h = O.histogram(w)
    _, cov = O.select_window(h)
    assert O.coverage_ratio_topk(h, 3) == pytest.approx(cov / h.sum(), abs=1e-15)
    # ... and r_3 of the sampled histogram agrees with the Appendix A pmf (bf16 rounding and
    # sampling error only)
    ps = np.sort(np.array([O.gaussian_pmf(0.02, x) for x in range(-60, 11)]))[::-1]
    assert O.coverage_ratio_topk(h, 3) == pytest.approx(ps[:7].sum(), abs=3e-3)
