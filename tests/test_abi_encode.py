"""CPU tests of the boundary: libzs.so loads and exports every include/zs.h symbol, the host
encoder (zs_encode) is byte-identical to the oracle encoder, and validation errors are
returned synchronously (no GPU needed, no compute call is made)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import zs_inputs as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def Z():
    from paper_2603_17435_b200 import build
    build.build()
    import paper_2603_17435_b200 as Zm
    Zm.lib()
    return Zm


def header_symbols():
    src = open(os.path.join(ROOT, "include", "zs.h")).read()
    return sorted(set(re.findall(r"^\s*(?:zs_status|size_t|int|const char \*)\s*(zs_\w+)\s*\(", src, re.M)))


def test_exports_every_header_symbol(Z):
    syms = header_symbols()
    assert set(syms) == set(Z.zs.EXPORTS)
    out = subprocess.check_output(["nm", "-D", "--defined-only", Z.zs.LIB_PATH]).decode()
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s
        getattr(Z.lib(), s)


def test_sass_is_blackwell_native(Z):
    sass = subprocess.check_output(["cuobjdump", "-sass", Z.zs.LIB_PATH]).decode()
    for mnem in ("UTCHMMA", "UBLKCP", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")


def test_status_strings(Z):
    L = Z.lib()
    assert L.zs_status_string(0) == b"ZS_OK"
    assert L.zs_status_string(7) == b"ZS_ERR_CAPACITY"


ENC_CASES = [
    lambda: G.gaussian_bf16(1, 1, 0.02, 1),
    lambda: G.gaussian_bf16(7, 9, 0.005, 2),
    lambda: G.special_patterns(G.gaussian_bf16(65, 63, 0.1, 3)),
    lambda: G.gaussian_bf16(300, 300, 0.02, 4),
    lambda: G.realistic_bf16(512, 1024, seed=5),
    G.all_patterns_256,
    lambda: np.zeros((64, 128), np.uint16),
    lambda: G.integer_weights(128, 256),
]


@pytest.mark.parametrize("i", range(len(ENC_CASES)))
def test_encoder_byte_equal_to_oracle(Z, i):
    w = ENC_CASES[i]()
    e = Z.encode(w)
    o = O.encode(w)
    assert e.base_exp == o.base_exp and e.pad_word == o.pad_word
    for a, b in ((e.b1, o.B1), (e.b2, o.B2), (e.b3, o.B3), (e.h, o.H), (e.l, o.L)):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(e.offsets[:-1], o.offsets)
    np.testing.assert_array_equal(e.offsets[-1], [o.H.size, 2 * o.L.size])   # sentinel
    s = e.sizes
    assert s["h_bytes"] == o.H.size and s["l_words"] == o.L.size
    off = e.offsets.astype(np.int64)
    assert s["max_h_seg_bytes"] == np.diff(off[:, 0]).max()
    assert s["max_l_seg_bytes"] == np.diff(off[:, 1]).max()
    start, cov = O.select_window(O.histogram(w))
    assert e.covered == cov


def test_encoder_forced_base_exp(Z):
    w = G.gaussian_bf16(100, 130, 0.02, 7)
    for be in (-1, 0, 100, 248):
        e = Z.encode(w, base_exp=be)
        o = O.encode(w, base_exp=be)
        np.testing.assert_array_equal(e.h, o.H)
        np.testing.assert_array_equal(e.l, o.L)
        np.testing.assert_array_equal(e.b3, o.B3)


def test_encoder_full_size_accounting(Z):
    K, N = G.LAYERS["L8B.O"]
    w = G.gaussian_bf16(N, K, 0.02, G.seed_of("L8B.O"))
    e = Z.encode(w)
    assert e.base_exp == 115
    r = e.covered / w.size
    bpe = e.bits_per_element()
    assert 0 < bpe - O.average_bits(3, r) <= 0.2
    assert bpe / 16 <= 0.73


def test_validation_errors_without_gpu(Z):
    L = Z.lib()
    sz = Z.zs.zs_sizes()
    assert L.zs_encode_bound(0, 5, ctypes.byref(sz)) == 1
    assert L.zs_encode_bound(64, 64, ctypes.byref(sz)) == 0 and sz.l_words == 4096
    t = Z.zs.zs_tensor()
    assert L.zs_decompress(ctypes.byref(t), None, 0, None) == 1            # null pointers
    assert L.zs_gemm(None, 0, ctypes.byref(t), None, 0, 1, 1, 1, None, 0, None) == 1
    # capacity error: buffers too small for the encoding
    w = G.gaussian_bf16(64, 64, 0.02, 1)
    cap = Z.zs.zs_sizes()
    cap.n_fragtiles, cap.n_blocktiles, cap.h_bytes, cap.l_words = 64, 1, 16, 0
    b = np.zeros(64, np.uint64)
    h = np.zeros(16, np.uint8)
    off = np.zeros(4, np.uint64)
    act = Z.zs.zs_sizes()
    rc = L.zs_encode(w.ctypes.data_as(ctypes.c_void_p), 64, 64, 64, 115, ctypes.byref(cap),
                     *(b.ctypes.data_as(ctypes.c_void_p),) * 3, h.ctypes.data_as(ctypes.c_void_p), None,
                     off.ctypes.data_as(ctypes.c_void_p), ctypes.byref(act), None)
    assert rc == 7
    assert L.zs_gemm_workspace_bytes(32, 28672, 4096) >= 32 * 28672 * 4


def test_gemm_path_and_workspace_sizes(Z):
    # include/zs.h: M <= ZS_GEMM_LARGE_M runs the fused kernel with the fp32 split-K
    # workspace; larger M runs the decoupled path whose workspace holds the decoded W.
    L = Z.lib()
    hdr = open(os.path.join(ROOT, "include", "zs.h")).read()
    large = int(re.search(r"#define ZS_GEMM_LARGE_M (\d+)", hdr).group(1))
    small_nk = eval(re.search(r"#define ZS_GEMM_SMALL_NK \((.*)\)", hdr).group(1).replace("ll", ""))
    small_m = int(re.search(r"#define ZS_GEMM_LARGE_M_SMALL_NK (\d+)", hdr).group(1))
    N, K = 28672, 4096
    assert N * K > small_nk
    for M in (1, 8, 32, large):
        assert L.zs_gemm_is_decoupled(M, N, K) == 0
        ws = L.zs_gemm_workspace_bytes(M, N, K)
        assert ws >= 4 * min(M, 256) * N and ws % 256 == 0
    for M in (large + 1, 1024, 8192):
        assert L.zs_gemm_is_decoupled(M, N, K) == 1
        assert L.zs_gemm_workspace_bytes(M, N, K) >= 2 * N * K
    # small matrices (8B QKV: 6144 x 4096) switch earlier
    assert 6144 * 4096 <= small_nk
    assert L.zs_gemm_is_decoupled(small_m, 6144, 4096) == 0
    assert L.zs_gemm_is_decoupled(small_m + 1, 6144, 4096) == 1
    assert L.zs_gemm_workspace_bytes(0, N, K) == 0
    # K is padded to a multiple of 8 elements (16-B rows of the decoded operand)
    assert L.zs_gemm_workspace_bytes(large + 1, 100, 1001) >= 2 * 100 * 1008


def test_selector_table_matches_generator():
    # csrc/zs_lut.h must be exactly what scripts/gen_lut.py derives from the rank definition
    # (Alg. 2: idx_H = popc(M & ((1 << p) - 1)), fallback rank p - idx_H)
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_lut", os.path.join(ROOT, "scripts", "gen_lut.py"))
    gl = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gl)
    src = open(os.path.join(ROOT, "paper_2603_17435_b200", "csrc", "zs_lut.h")).read()
    rows = re.findall(r"\{0x([0-9A-F]{8})u, 0x([0-9A-F]{8})u, 0x([0-9A-F]{8})u, 0x([0-9A-F]{8})u\}", src)
    assert len(rows) == 256
    for m, r in enumerate(rows):
        assert [int(v, 16) for v in r] == gl.entry(m)
    # spot-check the rank semantics: m = 0b10110101 -> element 2 is in-window with H rank 1
    e = gl.entry(0b10110101)
    assert (e[1] & 0xF) == 1                      # word 1, low byte <- H byte of rank 1
