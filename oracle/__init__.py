"""CPU oracle for TCA-TBE / ZipGEMM (arxiv 2603.17435).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``bench.py`` CPU legs (``cpu_baseline`` and ``--impl reference``) may import this
package.  It shares no code with the product package ``paper_2603_17435_b200``;
the only common dependency is the seeded input generator ``zs_inputs`` (which
holds none of the method's arithmetic).

The codec, decoders and fp64 GEMM live in plain C (``zs_oracle.c``); this module
only marshals numpy arrays.  Closed forms of the paper (AverageBits, the
compute-intensity model, the Appendix-A pmf) are written out here in Python.

Parity status per function ("Oracle pins"):
  encode / decode_sequential / decode_lanes / gemm_f64 / round_bf16 ... pinned
  average_bits / ci_* / gaussian_pmf / entropy ........................... pinned
Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "zs_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile zs_oracle.c with plain gcc -O2 (no intrinsics, single thread)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, u16, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint16, ctypes.c_void_p
        L.or_encode.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp, i64, vp, i64, vp, vp]
        L.or_encode.restype = ctypes.c_int
        L.or_encode_bound.argtypes = [i64, i64, vp]
        L.or_histogram.argtypes = [vp, i64, vp]
        L.or_select_window.argtypes = [vp, vp, vp]
        L.or_select_window.restype = ctypes.c_int
        dec = [i64, i64, i32, vp, vp, vp, vp, i64, vp, i64, vp, vp]
        L.or_decode_sequential.argtypes = dec
        L.or_decode_sequential.restype = ctypes.c_int
        L.or_decode_lanes.argtypes = dec
        L.or_decode_lanes.restype = ctypes.c_int
        L.or_decode_lane.argtypes = [ctypes.c_uint64] * 3 + [vp, i64, i64, vp, i64, i64, i32, ctypes.c_int, vp]
        L.or_decode_lane.restype = ctypes.c_int
        L.or_gemm_f64.argtypes = [vp, i64, i64, vp, i64, vp]
        L.or_gemm_f64_cols.argtypes = [vp, i64, i64, vp, vp, i64, vp]
        L.or_round_bf16.argtypes = [ctypes.c_double]
        L.or_round_bf16.restype = u16
        L.or_bf16_to_double.argtypes = [u16]
        L.or_bf16_to_double.restype = ctypes.c_double
        L.or_split_fields.argtypes = [u16, vp, vp, vp]
        L.or_assemble_fields.argtypes = [ctypes.c_int] * 3 + [vp]
        L.or_assemble_fields.restype = ctypes.c_int
        L.or_pack_sm.argtypes = [ctypes.c_int, ctypes.c_int]
        L.or_pack_sm.restype = ctypes.c_uint8
        L.or_coords_of.argtypes = [i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ bf16 fields
def split_fields(w: int):
    s, e, m = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    lib().or_split_fields(w, ctypes.byref(s), ctypes.byref(e), ctypes.byref(m))
    return s.value, e.value, m.value


def assemble_fields(s: int, e: int, m: int) -> int:
    out = ctypes.c_uint16()
    rc = lib().or_assemble_fields(s, e, m, ctypes.byref(out))
    if rc:
        raise ValueError("field out of range")
    return out.value


def pack_sm(s: int, m: int) -> int:
    return lib().or_pack_sm(s, m)


def coords_of(br, bc, t, f, pos):
    r, c = ctypes.c_int64(), ctypes.c_int64()
    lib().or_coords_of(br, bc, t, f, pos, ctypes.byref(r), ctypes.byref(c))
    return r.value, c.value


# ------------------------------------------------------------------ Phase I (Alg. 1)
def histogram(w: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.uint16).reshape(-1)
    counts = np.zeros(256, dtype=np.int64)
    lib().or_histogram(_p(w), w.size, _p(counts))
    return counts


def select_window(counts: np.ndarray):
    """-> (start, covered); base_exp = start - 1 (Alg. 1 line 4)."""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    s, cov = ctypes.c_int(), ctypes.c_int64()
    if lib().or_select_window(_p(counts), ctypes.byref(s), ctypes.byref(cov)):
        raise ValueError("empty histogram")
    return s.value, cov.value


# ------------------------------------------------------------------ Phase II (Alg. 1)
@dataclass
class Encoded:
    rows: int
    cols: int
    padded_rows: int
    padded_cols: int
    base_exp: int
    pad_word: int
    B1: np.ndarray
    B2: np.ndarray
    B3: np.ndarray
    H: np.ndarray
    L: np.ndarray
    offsets: np.ndarray  # (n_blocktiles, 2) uint64: H start byte, L start byte

    @property
    def n_fragtiles(self):
        return self.B1.size

    @property
    def n_blocktiles(self):
        return self.offsets.shape[0]

    def payload_bits(self) -> int:
        """bit-planes + H + L + offsets + alignment padding, header excluded."""
        return 64 * 3 * self.n_fragtiles + 8 * self.H.size + 16 * self.L.size + 128 * self.n_blocktiles

    def bits_per_element(self) -> float:
        return self.payload_bits() / (self.rows * self.cols)

    def compression_ratio(self) -> float:
        return 16.0 * self.rows * self.cols / self.payload_bits()


def encode(w: np.ndarray, base_exp: int | None = None) -> Encoded:
    w = np.ascontiguousarray(w, dtype=np.uint16)
    assert w.ndim == 2
    rows, cols = w.shape
    bound = np.zeros(4, dtype=np.int64)
    lib().or_encode_bound(rows, cols, _p(bound))
    nft, nbt, hcap, lcap = (int(v) for v in bound)
    B1 = np.zeros(nft, np.uint64)
    B2 = np.zeros(nft, np.uint64)
    B3 = np.zeros(nft, np.uint64)
    H = np.zeros(max(hcap, 1), np.uint8)
    L = np.zeros(max(lcap, 1), np.uint16)
    off = np.zeros((nbt, 2), np.uint64)
    info = np.zeros(8, np.int64)
    be = -(2 ** 31) if base_exp is None else int(base_exp)
    rc = lib().or_encode(_p(w), rows, cols, be, _p(B1), _p(B2), _p(B3), _p(H), hcap, _p(L), lcap, _p(off), _p(info))
    if rc:
        raise ValueError(f"or_encode failed rc={rc}")
    return Encoded(rows, cols, int(info[0]), int(info[1]), int(info[2]), int(info[3]),
                   B1, B2, B3, H[: info[6]].copy(), L[: info[7]].copy(), off)


def _decode(fn, e: Encoded) -> np.ndarray:
    out = np.zeros((e.rows, e.cols), np.uint16)
    H = e.H if e.H.size else np.zeros(1, np.uint8)
    L = e.L if e.L.size else np.zeros(1, np.uint16)
    rc = fn(e.rows, e.cols, e.base_exp, _p(e.B1), _p(e.B2), _p(e.B3), _p(H), e.H.size, _p(L), e.L.size,
            _p(np.ascontiguousarray(e.offsets)), _p(out))
    if rc:
        raise ValueError(f"corrupt encoding rc={rc}")
    return out


def decode_sequential(e: Encoded) -> np.ndarray:
    """Sequential inverse of Alg. 1."""
    return _decode(lib().or_decode_sequential, e)


def decode_lanes(e: Encoded) -> np.ndarray:
    """Alg. 2 over 32 lockstep lanes per FragTile."""
    return _decode(lib().or_decode_lanes, e)


def decode_lane(B1, B2, B3, H, h_start, h_end, L, l_start, l_end, base_exp, lane):
    """Alg. 2 for a single lane -> (w at p=2l, w at p=2l+1)."""
    H = np.ascontiguousarray(H, np.uint8) if len(H) else np.zeros(1, np.uint8)
    L = np.ascontiguousarray(L, np.uint16) if len(L) else np.zeros(1, np.uint16)
    out = np.zeros(2, np.uint16)
    rc = lib().or_decode_lane(B1, B2, B3, _p(H), h_start, h_end, _p(L), l_start, l_end, base_exp, lane, _p(out))
    if rc:
        raise ValueError("index past segment end")
    return int(out[0]), int(out[1])


# ------------------------------------------------------------------ fp64 GEMM
def gemm_f64(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Y[m][n] = sum_k X[m][k] W[n][k] accumulated in fp64; X, W are bf16 bit patterns."""
    x = np.ascontiguousarray(x, np.uint16)
    w = np.ascontiguousarray(w, np.uint16)
    M, K = x.shape
    N, K2 = w.shape
    assert K == K2
    y = np.zeros((M, N), np.float64)
    lib().or_gemm_f64(_p(x), M, K, _p(w), N, _p(y))
    return y


def gemm_f64_cols(x: np.ndarray, w: np.ndarray, cols: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.uint16)
    w = np.ascontiguousarray(w, np.uint16)
    cols = np.ascontiguousarray(cols, np.int64)
    M, K = x.shape
    y = np.zeros((M, cols.size), np.float64)
    lib().or_gemm_f64_cols(_p(x), M, K, _p(w), _p(cols), cols.size, _p(y))
    return y


def bf16_to_double(w: int) -> float:
    return lib().or_bf16_to_double(w)


def round_bf16(v: float) -> int:
    return int(lib().or_round_bf16(float(v)))


def round_bf16_array(a: np.ndarray) -> np.ndarray:
    f = lib().or_round_bf16
    flat = np.asarray(a, np.float64).reshape(-1)
    return np.fromiter((f(float(v)) for v in flat), dtype=np.uint16, count=flat.size).reshape(np.shape(a))


def bf16_array_to_double(w: np.ndarray) -> np.ndarray:
    """Vectorised exact bf16 -> fp64 (bit placement into fp32; every bf16 is an fp32)."""
    w = np.asarray(w, np.uint16)
    return (w.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


# ------------------------------------------------------------------ closed forms
def average_bits(n: int, r: float) -> float:
    """AverageBits(n) = r (n + 8) + (1 - r)(n + 16)."""
    return r * (n + 8) + (1 - r) * (n + 16)


def ci_gemm(M: float, N: float, K: float) -> float:
    """Eq. 1: MNK / (MK + KN + MN)."""
    return M * N * K / (M * K + K * N + M * N)


def ci_decoupled(M: float, N: float, K: float, CR: float) -> float:
    """Eq. 2: 2MNK / (MK (2/CR + 4) + 2 (KN + MN))."""
    return 2 * M * N * K / (M * K * (2 / CR + 4) + 2 * (K * N + M * N))


def ci_fused(M: float, N: float, K: float, CR: float) -> float:
    """Eq. 3: 2MNK / (MK 2/CR + 2 (KN + MN))."""
    return 2 * M * N * K / (M * K * (2 / CR) + 2 * (K * N + M * N))


def gaussian_pmf(sigma: float, x: int) -> float:
    """Appendix A: erf(2^(x+1)/(sigma sqrt2)) - erf(2^x/(sigma sqrt2))."""
    if sigma <= 0:
        raise ValueError("sigma must be positive")
    s = sigma * math.sqrt(2.0)
    return math.erf(2.0 ** (x + 1) / s) - math.erf(2.0 ** x / s)


def shannon_entropy(counts: np.ndarray) -> float:
    c = np.asarray(counts, np.float64)
    p = c[c > 0] / c.sum()
    return float(-(p * np.log2(p)).sum())


def coverage_ratio_topk(counts: np.ndarray, n: int) -> float:
    """r_n: fraction covered by the 2^n - 1 largest counts."""
    c = np.sort(np.asarray(counts, np.int64))[::-1]
    return float(c[: 2 ** n - 1].sum() / c.sum())
