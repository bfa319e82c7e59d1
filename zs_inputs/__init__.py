"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no histogram, window, encoding or
decoding).  It only draws numbers and rounds fp32 -> bf16 (round to nearest even,
the same as ``tensor.to(torch.bfloat16)``).  Recipes ("Input recipe"):

* ``gaussian_bf16``: W ~ N(0, sigma^2) drawn in fp32, rounded to bf16.  sigma = 0.02
  is the LLaMA-like default (Appendix A models weights as zero-mean Gaussians).
* ``realistic_bf16``: per-row sigma_n = sigma * 2^U(-1, 1) plus a fraction of outliers
  at 20 sigma -- the "real-model-like" variant of SURVEY.md section 8(d).
* ``activations_bf16``: X ~ N(0, 1) rounded to bf16.
* ``special_patterns``: NaN / Inf / subnormal / -0 injection (SPEC acceptance #1).
* ``all_patterns_256``: every one of the 65,536 bf16 bit patterns as a 256x256 matrix.
* ``LAYERS``: the layer shapes (K = in features, N = out features) of the configs.
"""
from __future__ import annotations

import zlib

import numpy as np

# Layer shapes, build convention Y[M][N] = X[M][K] W[N][K]^T.
LAYERS = {
    "L8B.QKV": (4096, 6144),
    "L8B.O": (4096, 4096),
    "L8B.GateUp": (4096, 28672),
    "L8B.Down": (14336, 4096),
    "L70B.QKV": (8192, 10240),
    "L70B.O": (8192, 8192),
    "L70B.GateUp": (8192, 57344),
    "L70B.Down": (28672, 8192),
    "Q32B.QKV": (5120, 10240),
    "Q32B.O": (8192, 5120),
    "Q32B.GateUp": (5120, 51200),
    "Q32B.Down": (25600, 5120),
    # per-rank column shards of the 70B layers at 8 GPUs (N / 8 output features each, 8(e))
    "L70B.QKV.w8": (8192, 1280),
    "L70B.O.w8": (8192, 1024),
    "L70B.GateUp.w8": (8192, 7168),
    "L70B.Down.w8": (28672, 1024),
    # f4: Gemma-3-27B (hidden 5376, intermediate 21504, 32 q / 16 kv heads
    # of 128), Qwen2.5-7B (hidden 3584, intermediate 18944, 28 q / 4 kv heads of 128);
    # Mistral-7B-v0.1's linear layers have exactly the LLaMA-3.1-8B shapes above
    "G3-27B.QKV": (5376, 8192),
    "G3-27B.O": (4096, 5376),
    "G3-27B.GateUp": (5376, 43008),
    "G3-27B.Down": (21504, 5376),
    "Q2.5-7B.QKV": (3584, 4608),
    "Q2.5-7B.O": (3584, 3584),
    "Q2.5-7B.GateUp": (3584, 37888),
    "Q2.5-7B.Down": (18944, 3584),
    # LM head of LLaMA-3.1-8B (vocabulary 128256, P:493 lists the LM head among the layers)
    "L8B.LMHead": (4096, 128256),
    # fixed-cost probes: one unit (128 x 64) and one 128-row band of K = 4096
    "T.1unit": (64, 128),
    "T.1band": (4096, 128),
}


def seed_of(name: str) -> int:
    """Stable per-(model, layer) seed (crc32 of the name)."""
    return zlib.crc32(name.encode()) & 0x7FFFFFFF


def fp32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (nearest, ties to even); NaNs become a quiet NaN."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(a)
    if nan.any():
        r[nan] = (0x7FC0 | ((u[nan] >> 16) & 0x8000)).astype(np.uint16)
    return r


def bf16_bits_to_fp32(w: np.ndarray) -> np.ndarray:
    return (np.asarray(w, np.uint16).astype(np.uint32) << 16).view(np.float32)


def gaussian_bf16(rows: int, cols: int, sigma: float = 0.02, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return fp32_to_bf16_bits(rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(sigma))


def realistic_bf16(rows: int, cols: int, sigma: float = 0.02, spread: float = 1.0,
                   outlier_frac: float = 1e-3, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    row_sigma = (sigma * 2.0 ** rng.uniform(-spread, spread, size=(rows, 1))).astype(np.float32)
    a = rng.standard_normal((rows, cols), dtype=np.float32) * row_sigma
    if outlier_frac > 0:
        mask = rng.random((rows, cols)) < outlier_frac
        a[mask] = (20.0 * sigma * np.sign(rng.standard_normal(int(mask.sum())))).astype(np.float32)
    return fp32_to_bf16_bits(a)


def activations_bf16(M: int, K: int, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return fp32_to_bf16_bits(rng.standard_normal((M, K), dtype=np.float32))


SPECIALS = np.array([0x7FC0, 0xFFC0, 0x7F80, 0xFF80, 0x0001, 0x8001, 0x007F, 0x8000, 0x0000, 0x7F81],
                    dtype=np.uint16)


def special_patterns(w: np.ndarray, frac: float = 0.05, seed: int = 3) -> np.ndarray:
    """Inject NaN / Inf / subnormal / signed-zero patterns into a copy of w."""
    rng = np.random.default_rng(seed)
    w = np.array(w, dtype=np.uint16, copy=True)
    mask = rng.random(w.shape) < frac
    w[mask] = rng.choice(SPECIALS, size=int(mask.sum()))
    return w


def all_patterns_256() -> np.ndarray:
    return np.arange(65536, dtype=np.uint32).astype(np.uint16).reshape(256, 256)


def integer_weights(rows: int, cols: int, seed: int = 5) -> np.ndarray:
    """W in {0, +-1, +-2, +-3, +-4} (exact-sum pin)."""
    rng = np.random.default_rng(seed)
    v = rng.integers(-4, 5, size=(rows, cols)).astype(np.float32)
    return fp32_to_bf16_bits(v)


def integer_activations(M: int, K: int, seed: int = 6) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = rng.integers(-4, 5, size=(M, K)).astype(np.float32)
    return fp32_to_bf16_bits(v)


def one_hot_activations(M: int, K: int, ks) -> np.ndarray:
    """X[m][ks[m]] = 1.0, zeros elsewhere."""
    x = np.zeros((M, K), np.uint16)
    for m, k in enumerate(ks):
        x[m, k] = 0x3F80
    return x
