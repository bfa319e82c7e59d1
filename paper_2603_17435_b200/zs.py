"""Thin Python binding of libzs.so (include/zs.h): argument marshalling only.

Every step of the hot path (encode on the host; decompress and ZipGEMM on the GPU)
runs inside libzs.so.  PyTorch is used for device memory and streams only.  There is
no fallback: if libzs.so is missing or the GPU is not sm_100a, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZS_LIB") or os.path.join(_PKG, "libzs.so")   # ZS_LIB: debug builds

ZS_STATUS = {0: "ZS_OK", 1: "ZS_ERR_INVALID_ARG", 2: "ZS_ERR_SHAPE", 3: "ZS_ERR_ALIGNMENT",
             4: "ZS_ERR_UNSUPPORTED", 5: "ZS_ERR_CORRUPT", 6: "ZS_ERR_CUDA", 7: "ZS_ERR_CAPACITY"}

# every symbol include/zs.h declares (checked by tests/test_abi_encode.py)
EXPORTS = ["zs_encode_bound", "zs_encode_measure", "zs_encode", "zs_decompress", "zs_gemm_workspace_bytes",
           "zs_gemm_is_decoupled", "zs_gemm", "zs_last_launch_count", "zs_status_string",
           "zs_encode_device_workspace_bytes", "zs_encode_measure_device", "zs_encode_device",
           "zs_gemm_peer_workspace_bytes", "zs_gemm_peer", "zs_peer_wait", "zs_ipc_get_handle", "zs_ipc_open",
           "zs_ipc_close"]

MAX_PEERS = 8            # ZS_MAX_PEERS
IPC_HANDLE_BYTES = 64    # ZS_IPC_HANDLE_BYTES


class ZsError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {ZS_STATUS.get(code, code)}")
        self.code = code


class zs_sizes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "rows", "cols", "padded_rows", "padded_cols", "n_fragtiles", "n_blocktiles",
        "h_bytes", "l_words", "max_h_seg_bytes", "max_l_seg_bytes")]


class zs_tensor(ctypes.Structure):
    _fields_ = [("sz", zs_sizes), ("base_exp", ctypes.c_int32), ("pad_word", ctypes.c_uint16),
                ("reserved", ctypes.c_uint16),
                ("b1", ctypes.c_void_p), ("b2", ctypes.c_void_p), ("b3", ctypes.c_void_p),
                ("h", ctypes.c_void_p), ("l", ctypes.c_void_p), ("offsets", ctypes.c_void_p)]


class zs_peer_out(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("y", ctypes.c_void_p * MAX_PEERS),
                ("ldy", ctypes.c_int64), ("col0", ctypes.c_int64), ("flags", ctypes.c_void_p * MAX_PEERS),
                ("epoch", ctypes.c_uint32)]


_lib = None


def lib():
    """Load libzs.so; raises (no fallback) if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2603_17435_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.zs_encode_bound.argtypes = [i64, i64, ctypes.POINTER(zs_sizes)]
        L.zs_encode_measure.argtypes = [vp, i64, i64, i64, ctypes.POINTER(i32), ctypes.POINTER(i64),
                                        ctypes.POINTER(zs_sizes)]
        L.zs_encode.argtypes = [vp, i64, i64, i64, i32, ctypes.POINTER(zs_sizes), vp, vp, vp, vp, vp, vp,
                                ctypes.POINTER(zs_sizes), ctypes.POINTER(ctypes.c_uint16)]
        L.zs_decompress.argtypes = [ctypes.POINTER(zs_tensor), vp, i64, vp]
        L.zs_gemm_workspace_bytes.argtypes = [i64, i64, i64]
        L.zs_gemm_workspace_bytes.restype = ctypes.c_size_t
        L.zs_gemm_is_decoupled.argtypes = [i64, i64, i64]
        L.zs_gemm_is_decoupled.restype = ctypes.c_int
        L.zs_gemm.argtypes = [vp, i64, ctypes.POINTER(zs_tensor), vp, i64, i64, i64, i64, vp, ctypes.c_size_t, vp]
        L.zs_status_string.argtypes = [ctypes.c_int]
        L.zs_status_string.restype = ctypes.c_char_p
        L.zs_encode_device_workspace_bytes.argtypes = [i64, i64]
        L.zs_encode_device_workspace_bytes.restype = ctypes.c_size_t
        L.zs_encode_measure_device.argtypes = [vp, i64, i64, i64, vp, ctypes.c_size_t, vp, ctypes.POINTER(i32),
                                               ctypes.POINTER(i64), ctypes.POINTER(zs_sizes)]
        L.zs_encode_device.argtypes = [vp, i64, i64, i64, i32, ctypes.POINTER(zs_sizes), vp, vp, vp, vp, vp, vp,
                                       ctypes.POINTER(zs_sizes), ctypes.POINTER(ctypes.c_uint16), vp, ctypes.c_size_t,
                                       vp]
        L.zs_gemm_peer_workspace_bytes.argtypes = [i64, i64, i64]
        L.zs_gemm_peer_workspace_bytes.restype = ctypes.c_size_t
        L.zs_gemm_peer.argtypes = [vp, i64, ctypes.POINTER(zs_tensor), ctypes.POINTER(zs_peer_out), i64, i64, i64,
                                   vp, ctypes.c_size_t, vp]
        L.zs_peer_wait.argtypes = [vp, i32, ctypes.c_uint32, vp]
        L.zs_ipc_get_handle.argtypes = [vp, vp, ctypes.POINTER(i64)]
        L.zs_ipc_open.argtypes = [vp, ctypes.POINTER(vp)]
        L.zs_ipc_close.argtypes = [vp]
        for f in ("zs_encode_bound", "zs_encode_measure", "zs_encode", "zs_decompress", "zs_gemm",
                  "zs_encode_measure_device", "zs_encode_device", "zs_gemm_peer", "zs_peer_wait",
                  "zs_ipc_get_handle", "zs_ipc_open", "zs_ipc_close"):
            getattr(L, f).restype = ctypes.c_int
        L.zs_last_launch_count.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(fn, rc):
    if rc != 0:
        raise ZsError(fn, rc)


def _np_ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else None


def _as_u16(w) -> np.ndarray:
    try:
        import torch
        if isinstance(w, torch.Tensor):
            assert w.dtype == torch.bfloat16 and w.device.type == "cpu"
            return w.contiguous().view(torch.int16).numpy().view(np.uint16)
    except ImportError:  # pragma: no cover
        pass
    return np.ascontiguousarray(w, dtype=np.uint16)


# ------------------------------------------------------------------ host encoding
@dataclass
class ZsHost:
    """A TCA-TBE-encoded matrix in host memory (numpy arrays, include/zs.h layout)."""
    sizes: dict
    base_exp: int
    pad_word: int
    covered: int
    b1: np.ndarray
    b2: np.ndarray
    b3: np.ndarray
    h: np.ndarray
    l: np.ndarray
    offsets: np.ndarray  # (n_blocktiles + 1, 2) uint64 incl. sentinel

    @property
    def rows(self):
        return self.sizes["rows"]

    @property
    def cols(self):
        return self.sizes["cols"]

    def nbytes(self) -> int:
        return self.b1.nbytes * 3 + self.h.nbytes + self.l.nbytes + self.offsets.nbytes

    def bits_per_element(self) -> float:
        return 8.0 * self.nbytes() / (self.rows * self.cols)

    def to(self, device) -> "ZsDevice":
        import torch
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64 if a.dtype == np.uint64 else
                                                                    (np.int16 if a.dtype == np.uint16 else np.uint8))
                                       ).to(device)
        pad16 = lambda a: a if a.size else np.zeros(8, a.dtype)
        return ZsDevice(dict(self.sizes), self.base_exp, self.pad_word, t(self.b1), t(self.b2), t(self.b3),
                        t(pad16(self.h)), t(pad16(self.l)), t(self.offsets.reshape(-1)))


def encode(w, base_exp: int | None = None) -> ZsHost:
    """zs_encode_measure + zs_encode (Alg. 1) on a host [rows][cols] bf16 matrix."""
    L = lib()
    w = _as_u16(w)
    assert w.ndim == 2
    rows, cols = w.shape
    sz = zs_sizes()
    be = ctypes.c_int32()
    cov = ctypes.c_int64()
    _check("zs_encode_measure", L.zs_encode_measure(_np_ptr(w), rows, cols, cols, ctypes.byref(be),
                                                    ctypes.byref(cov), ctypes.byref(sz)))
    if base_exp is not None and base_exp != be.value:
        be = ctypes.c_int32(base_exp)
        _check("zs_encode_bound", L.zs_encode_bound(rows, cols, ctypes.byref(sz)))
    nft, nbt = sz.n_fragtiles, sz.n_blocktiles
    b1, b2, b3 = (np.empty(nft, np.uint64) for _ in range(3))
    h = np.empty(max(sz.h_bytes, 0), np.uint8)
    l = np.empty(max(sz.l_words, 0), np.uint16)
    off = np.empty((nbt + 1, 2), np.uint64)
    act = zs_sizes()
    pad = ctypes.c_uint16()
    _check("zs_encode", L.zs_encode(_np_ptr(w), rows, cols, cols, be.value, ctypes.byref(sz), _np_ptr(b1),
                                    _np_ptr(b2), _np_ptr(b3), _np_ptr(h), _np_ptr(l), _np_ptr(off),
                                    ctypes.byref(act), ctypes.byref(pad)))
    sizes = {f: getattr(act, f) for f, _ in zs_sizes._fields_}
    return ZsHost(sizes, be.value, pad.value, cov.value if base_exp is None else -1, b1, b2, b3,
                  h[: act.h_bytes].copy(), l[: act.l_words].copy(), off)


# ------------------------------------------------------------------ device tensors
@dataclass
class ZsDevice:
    """A TCA-TBE matrix resident in device memory (torch tensors as raw storage)."""
    sizes: dict
    base_exp: int
    pad_word: int
    b1: "object"
    b2: "object"
    b3: "object"
    h: "object"
    l: "object"
    offsets: "object"

    @property
    def rows(self):
        return self.sizes["rows"]

    @property
    def cols(self):
        return self.sizes["cols"]

    @property
    def device(self):
        return self.b1.device

    def nbytes(self) -> int:
        return int(self.b1.numel() * 8 * 3 + self.sizes["h_bytes"] + 2 * self.sizes["l_words"]
                   + 16 * (self.sizes["n_blocktiles"] + 1))

    def c_struct(self) -> zs_tensor:
        # the encoded tensors are immutable: build the ABI view once per ZsDevice
        t = self.__dict__.get("_ct")
        if t is not None:
            return t
        t = zs_tensor()
        for f, _ in zs_sizes._fields_:
            setattr(t.sz, f, int(self.sizes[f]))
        t.base_exp = self.base_exp
        t.pad_word = self.pad_word
        t.b1, t.b2, t.b3 = self.b1.data_ptr(), self.b2.data_ptr(), self.b3.data_ptr()
        t.h, t.l, t.offsets = self.h.data_ptr(), self.l.data_ptr(), self.offsets.data_ptr()
        self.__dict__["_ct"] = t
        return t


def encode_device(w, base_exp: int | None = None, stream=None) -> "ZsDevice":
    """GPU-side encoder: a device torch.bfloat16 [rows][cols] matrix -> ZsDevice on the same
    device, byte-identical to encode(w.cpu()).to(device)."""
    import torch
    assert w.dtype == torch.bfloat16 and w.dim() == 2 and w.stride(1) == 1 and w.is_cuda
    L = lib()
    rows, cols = w.shape
    dev = w.device
    sp = _stream_ptr(stream, dev)
    wsb = int(L.zs_encode_device_workspace_bytes(rows, cols))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    wp = ctypes.c_void_p(w.data_ptr())
    sz = zs_sizes()
    be = ctypes.c_int32()
    cov = ctypes.c_int64()
    _check("zs_encode_measure_device", L.zs_encode_measure_device(wp, rows, cols, w.stride(0), ctypes.c_void_p(ws.data_ptr()),
                                                                  ws.numel(), sp, ctypes.byref(be), ctypes.byref(cov),
                                                                  ctypes.byref(sz)))
    if base_exp is not None and base_exp != be.value:
        be = ctypes.c_int32(base_exp)
        _check("zs_encode_bound", L.zs_encode_bound(rows, cols, ctypes.byref(sz)))
    nft, nbt = sz.n_fragtiles, sz.n_blocktiles
    planes = [torch.empty(nft, dtype=torch.int64, device=dev) for _ in range(3)]
    h = torch.empty(max(sz.h_bytes, 16), dtype=torch.uint8, device=dev)
    l = torch.empty(max(sz.l_words, 8), dtype=torch.int16, device=dev)
    off = torch.empty(2 * (nbt + 1), dtype=torch.int64, device=dev)
    act = zs_sizes()
    pad = ctypes.c_uint16()
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())
    _check("zs_encode_device", L.zs_encode_device(wp, rows, cols, w.stride(0), be.value, ctypes.byref(sz),
                                                  ptr(planes[0]), ptr(planes[1]), ptr(planes[2]), ptr(h), ptr(l),
                                                  ptr(off), ctypes.byref(act), ctypes.byref(pad),
                                                  ctypes.c_void_p(ws.data_ptr()), ws.numel(), sp))
    sizes = {f: getattr(act, f) for f, _ in zs_sizes._fields_}
    return ZsDevice(sizes, be.value, pad.value, planes[0], planes[1], planes[2], h, l, off)


def _stream_ptr(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def decompress(w: ZsDevice, out=None, stream=None):
    """ZipServ-Decomp: -> torch.bfloat16 [rows][cols] on w's device (bit-exact)."""
    import torch
    if out is None:
        out = torch.empty((w.rows, w.cols), dtype=torch.bfloat16, device=w.device)
    assert out.dtype == torch.bfloat16 and out.stride(1) == 1
    t = w.c_struct()
    _check("zs_decompress", lib().zs_decompress(ctypes.byref(t), ctypes.c_void_p(out.data_ptr()), out.stride(0),
                                                _stream_ptr(stream, w.device)))
    return out


_WS = {}


def _stream_key(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return int(stream.cuda_stream)


def workspace(M: int, N: int, K: int, device, stream=None):
    """zs_gemm workspace, kept per (device, stream, path) and grown on demand: the
    zero-initialised, self-cleaning split-K buffer of the fused path, or the decoded-weight
    scratch of the decoupled (large-M) path -- separate buffers, since the latter is left dirty.
    include/zs.h allows a workspace to be reused only in stream order, so each stream gets
    its own; a buffer replaced by a larger one is released only after a synchronisation of
    its stream (a kernel queued on it may still use it)."""
    import torch
    need = int(lib().zs_gemm_workspace_bytes(M, N, K))
    key = (str(device), _stream_key(stream, device), int(lib().zs_gemm_is_decoupled(M, N, K)))
    ws = _WS.get(key)
    if ws is None or ws.numel() < need:
        if ws is not None:
            torch.cuda.synchronize(device)
        ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def gemm(x, w: ZsDevice, out=None, ws=None, stream=None):
    """ZipGEMM: Y = X @ W^T with X torch.bfloat16 [M][K] on the GPU -> Y [M][N] bf16."""
    import torch
    assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1
    M, K = x.shape
    N = w.rows
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=x.device)
    if ws is None:
        ws = workspace(M, N, K, x.device, stream)
    t = w.c_struct()
    _check("zs_gemm", lib().zs_gemm(ctypes.c_void_p(x.data_ptr()), x.stride(0), ctypes.byref(t),
                                    ctypes.c_void_p(out.data_ptr()), out.stride(0), M, N, K,
                                    ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream, x.device)))
    return out


def peer_workspace(M: int, N: int, K: int, device, stream=None):
    """zs_gemm_peer workspace (zeroed once, self-cleaning counter + zs_gemm's workspace), kept
    per (device, stream, path) like workspace()."""
    import torch
    need = int(lib().zs_gemm_peer_workspace_bytes(M, N, K))
    key = (str(device), _stream_key(stream, device), int(lib().zs_gemm_is_decoupled(M, N, K)), "peer")
    ws = _WS.get(key)
    if ws is None or ws.numel() < need:
        if ws is not None:
            torch.cuda.synchronize(device)
        ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def gemm_peer(x, w: ZsDevice, ys, flags, rank: int, col0: int, epoch: int, ldy: int | None = None, ws=None,
              stream=None):
    """Column-sharded ZipGEMM with the output exchange fused into the kernel (zs_gemm_peer):
    stores X @ W_shard^T into columns [col0, col0 + w.rows) of EVERY rank's Y and signals each
    rank's flags[rank] = epoch.  ys / flags: per rank, a torch tensor on this device or an int
    device address valid in this process (IPC-mapped peer memory)."""
    import torch
    assert x.dtype == torch.bfloat16 and x.dim() == 2 and x.stride(1) == 1
    world = len(ys)
    assert len(flags) == world and world <= MAX_PEERS   # the rest is validated by zs_gemm_peer
    M, K = x.shape
    N = w.rows
    if ldy is None:
        ldy = ys[rank].stride(0)
    # Y buffers are [M][ldy]: the kernel stores M rows into every rank's buffer, so every
    # buffer this process can see must have them (peer buffers are the same shape by contract)
    for r in range(world):
        if not isinstance(ys[r], int):
            assert ys[r].shape[0] >= M and ys[r].stride(0) == ldy, f"ys[{r}] smaller than [M={M}][ldy={ldy}]"
    o = zs_peer_out()
    o.world, o.rank, o.ldy, o.col0, o.epoch = world, rank, ldy, col0, epoch & 0xFFFFFFFF
    for r in range(world):
        o.y[r] = ys[r] if isinstance(ys[r], int) else ys[r].data_ptr()
        o.flags[r] = flags[r] if isinstance(flags[r], int) else flags[r].data_ptr()
    if ws is None:
        ws = peer_workspace(M, N, K, x.device, stream)
    t = w.c_struct()
    _check("zs_gemm_peer", lib().zs_gemm_peer(ctypes.c_void_p(x.data_ptr()), x.stride(0), ctypes.byref(t),
                                              ctypes.byref(o), M, N, K, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                              _stream_ptr(stream, x.device)))


def peer_wait(flags, world: int, epoch: int, stream=None):
    """Block the stream until this rank's flags[0..world) reached epoch (zs_peer_wait)."""
    _check("zs_peer_wait", lib().zs_peer_wait(ctypes.c_void_p(flags.data_ptr()), world, epoch & 0xFFFFFFFF,
                                              _stream_ptr(stream, flags.device)))


def ipc_handle(t) -> tuple[bytes, int]:
    """(handle bytes, byte offset) of the CUDA allocation holding torch tensor t."""
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    off = ctypes.c_int64()
    _check("zs_ipc_get_handle", lib().zs_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)))
    return h.raw, off.value


def ipc_open(handle: bytes) -> int:
    """Map a peer's allocation (another process); returns its base address in this process."""
    base = ctypes.c_void_p()
    _check("zs_ipc_open", lib().zs_ipc_open(ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES),
                                            ctypes.byref(base)))
    return base.value


def ipc_close(base: int):
    _check("zs_ipc_close", lib().zs_ipc_close(ctypes.c_void_p(base)))


def last_launch_count() -> int:
    return lib().zs_last_launch_count()
