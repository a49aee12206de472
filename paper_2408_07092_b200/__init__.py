"""Double Sparsity decode attention (arXiv 2408.07092), native on NVIDIA B200.

Thin Python binding over the C ABI of ``libds.so`` (``include/ds.h``): the
functions below have the C names and only marshal arguments (torch tensors
-> device pointers, the current CUDA stream).  Every step of the method runs
in the sm_100a kernels under ``csrc/``.  There is no CPU fallback: if the
library is missing or the device is not a CUDA device, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DS_LIB") or os.path.join(_PKG, "libds.so")  # DS_LIB: debug builds only

DS_OK, DS_ERR_INVALID_ARGUMENT, DS_ERR_UNSUPPORTED, DS_ERR_GQA_INCOMPATIBLE, \
    DS_ERR_WORKSPACE_TOO_SMALL, DS_ERR_CUDA = range(6)
DS_FP16, DS_BF16, DS_FP32 = 0, 1, 2
DS_CALIB_QK, DS_CALIB_Q, DS_CALIB_K, DS_CALIB_RANDOM = 0, 1, 2, 3
DS_LABEL_NATIVE, DS_LABEL_INT4, DS_LABEL_NONE = 0, 1, 2
_LF = {"native": DS_LABEL_NATIVE, "int4": DS_LABEL_INT4, "none": DS_LABEL_NONE}
DS_GROUP_SUM, DS_GROUP_MAX, DS_GROUP_PER_HEAD = 0, 1, 2
_GR = {"sum": DS_GROUP_SUM, "max": DS_GROUP_MAX, "per_head": DS_GROUP_PER_HEAD}

_DT = {torch.float16: DS_FP16, torch.bfloat16: DS_BF16, torch.float32: DS_FP32}


class DsError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {ds_status_string(status)}")
        self.status = status


class GqaIncompatible(DsError):
    pass


class ds_cache(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("num_pages", ctypes.c_int32),
                ("max_pages_per_seq", ctypes.c_int32), ("max_seq_len", ctypes.c_int32),
                ("r", ctypes.c_int32), ("dtype", ctypes.c_int),
                ("k_pool", ctypes.c_void_p), ("v_pool", ctypes.c_void_p),
                ("block_table", ctypes.c_void_p), ("seq_lens", ctypes.c_void_p),
                ("label", ctypes.c_void_p), ("channel_idx", ctypes.c_void_p),
                ("label_format", ctypes.c_int), ("label_scale", ctypes.c_void_p),
                ("group_reduce", ctypes.c_int)]


_lib = None


def lib():
    """Load libds.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2408_07092_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        C = ctypes.POINTER(ds_cache)
        L.ds_status_string.argtypes = [ctypes.c_int]
        L.ds_status_string.restype = ctypes.c_char_p
        L.ds_version.restype = ctypes.c_char_p
        L.ds_calibrate_channels.argtypes = [P, P, I32, I32, I32, I32, ctypes.c_int, ctypes.c_int, I32,
                                            ctypes.c_uint64, P, P]
        L.ds_append_kv.argtypes = [C, P, P, P, I32, P]
        L.ds_decode_workspace_size.argtypes = [C, I32]
        L.ds_decode_workspace_size.restype = SZ
        L.ds_decode_attention.argtypes = [C, P, I32, P, P, P, SZ, P]
        L.ds_approx_scores.argtypes = [C, P, P, P]
        L.ds_decode_attention_append.argtypes = [C, P, P, P, P, I32, P, P, P, SZ, P]
        L.ds_decode_attention_append.restype = ctypes.c_int
        SL = ctypes.POINTER(ds_prefetch_slot)
        L.ds_prefetch_next_layer.argtypes = [C, P, I32, SL, P]
        L.ds_decode_attention_prefetched.argtypes = [C, P, SL, P, P]
        L.ds_prefetch_next_layer.restype = ctypes.c_int
        L.ds_decode_attention_prefetched.restype = ctypes.c_int
        L.ds_decode_launches.argtypes = [C, I32]
        L.ds_decode_launches.restype = I32
        L.ds_dense_workspace_size.argtypes = [C]
        L.ds_dense_workspace_size.restype = SZ
        L.ds_dense_decode_attention.argtypes = [C, P, P, P, SZ, P]
        for f in ("ds_calibrate_channels", "ds_append_kv", "ds_decode_attention", "ds_approx_scores",
                  "ds_dense_decode_attention"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


EXPORTS = ("ds_status_string", "ds_version", "ds_calibrate_channels", "ds_append_kv",
           "ds_decode_workspace_size", "ds_decode_attention", "ds_approx_scores",
           "ds_dense_workspace_size", "ds_dense_decode_attention", "ds_decode_launches",
           "ds_prefetch_next_layer", "ds_decode_attention_prefetched", "ds_decode_attention_append")


def ds_status_string(s: int) -> str:
    return lib().ds_status_string(s).decode()


def ds_version() -> str:
    return lib().ds_version().decode()


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda and not t.is_pinned():  # pinned host memory is device-addressable (offload pools)
        raise ValueError("libds takes device tensors or pinned host tensors (no CPU path)")
    if not t.is_contiguous():
        raise ValueError("libds takes contiguous tensors")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check(status: int, what: str):
    if status == DS_ERR_GQA_INCOMPATIBLE:
        raise GqaIncompatible(status, what)
    if status != DS_OK:
        raise DsError(status, what)


@dataclass
class LayerCache:
    """Device buffers of one layer's cache (the ds_cache struct of ds.h).
    Allocation is plumbing (torch); contents are written by ds_append_kv."""
    batch: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    page_size: int
    max_seq_len: int
    r: int
    dtype: torch.dtype
    k_pool: torch.Tensor
    v_pool: torch.Tensor
    block_table: torch.Tensor
    seq_lens: torch.Tensor
    label: torch.Tensor
    channel_idx: torch.Tensor
    label_format: int = DS_LABEL_NATIVE
    label_scale: torch.Tensor | None = None
    group_reduce: int = DS_GROUP_SUM

    @staticmethod
    def allocate(batch, num_q_heads, num_kv_heads, head_dim, max_seq_len, r, dtype, block_table,
                 num_pages=None, page_size=16, device="cuda", channel_idx=None, host_kv=False,
                 label_format="native", group_reduce="sum"):
        """host_kv: K/V pools in pinned host memory (Double Sparsity-Offload,
        P:192): the kernels read them over the host link; label stays on device.
        label_format: "native" (label in K's dtype), "int4" (packed 4-bit
        codes uint8 [B][Hkv][S][ceil(r/2)] + a per-token scale [B][Hkv][S],
        P:171) or "none" (no label cache, the Table 4 ablation); ds.h
        ds_label_format.  group_reduce: "sum" (reading R3), "max" or
        "per_head" (ds.h ds_group_reduce)."""
        bt = torch.as_tensor(block_table, dtype=torch.int32).to(device).contiguous()
        npages = int(num_pages if num_pages is not None else int(bt.max()) + 1)
        pool = (npages, num_kv_heads, page_size, head_dim)

        def pool_buf():
            if host_kv:
                return torch.empty(pool, dtype=dtype, pin_memory=True)
            return torch.empty(pool, dtype=dtype, device=device)
        lf = _LF[label_format] if isinstance(label_format, str) else int(label_format)
        if lf == DS_LABEL_NONE:  # no label cache (Table 4 ablation): a 16-B placeholder, never read
            label = torch.empty(16, dtype=torch.uint8, device=device)
            scale = None
        elif lf == DS_LABEL_INT4:
            label = torch.empty((batch, num_kv_heads, max_seq_len, (r + 1) // 2), dtype=torch.uint8, device=device)
            scale = torch.empty((batch, num_kv_heads, max_seq_len), dtype=dtype, device=device)
        else:
            label = torch.empty((batch, num_kv_heads, max_seq_len, r), dtype=dtype, device=device)
            scale = None
        return LayerCache(
            batch, num_q_heads, num_kv_heads, head_dim, page_size, max_seq_len, r, dtype,
            pool_buf(), pool_buf(),
            bt, torch.zeros(batch, dtype=torch.int32, device=device), label,
            (torch.as_tensor(channel_idx, dtype=torch.int32).to(device).contiguous() if channel_idx is not None
             else torch.zeros((num_kv_heads, r), dtype=torch.int32, device=device)),
            lf, scale, _GR[group_reduce] if isinstance(group_reduce, str) else int(group_reduce))

    @property
    def num_pages(self):
        return self.k_pool.shape[0]

    def struct(self) -> ds_cache:
        return ds_cache(self.batch, self.num_q_heads, self.num_kv_heads, self.head_dim, self.page_size,
                        self.num_pages, self.block_table.shape[1], self.max_seq_len, self.r,
                        _DT[self.dtype], _ptr(self.k_pool), _ptr(self.v_pool), _ptr(self.block_table),
                        _ptr(self.seq_lens), _ptr(self.label), _ptr(self.channel_idx), self.label_format,
                        _ptr(self.label_scale), self.group_reduce)

    @property
    def label_bytes(self) -> int:
        n = self.label.numel() * self.label.element_size()
        return n + (self.label_scale.numel() * self.label_scale.element_size() if self.label_scale is not None else 0)


def ds_calibrate_channels(q_calib, k_calib, num_kv_heads, r, mode=DS_CALIB_QK, seed=0, out=None, stream=None):
    """Offline channel calibration. q_calib [n][Hq][d], k_calib [n][Hkv][d] -> int32 [Hkv][r]."""
    n, hq, d = q_calib.shape
    if out is None:
        out = torch.empty((num_kv_heads, r), dtype=torch.int32, device=q_calib.device)
    st = lib().ds_calibrate_channels(_ptr(q_calib), _ptr(k_calib), n, hq, num_kv_heads, d, _DT[q_calib.dtype],
                                     mode, r, ctypes.c_uint64(seed), _ptr(out), _stream(stream))
    _check(st, "ds_calibrate_channels")
    return out


def ds_append_kv(cache: LayerCache, k_new, v_new, positions, stream=None, cs=None):
    """Write K/V rows + label rows of n_new tokens per sequence. k_new [B][n_new][Hkv][d]."""
    cs = cs if cs is not None else cache.struct()
    st = lib().ds_append_kv(ctypes.byref(cs), _ptr(k_new), _ptr(v_new), _ptr(positions), k_new.shape[1],
                            _stream(stream))
    _check(st, "ds_append_kv")


def ds_decode_workspace_size(cache: LayerCache, k: int) -> int:
    return lib().ds_decode_workspace_size(ctypes.byref(cache.struct()), k)


def ds_decode_launches(cache: LayerCache, k: int) -> int:
    """Kernels one ds_decode_attention call enqueues: 1 (fused) or 2."""
    return lib().ds_decode_launches(ctypes.byref(cache.struct()), k)


def ds_dense_workspace_size(cache: LayerCache) -> int:
    return lib().ds_dense_workspace_size(ctypes.byref(cache.struct()))


def workspace(nbytes: int, device="cuda") -> torch.Tensor:
    """Zero-filled workspace (ds.h: zero before first use; the library leaves it zeroed)."""
    return torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=device)


def ds_decode_attention(cache: LayerCache, q, k, out=None, topk_idx_out=None, ws=None, stream=None, cs=None):
    """Algorithm 1. q [B][Hq][d] -> out [B][Hq][d]."""
    cs = cs if cs is not None else cache.struct()
    if out is None:
        out = torch.empty_like(q)
    if ws is None:
        ws = workspace(lib().ds_decode_workspace_size(ctypes.byref(cs), k), q.device)
    st = lib().ds_decode_attention(ctypes.byref(cs), _ptr(q), k, _ptr(out), _ptr(topk_idx_out), _ptr(ws),
                                   ws.numel(), _stream(stream))
    _check(st, "ds_decode_attention")
    return out


def ds_decode_attention_append(cache: LayerCache, k_new, v_new, positions, q, k, out=None, topk_idx_out=None,
                               ws=None, stream=None, cs=None):
    """One decode step in one launch: ds_append_kv of one token per sequence
    (k_new, v_new [B][1][Hkv][d], positions [B]) then Algorithm 1.  The
    caller has already set seq_lens to include the new token."""
    cs = cs if cs is not None else cache.struct()
    if out is None:
        out = torch.empty_like(q)
    if ws is None:
        ws = workspace(lib().ds_decode_workspace_size(ctypes.byref(cs), k), q.device)
    st = lib().ds_decode_attention_append(ctypes.byref(cs), _ptr(k_new), _ptr(v_new), _ptr(positions), _ptr(q), k,
                                          _ptr(out), _ptr(topk_idx_out), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "ds_decode_attention_append")
    return out


class ds_prefetch_slot(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("idx", ctypes.c_void_p), ("count", ctypes.c_void_p),
                ("table", ctypes.c_void_p), ("k_rows", ctypes.c_void_p), ("v_rows", ctypes.c_void_p)]


@dataclass
class PrefetchSlot:
    """One half of the offload double buffer (ds_prefetch_slot, device memory)."""
    k: int
    idx: torch.Tensor
    count: torch.Tensor
    table: torch.Tensor
    k_rows: torch.Tensor
    v_rows: torch.Tensor

    @staticmethod
    def allocate(cache: LayerCache, k: int, device="cuda"):
        B, H, d = cache.batch, cache.num_kv_heads, cache.head_dim
        return PrefetchSlot(k, torch.empty((B, H, k), dtype=torch.int32, device=device),
                            torch.zeros(B, dtype=torch.int32, device=device),
                            torch.zeros(B, dtype=torch.int32, device=device),
                            torch.empty((B, H, k, d), dtype=cache.dtype, device=device),
                            torch.empty((B, H, k, d), dtype=cache.dtype, device=device))

    def struct(self) -> ds_prefetch_slot:
        return ds_prefetch_slot(self.k, _ptr(self.idx), _ptr(self.count), _ptr(self.table), _ptr(self.k_rows),
                                _ptr(self.v_rows))


def ds_prefetch_next_layer(next_cache: LayerCache, q_pred, k, slot: PrefetchSlot = None, stream=None):
    """a6: select with the predicted query, gather the rows into a device slot."""
    slot = slot if slot is not None else PrefetchSlot.allocate(next_cache, k, q_pred.device)
    ss = slot.struct()
    st = lib().ds_prefetch_next_layer(ctypes.byref(next_cache.struct()), _ptr(q_pred), k, ctypes.byref(ss),
                                      _stream(stream))
    _check(st, "ds_prefetch_next_layer")
    return slot


def ds_decode_attention_prefetched(cache: LayerCache, q, slot: PrefetchSlot, out=None, stream=None):
    """Lines 4-5 with the true query over a prefetched slot."""
    if out is None:
        out = torch.empty_like(q)
    ss = slot.struct()
    st = lib().ds_decode_attention_prefetched(ctypes.byref(cache.struct()), _ptr(q), ctypes.byref(ss), _ptr(out),
                                              _stream(stream))
    _check(st, "ds_decode_attention_prefetched")
    return out


def ds_approx_scores(cache: LayerCache, q, out=None, stream=None):
    """Lines 1-2 of Alg. 1 only: fp32 [B][Hkv][max_seq_len]."""
    if out is None:
        out = torch.full((cache.batch, cache.num_kv_heads, cache.max_seq_len), float("nan"),
                         dtype=torch.float32, device=q.device)
    st = lib().ds_approx_scores(ctypes.byref(cache.struct()), _ptr(q), _ptr(out), _stream(stream))
    _check(st, "ds_approx_scores")
    return out


def ds_dense_decode_attention(cache: LayerCache, q, out=None, ws=None, stream=None, cs=None):
    """Dense decode baseline on the same paged layout."""
    cs = cs if cs is not None else cache.struct()
    if out is None:
        out = torch.empty_like(q)
    if ws is None:
        ws = workspace(lib().ds_dense_workspace_size(ctypes.byref(cs)), q.device)
    st = lib().ds_dense_decode_attention(ctypes.byref(cs), _ptr(q), _ptr(out), _ptr(ws), ws.numel(),
                                         _stream(stream))
    _check(st, "ds_dense_decode_attention")
    return out


def prefill(cache: LayerCache, K, V, seq_lens, stream=None):
    """Fill a cache from dense K, V [B][Hkv][S][d] through ds_append_kv (a0);
    sets seq_lens.  (Layout transpose to the append's [B][n][Hkv][d] is a
    torch copy: plumbing, not method arithmetic.)"""
    B = K.shape[0]
    kn = K.transpose(1, 2).contiguous()
    vn = V.transpose(1, 2).contiguous()
    pos = torch.zeros(B, dtype=torch.int32, device=K.device)
    ds_append_kv(cache, kn, vn, pos, stream=stream)
    cache.seq_lens.copy_(torch.as_tensor(seq_lens, dtype=torch.int32))


class CapturedStep:
    """A decode step built from the calls above (and torch copies), captured
    once in a CUDA graph on `stream` and replayed: one graph launch per step
    instead of a Python/ctypes call per kernel and copy.  The graph re-reads
    the same device and pinned host buffers on every replay, so a caller
    refreshes their contents between replays.  (Plumbing: the kernels are the
    ones the captured calls enqueue.)"""

    def __init__(self, fn, stream=None, warmup: int = 1):
        self.stream = stream if stream is not None else torch.cuda.Stream()
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                fn()
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            fn()

    def replay(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()
