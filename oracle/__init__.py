"""CPU oracle for the Double Sparsity decode hot path (arXiv 2408.07092).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this package.  The product package ``paper_2408_07092_b200`` never imports
it, and the two share no code (see ``ds_oracle.c`` for the arithmetic and
the paper passages each function follows).

This module only marshals numpy arrays into the plain-C oracle; it holds no
arithmetic of the method.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ds_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libds_oracle.so")
_lib = None

MODE_QK, MODE_Q, MODE_K, MODE_RANDOM = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile ds_oracle.c with gcc (IEEE fp32, no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + ".tmp.%d" % os.getpid()
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared",
             "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i = ctypes.c_int
        L.oracle_label_gather.argtypes = [P, i, i, P, i, P]
        L.oracle_query_label.argtypes = [P, i, i, P, i, P]
        L.oracle_approx_scores.argtypes = [P, P, i, i, P]
        L.oracle_argtopk.argtypes = [P, i, i, P, P]
        L.oracle_argtopk.restype = i
        L.oracle_attend.argtypes = [P, P, P, i, P, i, P]
        L.oracle_dense_attention.argtypes = [P, P, P, i, i, P]
        L.oracle_quantize_label_4bit.argtypes = [P, i, i, i, P, P]
        L.oracle_pack_int4.argtypes = [P, i, i, P]
        L.oracle_approx_scores_q4.argtypes = [P, P, P, i, i, P]
        L.oracle_ds_decode_unit.argtypes = [P, P, i, P, P, P, P, P, P, i, i, i, i, P, P, P, P]
        L.oracle_ds_decode_unit.restype = i
        L.oracle_ds_decode_unit_group.argtypes = [P, P, i, P, P, P, P, P, P, i, i, i, i, i, P, P, P]
        L.oracle_ds_decode_unit_group.restype = i
        L.oracle_decode_batch.argtypes = [P, P, P, P, P, P, P, P, P, i, i, i, i, i, i, i, i, P, P, i]
        L.oracle_decode_batch.restype = i
        L.oracle_calibrate.argtypes = [P, P, i, i, i, i, i, i, ctypes.c_uint64, P, P]
        L.oracle_calibrate.restype = i
        _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def label_gather(K, C):
    """a0: L[t][j] = K[t][C[j]]   (K [S][d], C [r]) -> [S][r]."""
    K, C = _f32(K), _i32(C)
    S, d = K.shape
    L = np.empty((S, C.shape[0]), np.float32)
    lib().oracle_label_gather(_p(K), S, d, _p(C), C.shape[0], _p(L))
    return L


def query_label(q, C):
    """a1: q [G][d] (or [d]) -> qlab [r] (group sum in g order)."""
    q = _f32(q)
    if q.ndim == 1:
        q = q[None]
    C = _i32(C)
    out = np.empty(C.shape[0], np.float32)
    lib().oracle_query_label(_p(q), q.shape[0], q.shape[1], _p(C), C.shape[0], _p(out))
    return out


def approx_scores(qlab, L):
    """a2: s_hat[t] = fma-chain_j qlab[j]*L[t][j]."""
    qlab, L = _f32(qlab), _f32(L)
    out = np.empty(L.shape[0], np.float32)
    lib().oracle_approx_scores(_p(qlab), _p(L), L.shape[0], L.shape[1], _p(out))
    return out


SCALE_FP16, SCALE_BF16, SCALE_FP32 = 0, 1, 2   # the ds_dtype numbering
SCALE_DTYPE = {"fp16": SCALE_FP16, "bf16": SCALE_BF16, "fp32": SCALE_FP32}


def quantize_label_4bit(L, scale_dtype):
    """f2 (reading R16): L [S][r] -> (codes int8 [S][r] in [-7, 7], scale fp32 [S])."""
    L = _f32(L)
    S, r = L.shape
    codes = np.empty((S, r), np.int8)
    scale = np.empty(S, np.float32)
    lib().oracle_quantize_label_4bit(_p(L), S, r, SCALE_DTYPE.get(scale_dtype, scale_dtype), _p(codes),
                                     _p(scale))
    return codes, scale


def pack_int4(codes):
    """The stored code bytes [S][ceil(r/2)]: code 2i low nibble, 2i+1 high nibble."""
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    S, r = codes.shape
    out = np.empty((S, (r + 1) // 2), np.uint8)
    lib().oracle_pack_int4(_p(codes), S, r, _p(out))
    return out


def approx_scores_q4(qlab, codes, scale):
    """a2 over a 4-bit label: s_hat[t] = (fma-chain_j qlab[j]*c[t][j]) * scale[t]."""
    qlab, scale = _f32(qlab), _f32(scale)
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    out = np.empty(codes.shape[0], np.float32)
    lib().oracle_approx_scores_q4(_p(qlab), _p(codes), _p(scale), codes.shape[0], codes.shape[1], _p(out))
    return out


def argtopk(scores, k):
    """a3: ascending indices of the k largest scores, ties -> lower index. Returns (idx, tau)."""
    s = _f32(scores)
    idx = np.empty(max(1, min(k, s.shape[0])), np.int32)
    tau = np.zeros(1, np.float32)
    n = lib().oracle_argtopk(_p(s), s.shape[0], k, _p(idx), _p(tau))
    return idx[:n], float(tau[0])


def attend(q, K, V, idx):
    """a4-a5 for one query head over the given rows."""
    q, K, V, idx = _f32(q), _f32(K), _f32(V), _i32(idx)
    y = np.empty(K.shape[1], np.float32)
    lib().oracle_attend(_p(q), _p(K), _p(V), K.shape[1], _p(idx), idx.shape[0], _p(y))
    return y


def dense_attention(q, K, V):
    q, K, V = _f32(q), _f32(K), _f32(V)
    y = np.empty(K.shape[1], np.float32)
    lib().oracle_dense_attention(_p(q), _p(K), _p(V), K.shape[0], K.shape[1], _p(y))
    return y


def ds_decode_unit(q, K, V, L, C, k, q_sel=None, codes=None, scale=None):
    """Algorithm 1 for one unit. q [G][d]. Returns (y [G][d], idx, shat, tau).
    codes/scale (from quantize_label_4bit): line 2 over the 4-bit label."""
    q = _f32(q)
    if q.ndim == 1:
        q = q[None]
    qs = q if q_sel is None else _f32(q_sel).reshape(q.shape)
    K, V, L, C = _f32(K), _f32(V), _f32(L), _i32(C)
    S, d = K.shape
    G = q.shape[0]
    y = np.empty((G, d), np.float32)
    idx = np.empty(max(1, min(k, S)), np.int32)
    shat = np.empty(max(1, S), np.float32)
    tau = np.zeros(1, np.float32)
    if scale is not None:
        codes = np.ascontiguousarray(codes, dtype=np.int8)
        scale = _f32(scale)
    n = lib().oracle_ds_decode_unit(_p(q), _p(qs), G, _p(K), _p(V), _p(L), _p(codes), _p(scale), _p(C), S,
                                    d, L.shape[1], k, _p(y), _p(idx), _p(shat), _p(tau))
    return y, idx[:n], shat[:S], float(tau[0])


GROUP_MODES = {"sum": 0, "max": 1, "per_head": 2}


def ds_decode_unit_group(q, K, V, L, C, k, group="sum", q_sel=None, codes=None, scale=None):
    """Algorithm 1 for one GQA unit under a group-reduction reading (R3 sum,
    R17 max / per_head).  Returns (y [G][d], idx, shat): idx [k_eff] and
    shat [S] for sum/max, idx [G][k] (-1 padded) and shat [G][S] per head."""
    q = _f32(q)
    if q.ndim == 1:
        q = q[None]
    qs = q if q_sel is None else _f32(q_sel).reshape(q.shape)
    K, V, L, C = _f32(K), _f32(V), _f32(L), _i32(C)
    if scale is not None:
        codes = np.ascontiguousarray(codes, dtype=np.int8)
        scale = _f32(scale)
    S, d = K.shape
    G = q.shape[0]
    mode = GROUP_MODES[group]
    y = np.empty((G, d), np.float32)
    idx = np.empty((G, max(k, 1)) if mode == 2 else (max(1, min(k, S)),), np.int32)
    shat = np.empty((G, max(S, 1)) if mode == 2 else (max(S, 1),), np.float32)
    n = lib().oracle_ds_decode_unit_group(_p(q), _p(qs), G, _p(K), _p(V), _p(L), _p(codes), _p(scale), _p(C), S,
                                          d, L.shape[1], k, mode, _p(y), _p(idx), _p(shat))
    if mode == 2:
        return y, idx[:, :k], shat[:, :S]
    return y, idx[:n], shat[:S]


def decode_batch(q, K, V, L, C, seq_lens, k, mode=0, q_sel=None, nthreads=1, codes=None, scale=None):
    """Batched oracle. q [B][Hq][d]; K,V [B][Hkv][Smax][d]; L [B][Hkv][Smax][r];
    C [Hkv][r]; seq_lens [B]. mode 0 = DS (Alg. 1), 1 = dense. Returns (y, idx).
    codes [B][Hkv][Smax][r] + scale [B][Hkv][Smax]: score over the 4-bit label."""
    q, K, V = _f32(q), _f32(K), _f32(V)
    B, Hq, d = q.shape
    Hkv, Smax = K.shape[1], K.shape[2]
    Lp = _f32(L) if L is not None else np.zeros((1,), np.float32)
    r = L.shape[3] if L is not None else 1
    C = _i32(C) if C is not None else np.zeros((Hkv, 1), np.int32)
    seq = _i32(seq_lens)
    qs = _f32(q_sel) if q_sel is not None else None
    y = np.zeros((B, Hq, d), np.float32)
    idx = np.full((B, Hkv, max(k, 1)), -1, np.int32)
    if scale is not None:
        codes = np.ascontiguousarray(codes, dtype=np.int8)
        scale = _f32(scale)
    rc = lib().oracle_decode_batch(_p(q), _p(qs), _p(K), _p(V), _p(Lp), _p(codes), _p(scale), _p(C), _p(seq),
                                   B, Hq, Hkv,
                                   Smax, d, r, k, mode, _p(y), _p(idx) if mode == 0 else None,
                                   nthreads)
    if rc != 0:
        raise ValueError("oracle_decode_batch: bad arguments")
    return y, idx


class GqaIncompatible(ValueError):
    pass


def calibrate(Qc, Kc, Hq, Hkv, r, mode=MODE_QK, seed=0, return_importance=False):
    """Offline channel calibration. Qc [n][Hq][d], Kc [n][Hkv][d] -> C [Hkv][r] ascending."""
    Qc, Kc = _f32(Qc), _f32(Kc)
    n, _, d = Qc.shape
    C = np.empty((Hkv, r), np.int32)
    imp = np.empty((Hkv, d), np.float64)
    rc = lib().oracle_calibrate(_p(Qc), _p(Kc), n, Hq, Hkv, d, mode, r, ctypes.c_uint64(seed),
                                _p(C), _p(imp))
    if rc == -2:
        raise GqaIncompatible("k-outlier calibration is N/A for GQA (paper Table 3)")
    if rc != 0:
        raise ValueError("oracle_calibrate: bad arguments")
    return (C, imp) if return_importance else C
