"""Algorithmic-bytes model of the decode hot path (measurement, not method).

Sec. 5.3: memory access is O(d) for Q, O(S*r) for the label
cache and O(2*k*d) for the KV cache.  Per (b, KV head) unit with element
size e (the label has K's dtype, DESIGN reading R8):

    B_alg   = S*r*e + 2*k*d*e                     (north_star's counted bytes)
    B_all   = B_alg + G*d*e (q) + G*d*e (out) + 4*k (block-table entries, upper bound)
    B_dense = 2*S*d*e                             (+ q/out, same as above)

Top-k moves no algorithmic bytes.  k is per sequence:
k_eff = min(k, S_b).  With the 4-bit label (reading R16) a label row
is ceil(r/2) code bytes + one e-byte scale: S*r*e becomes S*(ceil(r/2) + e).
"""
from __future__ import annotations


def label_row_bytes(r: int, e: int, label: str = "native") -> int:
    return (r + 1) // 2 + e if label == "int4" else r * e


def unit_bytes_alg(S: int, d: int, r: int, k: int, e: int, label: str = "native") -> int:
    keff = min(k, S)
    return S * label_row_bytes(r, e, label) + 2 * keff * d * e


def unit_bytes_all(S: int, d: int, r: int, k: int, e: int, G: int, label: str = "native") -> int:
    keff = min(k, S)
    return unit_bytes_alg(S, d, r, k, e, label) + 2 * G * d * e + 4 * keff


def unit_bytes_dense(S: int, d: int, e: int) -> int:
    return 2 * S * d * e


def layer_bytes_alg(cfg, label: str = "native") -> int:
    return cfg.B * cfg.Hkv * unit_bytes_alg(cfg.S, cfg.d, cfg.r, cfg.k, cfg.elem, label)


def layer_bytes_dense(cfg) -> int:
    return cfg.B * cfg.Hkv * unit_bytes_dense(cfg.S, cfg.d, cfg.elem)


def byte_ratio_ceiling(cfg, label: str = "native") -> float:
    """Upper bound of the sparse/dense speedup at equal achieved bandwidth."""
    return layer_bytes_dense(cfg) / layer_bytes_alg(cfg, label)
