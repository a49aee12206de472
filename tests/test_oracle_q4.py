"""Pins of the oracle's 4-bit label (reading R16 in
DESIGN.md): worked examples (tests/golden), brute-force nearest-grid-point
characterisation of the codes, the scale rounding against torch's dtype
conversion, the packing against a hand-worked byte string and an
independent numpy unpack, and the score degradation bound of SPEC S:231."""
import json
import os

import numpy as np
import pytest
import torch

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
TD = {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}


@pytest.mark.parametrize("name", ["quantize_4bit_spec_row", "quantize_4bit_zero_row"])
@pytest.mark.parametrize("dt", ["fp16", "bf16", "fp32"])
def test_quantize_spec_examples(name, dt):
    g = GOLD[name]
    codes, scale = oracle.quantize_label_4bit(np.array([g["row"]], np.float32), dt)
    assert codes[0].tolist() == g["codes"] and scale[0] == g["scale"]


def test_quantize_hand_example_fp32_scale():
    g = GOLD["quantize_4bit_hand"]
    codes, scale = oracle.quantize_label_4bit(np.array([g["row"]], np.float32), "fp32")
    assert codes[0].tolist() == g["codes"]
    assert scale[0] == np.float32(np.float32(1.4) / np.float32(7))
    assert abs(float(scale[0]) - g["scale_fp32"]) < 1e-7


def test_pack_hand_example():
    g = GOLD["pack_int4_hand"]
    assert oracle.pack_int4(np.array([g["codes"]], np.int8))[0].tolist() == g["bytes"]


def _unpack_numpy(b, r):
    lo = (b & 15).astype(np.int16)
    hi = (b >> 4).astype(np.int16)
    lo = np.where(lo > 7, lo - 16, lo)
    hi = np.where(hi > 7, hi - 16, hi)
    out = np.stack([lo, hi], axis=-1).reshape(b.shape[0], -1)
    return out[:, :r]


@pytest.mark.parametrize("r", [1, 3, 8, 16])
def test_pack_roundtrip(r):
    g = np.random.default_rng(r)
    codes = g.integers(-7, 8, size=(200, r)).astype(np.int8)
    packed = oracle.pack_int4(codes)
    assert packed.shape == (200, (r + 1) // 2)
    assert (_unpack_numpy(packed, r) == codes).all()
    if r % 2:
        assert (packed[:, -1] >> 4 == 0).all()


def _rows(seed, n=3000, r=8):
    g = np.random.default_rng(seed)
    x = g.standard_normal((n, r)).astype(np.float32) * np.exp(g.uniform(-6, 6, size=(n, 1))).astype(np.float32)
    x[::37] = 0.0                                # zero rows
    x[5::41, 3] = 0.0                            # zero entries
    x[7::43] = np.round(x[7::43])                # integer rows (ties at .5 appear after scaling)
    x[11::47] = np.array([7.0, 3.5, -3.5, 0.5, -0.5, 1.5, 2.5, -6.5], np.float32)[:r]  # scale 1: .5 ties
    return x


@pytest.mark.parametrize("dt", ["fp16", "bf16", "fp32"])
def test_scale_is_rounded_max_over_seven(dt):
    x = _rows(1)
    if dt == "fp16":
        x = np.clip(x, -60000, 60000)
    _, scale = oracle.quantize_label_4bit(x, dt)
    a = np.abs(x).max(axis=1)
    s32 = np.where(a == 0, np.float32(1), a / np.float32(7)).astype(np.float32)
    want = torch.from_numpy(s32).to(TD[dt]).float().numpy()   # torch's RNE dtype conversion
    want = np.where(want == 0, np.float32(1), want)
    assert (scale == want).all()


@pytest.mark.parametrize("dt", ["fp16", "bf16", "fp32"])
def test_codes_are_nearest_grid_point_brute_force(dt):
    """Every code is the c in [-7, 7] minimising |x/s - c| (in the fp32
    quotient), ties away from zero: a brute-force restatement of R16."""
    x = _rows(2)
    if dt == "fp16":
        x = np.clip(x, -60000, 60000)
    codes, scale = oracle.quantize_label_4bit(x, dt)
    v = (x / scale[:, None]).astype(np.float32).astype(np.float64)
    cand = np.arange(-7, 8, dtype=np.float64)
    dist = np.abs(v[..., None] - cand)
    best = dist.min(axis=-1, keepdims=True)
    ok = dist == best
    # among equidistant candidates take the one of larger magnitude
    mag = np.where(ok, np.abs(cand), -1)
    pick = cand[np.argmax(mag, axis=-1)]
    assert (codes == pick.astype(np.int8)).all()
    assert codes.min() >= -7 and codes.max() <= 7


def test_reconstruction_error_within_half_scale_fp32():
    x = _rows(3)
    codes, scale = oracle.quantize_label_4bit(x, "fp32")
    err = np.abs(codes.astype(np.float64) * scale[:, None] - x.astype(np.float64))
    assert (err <= scale[:, None].astype(np.float64) / 2 * (1 + 1e-6) + 1e-30).all()


def test_scores_q4_definition_and_degradation_bound():
    """s_hat_q = (sum_j qlab_j c_j) s up to fp32 rounding, and
    |s_hat_q - s_hat_float| <= sum_j |qlab_j| s/2 (triangle inequality)."""
    g = np.random.default_rng(4)
    for r in (1, 4, 8, 16):
        L = g.standard_normal((500, r)).astype(np.float32) * 3
        qlab = g.standard_normal(r).astype(np.float32)
        codes, scale = oracle.quantize_label_4bit(L, "fp32")
        sq = oracle.approx_scores_q4(qlab, codes, scale)
        exact = (codes.astype(np.float64) @ qlab.astype(np.float64)) * scale.astype(np.float64)
        mag = (np.abs(codes.astype(np.float64)) @ np.abs(qlab.astype(np.float64))) * scale
        assert np.all(np.abs(sq - exact) <= (r + 1) * 2.0 ** -24 * mag + 1e-30)
        sf = oracle.approx_scores(qlab, L)
        bound = np.abs(qlab).astype(np.float64).sum() * scale / 2
        assert np.all(np.abs(sq.astype(np.float64) - sf) <= bound * (1 + 1e-5) + 1e-5 * np.abs(sf))


def test_scores_q4_unit_scale_integer_label_equals_float_label_bitwise():
    """Special case: integer labels in [-7, 7] with max |.| = 7 quantise to
    themselves with scale 1, so line 2 over the 4-bit label is the 16-bit
    fma chain bit for bit."""
    g = np.random.default_rng(5)
    L = g.integers(-7, 8, size=(300, 8)).astype(np.float32)
    L[:, 0] = 7.0
    codes, scale = oracle.quantize_label_4bit(L, "bf16")
    assert (scale == 1).all() and (codes == L).all()
    qlab = g.standard_normal(8).astype(np.float32)
    assert (oracle.approx_scores_q4(qlab, codes, scale) == oracle.approx_scores(qlab, L)).all()


def test_decode_unit_q4_uses_q4_scores():
    g = np.random.default_rng(6)
    S, d, r, k, G = 300, 16, 4, 20, 2
    K = g.standard_normal((S, d)).astype(np.float32)
    V = g.standard_normal((S, d)).astype(np.float32)
    q = g.standard_normal((G, d)).astype(np.float32)
    C = np.array([1, 5, 9, 12], np.int32)
    L = oracle.label_gather(K, C)
    codes, scale = oracle.quantize_label_4bit(L, "fp16")
    y, idx, shat, tau = oracle.ds_decode_unit(q, K, V, L, C, k, codes=codes, scale=scale)
    want = oracle.approx_scores_q4(oracle.query_label(q, C), codes, scale)
    assert (shat == want).all()
    ref_idx, ref_tau = oracle.argtopk(want, k)
    assert (idx == ref_idx).all() and tau == ref_tau
    for gg in range(G):
        assert np.array_equal(y[gg], oracle.attend(q[gg], K, V, idx))
    # the batch driver agrees with the unit
    yb, ib = oracle.decode_batch(q[None, :, :], K[None, None], V[None, None], L[None, None], C[None], [S], k,
                                 codes=codes[None, None], scale=scale[None, None])
    assert np.array_equal(yb[0], y) and (ib[0, 0] == idx).all()
