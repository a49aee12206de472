"""Pins for the CPU oracle (-m "not gpu").

Each test ties an oracle function to something other than itself: a worked
example from SPEC.md / the paper (tests/golden/spec_examples.json), a closed
form, a brute-force definition on tiny inputs, a library routine (torch SDPA
in fp64, numpy indexing) or an invariant the paper fixes.  Chosen so that a
dropped term, wrong sign/index or transposed operand in oracle/ds_oracle.c
fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- golden
@pytest.mark.parametrize("name", ["full_attention_zero_query", "full_attention_single_token",
                                  "full_attention_d2_closed_form"])
def test_dense_attention_worked_examples(name):
    ex = GOLD[name]
    y = oracle.dense_attention(np.array(ex["q"]), np.array(ex["K"]), np.array(ex["V"]))
    np.testing.assert_allclose(y, ex["y"], rtol=0, atol=ex["atol"] + 1e-7)


def test_approx_scores_worked_example():
    ex = GOLD["approx_scores_d4"]
    qlab = oracle.query_label(np.array(ex["q"]), np.array(ex["C"]))
    s = oracle.approx_scores(qlab, np.array(ex["L"]))
    np.testing.assert_array_equal(s, np.array(ex["shat"], np.float32))


@pytest.mark.parametrize("name", ["argtopk_tie_lower_index", "argtopk_all", "argtopk_signed_zero"])
def test_argtopk_worked_examples(name):
    ex = GOLD[name]
    idx, _ = oracle.argtopk(np.array(ex["scores"], np.float32), ex["k"])
    assert idx.tolist() == ex["idx"]


@pytest.mark.parametrize("name", ["select_channels_importance", "calibrate_one_hot_qk"])
def test_calibration_worked_examples(name):
    ex = GOLD[name]
    Qc, Kc = np.array(ex["Qc"]), np.array(ex["Kc"])
    C, imp = oracle.calibrate(Qc, Kc, Qc.shape[1], Kc.shape[1], ex["r"], mode=ex["mode"],
                              return_importance=True)
    assert C.tolist() == ex["C"]
    if "importance" in ex:
        np.testing.assert_array_equal(imp, np.array(ex["importance"]))


# ------------------------------------------------------------ a0 label
def test_label_gather_matches_fancy_indexing_bitwise():
    rng = np.random.default_rng(0)
    K = rng.standard_normal((97, 128)).astype(np.float32)
    K[3, 5] = -0.0
    C = np.sort(rng.choice(128, 8, replace=False)).astype(np.int32)
    C[0] = 5
    C = np.sort(C)
    L = oracle.label_gather(K, C)
    assert np.array_equal(L.view(np.uint32), np.ascontiguousarray(K[:, C]).view(np.uint32))


def test_label_full_channel_set_is_K():
    rng = np.random.default_rng(1)
    K = rng.standard_normal((33, 16)).astype(np.float32)
    L = oracle.label_gather(K, np.arange(16))
    assert np.array_equal(L.view(np.uint32), K.view(np.uint32))


# ------------------------------------------------------ a1 / a2 scores
def test_query_label_mha_is_channel_gather():
    rng = np.random.default_rng(2)
    q = rng.standard_normal((1, 64)).astype(np.float32)
    C = np.array([1, 7, 9, 33], np.int32)
    assert np.array_equal(oracle.query_label(q, C), q[0, C])


def test_query_label_gqa_group_sum():
    # closed form on exactly representable values: sum of the G heads
    q = np.zeros((4, 8), np.float32)
    for g in range(4):
        q[g] = np.arange(8) * (g + 1)       # integers: sums are exact
    C = np.array([0, 3, 7], np.int32)
    np.testing.assert_array_equal(oracle.query_label(q, C), np.array([0, 30, 70], np.float32))


def test_scores_full_channels_equal_exact_qk_within_fma_bound():
    # r = d, C = identity: s_hat = q.K^T; error bound of an
    # r-term fp32 fma chain: gamma_r * sum |q_j K_tj|
    rng = np.random.default_rng(3)
    d, S = 128, 500
    q = rng.standard_normal(d).astype(np.float32)
    K = rng.standard_normal((S, d)).astype(np.float32)
    C = np.arange(d, dtype=np.int32)
    s = oracle.approx_scores(oracle.query_label(q, C), oracle.label_gather(K, C))
    exact = K.astype(np.float64) @ q.astype(np.float64)
    bound = d * 2.0 ** -24 / (1 - d * 2.0 ** -24) * (np.abs(K.astype(np.float64)) @ np.abs(q.astype(np.float64)))
    assert np.all(np.abs(s - exact) <= bound)
    # a transposed operand / wrong channel would be far off
    assert np.max(np.abs(s - exact)) < 1e-3


def test_scores_zero_query_are_zero():
    L = np.random.default_rng(4).standard_normal((50, 8)).astype(np.float32)
    assert np.all(oracle.approx_scores(np.zeros(8, np.float32), L) == 0)


def test_scores_use_only_label_channels():
    # changing K outside C must not change s_hat (channel sparsity)
    rng = np.random.default_rng(5)
    K = rng.standard_normal((40, 32)).astype(np.float32)
    q = rng.standard_normal(32).astype(np.float32)
    C = np.array([2, 11, 30], np.int32)
    s1 = oracle.approx_scores(oracle.query_label(q, C), oracle.label_gather(K, C))
    K2 = K.copy()
    K2[:, [0, 1, 3, 12, 31]] += 100
    s2 = oracle.approx_scores(oracle.query_label(q, C), oracle.label_gather(K2, C))
    assert np.array_equal(s1, s2)


# ------------------------------------------------------------ a3 topk
def _rank_definition(scores, k):
    """Brute force: t is selected iff fewer than k tokens beat it, where t'
    beats t if s[t'] > s[t] or (s[t'] == s[t] and t' < t)."""
    S = len(scores)
    sel = []
    for t in range(S):
        beat = sum(1 for u in range(S) if scores[u] > scores[t] or (scores[u] == scores[t] and u < t))
        if beat < k:
            sel.append(t)
    return sel


def test_argtopk_matches_rank_definition_random_with_duplicates():
    rng = np.random.default_rng(6)
    for trial in range(3000):
        S = int(rng.integers(1, 40))
        vals = rng.integers(-4, 5, S).astype(np.float32) * 0.5  # many duplicates
        if trial % 3 == 0:
            vals = rng.standard_normal(S).astype(np.float32)
        if trial % 7 == 0:
            vals[rng.integers(0, S)] = -0.0
        k = int(rng.integers(1, S + 3))
        idx, _ = oracle.argtopk(vals, k)
        assert idx.tolist() == _rank_definition(vals.tolist(), min(k, S))


def test_argtopk_exhaustive_tiny():
    # every score pattern over {-1,0,1}^5 and every k
    for pat in itertools.product([-1.0, 0.0, 1.0], repeat=5):
        s = np.array(pat, np.float32)
        for k in range(1, 6):
            assert oracle.argtopk(s, k)[0].tolist() == _rank_definition(pat, k)


def test_argtopk_all_equal_and_k_ge_S():
    s = np.full(10, 3.25, np.float32)
    assert oracle.argtopk(s, 4)[0].tolist() == [0, 1, 2, 3]
    assert oracle.argtopk(s, 99)[0].tolist() == list(range(10))


def test_argtopk_tau_is_kth_largest():
    rng = np.random.default_rng(7)
    s = rng.standard_normal(1000).astype(np.float32)
    idx, tau = oracle.argtopk(s, 37)
    assert tau == np.sort(s)[::-1][36]
    assert set(idx.tolist()) == set(np.argsort(-s, kind="stable")[:37].tolist())


# --------------------------------------------------- a4 / a5 attention
def test_dense_attention_matches_torch_sdpa_fp64():
    rng = np.random.default_rng(8)
    for S, d in [(8, 4), (64, 16), (512, 64), (1000, 128)]:
        q = rng.standard_normal(d).astype(np.float32)
        K = (rng.standard_normal((S, d)) * 2).astype(np.float32)
        V = rng.standard_normal((S, d)).astype(np.float32)
        y = oracle.dense_attention(q, K, V)
        ref = torch.nn.functional.scaled_dot_product_attention(
            torch.from_numpy(q).double()[None, None, None], torch.from_numpy(K).double()[None, None],
            torch.from_numpy(V).double()[None, None])[0, 0, 0].numpy()
        np.testing.assert_allclose(y, ref, rtol=2e-5, atol=2e-6)


def test_attend_subset_matches_sdpa_on_gathered_rows():
    rng = np.random.default_rng(9)
    S, d = 300, 128
    q = rng.standard_normal(d).astype(np.float32)
    K = rng.standard_normal((S, d)).astype(np.float32) * 3
    V = rng.standard_normal((S, d)).astype(np.float32)
    idx = np.sort(rng.choice(S, 40, replace=False)).astype(np.int32)
    y = oracle.attend(q, K, V, idx)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q).double()[None, None, None], torch.from_numpy(K[idx]).double()[None, None],
        torch.from_numpy(V[idx]).double()[None, None])[0, 0, 0].numpy()
    np.testing.assert_allclose(y, ref, rtol=2e-5, atol=2e-6)


def test_attend_single_index_is_that_row():
    rng = np.random.default_rng(10)
    K = rng.standard_normal((20, 16)).astype(np.float32)
    V = rng.standard_normal((20, 16)).astype(np.float32)
    for t in [0, 7, 19]:
        assert np.array_equal(oracle.attend(rng.standard_normal(16), K, V, [t]), V[t])


def test_attention_weights_normalised_and_convex_hull():
    rng = np.random.default_rng(11)
    S, d = 200, 32
    q = rng.standard_normal(d).astype(np.float32) * 4
    K = rng.standard_normal((S, d)).astype(np.float32)
    idx = np.sort(rng.choice(S, 50, replace=False))
    ones = np.ones((S, d), np.float32)
    np.testing.assert_allclose(oracle.attend(q, K, ones, idx), 1.0, atol=1e-6)
    V = rng.standard_normal((S, d)).astype(np.float32)
    y = oracle.attend(q, K, V, idx)
    assert np.all(y <= V[idx].max(0) + 1e-6) and np.all(y >= V[idx].min(0) - 1e-6)


def test_scale_is_one_over_sqrt_d():
    # two tokens, logits differ by exactly dot/sqrt(d): weight ratio = exp(delta)
    d = 16
    q = np.zeros(d, np.float32)
    q[0] = 4.0
    K = np.zeros((2, d), np.float32)
    K[0, 0] = 1.0  # dot 4 -> logit 1
    V = np.array([[1.0] + [0] * 15, [0.0] * 16], np.float32)
    y = oracle.dense_attention(q, K, V)
    w0 = math.exp(1.0) / (math.exp(1.0) + 1.0)
    assert abs(y[0] - w0) < 1e-6


# ---------------------------------------------------- Algorithm 1 e2e
def test_ds_full_density_equals_dense_bitwise():
    # BJ north_star: "with r=d and k=S it must equal dense attention exactly"
    rng = np.random.default_rng(12)
    for S, d, G in [(8, 4, 1), (64, 16, 1), (512, 64, 1), (300, 128, 4)]:
        q = rng.standard_normal((G, d)).astype(np.float32)
        K = rng.standard_normal((S, d)).astype(np.float32)
        V = rng.standard_normal((S, d)).astype(np.float32)
        C = np.arange(d, dtype=np.int32)
        y, idx, _, _ = oracle.ds_decode_unit(q, K, V, oracle.label_gather(K, C), C, S)
        assert idx.tolist() == list(range(S))
        for g in range(G):
            assert np.array_equal(y[g], oracle.dense_attention(q[g], K, V))


def test_ds_full_channels_selects_exact_topk():
    # alpha=1 -> selection = argtopk of exact scores
    rng = np.random.default_rng(13)
    for _ in range(50):
        S, d = 128, 16
        q = rng.standard_normal(d).astype(np.float32)
        K = rng.standard_normal((S, d)).astype(np.float32)
        C = np.arange(d, dtype=np.int32)
        _, idx, _, _ = oracle.ds_decode_unit(q, K, K, oracle.label_gather(K, C), C, 16)
        exact = K.astype(np.float64) @ q.astype(np.float64)
        ref = np.sort(np.argsort(-exact, kind="stable")[:16])
        # fp32 fma vs fp64 can only swap near-ties
        sym = set(idx.tolist()) ^ set(ref.tolist())
        kth = np.sort(exact)[::-1][15]
        assert all(abs(exact[t] - kth) < 1e-4 for t in sym)


def test_ds_selection_then_truncated_attention_composes():
    rng = np.random.default_rng(14)
    S, d, r, k = 256, 64, 8, 32
    q = rng.standard_normal((2, d)).astype(np.float32)
    K = rng.standard_normal((S, d)).astype(np.float32)
    V = rng.standard_normal((S, d)).astype(np.float32)
    C = np.sort(rng.choice(d, r, replace=False)).astype(np.int32)
    L = oracle.label_gather(K, C)
    y, idx, shat, tau = oracle.ds_decode_unit(q, K, V, L, C, k)
    qlab = q[0, C].astype(np.float64) + q[1, C].astype(np.float64)
    np.testing.assert_allclose(shat, L.astype(np.float64) @ qlab, rtol=1e-5, atol=1e-5)
    assert idx.tolist() == _rank_definition(shat.tolist(), k)
    for g in range(2):
        np.testing.assert_array_equal(y[g], oracle.attend(q[g], K, V, idx))


def test_offload_selection_query_identity_collapses_to_ds():
    # q_hat = q -> identical selection and output
    rng = np.random.default_rng(15)
    S, d, r, k = 200, 32, 4, 25
    q = rng.standard_normal((1, d)).astype(np.float32)
    K = rng.standard_normal((S, d)).astype(np.float32)
    V = rng.standard_normal((S, d)).astype(np.float32)
    C = np.array([0, 5, 6, 20], np.int32)
    L = oracle.label_gather(K, C)
    a = oracle.ds_decode_unit(q, K, V, L, C, k)
    b = oracle.ds_decode_unit(q, K, V, L, C, k, q_sel=q.copy())
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = oracle.ds_decode_unit(q, K, V, L, C, k, q_sel=-q)
    assert not np.array_equal(a[1], c[1])


def test_decode_batch_equals_per_unit_and_threads_agree():
    cfg = synth.Config("t", B=2, Hq=8, Hkv=2, d=32, S=96, r=4, k=12, dtype="bf16")
    lay = synth.make_layer(cfg, seed=5, seq_lens=[96, 50])
    q, K, V = lay.q.float().numpy(), lay.K.float().numpy(), lay.V.float().numpy()
    C = lay.C_plant.numpy()
    L = np.stack([np.stack([oracle.label_gather(K[b, h], C[h]) for h in range(2)]) for b in range(2)])
    y1, i1 = oracle.decode_batch(q, K, V, L, C, lay.seq_lens.numpy(), cfg.k, nthreads=1)
    y4, i4 = oracle.decode_batch(q, K, V, L, C, lay.seq_lens.numpy(), cfg.k, nthreads=3)
    assert np.array_equal(y1, y4) and np.array_equal(i1, i4)
    for b in range(2):
        S = int(lay.seq_lens[b])
        for h in range(2):
            y, idx, _, _ = oracle.ds_decode_unit(q[b, h * 4:(h + 1) * 4], K[b, h, :S], V[b, h, :S],
                                                 L[b, h, :S], C[h], cfg.k)
            assert np.array_equal(y1[b, h * 4:(h + 1) * 4], y)
            assert i1[b, h, :len(idx)].tolist() == idx.tolist()
    yd, _ = oracle.decode_batch(q, K, V, None, None, lay.seq_lens.numpy(), cfg.k, mode=1)
    np.testing.assert_array_equal(yd[1, 0], oracle.dense_attention(q[1, 0], K[1, 0, :50], V[1, 0, :50]))


# --------------------------------------------------------- calibration
@pytest.mark.parametrize("mode", [oracle.MODE_QK, oracle.MODE_Q, oracle.MODE_K])
def test_calibration_recovers_planted_channels_mha(mode):
    for seed in range(20):
        cfg = synth.Config("t", B=1, Hq=4, Hkv=4, d=64, S=8, r=4, k=2, dtype="fp32")
        Qc, Kc = synth.make_calibration(cfg, n=64, seed=seed)
        C = oracle.calibrate(Qc.numpy(), Kc.numpy(), 4, 4, 4, mode=mode)
        assert np.array_equal(C, synth.plant_channels(cfg, seed).numpy())


@pytest.mark.parametrize("mode", [oracle.MODE_QK, oracle.MODE_Q])
def test_calibration_recovers_planted_channels_gqa(mode):
    for seed in range(20):
        cfg = synth.Config("t", B=1, Hq=8, Hkv=2, d=128, S=8, r=8, k=2, dtype="bf16")
        Qc, Kc = synth.make_calibration(cfg, n=128, seed=seed)
        C = oracle.calibrate(Qc.float().numpy(), Kc.float().numpy(), 8, 2, 8, mode=mode)
        assert np.array_equal(C, synth.plant_channels(cfg, seed).numpy())


def test_calibration_gqa_k_mode_incompatible():
    Qc = np.ones((2, 8, 16), np.float32)
    Kc = np.ones((2, 2, 16), np.float32)
    with pytest.raises(oracle.GqaIncompatible):
        oracle.calibrate(Qc, Kc, 8, 2, 4, mode=oracle.MODE_K)


def test_calibration_scale_invariance_and_full_r():
    rng = np.random.default_rng(16)
    Qc = rng.standard_normal((32, 4, 16)).astype(np.float32)
    Kc = rng.standard_normal((32, 2, 16)).astype(np.float32)
    C1 = oracle.calibrate(Qc, Kc, 4, 2, 5)
    C2 = oracle.calibrate(Qc * 4, Kc * 0.5, 4, 2, 5)
    assert np.array_equal(C1, C2)
    assert oracle.calibrate(Qc, Kc, 4, 2, 16).tolist() == [list(range(16))] * 2


def test_calibration_importance_is_separable_abs_sum():
    # P:149 decomposition, reading R5: imp_j = sum_{n,m,g} |Q_ngj K_mj| = (sum|Q|)(sum|K|)
    rng = np.random.default_rng(17)
    Qc = rng.integers(-3, 4, (6, 2, 8)).astype(np.float32)
    Kc = rng.integers(-3, 4, (6, 1, 8)).astype(np.float32)
    _, imp = oracle.calibrate(Qc, Kc, 2, 1, 3, return_importance=True)
    brute = np.zeros(8)
    for n in range(6):
        for m in range(6):
            for g in range(2):
                brute += np.abs(Qc[n, g] * Kc[m, 0])
    np.testing.assert_array_equal(imp[0], brute)


def test_calibration_random_mode_deterministic_distinct():
    Qc = np.zeros((1, 2, 64), np.float32)
    Kc = np.zeros((1, 2, 64), np.float32)
    a = oracle.calibrate(Qc, Kc, 2, 2, 8, mode=oracle.MODE_RANDOM, seed=42)
    b = oracle.calibrate(Qc, Kc, 2, 2, 8, mode=oracle.MODE_RANDOM, seed=42)
    c = oracle.calibrate(Qc, Kc, 2, 2, 8, mode=oracle.MODE_RANDOM, seed=43)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    for row in a:
        assert len(set(row.tolist())) == 8 and list(row) == sorted(row) and row.min() >= 0 and row.max() < 64
