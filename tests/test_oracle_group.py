"""Pins of the oracle's GQA group-reduction readings (R3 sum, R17 max and
per head): a hand-worked example where the three readings
select different tokens, G = 1 collapse, identical-head collapse, the rank
definition of the max reading by brute force, and per-head = MHA."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_hand_example_three_readings_differ():
    g = GOLD["gqa_group_readings_hand"]
    q, K, C = np.array(g["q"]), np.array(g["K"]), np.array(g["C"])
    L = oracle.label_gather(K, C)
    for mode in ("sum", "max"):
        _, idx, _ = oracle.ds_decode_unit_group(q, K, K, L, C, g["k"], group=mode)
        assert idx.tolist() == g["idx"][mode], mode
    _, idx, _ = oracle.ds_decode_unit_group(q, K, K, L, C, g["k"], group="per_head")
    assert idx.tolist() == g["idx"]["per_head"]


def _unit(seed, G=4, S=300, d=32, r=4):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((S, d)).astype(np.float32)
    V = rng.standard_normal((S, d)).astype(np.float32)
    q = rng.standard_normal((G, d)).astype(np.float32)
    C = np.sort(rng.choice(d, r, replace=False)).astype(np.int32)
    return q, K, V, C, oracle.label_gather(K, C)


def test_single_head_all_readings_equal_bitwise():
    q, K, V, C, L = _unit(1, G=1)
    y0, i0, s0 = oracle.ds_decode_unit_group(q, K, V, L, C, 20, "sum")
    for mode in ("max", "per_head"):
        y, i, s = oracle.ds_decode_unit_group(q, K, V, L, C, 20, mode)
        assert np.array_equal(y, y0) and np.array_equal(np.asarray(i).ravel(), i0)
        assert np.array_equal(np.asarray(s).ravel(), s0)


def test_identical_heads_collapse():
    """q_g all equal: max == per-head == sum selections (the sum scales the
    query label by G = 4, a power of two: scores scale exactly)."""
    q, K, V, C, L = _unit(2)
    q[:] = q[0]
    _, isum, _ = oracle.ds_decode_unit_group(q, K, V, L, C, 25, "sum")
    _, imax, smax = oracle.ds_decode_unit_group(q, K, V, L, C, 25, "max")
    _, iph, _ = oracle.ds_decode_unit_group(q, K, V, L, C, 25, "per_head")
    assert np.array_equal(isum, imax) and all(np.array_equal(iph[g], imax) for g in range(4))


def test_max_reading_rank_definition_brute_force():
    for seed in range(20):
        q, K, V, C, L = _unit(10 + seed, S=40, d=8, r=3)
        k = 1 + seed % 12
        _, idx, shat = oracle.ds_decode_unit_group(q, K, V, L, C, k, "max")
        per = np.stack([oracle.approx_scores(oracle.query_label(q[g], C), L) for g in range(4)])
        assert np.array_equal(shat, per.max(axis=0))
        sel = set(idx.tolist())
        # every selected token outranks every other under (score desc, index asc)
        for t in sel:
            for u in set(range(40)) - sel:
                assert shat[t] > shat[u] or (shat[t] == shat[u] and t < u)


def test_per_head_is_mha_over_shared_kv():
    q, K, V, C, L = _unit(3)
    y, idx, shat = oracle.ds_decode_unit_group(q, K, V, L, C, 30, "per_head")
    for g in range(4):
        yg, ig, sg, _ = oracle.ds_decode_unit(q[g], K, V, L, C, 30)
        assert np.array_equal(y[g], yg[0]) and np.array_equal(idx[g], ig) and np.array_equal(shat[g], sg)
