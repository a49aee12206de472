"""GPU parity: the CUDA path through the C ABI vs the CPU oracle (-m gpu).

Small shapes the oracle finishes in seconds that still span several CTAs,
clusters and ragged tails; edge cases (k >= S, k = 1, S = 1, S = 0, ties,
odd page sizes); and BASELINE.json's full sizes in the bench launch
configuration with sampled units.  Tolerances: DESIGN.md R13/R14."""
import numpy as np
import pytest
import torch

import oracle
import paper_2408_07092_b200 as ds
import synth
from parity import build_cache, check_output, check_units, sample_units, unit_host

pytestmark = pytest.mark.gpu


def all_units(cfg):
    return [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]


def run_decode(cache, lay, k):
    cfg = lay.cfg
    idx = torch.empty((cfg.B, cfg.Hkv, k), dtype=torch.int32, device="cuda")
    y = ds.ds_decode_attention(cache, lay.q, k, topk_idx_out=idx)
    torch.cuda.synchronize()
    return y, idx


SMALL = [
    # name, cfg, seq_lens, k
    ("c1", synth.CONFIGS["c1"], None, 64),
    ("gqa4_bf16_ragged", synth.Config("g4", B=3, Hq=8, Hkv=2, d=128, S=3000, r=8, k=300, dtype="bf16"),
     [3000, 1777, 65], 300),
    ("mha_fp16", synth.Config("m", B=2, Hq=4, Hkv=4, d=128, S=2048, r=8, k=128, dtype="fp16"), None, 128),
    ("gqa8_bf16", synth.Config("g8", B=2, Hq=16, Hkv=2, d=128, S=1500, r=8, k=100, dtype="bf16"), [1500, 999], 100),
    ("gqa2_fp16_d64", synth.Config("g2", B=2, Hq=4, Hkv=2, d=64, S=1000, r=4, k=77, dtype="fp16"), [1000, 513], 77),
    ("page7_bf16", synth.Config("p7", B=2, Hq=4, Hkv=1, d=128, S=777, r=8, k=50, dtype="bf16", page_size=7),
     [777, 400], 50),
    ("fp32_gqa4", synth.Config("f", B=1, Hq=4, Hkv=1, d=128, S=600, r=16, k=40, dtype="fp32"), None, 40),
    ("r3_bf16", synth.Config("r3", B=1, Hq=2, Hkv=1, d=128, S=500, r=3, k=31, dtype="bf16"), None, 31),
]


@pytest.mark.parametrize("name,cfg,seq_lens,k", SMALL, ids=[s[0] for s in SMALL])
def test_decode_parity_small(name, cfg, seq_lens, k):
    lay, cache, C = build_cache(cfg, seq_lens=seq_lens)
    y, idx = run_decode(cache, lay, k)
    check_units(lay, cache, C, k, all_units(cfg), y, idx)


@pytest.mark.parametrize("structure", ["clustered"])
def test_decode_parity_clustered(structure):
    cfg = synth.Config("cl", B=2, Hq=8, Hkv=2, d=128, S=4096, r=8, k=256, dtype="bf16")
    lay, cache, C = build_cache(cfg, structure=structure, seq_lens=[4096, 3001])
    y, idx = run_decode(cache, lay, 256)
    check_units(lay, cache, C, 256, all_units(cfg), y, idx)


def test_label_cache_and_pool_bit_exact():
    """a0: label == channel gather of K (bit-exact), pool rows == K/V rows."""
    cfg = synth.Config("a0", B=2, Hq=8, Hkv=2, d=128, S=300, r=8, k=10, dtype="bf16", page_size=16)
    lay, cache, C = build_cache(cfg, seq_lens=[300, 123])
    lab = cache.label.cpu()
    kp, vp = cache.k_pool.cpu(), cache.v_pool.cpu()
    bt = lay.block_table
    for b in range(cfg.B):
        S = int(lay.seq_lens[b])
        for h in range(cfg.Hkv):
            K = lay.K[b, h, :S].cpu()
            exp = oracle.label_gather(K.float().numpy(), C[h].numpy())
            got = lab[b, h, :S].float().numpy()
            assert np.array_equal(got.view(np.uint32), exp.view(np.uint32))
            t = torch.arange(S)
            pages = bt[b, t // cfg.page_size].long()
            assert torch.equal(kp[pages, h, t % cfg.page_size], K)
            assert torch.equal(vp[pages, h, t % cfg.page_size], lay.V[b, h, :S].cpu())


def test_append_one_by_one_equals_bulk():
    """Incremental decode appends == prefill append, bit-exact."""
    cfg = synth.Config("inc", B=2, Hq=4, Hkv=2, d=64, S=40, r=4, k=8, dtype="fp16", page_size=8)
    lay, cache, C = build_cache(cfg)
    c2 = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, torch.float16, lay.block_table,
                                num_pages=lay.num_pages, page_size=8, channel_idx=C)
    c2.label.zero_()
    c2.k_pool.zero_()
    c2.v_pool.zero_()
    cache2 = c2
    for t in range(cfg.S):
        kn = lay.K[:, :, t:t + 1].transpose(1, 2).contiguous()
        vn = lay.V[:, :, t:t + 1].transpose(1, 2).contiguous()
        ds.ds_append_kv(cache2, kn, vn, torch.full((cfg.B,), t, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(cache2.label, cache.label)
    assert torch.equal(cache2.k_pool, cache.k_pool) and torch.equal(cache2.v_pool, cache.v_pool)


@pytest.mark.parametrize("cfgname", ["c1", "gqa"])
def test_approx_scores_bit_exact(cfgname):
    """a1+a2: s_hat is the same fp32 fma chain as the oracle -> bit-identical."""
    cfg = synth.CONFIGS["c1"] if cfgname == "c1" else synth.Config("s", B=2, Hq=8, Hkv=2, d=128, S=2000, r=8, k=9,
                                                                   dtype="bf16")
    lay, cache, C = build_cache(cfg, seq_lens=None)
    s = ds.ds_approx_scores(cache, lay.q).cpu().numpy()
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            q, K, V = unit_host(lay, b, h)
            ref = oracle.approx_scores(oracle.query_label(q, C[h].numpy()), oracle.label_gather(K, C[h].numpy()))
            assert np.array_equal(s[b, h, :K.shape[0]].view(np.uint32), ref.view(np.uint32))


def test_full_density_equals_dense():
    """r = d, C = identity, k = S: Algorithm 1 must reduce to dense attention."""
    cfg = synth.Config("fd", B=2, Hq=8, Hkv=2, d=64, S=700, r=64, k=700, dtype="bf16")
    C = torch.arange(64, dtype=torch.int32)[None].repeat(2, 1)
    lay, cache, _ = build_cache(cfg, C=C, seq_lens=[700, 333])
    y, idx = run_decode(cache, lay, 700)
    yd = ds.ds_dense_decode_attention(cache, lay.q)
    torch.cuda.synchronize()
    assert idx[1, 0, :333].tolist() == list(range(333)) and (idx[1, 0, 333:] == -1).all()
    for b in range(2):
        for h in range(2):
            q, K, V = unit_host(lay, b, h)
            for g in range(4):
                ref = oracle.dense_attention(q[g], K, V)
                check_output(y[b, h * 4 + g].float().cpu().numpy(), ref, "bf16")
                check_output(yd[b, h * 4 + g].float().cpu().numpy(), ref, "bf16")


@pytest.mark.parametrize("k", [1, 2, 5000])
def test_k_edge_cases(k):
    cfg = synth.Config("ke", B=2, Hq=4, Hkv=1, d=128, S=5000, r=8, k=k, dtype="bf16")
    lay, cache, C = build_cache(cfg, seq_lens=[5000, 1])
    y, idx = run_decode(cache, lay, k)
    check_units(lay, cache, C, k, all_units(cfg), y, idx)


def test_all_scores_tied_takes_lowest_indices():
    """q = 0 -> every s_hat is 0: the selection must be tokens 0..k-1 across all
    CTAs of the cluster (tie-break R6), and the output the mean of their V."""
    cfg = synth.Config("tie", B=1, Hq=4, Hkv=1, d=128, S=20000, r=8, k=1500, dtype="bf16")
    lay, cache, C = build_cache(cfg)
    lay.q.zero_()
    y, idx = run_decode(cache, lay, 1500)
    assert idx[0, 0].tolist() == list(range(1500))
    ref = lay.V[0, 0, :1500].float().mean(0).cpu().numpy()
    for g in range(4):
        check_output(y[0, g].float().cpu().numpy(), ref, "bf16")


def test_duplicate_scores_tie_break():
    """Many exactly equal scores straddling the threshold (label values from
    a tiny set) -> tie-break by lower index, matching the oracle exactly."""
    cfg = synth.Config("dup", B=1, Hq=1, Hkv=1, d=128, S=9000, r=8, k=1000, dtype="bf16")
    lay, cache, C = build_cache(cfg)
    g = torch.Generator(device="cuda").manual_seed(9)
    vals = torch.randint(-2, 3, (9000, 8), generator=g, device="cuda").to(torch.bfloat16)
    Kd = lay.K.clone()
    Kd[0, 0][:, C[0].long().cuda()] = vals
    lay.K.copy_(Kd)
    ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
    lay.q[0, 0, C[0].long().cuda()] = torch.tensor([1, 2, 1, 1, 2, 1, 1, 1], dtype=torch.bfloat16, device="cuda")
    y, idx = run_decode(cache, lay, 1000)
    q, K, V = unit_host(lay, 0, 0)
    L = oracle.label_gather(K, C[0].numpy())
    _, idx_ref, _, _ = oracle.ds_decode_unit(q, K, V, L, C[0].numpy(), 1000)
    assert idx[0, 0].cpu().numpy().tolist() == idx_ref.tolist()


def test_empty_sequence_gives_zero_output():
    cfg = synth.Config("z", B=2, Hq=4, Hkv=1, d=128, S=256, r=8, k=16, dtype="bf16")
    lay, cache, C = build_cache(cfg, seq_lens=[256, 0])
    y, idx = run_decode(cache, lay, 16)
    assert (y[1] == 0).all() and (idx[1] == -1).all()
    check_units(lay, cache, C, 16, [(0, 0)], y, idx)


@pytest.mark.parametrize("mode", [ds.DS_CALIB_QK, ds.DS_CALIB_Q, ds.DS_CALIB_K, ds.DS_CALIB_RANDOM])
def test_calibration_matches_oracle(mode):
    Hq = 8 if mode != ds.DS_CALIB_K else 4
    cfg = synth.Config("cal", B=1, Hq=Hq, Hkv=4 if mode == ds.DS_CALIB_K else 2, d=128, S=8, r=8, k=2,
                       dtype="bf16")
    Qc, Kc = synth.make_calibration(cfg, n=512, seed=7, device="cuda")
    got = ds.ds_calibrate_channels(Qc, Kc, cfg.Hkv, cfg.r, mode=mode, seed=11).cpu().numpy()
    exp = oracle.calibrate(Qc.float().cpu().numpy(), Kc.float().cpu().numpy(), cfg.Hq, cfg.Hkv, cfg.r,
                           mode=mode, seed=11)
    assert np.array_equal(got, exp)
    if mode != ds.DS_CALIB_RANDOM:
        assert np.array_equal(got, synth.plant_channels(cfg, 7).numpy())


def test_calibration_gqa_k_raises():
    Qc = torch.ones((4, 8, 128), dtype=torch.bfloat16, device="cuda")
    Kc = torch.ones((4, 2, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ds.GqaIncompatible):
        ds.ds_calibrate_channels(Qc, Kc, 2, 8, mode=ds.DS_CALIB_K)


def test_dense_parity_ragged():
    cfg = synth.Config("dn", B=3, Hq=8, Hkv=2, d=128, S=5000, r=8, k=8, dtype="bf16")
    lay, cache, C = build_cache(cfg, seq_lens=[5000, 2345, 17])
    yd = ds.ds_dense_decode_attention(cache, lay.q).float().cpu().numpy()
    for b in range(3):
        for h in range(2):
            q, K, V = unit_host(lay, b, h)
            for g in range(4):
                check_output(yd[b, h * 4 + g], oracle.dense_attention(q[g], K, V), "bf16")


# ------------------------------------------------ full BASELINE sizes
FULL = ["c2_32k", "c3", "c4", "c5"]


@pytest.mark.parametrize("name", FULL)
def test_full_size_sampled_units(name):
    """BASELINE.json sizes in the bench launch configuration; the oracle
    checks a sample of units (first, last and ten seeded random ones)."""
    cfg = synth.CONFIGS[name]
    lay, cache, C = build_cache(cfg)
    y, idx = run_decode(cache, lay, cfg.k)
    check_units(lay, cache, C, cfg.k, sample_units(cfg, n=12), y, idx)
    # properties at every unit: ascending, distinct, in range, exact count
    iv = idx.cpu()
    assert (iv[..., 1:] > iv[..., :-1]).all() and (iv >= 0).all() and (iv < cfg.S).all()
    del cache, lay
    torch.cuda.empty_cache()


@pytest.mark.parametrize("S,k", [(300000, 18750), (40000, 2500)])
def test_long_sequence_large_cluster(S, k):
    """S beyond 8 x 32K keys: a non-portable cluster of ceil(S / 32K) CTAs
    per unit (10 at S = 300K, after the occupancy check), and a ragged
    second sequence; every unit against the oracle."""
    cfg = synth.Config("ls", B=2, Hq=4, Hkv=1, d=128, S=S, r=8, k=k, dtype="bf16")
    lay, cache, C = build_cache(cfg, seq_lens=[S, S - 4321])
    assert ds.ds_decode_launches(cache, k) == 1, "expected the single-kernel cluster path"
    y, idx = run_decode(cache, lay, k)
    check_units(lay, cache, C, k, all_units(cfg), y, idx)


EXT = [
    # name, cfg, seq_lens, k: more selected rows per CTA than the 2112-entry list,
    # continued in the dead candidate buffer (one CTA, and 8-CTA clusters)
    ("cta_k2150", synth.Config("x1", B=2, Hq=8, Hkv=1, d=128, S=8000, r=8, k=2150, dtype="bf16"), [8000, 7001], 2150),
    ("cta_k3000", synth.Config("x2", B=2, Hq=8, Hkv=1, d=128, S=8000, r=8, k=3000, dtype="bf16"), [8000, 6500], 3000),
    # (one unit of S=64K: 16 CTAs of 4K tokens; two of S=40000: 9 CTAs of 4.4K)
    ("cluster16_k36000", synth.Config("x3", B=1, Hq=4, Hkv=1, d=128, S=65536, r=8, k=36000, dtype="bf16"), None,
     36000),
    ("cluster9_ragged", synth.Config("x4", B=2, Hq=4, Hkv=1, d=128, S=40000, r=8, k=21000, dtype="fp16"),
     [40000, 33333], 21000),
]


@pytest.mark.parametrize("name,cfg,seq_lens,k", EXT, ids=[e[0] for e in EXT])
def test_extended_row_list(name, cfg, seq_lens, k):
    lay, cache, C = build_cache(cfg, seq_lens=seq_lens)
    assert ds.ds_decode_launches(cache, k) == 1
    y, idx = run_decode(cache, lay, k)
    check_units(lay, cache, C, k, all_units(cfg), y, idx)
