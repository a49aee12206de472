"""GPU parity of the single-kernel decode path (decode.cu): shapes with
enough (b, KV head) units that ds_decode_attention runs Algorithm 1 as one
kernel with one CTA per unit (ds_decode_launches == 1).  Same oracle and
tolerances as test_gpu_parity.py (R13/R14); the cases target the
kernel's branches: k >= S (everything selected), a boundary digit taken
whole, the candidate ranking, the digit-3 / token-order tie path, a
candidate list overflow, several attention rounds, G in {1, 2, 4, 8},
d in {64, 128}, non-power-of-two pages, empty and length-1 sequences."""
import numpy as np
import pytest
import torch

import oracle
import paper_2408_07092_b200 as ds
import synth
from parity import build_cache, check_output, check_units, unit_host

pytestmark = pytest.mark.gpu


def run(cache, lay, k, with_idx=True):
    cfg = lay.cfg
    assert ds.ds_decode_launches(cache, k) == 1, "expected the single-kernel path"
    idx = torch.empty((cfg.B, cfg.Hkv, k), dtype=torch.int32, device="cuda") if with_idx else None
    y = ds.ds_decode_attention(cache, lay.q, k, topk_idx_out=idx)
    torch.cuda.synchronize()
    return y, idx


def ragged(B, S, seed):
    g = np.random.default_rng(seed)
    lens = g.integers(1, S + 1, size=B)
    lens[0], lens[1], lens[2], lens[3] = S, 0, 1, max(1, S // 40)
    return [int(x) for x in lens]


def sample_units(cfg, n=12, seed=0):
    g = np.random.default_rng(seed)
    units = {(0, 0), (1, 0), (2, cfg.Hkv - 1), (3, 1), (cfg.B - 1, cfg.Hkv - 1)}
    n = min(n, cfg.B * cfg.Hkv)
    while len(units) < n:
        units.add((int(g.integers(cfg.B)), int(g.integers(cfg.Hkv))))
    return sorted(units)


CASES = [
    # name, cfg, k, structure
    ("gqa4_bf16", synth.Config("f4", B=16, Hq=32, Hkv=8, d=128, S=2048, r=8, k=128, dtype="bf16"), 128, "iid"),
    ("mha_fp16_d64_r4_page7",
     synth.Config("f1", B=16, Hq=8, Hkv=8, d=64, S=1500, r=4, k=90, dtype="fp16", page_size=7), 90, "iid"),
    ("gqa8_bf16_clustered", synth.Config("f8", B=16, Hq=64, Hkv=8, d=128, S=4096, r=8, k=256, dtype="bf16"), 256,
     "clustered"),
    ("gqa2_fp16_rounds", synth.Config("f2", B=16, Hq=16, Hkv=8, d=128, S=8192, r=8, k=4096, dtype="fp16"), 4096,
     "iid"),
    ("k1_bf16", synth.Config("k1", B=16, Hq=32, Hkv=8, d=128, S=1024, r=8, k=1, dtype="bf16"), 1, "iid"),
    ("kS_bf16", synth.Config("kS", B=16, Hq=32, Hkv=8, d=128, S=700, r=8, k=700, dtype="bf16"), 700, "iid"),
    # few units -> a cluster of CTAs per unit (DSMEM histograms, cluster merge)
    ("cl4_mha_fp16", synth.Config("c4u", B=4, Hq=32, Hkv=8, d=128, S=9000, r=8, k=375, dtype="fp16"), 375, "iid"),
    ("cl8_gqa_bf16_d64", synth.Config("c8u", B=4, Hq=8, Hkv=2, d=64, S=9000, r=4, k=500, dtype="bf16",
                                      page_size=7), 500, "clustered"),
]


@pytest.mark.parametrize("name,cfg,k,structure", CASES, ids=[c[0] for c in CASES])
def test_fused_parity(name, cfg, k, structure):
    lay, cache, C = build_cache(cfg, structure=structure, seq_lens=ragged(cfg.B, cfg.S, hash(name) % 1000))
    y, idx = run(cache, lay, k)
    check_units(lay, cache, C, k, sample_units(cfg), y, idx)
    iv = idx.cpu()
    lens = lay.seq_lens.cpu()
    for b in range(cfg.B):  # every unit: ascending, in range, exactly k_eff entries
        ke = min(k, int(lens[b]))
        v = iv[b, :, :ke]
        assert (v[..., 1:] > v[..., :-1]).all() and (v >= 0).all() and (v < int(lens[b])).all()
        assert (iv[b, :, ke:] == -1).all()
    assert (y[1] == 0).all(), "empty sequence -> y = 0"


def test_fused_without_index_output_matches():
    cfg = synth.Config("ni", B=16, Hq=32, Hkv=8, d=128, S=3000, r=8, k=200, dtype="bf16")
    lay, cache, C = build_cache(cfg, seq_lens=ragged(cfg.B, cfg.S, 5))
    y1, _ = run(cache, lay, 200, with_idx=False)
    y2, idx = run(cache, lay, 200)
    check_units(lay, cache, C, 200, sample_units(cfg, 6), y1, idx)
    check_output(y1.float().cpu().numpy(), y2.float().cpu().numpy(), "bf16")


def test_fused_all_tied_takes_lowest_indices():
    """q = 0: every score ties at 0 -> digit-3 and token-order tie path;
    the selection must be tokens 0..k-1 and y the mean of their V rows."""
    cfg = synth.Config("ft", B=16, Hq=32, Hkv=8, d=128, S=6000, r=8, k=1500, dtype="bf16")
    lay, cache, C = build_cache(cfg)
    lay.q.zero_()
    y, idx = run(cache, lay, 1500)
    assert (idx.cpu() == torch.arange(1500, dtype=torch.int32)).all()
    for b, h in [(0, 0), (15, 7), (7, 3)]:
        ref = lay.V[b, h, :1500].float().mean(0).cpu().numpy()
        for g in range(4):
            check_output(y[b, h * 4 + g].float().cpu().numpy(), ref, "bf16")


TIE_CFGS = {
    "one_cta": (synth.Config("fd", B=16, Hq=32, Hkv=8, d=128, S=5000, r=8, k=600, dtype="bf16"), 600),
    # 8 units -> clusters of 8 CTAs: the cluster-local tail (the D1 bin fits
    # one list) with members / digit-3 ties, and the exchange tail ("narrow")
    "cluster9k": (synth.Config("fc", B=2, Hq=16, Hkv=4, d=128, S=9000, r=8, k=1080, dtype="bf16"), 1080),
    "cluster12k": (synth.Config("fe", B=2, Hq=16, Hkv=4, d=128, S=12000, r=8, k=1440, dtype="bf16"), 1440),
}


@pytest.mark.parametrize("geom", list(TIE_CFGS))
@pytest.mark.parametrize("span", ["duplicates", "narrow"])
def test_fused_duplicate_and_narrow_scores(span, geom):
    """Label values from a tiny set: many exactly equal scores at the
    boundary ("duplicates": members + ties) and, for "narrow", all scores in
    one 12-bit digit so the candidate list overflows (key-scan path)."""
    cfg, k = TIE_CFGS[geom]
    lay, cache, C = build_cache(cfg)
    g = torch.Generator(device="cuda").manual_seed(3)
    if span == "duplicates":
        vals = torch.randint(-2, 3, (cfg.B, cfg.Hkv, cfg.S, 8), generator=g, device="cuda").float()
    else:
        vals = 1.0 + torch.randint(0, 4, (cfg.B, cfg.Hkv, cfg.S, 8), generator=g, device="cuda").float() / 128
    Kd = lay.K.clone()
    for h in range(cfg.Hkv):
        Kd[:, h][..., C[h].long().cuda()] = vals[:, h].to(torch.bfloat16)
    lay.K.copy_(Kd)
    ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
    lay.q.zero_()
    for h in range(cfg.Hkv):  # q_lab = 1 on every channel (head 0 of the group carries it)
        lay.q[:, h * cfg.G, C[h].long().cuda()] = 1.0
    y, idx = run(cache, lay, k)
    units = [(0, 0), (9, 5), (15, 7)] if cfg.B == 16 else [(0, 0), (1, 3), (1, 1)]
    for b, h in units:
        q, K, V = unit_host(lay, b, h)
        L = oracle.label_gather(K, C[h].numpy())
        yr, idx_ref, _, _ = oracle.ds_decode_unit(q, K, V, L, C[h].numpy(), k)
        assert idx[b, h].cpu().numpy().tolist() == idx_ref.tolist()
        for gq in range(cfg.G):
            check_output(y[b, h * cfg.G + gq].float().cpu().numpy(), yr[gq], "bf16")


def test_fused_full_density_equals_dense():
    """r = d, C = identity, k = S through the single-kernel path."""
    cfg = synth.Config("fdd", B=16, Hq=32, Hkv=8, d=64, S=600, r=64, k=600, dtype="bf16")
    C = torch.arange(64, dtype=torch.int32)[None].repeat(8, 1)
    lay, cache, _ = build_cache(cfg, C=C, seq_lens=[600, 333] + [600 - 7 * i for i in range(14)])
    y, idx = run(cache, lay, 600)
    yd = ds.ds_dense_decode_attention(cache, lay.q)
    torch.cuda.synchronize()
    assert idx[1, 0, :333].tolist() == list(range(333)) and (idx[1, 0, 333:] == -1).all()
    for b, h in [(0, 0), (1, 7), (9, 2)]:
        q, K, V = unit_host(lay, b, h)
        for g in range(4):
            ref = oracle.dense_attention(q[g], K, V)
            check_output(y[b, h * 4 + g].float().cpu().numpy(), ref, "bf16")
            check_output(yd[b, h * 4 + g].float().cpu().numpy(), ref, "bf16")


def test_path_choice():
    """16-bit caches take the single kernel (one CTA per unit for many units,
    a cluster of CTAs per unit for few units or long sequences); fp32 takes
    the two-kernel path."""
    small = synth.Config("s", B=2, Hq=8, Hkv=2, d=128, S=1024, r=8, k=64, dtype="bf16")
    lay, cache, _ = build_cache(small)
    assert ds.ds_decode_launches(cache, 64) == 1
    f32 = synth.Config("f", B=16, Hq=32, Hkv=8, d=128, S=256, r=16, k=16, dtype="fp32")
    lay, cache, _ = build_cache(f32)
    assert ds.ds_decode_launches(cache, 16) == 2
