"""f2: the 4-bit label cache (DESIGN reading R16) on the GPU vs the
oracle (-m gpu).

- a0: the packed codes and scales ds_append_kv writes are the oracle's
  quantize_label_4bit + pack_int4 of the channel gather of K, byte for byte
  (every dtype, even / odd / > 32 channels); one-by-one appends == bulk.
- a1+a2: ds_approx_scores over the 4-bit label is bit-identical to the
  oracle's (fma chain of q_label * codes) * scale.
- Algorithm 1 end to end with the 4-bit label: selection bit-exact (R13),
  output within R14, through the single-kernel path (one CTA per unit and
  clusters, vector and scalar label reads), the fp32 two-kernel path, the
  offload prefetch, and BASELINE sizes with sampled units."""
import numpy as np
import pytest
import torch

import oracle
import paper_2408_07092_b200 as ds
import synth
from parity import build_cache, check_units, unit_host

pytestmark = pytest.mark.gpu


def all_units(cfg):
    return [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]


def oracle_label_q4(lay, C, b, h, dtype):
    _, K, _ = unit_host(lay, b, h)
    codes, scale = oracle.quantize_label_4bit(oracle.label_gather(K, C[h].numpy()), dtype)
    return codes, scale


APPEND = [
    synth.Config("q4a", B=2, Hq=8, Hkv=2, d=128, S=300, r=8, k=10, dtype="bf16"),
    synth.Config("q4b", B=2, Hq=4, Hkv=2, d=64, S=257, r=3, k=10, dtype="fp16", page_size=7),
    synth.Config("q4c", B=1, Hq=2, Hkv=1, d=128, S=100, r=16, k=10, dtype="fp32"),
    synth.Config("q4d", B=1, Hq=2, Hkv=1, d=128, S=90, r=41, k=10, dtype="bf16"),
]


@pytest.mark.parametrize("cfg", APPEND, ids=[c.name for c in APPEND])
def test_append_codes_and_scales_bit_exact(cfg):
    lay, cache, C = build_cache(cfg, seq_lens=[cfg.S, cfg.S // 3][:cfg.B], label_format="int4")
    assert cache.label.dtype == torch.uint8 and cache.label.shape[-1] == (cfg.r + 1) // 2
    lab, scl = cache.label.cpu().numpy(), cache.label_scale.float().cpu().numpy()
    for b in range(cfg.B):
        S = int(lay.seq_lens[b])
        for h in range(cfg.Hkv):
            codes, scale = oracle_label_q4(lay, C, b, h, cfg.dtype)
            assert np.array_equal(lab[b, h, :S], oracle.pack_int4(codes))
            assert np.array_equal(scl[b, h, :S].view(np.uint32), scale.view(np.uint32))


def test_append_one_by_one_equals_bulk_q4():
    cfg = synth.Config("inc4", B=2, Hq=4, Hkv=2, d=64, S=40, r=5, k=8, dtype="fp16", page_size=8)
    lay, cache, C = build_cache(cfg, label_format="int4")
    c2 = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, torch.float16, lay.block_table,
                                num_pages=lay.num_pages, page_size=8, channel_idx=C, label_format="int4")
    c2.label.zero_()
    c2.label_scale.zero_()
    for t in range(cfg.S):
        kn = lay.K[:, :, t:t + 1].transpose(1, 2).contiguous()
        vn = lay.V[:, :, t:t + 1].transpose(1, 2).contiguous()
        ds.ds_append_kv(c2, kn, vn, torch.full((cfg.B,), t, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(c2.label, cache.label) and torch.equal(c2.label_scale, cache.label_scale)


def test_append_zero_and_tiny_rows():
    """A zero row gets scale 1 and codes 0; a row whose max/7 underflows the
    fp16 scale also gets scale 1 (R16) -- bit-exact with the oracle."""
    cfg = synth.Config("z4", B=1, Hq=1, Hkv=1, d=128, S=64, r=8, k=4, dtype="fp16")
    lay = synth.make_layer(cfg, 1, device="cuda")
    C = lay.C_plant
    K = lay.K.clone()
    cols = C[0].long().cuda()
    K[0, 0, :8][:, cols] = 0.0
    K[0, 0, 8:16][:, cols] = torch.tensor(3e-8, dtype=torch.float16, device="cuda")  # fp16 subnormal
    lay.K.copy_(K)
    cache = ds.LayerCache.allocate(1, 1, 1, 128, 64, 8, torch.float16, lay.block_table, num_pages=lay.num_pages,
                                   channel_idx=C, label_format="int4")
    ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
    torch.cuda.synchronize()
    codes, scale = oracle_label_q4(lay, C, 0, 0, "fp16")
    assert (scale[:16] == 1).all() and (codes[:16] == 0).all()
    assert np.array_equal(cache.label[0, 0].cpu().numpy(), oracle.pack_int4(codes))
    assert np.array_equal(cache.label_scale[0, 0].float().cpu().numpy(), scale)


@pytest.mark.parametrize("cfg", [
    synth.Config("s4", B=2, Hq=8, Hkv=2, d=128, S=2000, r=8, k=9, dtype="bf16"),
    synth.Config("s4o", B=1, Hq=2, Hkv=1, d=128, S=999, r=3, k=9, dtype="fp16"),
    synth.CONFIGS["c1"],
], ids=["bf16_r8", "fp16_r3", "c1_fp32"])
def test_approx_scores_q4_bit_exact(cfg):
    lay, cache, C = build_cache(cfg, label_format="int4")
    s = ds.ds_approx_scores(cache, lay.q).cpu().numpy()
    for b in range(cfg.B):
        for h in range(cfg.Hkv):
            q, K, _ = unit_host(lay, b, h)
            codes, scale = oracle_label_q4(lay, C, b, h, cfg.dtype)
            ref = oracle.approx_scores_q4(oracle.query_label(q, C[h].numpy()), codes, scale)
            assert np.array_equal(s[b, h, :K.shape[0]].view(np.uint32), ref.view(np.uint32))


def ragged(B, S, seed):
    g = np.random.default_rng(seed)
    lens = g.integers(1, S + 1, size=B)
    lens[0] = S
    if B > 3:
        lens[1], lens[2], lens[3] = 0, 1, max(1, S // 40)
    return [int(x) for x in lens]


DECODE = [
    # single-kernel path, one CTA per unit (vector label reads: Smax % 4 == 0)
    ("gqa4_bf16", synth.Config("d4a", B=16, Hq=32, Hkv=8, d=128, S=2048, r=8, k=128, dtype="bf16"), "iid"),
    # Smax % 4 != 0: scalar label reads
    ("gqa8_bf16_odd_smax", synth.Config("d4b", B=16, Hq=64, Hkv=8, d=128, S=4097, r=8, k=256, dtype="bf16"),
     "clustered"),
    ("mha_fp16_d64_r4", synth.Config("d4c", B=16, Hq=8, Hkv=8, d=64, S=1500, r=4, k=90, dtype="fp16",
                                     page_size=7), "iid"),
    ("kS_bf16", synth.Config("d4d", B=16, Hq=32, Hkv=8, d=128, S=700, r=8, k=700, dtype="bf16"), "iid"),
    # clusters of CTAs per unit
    ("cl_mha_fp16", synth.Config("d4e", B=4, Hq=32, Hkv=8, d=128, S=9000, r=8, k=375, dtype="fp16"), "iid"),
    ("cl_gqa_bf16_d64", synth.Config("d4f", B=4, Hq=8, Hkv=2, d=64, S=9000, r=4, k=500, dtype="bf16",
                                     page_size=7), "clustered"),
    # fp32: the two-kernel path
    ("c1_fp32", synth.CONFIGS["c1"], "iid"),
]


@pytest.mark.parametrize("name,cfg,structure", DECODE, ids=[d[0] for d in DECODE])
def test_decode_parity_q4(name, cfg, structure):
    lay, cache, C = build_cache(cfg, structure=structure, seq_lens=ragged(cfg.B, cfg.S, len(name)),
                                label_format="int4")
    idx = torch.empty((cfg.B, cfg.Hkv, cfg.k), dtype=torch.int32, device="cuda")
    y = ds.ds_decode_attention(cache, lay.q, cfg.k, topk_idx_out=idx)
    torch.cuda.synchronize()
    units = all_units(cfg)
    if len(units) > 16:
        rng = np.random.default_rng(1)
        units = sorted({units[0], units[-1], (1, 0), (2, 0), (3, 0)} |
                       {units[i] for i in rng.choice(len(units), 8, replace=False)})
    check_units(lay, cache, C, cfg.k, units, y, idx)


def test_prefetch_q4_true_query_equals_decode():
    cfg = synth.Config("off4", B=4, Hq=16, Hkv=4, d=128, S=6000, r=8, k=375, dtype="bf16")
    lay = synth.make_layer(cfg, cfg.seed_base, device="cuda", seq_lens=[6000, 4321, 100, 1])
    cache = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, torch.bfloat16, lay.block_table,
                                   num_pages=lay.num_pages, channel_idx=lay.C_plant, host_kv=True,
                                   label_format="int4")
    ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
    slot = ds.ds_prefetch_next_layer(cache, lay.q, cfg.k)
    idx = torch.empty((cfg.B, cfg.Hkv, cfg.k), dtype=torch.int32, device="cuda")
    y = ds.ds_decode_attention(cache, lay.q, cfg.k, topk_idx_out=idx)
    torch.cuda.synchronize()
    assert torch.equal(slot.idx, idx)
    check_units(lay, cache, lay.C_plant, cfg.k, all_units(cfg), y, idx)


@pytest.mark.parametrize("name", ["c2_32k", "c3", "c5"])
def test_full_size_sampled_units_q4(name):
    cfg = synth.CONFIGS[name]
    lay, cache, C = build_cache(cfg, label_format="int4")
    idx = torch.empty((cfg.B, cfg.Hkv, cfg.k), dtype=torch.int32, device="cuda")
    y = ds.ds_decode_attention(cache, lay.q, cfg.k, topk_idx_out=idx)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    units = {(0, 0), (cfg.B - 1, cfg.Hkv - 1)}
    while len(units) < 4:
        units.add((int(rng.integers(cfg.B)), int(rng.integers(cfg.Hkv))))
    check_units(lay, cache, C, cfg.k, sorted(units), y, idx)
    iv = idx.cpu()
    assert (iv[..., 1:] > iv[..., :-1]).all() and (iv >= 0).all() and (iv < cfg.S).all()
    del cache, lay
    torch.cuda.empty_cache()
