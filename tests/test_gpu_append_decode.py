"""ds_decode_attention_append (one launch per decode step: a0 for one new
token per sequence, then Algorithm 1) against the two calls it fuses,
ds_append_kv + ds_decode_attention, on identical caches (-m gpu): the same
index sets bit for bit, the same outputs within R14 (the attention visits
rows in a run-dependent order), and the same cache contents byte for byte
afterwards.  The new token differs from what the prefill left at its
position, so the fused path must not score the stale label row.

The fused call (the one bench.py times) is also checked against the oracle
directly: Algorithm 1 on the post-append host K/V -- the
prefilled tokens plus the new token at its position -- with exact index
sets (R13) and outputs within R14, for every unit of the small cases and a
seeded sample of units at c3's full size."""
import numpy as np
import pytest
import torch

import paper_2408_07092_b200 as ds
import synth
from parity import check_output, check_units, check_units_group, sample_units

pytestmark = pytest.mark.gpu

CASES = [
    ("gqa4_bf16", synth.Config("ad1", B=16, Hq=32, Hkv=8, d=128, S=2048, r=8, k=128, dtype="bf16"), "native", "sum"),
    ("cluster_mha_fp16", synth.Config("ad2", B=4, Hq=32, Hkv=8, d=128, S=9000, r=8, k=375, dtype="fp16"), "native",
     "sum"),
    ("int4_gqa4", synth.Config("ad3", B=16, Hq=32, Hkv=8, d=128, S=2048, r=8, k=128, dtype="bf16"), "int4", "sum"),
    ("int4_r3_fp16", synth.Config("ad4", B=4, Hq=8, Hkv=4, d=64, S=1500, r=3, k=90, dtype="fp16", page_size=7),
     "int4", "sum"),
    ("nolabel", synth.Config("ad5", B=4, Hq=16, Hkv=4, d=128, S=2500, r=8, k=150, dtype="bf16"), "none", "sum"),
    ("group_max", synth.Config("ad6", B=4, Hq=16, Hkv=4, d=128, S=2500, r=8, k=150, dtype="bf16"), "native", "max"),
    ("per_head_int4", synth.Config("ad7", B=4, Hq=16, Hkv=4, d=128, S=2500, r=8, k=150, dtype="bf16"), "int4",
     "per_head"),
    ("c1_fp32_two_kernel", synth.CONFIGS["c1"], "native", "sum"),
    # the bench's launch configuration: c3 at full size, 16-bit and 4-bit label
    ("c3_full", synth.CONFIGS["c3"], "native", "sum"),
    ("c3_full_int4", synth.CONFIGS["c3"], "int4", "sum"),
]


def cache_of(cfg, lay, label, group):
    c = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype], lay.block_table,
                               num_pages=lay.num_pages, page_size=cfg.page_size, channel_idx=lay.C_plant,
                               label_format=label, group_reduce=group)
    for t in (c.k_pool, c.v_pool, c.label, c.label_scale):  # unmapped pages stay comparable
        if t is not None:
            t.zero_()
    ds.prefill(c, lay.K, lay.V, lay.seq_lens)
    return c


@pytest.mark.parametrize("name,cfg,label,group", CASES, ids=[c[0] for c in CASES])
def test_fused_append_equals_append_then_decode(name, cfg, label, group):
    rng = np.random.default_rng(len(name))
    lens = [int(x) for x in rng.integers(1, cfg.S, size=cfg.B)]
    lens[0] = cfg.S - 1
    lay = synth.make_layer(cfg, cfg.seed_base + 1, device="cuda", seq_lens=lens)
    a, f = cache_of(cfg, lay, label, group), cache_of(cfg, lay, label, group)
    g = torch.Generator(device="cuda").manual_seed(5)
    dt = synth.DTYPES[cfg.dtype]
    k_new = (torch.randn((cfg.B, 1, cfg.Hkv, cfg.d), generator=g, device="cuda") * 3).to(dt)
    v_new = torch.randn((cfg.B, 1, cfg.Hkv, cfg.d), generator=g, device="cuda").to(dt)
    pos = torch.tensor(lens, dtype=torch.int32, device="cuda")
    for c in (a, f):
        c.seq_lens.copy_(pos + 1)
    nsel = cfg.Hq if group == "per_head" else cfg.Hkv
    ia = torch.empty((cfg.B, nsel, cfg.k), dtype=torch.int32, device="cuda")
    if_ = torch.empty_like(ia)
    ds.ds_append_kv(a, k_new, v_new, pos)
    ya = ds.ds_decode_attention(a, lay.q, cfg.k, topk_idx_out=ia)
    yf = ds.ds_decode_attention_append(f, k_new, v_new, pos, lay.q, cfg.k, topk_idx_out=if_)
    torch.cuda.synchronize()
    assert torch.equal(ia, if_)
    check_output(yf.float().cpu().numpy(), ya.float().cpu().numpy(), cfg.dtype)
    assert torch.equal(a.k_pool, f.k_pool) and torch.equal(a.v_pool, f.v_pool)
    if label != "none":
        assert torch.equal(a.label, f.label)
    if label == "int4":
        assert torch.equal(a.label_scale.view(torch.int16), f.label_scale.view(torch.int16))
    del a
    torch.cuda.empty_cache()
    # the new token is really there: its K row in the pool is k_new
    b = 0
    pg = int(lay.block_table[b, lens[b] // cfg.page_size])
    assert torch.equal(f.k_pool[pg, :, lens[b] % cfg.page_size], k_new[b, 0])
    # the fused call against the oracle on the post-append state (Alg. 1):
    # the host view of every sequence gains the new token at its position
    bi = torch.arange(cfg.B, device=lay.K.device)
    pi = pos.long().to(lay.K.device)
    lay.K[bi, :, pi] = k_new[:, 0]
    lay.V[bi, :, pi] = v_new[:, 0]
    lay.seq_lens = (pos + 1).cpu()
    units = sample_units(cfg, n=12, seed=len(name))
    if group == "sum":
        check_units(lay, f, lay.C_plant, cfg.k, units, yf, if_)
    else:
        check_units_group(lay, f, group, cfg.k, yf, if_, units)
