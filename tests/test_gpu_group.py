"""f4: GQA group-reduction readings on the GPU vs the oracle (-m gpu).
DS_GROUP_MAX (one set per KV head, scored by the max of the per-head
scores) and DS_GROUP_PER_HEAD (one set per query head), readings R17; the
default DS_GROUP_SUM (R3) is covered by every other parity test.  Selection
per R13 (exact, tau band), output per R14 against the oracle attention on
the GPU's own index sets."""
import numpy as np
import pytest
import torch

import oracle
import paper_2408_07092_b200 as ds
import synth
from parity import check_units_group, unit_host

pytestmark = pytest.mark.gpu


def build(cfg, group, label="native", seq_lens=None, structure="iid"):
    lay = synth.make_layer(cfg, cfg.seed_base, device="cuda", seq_lens=seq_lens, structure=structure)
    cache = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype],
                                   lay.block_table, num_pages=lay.num_pages, page_size=cfg.page_size,
                                   channel_idx=lay.C_plant, label_format=label, group_reduce=group)
    ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
    return lay, cache


def check(lay, cache, group, k, y, idx, units):
    check_units_group(lay, cache, group, k, y, idx, units)


CASES = [
    ("gqa4_bf16", synth.Config("g4", B=16, Hq=32, Hkv=8, d=128, S=2048, r=8, k=128, dtype="bf16"), "native", None),
    ("cl_gqa8_fp16", synth.Config("g8", B=2, Hq=16, Hkv=2, d=128, S=10000, r=8, k=300, dtype="fp16"), "native",
     [10000, 2222]),
    ("gqa2_int4_d64", synth.Config("g2", B=4, Hq=8, Hkv=4, d=64, S=3000, r=4, k=200, dtype="bf16"), "int4",
     [3000, 1, 0, 1500]),
    ("gqa4_nolabel", synth.Config("gn", B=4, Hq=16, Hkv=4, d=128, S=2500, r=8, k=150, dtype="bf16"), "none", None),
]


@pytest.mark.parametrize("group", ["max", "per_head"])
@pytest.mark.parametrize("name,cfg,label,lens", CASES, ids=[c[0] for c in CASES])
def test_group_reduce_parity(name, cfg, label, lens, group):
    lay, cache = build(cfg, group, label, lens)
    nsel = cfg.Hq if group == "per_head" else cfg.Hkv
    idx = torch.empty((cfg.B, nsel, cfg.k), dtype=torch.int32, device="cuda")
    y = ds.ds_decode_attention(cache, lay.q, cfg.k, topk_idx_out=idx)
    torch.cuda.synchronize()
    units = [(b, h) for b in range(cfg.B) for h in range(cfg.Hkv)]
    if len(units) > 12:
        rng = np.random.default_rng(0)
        units = sorted({units[0], units[-1]} | {units[i] for i in rng.choice(len(units), 10, replace=False)})
    check(lay, cache, group, cfg.k, y, idx, units)


def test_group_max_approx_scores_match_oracle():
    cfg = synth.Config("gs", B=2, Hq=8, Hkv=2, d=128, S=1000, r=8, k=9, dtype="bf16")
    lay, cache = build(cfg, "max")
    s = ds.ds_approx_scores(cache, lay.q).cpu().numpy()
    C = lay.C_plant.numpy()
    for b in range(2):
        for h in range(2):
            q, K, V = unit_host(lay, b, h)
            _, _, shat = oracle.ds_decode_unit_group(q, K, V, oracle.label_gather(K, C[h]), C[h], 9, group="max")
            assert np.array_equal(s[b, h, :K.shape[0]], shat)   # float equality (+0 == -0)


def test_group_variants_unsupported_paths():
    cfg = synth.Config("gu", B=1, Hq=4, Hkv=1, d=128, S=256, r=8, k=8, dtype="bf16")
    lay, cache = build(cfg, "per_head")
    with pytest.raises(ds.DsError):
        ds.ds_prefetch_next_layer(cache, lay.q, 8)
    with pytest.raises(ds.DsError):
        ds.ds_approx_scores(cache, lay.q)
    c32 = synth.Config("gu32", B=1, Hq=4, Hkv=1, d=128, S=256, r=8, k=8, dtype="fp32")
    lay32 = synth.make_layer(c32, 1, device="cuda")
    cache32 = ds.LayerCache.allocate(1, 4, 1, 128, 256, 8, torch.float32, lay32.block_table,
                                     num_pages=lay32.num_pages, channel_idx=lay32.C_plant, group_reduce="max")
    with pytest.raises(ds.DsError):
        ds.ds_decode_attention(cache32, lay32.q, 8)
