"""f3: the no-label-cache ablation (Appendix B.1, Table 4) on the
GPU (-m gpu).  DS_LABEL_NONE reads the r channels of every token straight
from its paged K row; those are the values the native label copies bit for
bit (a0), so line 2 gives the same scores and line 3 the same index sets
(both compared bit for bit against the native label path); lines 4-5 agree
within R14, and the oracle checks sampled units."""
import numpy as np
import pytest
import torch

import paper_2408_07092_b200 as ds
import synth
from parity import build_cache, check_output, check_units

pytestmark = pytest.mark.gpu

CASES = [
    ("gqa4_bf16", synth.Config("n4a", B=16, Hq=32, Hkv=8, d=128, S=2048, r=8, k=128, dtype="bf16"), None),
    ("cl_mha_fp16", synth.Config("n4b", B=4, Hq=32, Hkv=8, d=128, S=9000, r=8, k=375, dtype="fp16"),
     [9000, 3001, 1, 0]),
    ("d64_r4_page7_long", synth.Config("n4c", B=2, Hq=8, Hkv=2, d=64, S=30000, r=4, k=1000, dtype="bf16",
                                       page_size=7), [30000, 12345]),
    ("c1_fp32", synth.CONFIGS["c1"], None),
]


def decode(cache, lay, k):
    cfg = lay.cfg
    idx = torch.empty((cfg.B, cfg.Hkv, k), dtype=torch.int32, device="cuda")
    y = ds.ds_decode_attention(cache, lay.q, k, topk_idx_out=idx)
    torch.cuda.synchronize()
    return y, idx


@pytest.mark.parametrize("name,cfg,lens", CASES, ids=[c[0] for c in CASES])
def test_no_label_equals_native_label_bitwise(name, cfg, lens):
    lay, native, C = build_cache(cfg, seq_lens=lens)
    none = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype],
                                  lay.block_table, num_pages=lay.num_pages, page_size=cfg.page_size,
                                  channel_idx=C, label_format="none")
    ds.prefill(none, lay.K, lay.V, lay.seq_lens)
    y0, i0 = decode(native, lay, cfg.k)
    y1, i1 = decode(none, lay, cfg.k)
    assert torch.equal(i0, i1)
    # same rows, but the attention warps visit them in a run-dependent order
    # (shared cursor, candidate list slots), so the fp32 sums round differently
    check_output(y1.float().cpu().numpy(), y0.float().cpu().numpy(), cfg.dtype)
    s0 = ds.ds_approx_scores(native, lay.q)
    s1 = ds.ds_approx_scores(none, lay.q)
    for b in range(cfg.B):
        n = int(lay.seq_lens[b])
        assert torch.equal(s0[b, :, :n].view(torch.int32), s1[b, :, :n].view(torch.int32))
    units = [(0, 0), (cfg.B - 1, cfg.Hkv - 1)]
    check_units(lay, none, C, cfg.k, units, y1, i1)
