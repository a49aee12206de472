"""a6 / f1: Double Sparsity-Offload -- K/V pools in pinned host
memory, the label cache on the device.  ds_prefetch_next_layer selects with a
predicted query and gathers the k rows into a device slot;
ds_decode_attention_prefetched attends with the true query over the slot.
Pins: q_hat = q gives the same index sets and output as
ds_decode_attention; the gathered rows are the pool rows bit for bit; with
q_hat != q the selection is the oracle's argtopk under q_hat and the output
the oracle attention of the true q over those rows."""
import numpy as np
import pytest
import torch

import oracle
import paper_2408_07092_b200 as ds
import synth
from parity import check_output, check_selection, sample_units, unit_host

pytestmark = pytest.mark.gpu

CFG = synth.Config("off", B=4, Hq=16, Hkv=4, d=128, S=6000, r=8, k=375, dtype="bf16")


def host_cache(cfg, seq_lens):
    lay = synth.make_layer(cfg, cfg.seed_base, device="cuda", seq_lens=seq_lens)
    cache = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype],
                                   lay.block_table, num_pages=lay.num_pages, page_size=cfg.page_size,
                                   channel_idx=lay.C_plant, host_kv=True)
    assert not cache.k_pool.is_cuda and cache.k_pool.is_pinned()
    ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
    torch.cuda.synchronize()
    return lay, cache


def test_prefetch_with_true_query_equals_decode():
    lay, cache = host_cache(CFG, [6000, 4321, 100, 1])
    k = CFG.k
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        slot = ds.ds_prefetch_next_layer(cache, lay.q, k, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    y_pf = ds.ds_decode_attention_prefetched(cache, lay.q, slot)
    idx = torch.empty((CFG.B, CFG.Hkv, k), dtype=torch.int32, device="cuda")
    y = ds.ds_decode_attention(cache, lay.q, k, topk_idx_out=idx)
    torch.cuda.synchronize()
    assert torch.equal(slot.idx, idx)
    assert slot.count.tolist() == [min(k, int(x)) for x in lay.seq_lens.tolist()]
    check_output(y_pf.float().cpu().numpy(), y.float().cpu().numpy(), "bf16")
    # the slot rows are the pool rows of the selected tokens, bit for bit
    for b in range(CFG.B):
        ke = int(slot.count[b])
        for h in range(CFG.Hkv):
            t = slot.idx[b, h, :ke].long()
            assert torch.equal(slot.k_rows[b, h, :ke], lay.K[b, h, t])
            assert torch.equal(slot.v_rows[b, h, :ke], lay.V[b, h, t])


C5 = synth.CONFIGS["c5"]


@pytest.mark.parametrize("cfg,lens", [(CFG, [6000, 5000, 2222, 375]),
                                      # c5's full size: S=128K, a cluster of CTAs per unit (select-only)
                                      (C5, [C5.S, C5.S - 1, 77777, 40000])], ids=["S6000", "c5_full"])
def test_prefetch_with_predicted_query_matches_oracle(cfg, lens):
    lay, cache = host_cache(cfg, lens)
    q_hat = synth.predicted_query(lay.q, 0.95, seed=3)
    slot = ds.ds_prefetch_next_layer(cache, q_hat, cfg.k)
    y = ds.ds_decode_attention_prefetched(cache, lay.q, slot)
    torch.cuda.synchronize()
    C = lay.C_plant.numpy()
    G = cfg.G
    jac = []
    for b, h in sample_units(cfg, n=12):
        q, K, V = unit_host(lay, b, h)
        qh = q_hat[b, h * G:(h + 1) * G].float().cpu().numpy()
        L = oracle.label_gather(K, C[h])
        shat = oracle.approx_scores(oracle.query_label(qh, C[h]), L)
        ref_idx, tau = oracle.argtopk(shat, cfg.k)
        ke = min(cfg.k, K.shape[0])
        sel = slot.idx[b, h].cpu().numpy()
        check_selection(sel, ref_idx, shat, tau, ke)
        for g in range(G):
            check_output(y[b, h * G + g].float().cpu().numpy(), oracle.attend(q[g], K, V, sel[:ke]), "bf16")
        _, true_idx, _, _ = oracle.ds_decode_unit(q, K, V, L, C[h], cfg.k)
        sa, st = set(sel[:ke].tolist()), set(true_idx.tolist())
        jac.append(len(sa & st) / len(sa | st))
    assert np.mean(jac) > 0.2  # the predicted query selects overlapping tokens (diagnostic floor)
