"""Small decode calls for compute-sanitizer (memcheck / synccheck): single CTA
per unit, cluster, 4-bit label, no label, group max, per head, fused append,
prefetch, fp32 two-kernel path and dense."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_07092_b200 as ds  # noqa: E402
import synth  # noqa: E402

cases = [
    (synth.Config("s1", B=4, Hq=16, Hkv=4, d=128, S=3000, r=8, k=200, dtype="bf16"), "native", "sum"),
    (synth.Config("s2", B=1, Hq=8, Hkv=2, d=128, S=12000, r=8, k=700, dtype="fp16"), "native", "sum"),
    (synth.Config("s3", B=2, Hq=8, Hkv=2, d=64, S=2500, r=4, k=100, dtype="bf16", page_size=7), "int4", "max"),
    (synth.Config("s4", B=2, Hq=8, Hkv=2, d=128, S=2500, r=8, k=100, dtype="bf16"), "none", "per_head"),
    (synth.Config("s5", B=1, Hq=4, Hkv=1, d=128, S=1500, r=16, k=64, dtype="fp32"), "native", "sum"),
]
for cfg, label, group in cases:
    lens = [cfg.S - 1] + [max(1, cfg.S // (i + 2)) for i in range(cfg.B - 1)]
    lay = synth.make_layer(cfg, 7, device="cuda", seq_lens=lens)
    c = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype], lay.block_table,
                               num_pages=lay.num_pages, page_size=cfg.page_size, channel_idx=lay.C_plant,
                               label_format=label, group_reduce=group)
    # the label rows past a sequence's length are read in whole 16-B vectors
    # and discarded (ds.h): zero them so initcheck reports only other reads
    c.label.zero_()
    if c.label_scale is not None:
        c.label_scale.zero_()
    ds.prefill(c, lay.K, lay.V, lay.seq_lens)
    nsel = cfg.Hq if group == "per_head" else cfg.Hkv
    idx = torch.empty((cfg.B, nsel, cfg.k), dtype=torch.int32, device="cuda")
    ds.ds_decode_attention(c, lay.q, cfg.k, topk_idx_out=idx)
    pos = torch.tensor(lens, dtype=torch.int32, device="cuda")
    c.seq_lens.copy_(pos + 1)
    kn = lay.K[:, :, :1].transpose(1, 2).contiguous()
    vn = lay.V[:, :, :1].transpose(1, 2).contiguous()
    ds.ds_decode_attention_append(c, kn, vn, pos, lay.q, cfg.k, topk_idx_out=idx)
    ds.ds_dense_decode_attention(c, lay.q)
    if group != "per_head" and cfg.dtype != "fp32":
        ds.ds_approx_scores(c, lay.q)
    torch.cuda.synchronize()
    print("ok", cfg.name, label, group, flush=True)
# offload prefetch
cfg = synth.Config("s6", B=2, Hq=8, Hkv=2, d=128, S=3000, r=8, k=200, dtype="bf16")
lay = synth.make_layer(cfg, 8, device="cuda")
c = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, torch.bfloat16, lay.block_table,
                           num_pages=lay.num_pages, channel_idx=lay.C_plant, host_kv=True)
c.label.zero_()
ds.prefill(c, lay.K, lay.V, lay.seq_lens)
slot = ds.ds_prefetch_next_layer(c, lay.q, cfg.k)
ds.ds_decode_attention_prefetched(c, lay.q, slot)
torch.cuda.synchronize()
print("ok offload", flush=True)
