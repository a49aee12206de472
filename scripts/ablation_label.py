"""f3: label-cache ablation on B200 (the analogue of the paper's Table 4,
Appendix B.1: decode latency with vs without the label cache at
batch 4 / 32 and S = 2K..16K).  Shape: Llama-2-7B attention (32 heads MHA,
d=128, fp16), r = 8 (1/16 of the channels), k = S/16 (1/16 of the tokens).

For every shape: ds_decode_attention per layer with the native 16-bit
label, the 4-bit label (f2) and no label (channels read from the
paged K rows), and our dense flash-decode, each a CUDA graph over enough
resident layers that every replay touches > 2x the 126 MB L2.  Prints one
JSON object (also written to profiles/r1_ablation_label.json by default).

usage: python scripts/ablation_label.py [--out PATH] [--quick]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_07092_b200 as ds  # noqa: E402
import synth  # noqa: E402
from paper_2408_07092_b200 import ledger  # noqa: E402

L2 = 126 * 2**20


def time_graph(fn, reps, stream):
    with torch.cuda.stream(stream):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    with torch.cuda.stream(stream):
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_shape(B, S, reps=20):
    cfg = synth.Config(f"t4_b{B}_s{S}", B=B, Hq=32, Hkv=32, d=128, S=S, r=8, k=S // 16, dtype="fp16")
    touched = ledger.layer_bytes_alg(cfg)
    L = max(2, -(-2 * L2 // touched))
    lib = ds.lib()
    P = ctypes.c_void_p
    stream = torch.cuda.Stream()
    sp = P(stream.cuda_stream)
    res = {"B": B, "S": S, "k": cfg.k, "layers": L}
    caches = {f: [] for f in ("native", "int4", "none")}
    qs = []
    for l in range(L):
        lay = synth.make_layer(cfg, cfg.seed_base + 31 * l, device="cuda")
        for f in caches:
            c = ds.LayerCache.allocate(B, 32, 32, 128, S, 8, torch.float16, lay.block_table,
                                       num_pages=lay.num_pages, page_size=cfg.page_size, channel_idx=lay.C_plant,
                                       label_format=f)
            ds.prefill(c, lay.K, lay.V, lay.seq_lens)
            caches[f].append(c)
        qs.append(lay.q.contiguous())
        del lay
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    out = torch.empty_like(qs[0])
    ws = ds.workspace(ds.ds_decode_workspace_size(caches["native"][0], cfg.k))
    idx = {}
    for f, cl in caches.items():
        structs = [c.struct() for c in cl]

        def fn(structs=structs):
            for s, q in zip(structs, qs):
                lib.ds_decode_attention(ctypes.byref(s), P(q.data_ptr()), cfg.k, P(out.data_ptr()), None,
                                        P(ws.data_ptr()), ws.numel(), sp)
        res[f"{f}_us"] = round(time_graph(fn, reps, stream) * 1e3 / L, 3)
        ii = torch.empty((B, 32, cfg.k), dtype=torch.int32, device="cuda")
        ds.ds_decode_attention(cl[0], qs[0], cfg.k, topk_idx_out=ii)
        idx[f] = ii
    structs = [c.struct() for c in caches["native"]]

    def dense():
        for s, q in zip(structs, qs):
            lib.ds_dense_decode_attention(ctypes.byref(s), P(q.data_ptr()), P(out.data_ptr()), None, 0, sp)
    res["dense_us"] = round(time_graph(dense, max(3, reps // 4), stream) * 1e3 / L, 3)
    torch.cuda.synchronize()
    res["same_selection_none_vs_native"] = bool(torch.equal(idx["none"], idx["native"]))
    res["speedup_label_vs_none"] = round(res["none_us"] / res["native_us"], 2)
    res["speedup_int4_vs_none"] = round(res["none_us"] / res["int4_us"], 2)
    res["speedup_native_vs_dense"] = round(res["dense_us"] / res["native_us"], 2)
    res["speedup_int4_vs_dense"] = round(res["dense_us"] / res["int4_us"], 2)
    res["label_bytes_native"] = B * 32 * S * ledger.label_row_bytes(8, 2)
    res["label_bytes_int4"] = B * 32 * S * ledger.label_row_bytes(8, 2, "int4")
    del caches, qs
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_ablation_label.json"))
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    shapes = [(4, 2048), (32, 4096)] if a.quick else [(b, s) for b in (4, 32) for s in (2048, 4096, 8192, 16384)]
    rows = [run_shape(b, s) for b, s in shapes]
    doc = {"what": "label-cache ablation (paper Table 4 analogue), Llama-2-7B attention shape, fp16, r=8, k=S/16, "
                   "us per ds_decode_attention per layer, 1 x B200",
           "paper_table4_ms": {"note": "paper: A100-era GPU, its own kernels; with/without label speedup 1.7-4.2x"},
           "rows": rows}
    print(json.dumps(doc))
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        json.dump(doc, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
