"""f4 diagnostic: accuracy grid of the GQA group-reduction readings (R3 sum,
R17 max / per head) over the channel ratio alpha = r/d and the token ratio
beta = k/S (the analogue of the paper's Fig. 1 / Fig. 8 sparsity sweeps,
P:129-131) on synthetic Llama-3-8B-shaped GQA data (seeded N(0,1)
q/K/V with 8 planted outlier channels per KV head, the bench recipe).

Per cell and reading: the relative L2 error of the Double Sparsity output vs
dense attention (both from libds), and the recall of each query head's exact
top-k tokens (by q_g . K) inside the set that head attends.  Not a parity
gate: how well DS approximates dense attention is data dependent.

usage: python scripts/gqa_grid.py [--out profiles/r1_gqa_grid.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_07092_b200 as ds  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_gqa_grid.json"))
    a = ap.parse_args()
    base = synth.Config("grid", B=4, Hq=32, Hkv=8, d=128, S=4096, r=8, k=256, dtype="bf16")
    lay = synth.make_layer(base, base.seed_base + 5, device="cuda")
    Qc, Kc = synth.make_calibration(base, n=512, seed=base.seed_base + 5, device="cuda")
    G = base.G
    q = lay.q                                  # [B][Hq][d]
    Kf = lay.K.float()                          # [B][Hkv][S][d]
    # exact per-head logits q_g . K (the reference ranking of each head)
    qh = q.float().view(base.B, base.Hkv, G, base.d)
    logits = torch.einsum("bhgd,bhsd->bhgs", qh, Kf)
    rows = []
    dense = None
    for alpha in (1, 2, 4, 8, 16, 32):
        r = base.d // alpha
        C = ds.ds_calibrate_channels(Qc, Kc, base.Hkv, r)
        for beta in (2, 4, 8, 16, 32):
            k = base.S // beta
            cell = {"alpha": f"1/{alpha}", "beta": f"1/{beta}", "r": r, "k": k}
            for group in ("sum", "max", "per_head"):
                if group == "max" and G * r > 256:
                    cell[group] = None
                    continue
                cache = ds.LayerCache.allocate(base.B, base.Hq, base.Hkv, base.d, base.S, r, torch.bfloat16,
                                               lay.block_table, num_pages=lay.num_pages, channel_idx=C,
                                               group_reduce=group)
                ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
                if dense is None:
                    dense = ds.ds_dense_decode_attention(cache, q).float()
                nsel = base.Hq if group == "per_head" else base.Hkv
                idx = torch.empty((base.B, nsel, k), dtype=torch.int32, device="cuda")
                y = ds.ds_decode_attention(cache, q, k, topk_idx_out=idx).float()
                err = ((y - dense).norm(dim=-1) / dense.norm(dim=-1)).mean().item()
                # recall of each head's exact top-k inside the set it attends
                exact = logits.topk(k, dim=-1).indices                         # [B][Hkv][G][k]
                sel = idx.view(base.B, base.Hkv, G, k) if group == "per_head" else \
                    idx[:, :, None, :].expand(base.B, base.Hkv, G, k)
                hit = torch.zeros(base.B, base.Hkv, G, base.S, dtype=torch.bool, device="cuda")
                hit.scatter_(-1, sel.long(), True)
                recall = hit.gather(-1, exact).float().mean().item()
                cell[group] = {"rel_l2_err_vs_dense": round(err, 5), "recall_exact_topk": round(recall, 4)}
                del cache
            rows.append(cell)
            print(json.dumps(cell))
    doc = {"what": "GQA group-reduction readings: DS output error vs dense and per-head top-k recall, synthetic "
                   "Llama-3-8B-shaped data (B=4, Hq=32, Hkv=8, d=128, S=4096, bf16, 8 planted channels per KV head); "
                   "diagnostic only", "rows": rows}
    if a.out:
        json.dump(doc, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
