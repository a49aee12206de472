"""Library witness for a3 (SURVEY 8(c) pin table): flashinfer's radix top-k
with ties to the smaller index (tie_break=1), run on the approximate scores
s_hat of ds_approx_scores (bit-exact vs the oracle, test_gpu_parity), must pick
the same index SET as decode_kernel's on-chip selection (reading R6: the k
largest, ties to the lower index).  An independent GPU implementation of
argtopk; skipped if flashinfer cannot build its kernel on this box."""
import numpy as np
import pytest
import torch

import paper_2408_07092_b200 as ds
import synth
from parity import build_cache

pytestmark = pytest.mark.gpu

CASES = [
    ("c3_like", synth.Config("w3", B=2, Hq=8, Hkv=2, d=128, S=32768, r=8, k=2048, dtype="bf16"), "iid"),
    ("clustered", synth.Config("wc", B=2, Hq=8, Hkv=2, d=128, S=16384, r=8, k=1024, dtype="bf16"), "clustered"),
    ("ragged_fp16", synth.Config("wr", B=3, Hq=4, Hkv=4, d=128, S=9000, r=8, k=500, dtype="fp16"), "iid"),
]


@pytest.mark.parametrize("name,cfg,structure", CASES, ids=[c[0] for c in CASES])
def test_flashinfer_topk_same_sets(name, cfg, structure):
    try:
        import flashinfer
    except Exception as e:  # pragma: no cover
        pytest.skip(f"flashinfer unavailable: {e}")
    lens = [cfg.S] + [cfg.S - 17 * (i + 1) for i in range(cfg.B - 1)]
    lay, cache, C = build_cache(cfg, structure=structure, seq_lens=lens)
    idx = torch.empty((cfg.B, cfg.Hkv, cfg.k), dtype=torch.int32, device="cuda")
    ds.ds_decode_attention(cache, lay.q, cfg.k, topk_idx_out=idx)
    s = ds.ds_approx_scores(cache, lay.q)  # [B][Hkv][S] fp32, -inf-free for t < seq_len
    torch.cuda.synchronize()
    for b in range(cfg.B):
        n = lens[b]
        rows = s[b, :, :n].contiguous()
        try:
            _, wi = flashinfer.top_k(rows, min(cfg.k, n), tie_break=1)
        except Exception as e:  # JIT build not possible here
            pytest.skip(f"flashinfer.top_k failed to run: {type(e).__name__}: {str(e)[:120]}")
        wi = wi.cpu().numpy()
        ours = idx[b].cpu().numpy()
        for h in range(cfg.Hkv):
            a = np.sort(ours[h][ours[h] >= 0])
            w = np.sort(wi[h].astype(np.int64))
            assert np.array_equal(a, w), f"{name} b={b} h={h}: {len(set(a) ^ set(w))} tokens differ"
