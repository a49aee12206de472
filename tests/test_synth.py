"""The seeded input generators (shared by tests and bench; no method arithmetic)."""
import torch

import synth


def test_layer_shapes_determinism_and_plant():
    cfg = synth.Config("t", B=2, Hq=8, Hkv=2, d=64, S=100, r=4, k=8, dtype="bf16", page_size=16)
    a = synth.make_layer(cfg, seed=3)
    b = synth.make_layer(cfg, seed=3)
    assert a.q.shape == (2, 8, 64) and a.K.shape == (2, 2, 100, 64) and a.V.dtype == torch.bfloat16
    assert torch.equal(a.K, b.K) and torch.equal(a.q, b.q)
    assert a.block_table.shape == (2, 7) and a.num_pages == 14
    assert sorted(a.block_table.flatten().tolist()) == list(range(14))
    C = a.C_plant
    assert C.shape == (2, 4) and all(C[h].tolist() == sorted(set(C[h].tolist())) for h in range(2))
    # planted K channels have ~8x the magnitude of the others
    k0 = a.K[:, 0].float().abs().mean(dim=(0, 1))
    mask = torch.zeros(64, dtype=torch.bool)
    mask[C[0].long()] = True
    assert k0[mask].mean() > 5 * k0[~mask].mean()


def test_clustered_structure_and_ragged():
    cfg = synth.Config("t", B=2, Hq=2, Hkv=1, d=32, S=2048, r=4, k=128, dtype="fp16")
    a = synth.make_layer(cfg, seed=1, structure="clustered", seq_lens=[2048, 1000])
    assert a.seq_lens.tolist() == [2048, 1000]
    b = synth.make_layer(cfg, seed=1)
    diff = (a.K.float() - b.K.float()).abs().sum(dim=-1)[0, 0]
    changed = (diff > 0).nonzero().flatten()
    assert changed.min() == 0 and changed.max() == 2047 and 256 + 4 <= len(changed) <= 4 + 256 + 32 * 64


def test_predicted_query_cosine():
    q = torch.randn(4, 8, 128)
    qh = synth.predicted_query(q, 0.95, seed=0)
    cos = torch.nn.functional.cosine_similarity(q, qh, dim=-1)
    assert torch.allclose(cos, torch.full_like(cos, 0.95), atol=1e-4)
