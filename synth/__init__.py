"""Seeded synthetic inputs for the Double Sparsity decode hot path.

This module is shared by the tests, the bench and the oracle harness.  It
holds NO arithmetic of the method (no scores, no selection, no attention):
only the shapes of BASELINE.json's configs and seeded random tensors with
the value distribution and structure DESIGN.md states ("Input recipe"):

* q, K, V ~ N(0, 1); per KV head h a planted set of r outlier channels
  (seeded, ascending) where K is scaled x8 and the group's q heads x2, so
  the label score ranks tokens meaningfully (the paper's premise that a
  few channels dominate A = sum_i S_i).
* structure="clustered": tokens in 4 sink positions, the last 256 and 32
  random 64-token spans get their planted K channels pushed along the sign
  of the group's first q head, so the selection becomes mostly contiguous
  runs.  "iid" (default) is the headline, worst-locality case.
* a paged layout: page size P, each sequence's logical pages mapped to a
  seeded random permutation of the physical pool.

Values are drawn in fp32 (torch Philox on CUDA, mt19937 on CPU) and
rounded once (round-to-nearest-even) to the config dtype.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import torch

DTYPES = {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}


@dataclass(frozen=True)
class Config:
    name: str
    B: int
    Hq: int
    Hkv: int
    d: int
    S: int          # sequence length of every sequence (max_seq_len unless ragged)
    r: int
    k: int
    dtype: str
    page_size: int = 16
    seed_base: int = 0

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    @property
    def units(self) -> int:
        return self.B * self.Hkv

    @property
    def elem(self) -> int:
        return 4 if self.dtype == "fp32" else 2

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


# BASELINE.json configs (c1..c5); c2 is quoted at three sequence lengths.
CONFIGS = {
    "c1": Config("c1", B=1, Hq=1, Hkv=1, d=128, S=1024, r=16, k=64, dtype="fp32", seed_base=1000),
    "c2_4k": Config("c2_4k", B=1, Hq=32, Hkv=32, d=128, S=4096, r=8, k=256, dtype="fp16", seed_base=2000),
    "c2_16k": Config("c2_16k", B=1, Hq=32, Hkv=32, d=128, S=16384, r=8, k=1024, dtype="fp16", seed_base=2000),
    "c2_32k": Config("c2_32k", B=1, Hq=32, Hkv=32, d=128, S=32768, r=8, k=2048, dtype="fp16", seed_base=2000),
    "c3": Config("c3", B=16, Hq=32, Hkv=8, d=128, S=32768, r=8, k=2048, dtype="bf16", seed_base=3000),
    "c4": Config("c4", B=64, Hq=64, Hkv=8, d=128, S=16384, r=8, k=1024, dtype="bf16", seed_base=4000),
    "c5": Config("c5", B=4, Hq=32, Hkv=8, d=128, S=131072, r=8, k=8192, dtype="bf16", seed_base=5000),
}


def plant_channels(cfg: Config, seed: int) -> torch.Tensor:
    """[Hkv][r] int32, ascending distinct planted outlier channels per KV head."""
    g = torch.Generator().manual_seed(seed + 101)
    rows = [torch.sort(torch.randperm(cfg.d, generator=g)[: cfg.r]).values for _ in range(cfg.Hkv)]
    return torch.stack(rows).to(torch.int32)


def block_table(cfg: Config, seed: int, identity: bool = False):
    """(block_table [B][pages_per_seq] int32, num_pages). Pages are a seeded
    random permutation of the physical pool (identity=True: in order)."""
    pps = -(-cfg.S // cfg.page_size)
    n = cfg.B * pps
    if identity:
        perm = torch.arange(n, dtype=torch.int64)
    else:
        perm = torch.randperm(n, generator=torch.Generator().manual_seed(seed + 202))
    return perm.reshape(cfg.B, pps).to(torch.int32), n


@dataclass
class Layer:
    cfg: Config
    q: torch.Tensor         # [B][Hq][d]        cfg dtype
    K: torch.Tensor         # [B][Hkv][S][d]    cfg dtype (dense, logical order)
    V: torch.Tensor         # [B][Hkv][S][d]
    C_plant: torch.Tensor   # [Hkv][r] int32 (CPU)
    seq_lens: torch.Tensor  # [B] int32 (CPU)
    block_table: torch.Tensor  # [B][pages_per_seq] int32 (CPU)
    num_pages: int


def _randn(shape, gen, device):
    return torch.randn(shape, generator=gen, device=device, dtype=torch.float32)


def make_layer(cfg: Config, seed: int | None = None, device="cpu", structure: str = "iid",
               seq_lens=None, identity_pages: bool = False) -> Layer:
    """One layer's decode inputs for cfg.  seq_lens (list/tensor of B ints
    <= cfg.S) makes a ragged batch; tokens past a sequence's length are
    still generated (they are never read)."""
    seed = cfg.seed_base if seed is None else seed
    dev = torch.device(device)
    gen = torch.Generator(device=dev).manual_seed(seed)
    C = plant_channels(cfg, seed)
    q = _randn((cfg.B, cfg.Hq, cfg.d), gen, dev)
    K = _randn((cfg.B, cfg.Hkv, cfg.S, cfg.d), gen, dev)
    V = _randn((cfg.B, cfg.Hkv, cfg.S, cfg.d), gen, dev)
    G = cfg.G
    Cd = C.to(dev, torch.int64)
    for h in range(cfg.Hkv):
        K[:, h, :, Cd[h]] *= 8.0
        q[:, h * G:(h + 1) * G, Cd[h]] *= 2.0
    if structure == "clustered":
        tg = torch.Generator().manual_seed(seed + 303)
        mask = torch.zeros(cfg.S, dtype=torch.bool)
        mask[:4] = True
        mask[max(0, cfg.S - 256):] = True
        span = min(64, cfg.S)
        for s0 in torch.randint(0, max(1, cfg.S - span), (32,), generator=tg).tolist():
            mask[s0:s0 + span] = True
        tok = mask.nonzero().flatten().to(dev)
        for h in range(cfg.Hkv):
            sgn = torch.sign(q[:, h * G, Cd[h]])                      # [B][r]
            blk = K[:, h][:, tok][:, :, Cd[h]]                         # [B][T][r]
            K[:, h, tok[:, None], Cd[h][None, :]] = blk + 24.0 * sgn[:, None, :]
    elif structure != "iid":
        raise ValueError(structure)
    dt = DTYPES[cfg.dtype]
    if seq_lens is None:
        sl = torch.full((cfg.B,), cfg.S, dtype=torch.int32)
    else:
        sl = torch.as_tensor(seq_lens, dtype=torch.int32).reshape(cfg.B)
    bt, npages = block_table(cfg, seed, identity_pages)
    return Layer(cfg, q.to(dt), K.to(dt), V.to(dt), C, sl, bt, npages)


def make_calibration(cfg: Config, n: int = 512, seed: int | None = None, device="cpu"):
    """Calibration Q/K samples [n][Hq][d], [n][Hkv][d] with the same planted
    channels as make_layer(cfg, seed) (paper: "a small validation set")."""
    seed = cfg.seed_base if seed is None else seed
    dev = torch.device(device)
    gen = torch.Generator(device=dev).manual_seed(seed + 404)
    C = plant_channels(cfg, seed).to(dev, torch.int64)
    Qc = _randn((n, cfg.Hq, cfg.d), gen, dev)
    Kc = _randn((n, cfg.Hkv, cfg.d), gen, dev)
    G = cfg.G
    for h in range(cfg.Hkv):
        Kc[:, h, C[h]] *= 8.0
        Qc[:, h * G:(h + 1) * G, C[h]] *= 2.0
    dt = DTYPES[cfg.dtype]
    return Qc.to(dt), Kc.to(dt)


def predicted_query(q: torch.Tensor, cos: float, seed: int) -> torch.Tensor:
    """Synthetic next-layer query prediction q_hat with cos(q_hat, q) ~= cos per
    head (Double Sparsity-Offload; P:204 regime).  Pure input
    construction: q_hat = normalize(q/|q| * cos + e_perp * sin) * |q|."""
    qf = q.float()
    gen = torch.Generator(device=q.device).manual_seed(seed + 505)
    e = torch.randn(qf.shape, generator=gen, device=q.device, dtype=torch.float32)
    n = qf.norm(dim=-1, keepdim=True).clamp_min(1e-30)
    u = qf / n
    e = e - (e * u).sum(-1, keepdim=True) * u
    e = e / e.norm(dim=-1, keepdim=True).clamp_min(1e-30)
    s = math.sqrt(max(0.0, 1.0 - cos * cos))
    return ((u * cos + e * s) * n).to(q.dtype)
