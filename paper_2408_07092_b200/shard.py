"""Multi-GPU plumbing for the decode path.

Units (b, KV head) are independent (Algorithm 1 is per head), so the
path shards with no data-path exchange.  Two layouts:
  * weak:      each rank owns whole problems (its own batch of sequences);
               nothing is exchanged.
  * allgather: the KV heads of one problem are split into contiguous slices,
               rank r owning KV heads [h0, h1) and their G query heads; the
               only exchange is an all-gather of the head outputs (NCCL over
               NVLink on B200; gloo in the CPU tests), gathered as
               [world][B][Hq/world][d] and viewed as [B][Hq][d] by
               `heads_from_gathered`.
Host logic only: no kernels, no arithmetic of the method."""
from __future__ import annotations

import torch


def kv_head_slice(num_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous KV-head slice [h0, h1) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if num_kv_heads % world:
        raise ValueError(f"num_kv_heads ({num_kv_heads}) must be divisible by world ({world})")
    per = num_kv_heads // world
    return rank * per, (rank + 1) * per


def q_head_slice(num_q_heads: int, num_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """The query heads [g0, g1) of the rank's KV heads (G per KV head)."""
    G = num_q_heads // num_kv_heads
    h0, h1 = kv_head_slice(num_kv_heads, world, rank)
    return h0 * G, h1 * G


def allgather_heads(pg, out_local: torch.Tensor, gathered: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather [B][Hq/world][d] head outputs into [world][B][Hq/world][d]."""
    world = pg.get_world_size()
    if gathered is None:
        gathered = torch.empty((world,) + tuple(out_local.shape), dtype=out_local.dtype, device=out_local.device)
    if pg.get_backend() == "gloo":  # (the CPU tests; gloo has no all_gather_into_tensor of this shape)
        pg.all_gather(list(gathered.unbind(0)), out_local.contiguous())
    else:
        pg.all_gather_into_tensor(gathered, out_local.contiguous())
    return gathered


def heads_from_gathered(gathered: torch.Tensor) -> torch.Tensor:
    """[world][B][Hq/world][d] -> [B][Hq][d] (rank r's heads are slice r)."""
    n, B, hp, d = gathered.shape
    return gathered.permute(1, 0, 2, 3).reshape(B, n * hp, d)
