"""N>1 host logic on CPU with world-size-2 gloo process groups (no GPU):
the KV-head sharding covers every unit exactly once, the all-gather of head
outputs reassembles the single-process result bit-for-bit (the per-unit
computation is the oracle here, standing in for the kernel), and bench.py's
max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2408_07092_b200 import shard

CFG = synth.Config("mg", B=2, Hq=8, Hkv=4, d=64, S=96, r=4, k=12, dtype="bf16")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_outputs(lay, h_range):
    """y[B][heads of h_range][d] with the oracle (per unit), fp32."""
    G = CFG.G
    h0, h1 = h_range
    y = np.zeros((CFG.B, (h1 - h0) * G, CFG.d), np.float32)
    C = lay.C_plant.numpy()
    for b in range(CFG.B):
        S = int(lay.seq_lens[b])
        for h in range(h0, h1):
            q = lay.q[b, h * G:(h + 1) * G].float().numpy()
            K = lay.K[b, h, :S].float().numpy()
            V = lay.V[b, h, :S].float().numpy()
            L = oracle.label_gather(K, C[h])
            yu, _, _, _ = oracle.ds_decode_unit(q, K, V, L, C[h], CFG.k)
            y[b, (h - h0) * G:(h - h0 + 1) * G] = yu
    return y


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        lay = synth.make_layer(CFG, 11, device="cpu", seq_lens=[96, 70])
        h0, h1 = shard.kv_head_slice(CFG.Hkv, world, rank)
        y_local = torch.from_numpy(_oracle_outputs(lay, (h0, h1)))
        gathered = shard.allgather_heads(dist, y_local)
        y_full = shard.heads_from_gathered(gathered)
        # bench.py's timing reduction: max over ranks
        import bench
        d = bench.Dist()
        d.pg = dist
        mx = d.max(float(rank + 1) * 1.5)
        q.put((rank, y_full.numpy(), mx, (h0, h1)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the test
        q.put((rank, repr(e), None, None))


def test_kv_head_slices_partition_units():
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            h0, h1 = shard.kv_head_slice(8, world, r)
            seen += list(range(h0, h1))
            g0, g1 = shard.q_head_slice(32, 8, world, r)
            assert (g0, g1) == (h0 * 4, h1 * 4)
        assert seen == list(range(8))
    with pytest.raises(ValueError):
        shard.kv_head_slice(8, 3, 0)


def test_heads_from_gathered_layout():
    parts = [torch.arange(2 * 3 * 5).reshape(2, 3, 5) + 100 * r for r in range(2)]
    full = shard.heads_from_gathered(torch.stack(parts))
    assert torch.equal(full[:, :3], parts[0]) and torch.equal(full[:, 3:], parts[1])


def test_allgather_world2_gloo_reassembles_single_process_output():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, y, mx, hs in res:
        assert not isinstance(y, str), f"rank {rank} failed: {y}"
        assert mx == 3.0
    lay = synth.make_layer(CFG, 11, device="cpu", seq_lens=[96, 70])
    ref = _oracle_outputs(lay, (0, CFG.Hkv))
    for rank, y, _, _ in res:
        assert np.array_equal(y, ref), f"rank {rank}: gathered output differs"


def _bench_step_worker(rank, world, port, q):
    """bench.py's N>1 path on CPU: shard_plan's KV-head slice, make_step's
    per-layer call + all-gather (the oracle standing in for the kernel)."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        cfg, h0 = bench.shard_plan(CFG, world, rank, "allgather")
        layers = []
        for l in range(2):
            lay = synth.make_layer(CFG, 11 + l, device="cpu", seq_lens=[96, 70])
            layers.append(dict(lay=lay, out=torch.empty((CFG.B, cfg.Hq, CFG.d))))

        def call_layer(ly):
            ly["out"].copy_(torch.from_numpy(_oracle_outputs(ly["lay"], (h0, h0 + cfg.Hkv))))
        gathered = [torch.empty((world,) + tuple(ly["out"].shape)) for ly in layers]
        bench.make_step(layers, call_layer, dist, gathered)()
        q.put((rank, [shard.heads_from_gathered(g).numpy() for g in gathered], (cfg.Hkv, cfg.Hq, h0)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e), None))


def test_bench_step_world2_gloo_allgather_mode():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bench_step_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    refs = [_oracle_outputs(synth.make_layer(CFG, 11 + l, device="cpu", seq_lens=[96, 70]), (0, CFG.Hkv))
            for l in range(2)]
    for rank, ys, shp in res:
        assert not isinstance(ys, str), f"rank {rank} failed: {ys}"
        assert shp == (CFG.Hkv // world, CFG.Hq // world, rank * CFG.Hkv // world)
        for y, ref in zip(ys, refs):
            assert np.array_equal(y, ref), f"rank {rank}: gathered step output differs"


def test_shard_plan_modes():
    import bench
    c3 = synth.CONFIGS["c3"]
    for world in (1, 2, 4, 8):
        for rank in range(world):
            cfg, h0 = bench.shard_plan(c3, world, rank, "allgather")
            assert (cfg.Hkv, cfg.Hq, cfg.B, h0) == (8 // world, 32 // world, 16, rank * 8 // world)
            assert bench.shard_plan(c3, world, rank, "weak") == (c3, 0)
    c4 = synth.CONFIGS["c4"]
    cfg, h0 = bench.shard_plan(c4, 8, 5, "allgather")
    assert (cfg.Hkv, cfg.Hq, cfg.B, h0) == (1, 8, 64, 5)  # c4 at N=8: one KV head and all 64 sequences per rank
