#!/usr/bin/env python
"""Benchmark of the Double Sparsity decode hot path on B200 (BASELINE.json metric:
"sparse decode-attn us/layer & HBM GB/s vs dense, S=32K, 1/16 sparsity, 1-8 B200").

A step = one decode step of the whole hot path over L resident layer caches:
per layer a0 (the current token's K/V + label row) + a1..a5, as one ds_decode_attention_append.
Workload at N=1: c3 (Llama-3-8B GQA, B=16, H_q=32, H_kv=8, d=128, S=32768,
r=8, k=2048, bf16) -- the config BASELINE.json's metric names (S=32K, 1-8 B200).
N>1 (torchrun, one rank per GPU), default --mode allgather (north_star's
multi-GPU variant): the config's KV heads are split into
contiguous slices, rank r owning KV heads [r H_kv/N, (r+1) H_kv/N) with their
G query heads and all B sequences (c3 at N=8: one KV head per rank; c4 at N=8:
one KV head and all 64 sequences), and each layer's head outputs are
all-gathered over NCCL inside the captured step (the path's only exchange).
Strong scaling: the total work is the config's.  The kernel-only step (same
graph without the collective) is reported beside it.  --mode weak instead runs
a full independent batch per rank (no collective).

value = algorithmic HBM bytes (label S*r*e + gathered K/V 2*k*d*e per unit,
SURVEY 8(d)) of all layers of all ranks / max-over-ranks device time, GB/s.
Inputs are resident in HBM; every step touches L x 192 MiB >> 126 MB L2.

--impl reference: the CPU oracle (oracle/) timed on the host cores on bounded
samples of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2408_07092_b200 import ledger, shard  # noqa: E402

METRIC = "sparse decode-attn µs/layer & HBM GB/s vs dense, S=32K, 1/16 sparsity, 1-8 B200"
KERNELS_PER_APPEND = 1
# kernels per ds_decode_attention call: ds_decode_launches() (1 = fused decode_kernel,
# 2 = cluster score_select_kernel + attention kernel)
KERNELS_PER_DENSE = 1


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--structure", default="iid", choices=["iid", "clustered"])
    ap.add_argument("--pages", default="random", choices=["random", "identity"],
                    help="physical page order of each sequence (random: the headline, worst DRAM locality)")
    ap.add_argument("--no-dense-refs", action="store_true",
                    help="skip the library dense references (torch SDPA, flashinfer trtllm-gen)")
    ap.add_argument("--label", default="native", choices=["native", "int4"],
                    help="label cache storage: K's dtype (north_star's byte model) or 4-bit (P:171, f2)")
    ap.add_argument("--mode", default="allgather", choices=["weak", "allgather"],
                    help="N>1: allgather = KV-head shards + NCCL all-gather of head outputs (strong scaling), "
                         "weak = a full independent batch per rank")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--extra", action="store_true", help="also time c2 S=4K/16K/32K (reported under 'extra')")
    ap.add_argument("--offload-layers", type=int, default=32,
                    help="--offload: layers of pinned host K/V (capped by host memory)")
    ap.add_argument("--offload", action="store_true",
                    help="Double Sparsity-Offload pipeline on c5 (KV in pinned host memory); prints its own line")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_peak_gbs(dev, gib: float = 4.0, reps: int = 5) -> float:
    """Read-only streaming bandwidth on this box (context for the roofline:
    the decode kernel mostly reads, and a copy peak counts writes too):
    best of `reps` reductions of a `gib` GiB bf16 buffer, CUDA events."""
    n = int(gib * 2 ** 30) // 2
    x = torch.ones(n, dtype=torch.bfloat16, device=dev)
    best = float("inf")
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x.sum(dtype=torch.float32)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del x
    torch.cuda.empty_cache()
    return n * 2 / (best / 1e3) / 1e9


# ------------------------------------------------- per-kernel device times
def kernel_trace(fn, reps: int = 3):
    """Every kernel that fn() launches (fn run `reps` times, synchronised),
    with its device duration, as recorded by CUPTI through torch.profiler
    (kineto) -- CUDA-graph replays included.  Not a profiler replay: the
    kernels run once, in situ, at their normal clocks; only the activity
    records are collected.  Returns [{name, ts, dur (us), stream}]."""
    import tempfile
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    path = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(path)
    with open(path) as f:
        ev = json.load(f).get("traceEvents", [])
    os.unlink(path)
    out = [{"name": e["name"], "ts": float(e["ts"]), "dur": float(e["dur"]),
            "stream": e.get("args", {}).get("stream")} for e in ev if e.get("cat") == "kernel"]
    return sorted(out, key=lambda e: e["ts"])


def exclusive_times(ks):
    """Per launch, the device time no earlier launch already covers:
    end_i - max(start_i, latest end before it).  With programmatic dependent
    launch a kernel's CTAs start on idle SMs while its predecessor drains and
    then wait at griddepcontrol.wait, so raw durations overlap and over-count;
    the exclusive times sum to the union of the kernel intervals (<= the
    step's event time)."""
    out, end = [], float("-inf")
    for k in sorted(ks, key=lambda e: e["ts"]):
        e = k["ts"] + k["dur"]
        out.append(max(0.0, e - max(k["ts"], end)))
        end = max(end, e)
    return out


def summarize_kernels(ks, steps: int):
    """Per kernel name: launches, mean / median / min / max raw duration (us),
    the mean exclusive time (exclusive_times) and its share of the busy time;
    plus the busy (union) kernel time per step."""
    by, ex = {}, {}
    for k, x in zip(sorted(ks, key=lambda e: e["ts"]), exclusive_times(ks)):
        by.setdefault(k["name"], []).append(k["dur"])
        ex.setdefault(k["name"], []).append(x)
    tot = sum(sum(v) for v in ex.values())
    rows = {n: {"launches": len(v), "mean_us": round(statistics.mean(v), 3),
                "median_us": round(statistics.median(v), 3), "min_us": round(min(v), 3),
                "max_us": round(max(v), 3), "excl_mean_us": round(statistics.mean(ex[n]), 3),
                "share": round(sum(ex[n]) / tot, 4) if tot else None}
            for n, v in by.items()}
    return {"kernels": rows, "kernel_us_per_step": round(tot / max(1, steps), 3)}


def short_name(n: str) -> str:
    for key in ("decode_kernel", "attn_mma_kernel", "attn_simt_kernel", "score_select_kernel", "gather_rows_kernel",
                "append_kernel"):
        if key in n:
            return key
    return n[:80]


# ------------------------------------------------------------- dist plumbing
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend):
        self.backend = backend
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            if torch.cuda.is_available() and getattr(self, "backend", "nccl") == "nccl":
                self.pg.barrier(device_ids=[self.local])
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        dev = "cuda" if torch.cuda.is_available() and getattr(self, "backend", "nccl") == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def done(self):
        if self.pg:
            self.pg.destroy_process_group()


def shard_plan(cfg: synth.Config, world: int, rank: int, mode: str):
    """Units a rank owns and the first KV head of its slice.  weak: a full cfg
    batch per rank (seeded by rank).  allgather: a contiguous slice of KV heads
    (and their G query heads) of every sequence."""
    if mode == "weak" or world == 1:
        return cfg, 0
    try:
        h0, h1 = shard.kv_head_slice(cfg.Hkv, world, rank)
    except ValueError as e:
        raise SystemExit(f"--mode allgather: {e}")
    return cfg.with_(Hkv=h1 - h0, Hq=cfg.G * (h1 - h0)), h0


def make_step(layers, call_layer, pg=None, gathered=None):
    """One decode step over the resident layers: call_layer(layer) runs the
    hot path of one layer (one ds_decode_attention_append launch); with a
    process group, each layer's head outputs are then all-gathered into
    gathered[i] ([world][B][Hq/world][d]), the path's only exchange."""
    def step():
        for i, ly in enumerate(layers):
            call_layer(ly)
            if gathered is not None:
                shard.allgather_heads(pg, ly["out"], gathered[i])
    return step


# ------------------------------------------------------------------ clocks
class Clocks:
    """SM clock / throttle-reason sampler (NVML, every ~2 ms) running across the
    timed region; falls back to `nvidia-smi -lms 100` without pynvml."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int, path: str):
        import threading
        self.rows, self.path, self.proc, self.nv = [], path, None, None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.stop_ev = threading.Event()
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()
        except Exception:
            self.nv = None
            q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self.f = open(path, "w")
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=self.f, stderr=subprocess.DEVNULL)
            except Exception:
                self.proc = None

    def _loop(self):
        nv, h = self.nv, self.h
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.rows.append((float(sm), int(rs), pw))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        if self.nv is not None:
            self.stop_ev.set()
            self.th.join(timeout=2)
            if not self.rows:
                return None
            with open(self.path, "w") as f:
                f.write("sm_mhz,reasons_mask,power_w\n")
                for r in self.rows:
                    f.write(f"{r[0]},{r[1]:#x},{r[2]}\n")
            reasons = sorted({n for r in self.rows for bit, n in self.REASONS.items() if r[1] & bit})
            return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(self.rows), "power_w_max": max(r[2] for r in self.rows),
                    "source": "nvml, 2 ms"}
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        for ln in open(self.path):
            p = [x.strip() for x in ln.split(",")]
            if len(p) >= 9 and p[1].replace(".", "").isdigit():
                rows.append(p)
        if not rows:
            return None
        sm = [float(p[1]) for p in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in rows for i in range(4) if p[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "source": "nvidia-smi, 100 ms"}


# ----------------------------------------------------------- our GPU arm
def build_layers(cfg, L, rank, structure, device, label="native", identity_pages=False):
    import paper_2408_07092_b200 as ds
    layers = []
    for l in range(L):
        seed = cfg.seed_base + 97 * rank + l
        lay = synth.make_layer(cfg, seed, device=device, structure=structure, identity_pages=identity_pages)
        Qc, Kc = synth.make_calibration(cfg, n=512, seed=seed, device=device)
        C = ds.ds_calibrate_channels(Qc, Kc, cfg.Hkv, cfg.r)            # offline, untimed
        cache = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype],
                                       lay.block_table, num_pages=lay.num_pages, page_size=cfg.page_size,
                                       device=device, channel_idx=C, label_format=label)
        ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
        # the decode step's inputs: the current token (position S-1) and its query
        k_new = lay.K[:, :, cfg.S - 1:cfg.S].transpose(1, 2).contiguous()
        v_new = lay.V[:, :, cfg.S - 1:cfg.S].transpose(1, 2).contiguous()
        pos = torch.full((cfg.B,), cfg.S - 1, dtype=torch.int32, device=device)
        layers.append(dict(cache=cache, cs=cache.struct(), q=lay.q.contiguous(), k_new=k_new, v_new=v_new,
                           pos=pos, out=torch.empty_like(lay.q)))
        del lay, Qc, Kc
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return layers


def time_graph(fn, steps, warmup, dist, stream, sampler=None):
    """Capture fn() in a CUDA graph, replay W times, then time exactly K replays
    with events on the capture stream (barrier + sync on both sides).
    sampler(): started right before the timed replays, stopped right after;
    its result is returned as a third value.  If the capture fails (a
    collective the backend cannot capture), fn itself is timed the same way
    and the returned graph is None."""
    with torch.cuda.stream(stream):
        fn()                                   # eager warm-up (attribute setup, allocator, communicator)
    torch.cuda.synchronize()
    g, run = None, fn
    if getattr(dist, "backend", "nccl") != "gloo":  # (gloo collectives cannot be captured: eager)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        run = g.replay
    with torch.cuda.stream(stream):           # replay() launches on the current stream
        for _ in range(warmup):
            run()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        smp = sampler() if sampler else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
        sampled = smp.stop() if smp else None
    dist.barrier()
    if sampler:
        return e0.elapsed_time(e1), g, sampled
    return e0.elapsed_time(e1), g


def run_ours(args, dist):
    import paper_2408_07092_b200 as ds
    dev = torch.device("cuda", dist.local)
    torch.cuda.set_device(dev)
    full = synth.CONFIGS[args.config]
    cfg, h0 = shard_plan(full, dist.world, dist.rank, args.mode)
    hbm_peak, peak_src = peaks()
    # the layers swept per step must cover >= 4x the L2, so no
    # layer's bytes are still cached when it comes round again
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    bytes_layer = ledger.layer_bytes_alg(cfg, args.label)
    L = max(args.layers, -(-4 * l2 // bytes_layer))
    layers = build_layers(cfg, L, dist.rank if args.mode == "weak" else 0, args.structure, dev, args.label,
                          identity_pages=args.pages == "identity")
    assert L * bytes_layer >= 4 * l2, "swept footprint below 4x L2"
    k = cfg.k
    ws = ds.workspace(ds.ds_decode_workspace_size(layers[0]["cache"], k), dev)
    stream = torch.cuda.Stream(dev)
    gathered = None
    if args.mode == "allgather" and dist.world > 1:
        gathered = [torch.empty((dist.world,) + tuple(layers[0]["out"].shape), dtype=layers[0]["out"].dtype,
                                device=dev) for _ in range(L)]
    lib = ds.lib()
    sp = ctypes.c_void_p(stream.cuda_stream)
    P = ctypes.c_void_p

    def call_layer(ly):  # a0 + a1..a5 of one layer: ds_decode_attention_append (one launch)
        ds._check(lib.ds_decode_attention_append(ctypes.byref(ly["cs"]), P(ly["k_new"].data_ptr()),
                                                 P(ly["v_new"].data_ptr()), P(ly["pos"].data_ptr()),
                                                 P(ly["q"].data_ptr()), k, P(ly["out"].data_ptr()), None,
                                                 P(ws.data_ptr()), ws.numel(), sp), "append+decode")

    step = make_step(layers, call_layer, dist.pg, gathered)

    def decode_only_layer(ly):
        ds._check(lib.ds_decode_attention(ctypes.byref(ly["cs"]), P(ly["q"].data_ptr()), k, P(ly["out"].data_ptr()),
                                          None, P(ws.data_ptr()), ws.numel(), sp), "decode")

    def decode_only():
        for ly in layers:
            ds._check(lib.ds_decode_attention(ctypes.byref(ly["cs"]), P(ly["q"].data_ptr()), k,
                                              P(ly["out"].data_ptr()), None, P(ws.data_ptr()), ws.numel(), sp),
                      "decode")

    cpath = os.path.join(ROOT, "gpurun_out", f"clocks_rank{dist.rank}.csv")
    os.makedirs(os.path.dirname(cpath), exist_ok=True)
    ms_total, g_step, clocks = time_graph(step, args.steps, args.warmup, dist, stream,
                                          sampler=lambda: Clocks(dist.local, cpath))
    ms_step = dist.max(ms_total / args.steps)
    ms_kernel_step = None
    if gathered is not None:  # the same step without the collective: kernel-only time
        ms_k, _ = time_graph(make_step(layers, call_layer), args.steps, 2, dist, stream)
        ms_kernel_step = dist.max(ms_k / args.steps)

    # dominant launch group for the roofline: ds_decode_attention alone over the same layers
    ms_dec_total, g_dec = time_graph(decode_only, args.steps, 2, dist, stream)
    us_decode = dist.max(ms_dec_total / args.steps) / L * 1000.0

    # in-situ device time of every kernel of the two timed graphs (CUPTI via
    # torch.profiler, three more replays each), and of one decode launch in
    # isolation after an L2 flush
    with torch.cuda.stream(stream):
        ks_step = kernel_trace(g_step.replay if g_step is not None else step, reps=3)
        ks_dec = kernel_trace(g_dec.replay if g_dec is not None else decode_only, reps=3)
        flush = torch.ones(256 << 20, dtype=torch.bfloat16, device=dev)

        def iso():
            # 512 MiB READ: L2 (126 MB) holds nothing of layer 0 and no dirty
            # lines whose write-back the decode would pay for
            flush.sum(dtype=torch.float32)
            decode_only_layer(layers[0])
        ks_iso = [x for x in kernel_trace(iso, reps=10) if "decode_kernel" in x["name"]]
        del flush

    n_ranks = dist.world
    total_bytes = bytes_layer * L * (n_ranks if args.mode == "weak" else 1) if args.mode == "weak" else \
        ledger.layer_bytes_alg(full, args.label) * L
    value = total_bytes / (ms_step / 1e3) / 1e9
    us_layer = ms_step * 1000.0 / L
    res = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": n_ranks, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
        "scaling": "weak" if args.mode == "weak" else "strong", "vs_baseline": None, "dtype": cfg.dtype,
        "data": "synthetic (seeded N(0,1) q/K/V, 8 planted outlier channels per KV head, random page order)",
        "config": {"workload": f"{full.name}: B={full.B} Hq={full.Hq} Hkv={full.Hkv} d={full.d} S={full.S} "
                               f"r={full.r} k={full.k} {full.dtype}" + (" label=int4" if args.label == "int4" else ""),
                   "label": args.label, "layers_resident": L,
                   "structure": args.structure, "page_size": cfg.page_size, "page_order": args.pages,
                   "parallelism": (f"dp{n_ranks}" if args.mode == "weak" else f"kv-head-shard{n_ranks}+allgather"),
                   "l2": f"inputs > L2: each step touches {L} x {bytes_layer / 2**20:.1f} MiB of distinct layer caches "
                         f"= {L * bytes_layer / l2:.1f} x the {l2 / 2**20:.0f} MiB L2 (>= 4x asserted)"},
        "us_per_layer": round(us_layer, 3),
        "kernel_only_ms_per_step": round(ms_kernel_step, 5) if ms_kernel_step is not None else None,
        "step_graph_captured": g_step is not None,
        "tokens_per_s_attn": round(full.B * (n_ranks if args.mode == "weak" else 1) * 1e6 / (us_layer * 32), 1),
        "bytes_alg_per_layer": bytes_layer,
    }
    achieved = bytes_layer / (us_decode * 1e-6) / 1e9
    n_dec = ds.ds_decode_launches(layers[0]["cache"], cfg.k)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{full.name}" + ("_int4" if args.label == "int4" else "") + ".json")
    if os.path.exists(tpath) and cfg == full:  # (the captured launch is the full config's)
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch_group")
        except Exception:
            traffic = None
    res["roofline"] = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                       "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                       "kernel": ("decode_kernel (fused score+select+attention, one CTA per unit)" if n_dec == 1 else
                                  "ds_decode_attention launch group (score_select_kernel + attn_mma_kernel)"),
                       "us_per_launch": round(us_decode, 3), "peak_source": peak_src,
                       "algorithmic_bytes_per_launch": bytes_layer}
    # per layer: 1 fused launch on the single-kernel path, else append + 2 decode kernels
    res["gpu_launches"] = args.steps * L * (1 if n_dec == 1 else KERNELS_PER_APPEND + n_dec)
    # CUPTI in-situ durations: the dominant kernel's share of the step, and
    # the roofline fraction of its mean in-situ launch and of one isolated launch
    sd, ss = summarize_kernels(ks_dec, 3), summarize_kernels(ks_step, 3)
    dom = [n for n in sd["kernels"] if short_name(n) in ("decode_kernel", "score_select_kernel")]
    if dom:
        du = sd["kernels"][dom[0]]["excl_mean_us"]
        res["roofline"]["cupti_us_per_launch"] = du
        res["roofline"]["cupti_frac"] = round(bytes_layer / (du * 1e-6) / 1e9 / hbm_peak, 4)
    if ks_iso:
        iu = statistics.median(x["dur"] for x in ks_iso)
        res["roofline"]["isolated_us"] = round(iu, 3)
        res["roofline"]["isolated_frac"] = round(bytes_layer / (iu * 1e-6) / 1e9 / hbm_peak, 4)
    res["kernel_trace"] = {
        "source": "CUPTI kernel activity (torch.profiler), 3 extra replays of each timed graph",
        "step_graph": {short_name(n): v for n, v in ss["kernels"].items()},
        "step_kernel_us": ss["kernel_us_per_step"], "step_us_events": round(ms_step * 1e3, 3),
        "decode_graph": {short_name(n): v for n, v in sd["kernels"].items()},
        "decode_kernel_us": sd["kernel_us_per_step"], "decode_us_events": round(us_decode * L, 3)}
    tname = f"kernels_{full.name}" + ("_int4" if args.label == "int4" else "") + f"_rank{dist.rank}.json"
    with open(os.path.join(ROOT, "gpurun_out", tname), "w") as f:
        json.dump({"summary": res["kernel_trace"], "isolated_decode_us": [x["dur"] for x in ks_iso],
                   "step_graph_kernels": [{**x, "name": short_name(x["name"])} for x in ks_step]}, f, indent=1)
    rp = read_peak_gbs(dev)
    res["roofline"]["read_peak_gbs"] = round(rp, 1)  # torch bf16 sum over 4 GiB, context only
    res["roofline"]["frac_of_read_peak"] = round(achieved / rp, 4)
    if clocks:
        res["clocks"] = clocks

    if not args.no_dense:
        dws = ds.workspace(ds.ds_dense_workspace_size(layers[0]["cache"]), dev)

        def dense():
            for ly in layers:
                ds._check(lib.ds_dense_decode_attention(ctypes.byref(ly["cs"]), P(ly["q"].data_ptr()),
                                                        P(ly["out"].data_ptr()), P(dws.data_ptr()), dws.numel(), sp),
                          "dense")
        dsteps = max(3, args.steps // 4)
        ms_d, _ = time_graph(dense, dsteps, 2, dist, stream)
        us_dense = dist.max(ms_d / dsteps) * 1000.0 / L
        res["dense_us_per_layer"] = round(us_dense, 3)
        res["dense_gbs"] = round(ledger.layer_bytes_dense(cfg) / (us_dense * 1e-6) / 1e9, 1)
        res["speedup_vs_dense"] = round(us_dense / us_decode, 3)
        res["byte_ratio_ceiling"] = round(ledger.byte_ratio_ceiling(cfg, args.label), 3)
        del dws
        if not args.no_dense_refs:
            refs = dense_references(cfg, layers, args, dist, stream)
            refs["ours_dense_flash_decode"] = {"us_per_layer": round(us_dense, 3), "gbs": res["dense_gbs"]}
            res["dense_refs"] = refs
            fastest = min((v["us_per_layer"] for v in refs.values() if "us_per_layer" in v), default=None)
            if fastest:
                res["fastest_dense_us_per_layer"] = round(fastest, 3)
                res["speedup_vs_fastest_dense"] = round(fastest / us_decode, 3)

    if not args.no_e2e:
        res["e2e"] = e2e(args, dist, layers, ws, k, stream, cfg, gathered is not None)
    if args.extra and dist.world == 1:
        res["extra"] = extra_configs(args)
    del layers
    torch.cuda.empty_cache()
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(full, budget_s=12.0, label=args.label)
    return res


def dense_references(cfg, layers, args, dist, stream):
    """Dense decode attention over every token, by library kernels on the
    same shapes: torch SDPA on contiguous K/V [B][H_kv][S][d]
    (the paper's baseline; GQA through enable_gqa) and flashinfer's
    trtllm-gen decode kernel on our paged pools (HND layout, the same block
    tables).  Each is timed like ours (CUDA graph over the resident layers,
    events, max over ranks); a reference that cannot run reports its error."""
    import math

    import torch.nn.functional as F
    out = {}
    L = len(layers)
    dbytes = ledger.layer_bytes_dense(cfg)
    steps = max(3, args.steps // 4)
    dev = layers[0]["q"].device
    try:
        kv = [(torch.randn((cfg.B, cfg.Hkv, cfg.S, cfg.d), device=dev, dtype=layers[0]["q"].dtype),
               torch.randn((cfg.B, cfg.Hkv, cfg.S, cfg.d), device=dev, dtype=layers[0]["q"].dtype)) for _ in range(L)]
        qs = [ly["q"].view(cfg.B, cfg.Hq, 1, cfg.d) for ly in layers]

        def sdpa():
            for i in range(L):
                F.scaled_dot_product_attention(qs[i], kv[i][0], kv[i][1], enable_gqa=cfg.G > 1)
        ms, _ = time_graph(sdpa, steps, 2, dist, stream)
        us = dist.max(ms / steps) * 1e3 / L
        out["torch_sdpa"] = {"us_per_layer": round(us, 3), "gbs": round(dbytes / (us * 1e-6) / 1e9, 1),
                             "kv": "contiguous [B][H_kv][S][d]"}
        del kv
        torch.cuda.empty_cache()
    except Exception as e:
        out["torch_sdpa"] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
    try:
        from flashinfer.decode import trtllm_batch_decode_with_kv_cache
        wsb = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
        outs = [torch.empty_like(ly["q"]) for ly in layers]
        scale = 1.0 / math.sqrt(cfg.d)

        def fi():
            for i, ly in enumerate(layers):
                c = ly["cache"]
                trtllm_batch_decode_with_kv_cache(ly["q"], (c.k_pool, c.v_pool), wsb, c.block_table, c.seq_lens,
                                                  cfg.S, bmm1_scale=scale, bmm2_scale=1.0, out=outs[i],
                                                  kv_layout="HND", backend="trtllm-gen")
        ms, _ = time_graph(fi, steps, 2, dist, stream)
        us = dist.max(ms / steps) * 1e3 / L
        out["flashinfer_trtllm_gen"] = {"us_per_layer": round(us, 3), "gbs": round(dbytes / (us * 1e-6) / 1e9, 1),
                                        "kv": "our paged pools, HND, page 16"}
        del wsb, outs
    except Exception as e:
        out["flashinfer_trtllm_gen"] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
    return out


def e2e(args, dist, layers, ws, k, stream, cfg, allgather=False):
    """Same metric through the public Python API with host buffers: per step the
    current token's q/k_new/v_new of every layer are copied from pinned host
    memory and every layer's output is read back, inside the timed region.
    allgather: each layer's head outputs are all-gathered (every rank reads
    back all heads)."""
    import paper_2408_07092_b200 as ds
    # the step's inputs (every layer's q, k_new, v_new) packed in one pinned
    # host buffer and one device buffer, so each step is one H2D copy, the
    # layer calls on views of it, and one D2H copy of all outputs
    srcs = [t for ly in layers for t in (ly["q"], ly["k_new"], ly["v_new"])]
    nin = [t.numel() * t.element_size() for t in srcs]
    wmul = dist.world if allgather else 1
    nout = [ly["out"].numel() * ly["out"].element_size() * wmul for ly in layers]
    h_in = torch.empty(sum(nin), dtype=torch.uint8).pin_memory()
    h_out = torch.empty(sum(nout), dtype=torch.uint8).pin_memory()
    d_in = torch.empty(sum(nin), dtype=torch.uint8, device=layers[0]["q"].device)
    d_out = torch.empty(sum(nout), dtype=torch.uint8, device=layers[0]["q"].device)

    def views(buf, tensors, sizes):
        out, off = [], 0
        for t, n in zip(tensors, sizes):
            out.append(buf[off:off + n].view(t.dtype).view(t.shape))
            off += n
        return out
    dv = views(d_in, srcs, nin)
    for hv_, t in zip(views(h_in, srcs, nin), srcs):
        hv_.copy_(t.cpu())
    dq, dk, dvv = dv[0::3], dv[1::3], dv[2::3]
    if allgather:
        outs = [torch.empty((dist.world,) + tuple(ly["out"].shape), dtype=ly["out"].dtype) for ly in layers]
        gat = views(d_out, outs, nout)
        do = [torch.empty_like(ly["out"]) for ly in layers]
    else:
        do = views(d_out, [ly["out"] for ly in layers], nout)
    h2d, d2h = h_in.numel(), h_out.numel()

    # per layer, its inputs (q, k_new, v_new: adjacent in the packed buffers)
    # and its outputs, so the copies pipeline with the kernels: layer i waits
    # only for its own H2D copy (on the h2d stream), and its D2H copy (on the
    # d2h stream) runs while later layers compute
    lin = [sum(nin[3 * i:3 * i + 3]) for i in range(len(layers))]
    oin = [sum(lin[:i]) for i in range(len(layers))]
    oout = [sum(nout[:i]) for i in range(len(layers))]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in layers]
    ev_out = [torch.cuda.Event() for _ in layers]

    def one():
        cur = torch.cuda.current_stream()
        h2d_s.wait_stream(cur)
        d2h_s.wait_stream(cur)
        with torch.cuda.stream(h2d_s):
            for i in range(len(layers)):
                d_in[oin[i]:oin[i] + lin[i]].copy_(h_in[oin[i]:oin[i] + lin[i]], non_blocking=True)
                ev_in[i].record(h2d_s)
        for i, ly in enumerate(layers):
            cur.wait_event(ev_in[i])
            ds.ds_decode_attention_append(ly["cache"], dk[i], dvv[i], ly["pos"], dq[i], k, out=do[i], ws=ws,
                                          cs=ly["cs"])
            if allgather:
                shard.allgather_heads(dist.pg, do[i], gat[i])
            ev_out[i].record(cur)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_out[i])
                h_out[oout[i]:oout[i] + nout[i]].copy_(d_out[oout[i]:oout[i] + nout[i]], non_blocking=True)
        cur.wait_stream(h2d_s)
        cur.wait_stream(d2h_s)

    def timed(run):
        with torch.cuda.stream(stream):
            for _ in range(max(3, args.warmup)):
                run()
            torch.cuda.synchronize()
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                run()
            e1.record(stream)
            torch.cuda.synchronize()
        dist.barrier()
        return dist.max(e0.elapsed_time(e1) / args.steps)

    # Double buffering across steps: step s computes on input buffer s % 2
    # while the h2d stream copies step s+1's inputs into the other buffer;
    # every step still copies all its inputs in and all its outputs out.  Two
    # steps are captured as one graph (buffers 0 then 1).
    d_in2 = [d_in, torch.empty_like(d_in)]
    dv2 = [dv, views(d_in2[1], srcs, nin)]
    ev_ready = [torch.cuda.Event(), torch.cuda.Event()]

    def step_db(cb, first):
        cur = torch.cuda.current_stream()
        if not first:  # (the graph's first step: the previous replay joined its prefetch)
            cur.wait_event(ev_ready[cb])
        h2d_s.wait_stream(cur)
        d2h_s.wait_stream(cur)
        with torch.cuda.stream(h2d_s):  # the next step's inputs, under this step's kernels
            d_in2[cb ^ 1].copy_(h_in, non_blocking=True)
            ev_ready[cb ^ 1].record(h2d_s)
        xq, xk, xv = dv2[cb][0::3], dv2[cb][1::3], dv2[cb][2::3]
        for i, ly in enumerate(layers):
            ds.ds_decode_attention_append(ly["cache"], xk[i], xv[i], ly["pos"], xq[i], k, out=do[i], ws=ws,
                                          cs=ly["cs"])
            if allgather:
                shard.allgather_heads(dist.pg, do[i], gat[i])
            ev_out[i].record(cur)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_out[i])
                h_out[oout[i]:oout[i] + nout[i]].copy_(d_out[oout[i]:oout[i] + nout[i]], non_blocking=True)
        cur.wait_stream(h2d_s)
        cur.wait_stream(d2h_s)

    def two_steps():
        step_db(0, True)
        step_db(1, False)

    L = len(layers)
    nr = dist.world if args.mode == "weak" else 1
    per_step = ledger.layer_bytes_alg(cfg, args.label) * L * nr if args.mode == "weak" else \
        ledger.layer_bytes_alg(synth.CONFIGS[args.config], args.label) * L
    ms_eager = timed(one)
    # the same calls and copies captured once with the package's CapturedStep
    # (one graph launch per step; the copies stay inside every replay)
    if getattr(dist, "backend", "nccl") == "gloo":  # (one-GPU test mode: nothing to capture)
        ms = ms_one = ms_eager
    else:
        cap = ds.CapturedStep(one, stream=stream)
        ms_one = timed(cap.graph.replay)
        with torch.cuda.stream(stream):  # buffer 0 holds the first step's inputs
            d_in2[0].copy_(h_in, non_blocking=True)
        cap2 = ds.CapturedStep(two_steps, stream=stream)
        ms = timed(cap2.graph.replay) / 2.0
    return {"value": round(per_step / (ms / 1e3) / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 5),
            "api": "paper_2408_07092_b200.CapturedStep over ds_decode_attention_append; every step copies all its "
                   "inputs H2D from pinned memory (double-buffered: during the previous step, on an h2d stream) "
                   "and each layer's outputs D2H (d2h stream) as soon as the layer is done",
            "single_buffered": {"value": round(per_step / (ms_one / 1e3) / 1e9, 2), "ms_per_step": round(ms_one, 5),
                                "api": "the same with each step's H2D copies inside the step (per layer, pipelined "
                                       "with the kernels)"},
            "eager": {"value": round(per_step / (ms_eager / 1e3) / 1e9, 2), "ms_per_step": round(ms_eager, 5),
                      "api": "ds_decode_attention_append called per layer from Python (single-buffered)"}}


def extra_configs(args):
    """c2 (Llama-2-7B MHA, B=1, fp16) at S=4K/16K/32K: us/layer sparse vs dense."""
    import paper_2408_07092_b200 as ds
    out = {}
    stream = torch.cuda.Stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    P = ctypes.c_void_p
    lib = ds.lib()

    class _D:
        def barrier(self):
            pass
    for name in ("c2_4k", "c2_16k", "c2_32k"):
        cfg = synth.CONFIGS[name]
        L = 32
        layers = build_layers(cfg, L, 0, "iid", torch.device("cuda"))
        ws = ds.workspace(ds.ds_decode_workspace_size(layers[0]["cache"], cfg.k))
        dws = ds.workspace(ds.ds_dense_workspace_size(layers[0]["cache"]))

        def dec():
            for ly in layers:
                ds._check(lib.ds_decode_attention(ctypes.byref(ly["cs"]), P(ly["q"].data_ptr()), cfg.k,
                                                  P(ly["out"].data_ptr()), None, P(ws.data_ptr()), ws.numel(), sp),
                          "decode")

        def den():
            for ly in layers:
                ds._check(lib.ds_dense_decode_attention(ctypes.byref(ly["cs"]), P(ly["q"].data_ptr()),
                                                        P(ly["out"].data_ptr()), P(dws.data_ptr()), dws.numel(), sp),
                          "dense")
        ms_s, _ = time_graph(dec, 20, 3, _D(), stream)
        ms_d, _ = time_graph(den, 10, 2, _D(), stream)
        us_s, us_d = ms_s / 20 / L * 1e3, ms_d / 10 / L * 1e3
        out[name] = {"us_per_layer": round(us_s, 3), "dense_us_per_layer": round(us_d, 3),
                     "speedup_vs_dense": round(us_d / us_s, 3),
                     "gbs": round(ledger.layer_bytes_alg(cfg) / (us_s * 1e-6) / 1e9, 1)}
        del layers, ws, dws
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------ the oracle (CPU)
def oracle_sample(cfg: synth.Config, n_seq: int, seed: int, label="native"):
    """Host inputs for n_seq sequences of cfg (all H_kv units each); with
    label="int4" also the oracle's 4-bit codes and scales of the label."""
    import oracle
    sc = cfg.with_(B=n_seq)
    lay = synth.make_layer(sc, seed, device="cpu")
    q, K, V = lay.q.float().numpy(), lay.K.float().numpy(), lay.V.float().numpy()
    C = lay.C_plant.numpy()
    import numpy as np
    L = np.empty((sc.B, sc.Hkv, sc.S, sc.r), np.float32)
    q4 = None
    if label == "int4":
        q4 = dict(codes=np.empty((sc.B, sc.Hkv, sc.S, sc.r), np.int8), scale=np.empty((sc.B, sc.Hkv, sc.S), np.float32))
    for b in range(sc.B):
        for h in range(sc.Hkv):
            L[b, h] = oracle.label_gather(K[b, h], C[h])
            if q4 is not None:
                q4["codes"][b, h], q4["scale"][b, h] = oracle.quantize_label_4bit(L[b, h], cfg.dtype)
    return sc, q, K, V, L, C, lay.seq_lens.numpy(), (q4 or {})


def cpu_baseline(cfg: synth.Config, budget_s: float = 12.0, nthreads=None, label="native", one_core_s: float = 5.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the
    same workload: whole sequences (all KV heads) of cfg, as many as fit the
    time budget (pilot-timed); then the same oracle on ONE core over single
    units (SURVEY 8(d) asks for both)."""
    import oracle
    nthreads = nthreads or os.cpu_count() or 1
    n_seq = max(1, -(-nthreads // cfg.Hkv))            # enough units to occupy every core
    sc, q, K, V, L, C, sl, q4 = oracle_sample(cfg, n_seq, seed=cfg.seed_base + 777, label=label)
    nthreads = min(nthreads, sc.units)
    t = time.perf_counter()
    oracle.decode_batch(q, K, V, L, C, sl, cfg.k, nthreads=nthreads, **q4)
    pilot = time.perf_counter() - t
    reps = max(1, int(budget_s / max(pilot, 1e-3)))
    t = time.perf_counter()
    for _ in range(reps):
        oracle.decode_batch(q, K, V, L, C, sl, cfg.k, nthreads=nthreads, **q4)
    dt = time.perf_counter() - t
    units = sc.units * reps
    ubytes = ledger.unit_bytes_alg(cfg.S, cfg.d, cfg.r, cfg.k, cfg.elem, label)
    bytes_ = units * ubytes
    # one core: the first sequence's first KV head, repeated within one_core_s
    q1 = {kk: v[:1, :1] for kk, v in q4.items()}
    args1 = (q[:1, :cfg.G], K[:1, :1], V[:1, :1], L[:1, :1], C[:1], sl[:1], cfg.k)
    t = time.perf_counter()
    oracle.decode_batch(*args1, nthreads=1, **q1)
    p1 = time.perf_counter() - t
    r1 = max(1, int(one_core_s / max(p1, 1e-3)))
    t = time.perf_counter()
    for _ in range(r1):
        oracle.decode_batch(*args1, nthreads=1, **q1)
    d1 = time.perf_counter() - t
    return {"value": round(bytes_ / dt / 1e9, 4), "unit": "GB/s", "cores": nthreads, "kind": "oracle",
            "sample": f"{reps} x {sc.B} sequences ({sc.units} units of {cfg.name}, S={cfg.S}, k={cfg.k}), "
                      f"Algorithm 1 in plain fp32 C, {dt:.1f} s",
            "us_per_unit": round(dt / units * 1e6, 1),
            "one_core": {"value": round(r1 * ubytes / d1 / 1e9, 4), "unit": "GB/s", "cores": 1,
                         "us_per_unit": round(d1 / r1 * 1e6, 1),
                         "sample": f"{r1} x 1 unit of {cfg.name} on one thread, {d1:.1f} s"}}


def run_reference(args, dist):
    import oracle
    full = synth.CONFIGS[args.config]
    nthreads = os.cpu_count() or 1
    n_seq = max(1, -(-nthreads // full.Hkv))
    sc, q, K, V, L, C, sl, q4 = oracle_sample(full, n_seq, seed=full.seed_base + 777, label=args.label)
    nthreads = min(nthreads, sc.units)
    t = time.perf_counter()
    oracle.decode_batch(q, K, V, L, C, sl, full.k, nthreads=nthreads, **q4)
    pilot = time.perf_counter() - t
    reps = max(1, int(2.0 / max(pilot, 1e-3)))     # ~2 s of CPU work per step
    for _ in range(args.warmup):
        for _ in range(reps):
            oracle.decode_batch(q, K, V, L, C, sl, full.k, nthreads=nthreads, **q4)
    t = time.perf_counter()
    for _ in range(args.steps):
        for _ in range(reps):
            oracle.decode_batch(q, K, V, L, C, sl, full.k, nthreads=nthreads, **q4)
    dt = time.perf_counter() - t
    units = sc.units * reps * args.steps
    value = units * ledger.unit_bytes_alg(full.S, full.d, full.r, full.k, full.elem, args.label) / dt / 1e9
    ms_step = dt / args.steps * 1e3
    sample = f"{reps} x {sc.B} sequences ({sc.units} units) of {full.name} per step, plain fp32 C oracle"
    return {"metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": full.dtype, "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{full.name}: B={full.B} Hq={full.Hq} Hkv={full.Hkv} d={full.d} S={full.S} "
                                   f"r={full.r} k={full.k} {full.dtype}" + (" label=int4" if args.label == "int4" else ""),
                       "label": args.label, "sample_per_step": sample},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": nthreads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def link_peaks(dev, nbytes: int = 1 << 30, reps: int = 3):
    """Host-link ceilings in this run: pinned host -> device and device ->
    pinned host cudaMemcpy of `nbytes` (copy engine), best of `reps`, GB/s."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = {}
    for name, dst, src in (("h2d_gbs", d, h), ("d2h_gbs", h, d)):
        best = float("inf")
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = round(nbytes / (best / 1e3) / 1e9, 2)
    out["bytes"] = nbytes
    del h, d
    torch.cuda.empty_cache()
    return out


def _union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], b))
        else:
            out.append((a, b))
    return out


def _intersect(x, y):
    out, i, j = [], 0, 0
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            out.append((a, b))
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return out


def _measure(iv):
    return sum(b - a for a, b in _union(iv))


def run_offload(args, dist):
    """f1: Double Sparsity-Offload on c5.  K/V pools live in pinned
    host memory; per layer l, the main stream attends over slot l % 2 (rows
    prefetched earlier) while the side stream runs ds_prefetch_next_layer for
    layer l + 1 with a predicted query (cos ~0.95, reading R15) into the other
    slot.  Timed: exactly K steps of L layers after W warm-up steps (CUDA
    events on the main stream, after a join with the side stream)."""
    import paper_2408_07092_b200 as ds
    dev = torch.device("cuda", dist.local)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS["c5"]
    # L = 32 (Llama-3-8B) layers of pinned host K/V (2 GiB each), or as many
    # as half the available host memory holds
    host_kv_layer = 2 * cfg.B * cfg.Hkv * cfg.S * cfg.d * cfg.elem
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    L = max(2, min(args.offload_layers, int(0.5 * avail // host_kv_layer)))
    link = link_peaks(dev)
    layers = []
    for l in range(L):
        seed = cfg.seed_base + l
        lay = synth.make_layer(cfg, seed, device=dev)
        cache = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype],
                                       lay.block_table, num_pages=lay.num_pages, page_size=cfg.page_size,
                                       channel_idx=lay.C_plant, host_kv=True)
        ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
        torch.cuda.synchronize()
        q = lay.q.contiguous()
        layers.append(dict(cache=cache, q=q, q_hat=synth.predicted_query(q, 0.95, seed), out=torch.empty_like(q)))
        del lay
        torch.cuda.empty_cache()
    slots = [ds.PrefetchSlot.allocate(layers[0]["cache"], cfg.k, dev) for _ in range(2)]
    main_s, side_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    with torch.cuda.stream(side_s):                      # layer 0's rows before the first step
        ds.ds_prefetch_next_layer(layers[0]["cache"], layers[0]["q_hat"], cfg.k, slots[0], stream=side_s)
        ready[0].record(side_s)

    def step(base):
        for l in range(L):
            i = base + l
            s_cur, s_nxt = slots[i % 2], slots[(i + 1) % 2]
            nxt = layers[(l + 1) % L]
            with torch.cuda.stream(side_s):              # prefetch layer l+1 (slot freed by layer l-1)
                side_s.wait_event(free[(i + 1) % 2])
                ds.ds_prefetch_next_layer(nxt["cache"], nxt["q_hat"], cfg.k, s_nxt, stream=side_s)
                ready[(i + 1) % 2].record(side_s)
            with torch.cuda.stream(main_s):              # attention of layer l on its prefetched rows
                main_s.wait_event(ready[i % 2])
                ly = layers[l]
                ds.ds_decode_attention_prefetched(ly["cache"], ly["q"], s_cur, ly["out"], stream=main_s)
                free[i % 2].record(main_s)
    for w in range(args.warmup):
        step(w * L)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main_s)
    for st in range(args.steps):
        step((args.warmup + st) * L)
    main_s.wait_stream(side_s)
    e1.record(main_s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    us_layer = ms * 1e3 / L
    link_bytes = cfg.B * cfg.Hkv * cfg.k * 2 * cfg.d * cfg.elem          # K+V rows per layer over the link
    # overlap (CUPTI kernel activity over one more step): the share of the
    # attention kernels' time that the side stream's prefetch kernels cover
    ks = kernel_trace(lambda: step((args.warmup + args.steps) * L), reps=1)
    pre = [(k["ts"], k["ts"] + k["dur"]) for k in ks if short_name(k["name"]) in ("decode_kernel", "gather_rows_kernel")]
    att = [(k["ts"], k["ts"] + k["dur"]) for k in ks if short_name(k["name"]).startswith("attn")]
    overlap = {"attention_us": round(_measure(att), 2), "prefetch_us": round(_measure(pre), 2),
               "both_us": round(_measure(_intersect(_union(pre), _union(att))), 2)}
    overlap["attention_covered_frac"] = round(overlap["both_us"] / max(overlap["attention_us"], 1e-9), 4)
    overlap["source"] = "CUPTI kernel activity (torch.profiler), one step of L layers"
    # prefetch alone (one layer, side stream idle otherwise)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(side_s):
        t0.record(side_s)
        for _ in range(3):
            ds.ds_prefetch_next_layer(layers[0]["cache"], layers[0]["q_hat"], cfg.k, slots[0], stream=side_s)
        t1.record(side_s)
    torch.cuda.synchronize()
    us_pf = t0.elapsed_time(t1) / 3 * 1e3
    jac = []
    idx = torch.empty((cfg.B, cfg.Hkv, cfg.k), dtype=torch.int32, device=dev)
    ds.ds_decode_attention(layers[0]["cache"], layers[0]["q"], cfg.k, topk_idx_out=idx)
    ds.ds_prefetch_next_layer(layers[0]["cache"], layers[0]["q_hat"], cfg.k, slots[0])
    torch.cuda.synchronize()
    a, b = idx.cpu().numpy(), slots[0].idx.cpu().numpy()
    for bb in range(cfg.B):
        for h in range(cfg.Hkv):
            sa, sb = set(a[bb, h].tolist()), set(b[bb, h].tolist())
            jac.append(len(sa & sb) / max(1, len(sa | sb)))
    dev_bytes = sum(x.numel() * x.element_size() for sl in slots for x in (sl.k_rows, sl.v_rows, sl.idx)) + \
        L * layers[0]["cache"].label.numel() * layers[0]["cache"].label.element_size()
    return {"metric": "Double Sparsity-Offload decode µs/layer (c5, KV in pinned host memory)",
            "value": round(us_layer, 2), "unit": "µs/layer", "higher_is_better": False, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": f"c5: B={cfg.B} Hq={cfg.Hq} Hkv={cfg.Hkv} d={cfg.d} S={cfg.S} r={cfg.r} "
                                   f"k={cfg.k} {cfg.dtype}, K/V pools pinned host, {L} layers, q_hat cos 0.95"},
            "link_bytes_per_layer": link_bytes, "link_gbs": round(link_bytes / (us_layer * 1e-6) / 1e9, 2),
            "link_peak": link,
            "link_frac_of_h2d_peak": round(link_bytes / (us_layer * 1e-6) / 1e9 / link["h2d_gbs"], 4),
            "overlap": overlap, "layers": L,
            "prefetch_alone_us": round(us_pf, 2),
            "prefetch_alone_link_gbs": round(link_bytes / (us_pf * 1e-6) / 1e9, 2),
            "jaccard_qhat_vs_q_mean": round(float(np.mean(jac)), 4),
            "device_bytes_label_plus_slots": int(dev_bytes),
            "host_kv_bytes_per_layer": int(2 * layers[0]["cache"].k_pool.numel() * cfg.elem)}


def main():
    args = parse()
    dist = Dist()
    if args.impl == "reference":
        if dist.rank != 0:
            return 0
        print(json.dumps(run_reference(args, dist)), flush=True)
        return 0
    if not torch.cuda.is_available():
        raise SystemExit("bench.py (ours) needs a CUDA device; there is no CPU fallback")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    # DS_BENCH_ONE_GPU=1 (tests only): every rank on cuda:0 over gloo, to run
    # the N>1 code path on a one-GPU box (no graph capture of the collective)
    if os.environ.get("DS_BENCH_ONE_GPU") == "1":
        dist.local = 0
    torch.cuda.set_device(dist.local)  # before the NCCL communicator is created
    dist.init("gloo" if os.environ.get("DS_BENCH_ONE_GPU") == "1" else "nccl")
    res = run_offload(args, dist) if args.offload else run_ours(args, dist)
    if dist.rank == 0:
        print(json.dumps(res), flush=True)
    dist.done()
    return 0


if __name__ == "__main__":
    sys.exit(main())
