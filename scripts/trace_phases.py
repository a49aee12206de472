"""Per-CTA phase timeline of the decode kernels (needs libds_trace.so).

usage: DS_LIB=paper_2408_07092_b200/libds_trace.so python scripts/trace_phases.py [config]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2408_07092_b200 as ds
import synth

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = synth.CONFIGS[name]
for kv in sys.argv[2:]:  # overrides, e.g. B=1 Hkv=1 Hq=4
    key, val = kv.split("=")
    cfg = cfg.with_(**{key: int(val)})
print(cfg)
lay = synth.make_layer(cfg, cfg.seed_base, device="cuda", structure=os.environ.get("DS_STRUCTURE", "iid"))
cache = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, synth.DTYPES[cfg.dtype], lay.block_table,
                               num_pages=lay.num_pages, page_size=cfg.page_size, channel_idx=lay.C_plant,
                               label_format=os.environ.get("DS_LABEL", "native"))
ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
del lay.K, lay.V
L = ds.lib()
L.ds_debug_read_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
buf = np.zeros((3, 4096, 16), np.uint64)
for it in range(4):
    L.ds_debug_clear_trace()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ds.ds_decode_attention(cache, lay.q, cfg.k)
    e1.record()
    torch.cuda.synchronize()
    print(f"iter {it}: decode {e0.elapsed_time(e1) * 1e3:.1f} us (events, incl. launch)")
L.ds_debug_read_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)


def report_slots(kind, pairs):
    t = buf[kind].astype(np.int64)
    t = t[t[:, 0] > 0]
    for a, b_, nm in pairs:
        ok = (t[:, a] > 0) & (t[:, b_] > 0)
        if ok.any():
            d = (t[ok, b_] - t[ok, a]) / 1e3
            print(f"  sub {nm:14s} p50 {np.median(d):7.2f} p90 {np.percentile(d, 90):7.2f}")


def report(kind, names):
    t = buf[kind].astype(np.int64)
    t = t[t[:, 0] > 0]
    if len(t) == 0:
        print("no trace for kind", kind)
        return
    t0 = min(buf[k][buf[k][:, 0] > 0][:, 0].min() for k in range(3) if (buf[k][:, 0] > 0).any())
    print(f"\n{['score_select', 'fused decode', 'attention'][kind]}: {len(t)} CTAs")
    for i, n in enumerate(names):
        ok = t[:, i] > 0
        if not ok.any():
            continue
        v = (t[ok, i] - t0) / 1e3
        print(f"  {n:16s} (n={ok.sum():4d}) t(us) min {v.min():7.2f}  p50 {np.median(v):7.2f}  p90 {np.percentile(v, 90):7.2f}  max {v.max():7.2f}")
    for i in range(1, len(names)):
        ok = (t[:, i] > 0) & (t[:, i - 1] > 0)
        if ok.any():
            d = (t[ok, i] - t[ok, i - 1]) / 1e3
            print(f"  dur {names[i - 1]}->{names[i]:14s} p50 {np.median(d):7.2f} p90 {np.percentile(d, 90):7.2f} max {d.max():7.2f}")


if (buf[1][:, 0] > 0).any():  # fused kernel: kind 0 holds its exchange timestamps
    report_slots(0, [(0, 1, "xchg0 wait"), (1, 8, "L2 dsmem+bnd"), (8, 11, "L2 selsync"), (11, 14, "cand mark"),
                     (14, 2, "mark->xchg1"), (1, 2, "level2->xchg1"), (2, 3, "xchg1 wait"), (6, 7, "xchg3 wait")])
    report_slots(1, [(2, 0, "masks->xchg0")]) if False else None
report(0, ["start", "streamed", "S1 D1", "L2 pass", "members", "written", "published"])
report_slots(0, [(4, 7, "S3 sync"), (7, 8, "gather+rank"), (8, 10, "pre-write"), (10, 5, "write pass")])
_bc = buf[0][:, 9][buf[0][:, 0] > 0]
if len(_bc):
    print("  boundary-bin members p50", np.median(_bc), "p90", np.percentile(_bc, 90), "max", _bc.max())


def report1():
    t = buf[1].astype(np.int64)
    t = t[t[:, 0] > 0]
    names = {0: "start", 4: "pdl waited", 1: "staged", 5: "level1", 6: "level2", 7: "level3", 2: "radix done",
             8: "pass A", 9: "pass B", 3: "compacted"}
    order = [0, 4, 1, 5, 6, 7, 2, 8, 9, 3]
    prev = None
    print("\nselect phases (p50 of per-CTA durations, us):")
    for s_ in order:
        col = t[:, s_]
        ok = col > 0
        if prev is not None and ok.any():
            d = (col[ok] - t[ok, prev]) / 1e3
            print(f"  {names[prev]:>12s} -> {names[s_]:12s} p50 {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f}  (n={ok.sum()})")
        if ok.any():
            prev = s_
report(2, ["start", "rowids", "loop done", "cluster sync", "merged"])
report(1, ["start", "streamed", "masks", "tail done", "gt rows done", "all rows", "merged"])
report_slots(1, [(0, 12, "prologue"), (12, 13, "stream t0"), (13, 1, "stream sync"), (1, 7, "D1 boundary"), (7, 8, "mask loop w0"), (8, 9, "cand gather w0"), (9, 2, "sync"),
                 (2, 3, "tail"), (2, 14, "tail: level 2"), (14, 15, "tail: members"), (15, 3, "tail: rank+list"), (5, 10, "partials"), (10, 11, "weights"), (11, 6, "outputs")])
report_slots(2, [(0, 1, "sample sync")])
t1, t2 = buf[1].astype(np.int64), buf[2].astype(np.int64)
ok = (t1[:, 0] > 0) & (t2[:, 2] > 0) & (t2[:, 4] > 0)
if ok.any():  # fused decode prologue: start -> pdl waited -> n known -> tile waited -> stream starts (slot 12)
    for a, b_, nm in [((1, 0), (2, 2), "pro: pdl wait"), ((2, 2), (2, 3), "pro: n known"), ((2, 3), (2, 4), "pro: tile+sync"),
                      ((2, 4), (1, 12), "pro: qlab")]:
        d = (np.where(True, [t1, t2][b_[0] - 1][ok, b_[1]], 0) - [t1, t2][a[0] - 1][ok, a[1]]) / 1e3
        print(f"  sub {nm:14s} p50 {np.median(d):7.2f} p90 {np.percentile(d, 90):7.2f}")  # fused decode, high-mask threshold (kind 2's slots borrowed)

_nc = buf[2][:, 7].astype(np.int64)
_nc = _nc[(_nc > 0) & (_nc < 2000000)] - 1000000
if len(_nc):
    print("  D1-bin candidates ranked by the tail (per CTA, tail only): p50", np.median(_nc), "p90",
          np.percentile(_nc, 90), "max", _nc.max(), "n", len(_nc))
