"""Debug: do ctypes launches from libds.so get captured by torch.cuda.graph?"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2408_07092_b200 as ds
import synth

cfg = synth.CONFIGS["c3"].with_(B=4)
lay = synth.make_layer(cfg, 1, device="cuda")
cache = ds.LayerCache.allocate(cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.S, cfg.r, torch.bfloat16, lay.block_table,
                               num_pages=lay.num_pages, channel_idx=lay.C_plant)
ds.prefill(cache, lay.K, lay.V, lay.seq_lens)
cs = cache.struct()
ws = ds.workspace(ds.ds_decode_workspace_size(cache, cfg.k))
out = torch.zeros_like(lay.q)
st = torch.cuda.Stream()
lib = ds.lib()
P = ctypes.c_void_p


def call():
    r = lib.ds_decode_attention(ctypes.byref(cs), P(lay.q.data_ptr()), cfg.k, P(out.data_ptr()), None,
                                P(ws.data_ptr()), ws.numel(), P(st.cuda_stream))
    assert r == 0, r


with torch.cuda.stream(st):
    call()
torch.cuda.synchronize()
ref = out.clone()
print("eager nonzero", (ref != 0).float().mean().item())
for n in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with torch.cuda.stream(st):
        for _ in range(20):
            call()
    torch.cuda.synchronize()
    print("eager us/call", (time.perf_counter() - t) / 20 * 1e6)

g = torch.cuda.CUDAGraph()
g.enable_debug_mode()
out.zero_()
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=st):
    call()
torch.cuda.synchronize()
print("after capture nonzero (should be 0 if captured)", (out != 0).float().mean().item())
g.replay()
torch.cuda.synchronize()
print("after replay equal", torch.equal(out, ref))
g.debug_dump("gpurun_out/graph.dot")
print(open("gpurun_out/graph.dot").read()[:3000])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    g.replay()
e1.record(st)
torch.cuda.synchronize()
print("graph us/replay", e0.elapsed_time(e1) / 20 * 1e3)
