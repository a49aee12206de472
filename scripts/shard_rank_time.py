"""Per-rank kernel time of the KV-head-sharded configurations,
measured on one GPU: for N in {1, 2, 4, 8}, rank 0's slice of the config
(bench.shard_plan: H_kv / N KV heads with their G query heads, every
sequence) is built alone and its decode step (ds_decode_attention_append per
layer, the layers swept >= 4x L2, one CUDA graph) is timed with CUDA events.
No collective and no other rank run here: this is the kernel part of a
rank's step at N GPUs, not a multi-GPU measurement.

usage: python scripts/shard_rank_time.py [config ...]   (default c3 c4)
One JSON line per (config, N).  Cluster-size sweep (timing experiments only):
DS_LIB=<a build with -DDS_EXP_NCH_ENV> NCH_SWEEP=2,4,8 SHARDS=8 ... times each
slice once per forced cluster size.
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2408_07092_b200 import ledger  # noqa: E402


def main():
    import paper_2408_07092_b200 as ds
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist = bench.Dist()
    lib = ds.lib()
    P = ctypes.c_void_p
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    for name in sys.argv[1:] or ["c3", "c4"]:
        full = synth.CONFIGS[name]
        for n in [int(x) for x in os.environ.get("SHARDS", "1,2,4,8").split(",")]:
            if full.Hkv % n:
                continue
            cfg, h0 = bench.shard_plan(full, n, 0, "allgather")
            bl = ledger.layer_bytes_alg(cfg, "native")
            L = max(8, -(-4 * l2 // bl))
            layers = bench.build_layers(cfg, L, 0, "iid", dev)
            k = cfg.k
            ws = ds.workspace(ds.ds_decode_workspace_size(layers[0]["cache"], k), dev)
            stream = torch.cuda.Stream(dev)
            sp = P(stream.cuda_stream)

            def step():
                for ly in layers:
                    ds._check(lib.ds_decode_attention_append(
                        ctypes.byref(ly["cs"]), P(ly["k_new"].data_ptr()), P(ly["v_new"].data_ptr()),
                        P(ly["pos"].data_ptr()), P(ly["q"].data_ptr()), k, P(ly["out"].data_ptr()), None,
                        P(ws.data_ptr()), ws.numel(), sp), "append+decode")

            for nch in os.environ.get("NCH_SWEEP", "0").split(","):
                if nch != "0":
                    os.environ["DS_NCH"] = nch
                steps = 20
                ms, _ = bench.time_graph(step, steps, 5, dist, stream)
                us_layer = ms / steps / L * 1e3
                print(json.dumps({
                    "config": name, "n_gpus": n, "rank0_slice": f"Hkv={cfg.Hkv} (heads {h0}..{h0 + cfg.Hkv - 1}) "
                    f"Hq={cfg.Hq} B={cfg.B} S={cfg.S} k={cfg.k}",
                    "forced_ctas_per_unit": int(nch) or None,
                    "layers_resident": L, "us_per_layer_rank_kernel": round(us_layer, 3),
                    "rank_gbs": round(bl / (us_layer * 1e-6) / 1e9, 1),
                    "note": "rank 0's slice alone on one GPU: kernel time of one rank's step, no all-gather"}),
                    flush=True)
            del layers, ws
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
