"""Bytes model (closed forms) and bench host logic on CPU."""
import json
import os
import subprocess
import sys

import pytest

import synth
from paper_2408_07092_b200 import ledger

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_unit_bytes_closed_forms():
    # O(S*r) label + O(2*k*d) KV; 16-bit label (reading R8)
    assert ledger.unit_bytes_alg(S=1024, d=64, r=4, k=64, e=2) == 1024 * 4 * 2 + 2 * 64 * 64 * 2 == 24576
    assert ledger.unit_bytes_dense(S=1024, d=64, e=2) == 262144
    # k is clamped per sequence
    assert ledger.unit_bytes_alg(S=10, d=8, r=2, k=64, e=2) == 10 * 2 * 2 + 2 * 10 * 8 * 2
    # r = d, k = S: the sparse path is never cheaper than dense
    assert ledger.unit_bytes_alg(S=500, d=64, r=64, k=500, e=2) >= ledger.unit_bytes_dense(500, 64, 2)


def test_c3_layer_bytes_and_ceiling():
    c3 = synth.CONFIGS["c3"]
    assert ledger.layer_bytes_alg(c3) == 128 * (32768 * 8 * 2 + 2 * 2048 * 128 * 2) == 192 * 2 ** 20
    assert ledger.layer_bytes_dense(c3) == 2 * 2 ** 30
    assert abs(ledger.byte_ratio_ceiling(c3) - 10.6667) < 1e-3


def test_int4_label_bytes():
    """4-bit label (reading R16): ceil(r/2) code bytes + one e-byte scale per
    token, the layout ds.h documents and LayerCache allocates."""
    c3 = synth.CONFIGS["c3"]
    assert ledger.label_row_bytes(8, 2, "int4") == 4 + 2
    assert ledger.label_row_bytes(3, 2, "int4") == 2 + 2
    assert ledger.label_row_bytes(16, 4, "int4") == 8 + 4
    assert ledger.layer_bytes_alg(c3, "int4") == 128 * (32768 * 6 + 2 * 2048 * 128 * 2) == 152 * 2 ** 20
    assert abs(ledger.byte_ratio_ceiling(c3, "int4") - 2048 / 152) < 1e-9


def test_shard_plan_allgather_and_weak():
    sys.path.insert(0, ROOT)
    import bench
    c3 = synth.CONFIGS["c3"]
    cfg, h0 = bench.shard_plan(c3, 4, 3, "allgather")
    assert (cfg.Hkv, cfg.Hq, h0) == (2, 8, 6)
    cfg, h0 = bench.shard_plan(c3, 8, 5, "weak")
    assert cfg == c3 and h0 == 0
    with pytest.raises(SystemExit):
        bench.shard_plan(c3.with_(Hkv=3, Hq=12), 2, 0, "allgather")


def test_reference_arm_prints_contract_line():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "impl", "cpu_baseline", "e2e", "config"):
        assert key in line
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
