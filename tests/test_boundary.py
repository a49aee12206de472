"""The C-ABI boundary on CPU: libds.so loads, exports every symbol include/ds.h
declares, and host-side validation returns the documented status codes
(no kernel is launched by any call here)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2408_07092_b200 as ds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "ds.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ds_\w+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ("ds_calibrate_channels", "ds_append_kv", "ds_decode_attention"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    out = subprocess.check_output(["nm", "-D", "--defined-only", ds.LIB_PATH], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    assert set(ds.EXPORTS) <= exported


def test_library_loads_and_reports():
    L = ds.lib()
    for f in header_functions():
        assert hasattr(L, f)
    assert "sm_100a" in ds.ds_version()
    assert ds.ds_status_string(ds.DS_OK) == "DS_OK"
    assert "GQA" in ds.ds_status_string(ds.DS_ERR_GQA_INCOMPATIBLE)


def test_library_is_built_for_sm100a_only():
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ds.LIB_PATH], text=True)
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def _cache(**kw):
    base = dict(batch=1, num_q_heads=4, num_kv_heads=1, head_dim=128, page_size=16, num_pages=4,
                max_pages_per_seq=4, max_seq_len=64, r=8, dtype=ds.DS_BF16,
                k_pool=0x1000, v_pool=0x2000, block_table=0x3000, seq_lens=0x4000, label=0x5000,
                channel_idx=0x6000)
    base.update(kw)
    return ds.ds_cache(**base)


@pytest.mark.parametrize("kw,status", [
    (dict(head_dim=96), ds.DS_ERR_UNSUPPORTED),
    (dict(num_q_heads=12, num_kv_heads=1), ds.DS_ERR_UNSUPPORTED),      # G = 12
    (dict(num_q_heads=6, num_kv_heads=4), ds.DS_ERR_INVALID_ARGUMENT),   # not a multiple
    (dict(r=129), ds.DS_ERR_INVALID_ARGUMENT),
    (dict(max_pages_per_seq=2), ds.DS_ERR_INVALID_ARGUMENT),            # 32 < 64 tokens
    (dict(label=0x5008), ds.DS_ERR_INVALID_ARGUMENT),                    # misaligned
    (dict(dtype=7), ds.DS_ERR_UNSUPPORTED),
    (dict(label_format=3), ds.DS_ERR_INVALID_ARGUMENT),                  # unknown label format
    (dict(label=0), ds.DS_ERR_INVALID_ARGUMENT),                         # native label missing
    (dict(label_format=ds.DS_LABEL_INT4), ds.DS_ERR_INVALID_ARGUMENT),   # int4 without a scale array
    (dict(label_format=ds.DS_LABEL_INT4, label_scale=0xa008), ds.DS_ERR_INVALID_ARGUMENT),  # misaligned scale
])
def test_decode_validation(kw, status):
    c = _cache(**kw)
    st = ds.lib().ds_decode_attention(ctypes.byref(c), ctypes.c_void_p(0x7000), 8, ctypes.c_void_p(0x8000), None,
                                      ctypes.c_void_p(0x9000), 1 << 30, None)
    assert st == status


def test_decode_k_range_and_workspace():
    c = _cache()
    L = ds.lib()
    q, o, w = ctypes.c_void_p(0x7000), ctypes.c_void_p(0x8000), ctypes.c_void_p(0x9000)
    assert L.ds_decode_attention(ctypes.byref(c), q, 0, o, None, w, 1 << 30, None) == ds.DS_ERR_INVALID_ARGUMENT
    assert L.ds_decode_attention(ctypes.byref(c), q, 65, o, None, w, 1 << 30, None) == ds.DS_ERR_INVALID_ARGUMENT
    assert L.ds_decode_attention(ctypes.byref(c), q, 8, o, None, w, 16, None) == ds.DS_ERR_WORKSPACE_TOO_SMALL
    assert L.ds_decode_workspace_size(ctypes.byref(c), 8) > 0
    assert L.ds_decode_workspace_size(ctypes.byref(c), 0) == 0
    assert L.ds_dense_workspace_size(ctypes.byref(c)) == 0


def test_calibration_gqa_k_mode_rejected_on_host():
    st = ds.lib().ds_calibrate_channels(ctypes.c_void_p(0x1000), ctypes.c_void_p(0x2000), 8, 8, 2, 128, ds.DS_BF16,
                                        ds.DS_CALIB_K, 8, ctypes.c_uint64(0), ctypes.c_void_p(0x3000), None)
    assert st == ds.DS_ERR_GQA_INCOMPATIBLE
    st = ds.lib().ds_calibrate_channels(ctypes.c_void_p(0x1000), ctypes.c_void_p(0x2000), 8, 8, 2, 128, ds.DS_BF16,
                                        ds.DS_CALIB_QK, 200, ctypes.c_uint64(0), ctypes.c_void_p(0x3000), None)
    assert st == ds.DS_ERR_INVALID_ARGUMENT


def test_python_binding_refuses_cpu_tensors():
    import torch
    with pytest.raises(ValueError):
        ds._ptr(torch.zeros(4))


def test_ds_cache_struct_layout_matches_header():
    """The ctypes mirror of ds_cache has the header's field order; the two
    label fields added for the 4-bit label (ds_label_format) come last, so
    a zero-initialised struct keeps the native label."""
    names = [f[0] for f in ds.ds_cache._fields_]
    hdr = open(os.path.join(os.path.dirname(ds.LIB_PATH), "..", "include", "ds.h")).read()
    body = hdr[hdr.index("typedef struct {\n  int32_t batch"):]
    body = body[:body.index("} ds_cache;")]
    decl = re.findall(r"\*?\s*(\w+)\s*[,;]", body)   # declarators in order
    assert decl == names
    assert names[-3:] == ["label_format", "label_scale", "group_reduce"]
    assert ds.ds_cache().label_format == ds.DS_LABEL_NATIVE
