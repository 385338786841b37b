"""CPU-side checks of the C ABI boundary: the library loads, exports every symbol the header
declares, and validates arguments synchronously (no GPU needed: validation precedes any CUDA call)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sentencekv.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sentencekv_\w+)\s*\(", txt)))


def test_header_declares_the_three_hot_path_calls():
    names = declared()
    for n in ("sentencekv_prefill_compress", "sentencekv_decode_select", "sentencekv_decode_attend",
              "sentencekv_create", "sentencekv_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import paper_2504_00970_b200 as skv

    out = subprocess.run(["nm", "-D", "--defined-only", skv.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sentencekv_\w+)", out))
    assert set(declared()) <= exported, set(declared()) - exported
    # nothing else leaks from the library's C++ internals
    assert all(s.startswith("sentencekv_") for s in re.findall(r"\bT (\w+)", out) if not s.startswith("_"))
    for n in declared():
        assert hasattr(skv.lib, n)


def test_library_is_sm100a_cubin():
    import paper_2504_00970_b200 as skv

    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", skv.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_python_binding_has_abi_names():
    import paper_2504_00970_b200 as skv

    for n in ("sentencekv_create", "sentencekv_destroy", "sentencekv_prefill_compress", "sentencekv_decode_select",
              "sentencekv_decode_attend", "sentencekv_sync"):
        assert callable(getattr(skv, n))


def _create_status(**kw):
    import paper_2504_00970_b200 as skv

    base = dict(batch=1, layers=1, q_heads=8, kv_heads=2, head_dim=64, max_context=4096, token_budget=256)
    base.update(kw)
    cfg = skv.sentencekv_config_default(**base)
    ctx = ctypes.c_void_p()
    return skv.lib.sentencekv_create(ctypes.byref(cfg), ctypes.byref(ctx))


@pytest.mark.parametrize("kw,status", [
    (dict(q_heads=6, kv_heads=4), 1),          # Hq % G != 0
    (dict(token_budget=0), 1),                 # tau < 1
    (dict(semantic_factor=0.5), 1),            # r < 1
    (dict(batch=0), 1),
    (dict(kv_head_begin=1, kv_head_count=2), 1),  # shard out of range
    (dict(batch_begin=1), 1),
    (dict(head_dim=96), 3),                    # unsupported head dim
    (dict(q_heads=24, kv_heads=2), 3),         # grp = 12 unsupported
    (dict(obs_window=-1), 1),                  # N < 0
    (dict(obs_window=3), 3),                   # NEXT-1: window rows N * grp must be a multiple of 16
    (dict(obs_window=300), 3),                 # NEXT-1: N * grp <= 256
    (dict(residency=1, semantic_factor=1.5), 1),  # host residency needs r >= 2
])
def test_create_rejects_bad_configs(kw, status):
    assert _create_status(**kw) == status


def test_null_arguments_are_rejected():
    import paper_2504_00970_b200 as skv

    assert skv.lib.sentencekv_create(None, None) == 1
    assert skv.lib.sentencekv_prefill_compress(None, 0, None, 1, None, 0, None, None, 2.0, 1, None, None) == 1
    assert skv.lib.sentencekv_decode_select(None, 0, None, None, None, None, None, None) == 1
    assert skv.lib.sentencekv_set_band_log2(None, 19) == 1
    assert skv.lib.sentencekv_decode_attend(None, 0, None, None, None) == 1
    assert skv.lib.sentencekv_destroy(None) == 0
