"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every symbol
include/dscache.h declares, and rejects bad configurations before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dscache.h")


def _lib():
    from paper_2605_01858_b200 import _build
    _build.build()
    from paper_2605_01858_b200 import dscache
    return dscache.load_library(), dscache


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dscache_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ["dscache_create", "dscache_append_frame", "dscache_build_instant", "dscache_attend",
              "dscache_destroy"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib, dscache = _lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", dscache.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dscache_\w+)", out))
    assert set(declared_symbols()) <= exported
    assert set(dscache.EXPORTS) <= exported


def test_library_contains_tcgen05_sm100a_code():
    _, dscache = _lib()
    sass = subprocess.run(["cuobjdump", "-sass", dscache.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "LDTM" in sass and "STTM" in sass   # tcgen05.ld / st
    elf = subprocess.run(["cuobjdump", "-lelf", dscache.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


def _cfg(dscache, **kw):
    c = dict(num_streams=1, num_layers=1, num_q_heads=28, num_kv_heads=4, head_dim=128, kv_head_offset=0,
             tokens_per_frame=196, sink_tokens=4, past_frames=32, instant_frames=4, max_query_tokens=64,
             max_position=32768, rope_theta=1e6, rope_style=0, dtype=0, device=0, attn_impl=0)
    c.update(kw)
    return dscache.Config(**c)


@pytest.mark.parametrize("kw,status", [
    (dict(max_position=7000), -3),            # A+W+C+q_max = 7124 > 7000: E_POS_OVERFLOW
    # l_I = 0: the Eq. 5 update attention reaches id A+W+tpf-1 = 6471 > A+W+C+q_max-1 = 6283
    (dict(instant_frames=0, max_query_tokens=8, max_position=6300), -3),
    (dict(head_dim=96), -2),                  # E_CONFIG
    (dict(num_q_heads=30), -2),               # Hq % Hkv
    (dict(past_frames=0, instant_frames=0), -2),
    (dict(rope_theta=1.0), -2),
    (dict(attn_impl=1, head_dim=64), -2),     # tcgen05 forced on an ineligible shape (d = 64)
])
def test_create_validation_without_gpu(kw, status):
    lib, dscache = _lib()
    h = ctypes.c_void_p()
    cfg = _cfg(dscache, **kw)
    assert lib.dscache_create(ctypes.byref(cfg), ctypes.byref(h)) == status
    assert lib.dscache_last_error().decode() != ""
    assert not h.value


def test_null_arguments():
    lib, dscache = _lib()
    assert lib.dscache_create(None, None) == -1
    assert lib.dscache_append_frame(None, 0, 1, None, None, 4, None) == -1
    assert lib.dscache_destroy(None) == -1
    # checkpoint restore calls: null handle -> E_ARG before any device work
    assert lib.dscache_restore_ring(None, 0, 0, None, None) == -1
    assert lib.dscache_restore_sink(None, 0, 0, None, None) == -1
    assert lib.dscache_set_state(None, 0, 0, 1) == -1
