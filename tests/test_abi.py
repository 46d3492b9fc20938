"""CPU checks of the C-ABI library: it loads, exports every symbol include/cmb.h
declares, and its host-only entry points behave (no GPU compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cmb():
    from paper_2504_18082_b200 import _build
    _build.build()
    import paper_2504_18082_b200 as m
    return m


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cmb.h")).read()
    return sorted(set(re.findall(r"^CMB_API [^(]*?\b(cmb_\w+)\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("cmb_load_graph", "cmb_order_roots", "cmb_sample_blocks", "cmb_gather_features",
              "cmb_sage_mean_aggregate", "cmb_gather_aggregate"):
        assert s in syms


def test_library_exports_every_declared_symbol(cmb):
    L = cmb.lib()
    syms = declared_symbols()
    assert sorted(cmb.SYMBOLS) == syms
    for s in syms:
        assert hasattr(L, s), s


def test_host_only_entry_points(cmb):
    L = cmb.lib()
    assert L.cmb_version() == 1
    assert L.cmb_status_string(4) == b"CMB_ERR_CAPACITY"
    nc, ec = cmb.blocks_capacity(1024, [15, 10, 5], 2_449_029)
    assert nc == [1024, 16384, 180224, 1081344] and ec == [15360, 163840, 901120]
    nc, ec = cmb.blocks_capacity(64, [5, 5], 1000)
    assert nc == [64, 384, 1000] and ec == [320, 1920]
    assert L.cmb_graph_workspace_bytes(1000, 8) >= 1000 * 8 + 9 * 4 + 256
    # host-checkable argument errors return immediately, without touching a device
    out = ctypes.c_void_p()
    assert L.cmb_load_graph(None, None, ctypes.byref(out)) == 1
    assert b"null" in L.cmb_last_error_message()


def test_sm100a_code_in_library(cmb):
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", cmb.LIB_PATH],
                       capture_output=True, text=True)
    assert "sm_100a" in r.stdout
