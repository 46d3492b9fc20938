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


def test_layer_entry_points_host_checks(cmb):
    """NEXT-4 sizes and host-checked errors (no device work): image sizes follow the
    swizzle-atom layout, unsupported shapes report 0 / CMB_ERR_INVALID_ARGUMENT."""
    L = cmb.lib()
    # first layer: 2 halves x ceil(F/64) atoms x Fo rows x 128 B
    assert L.cmb_sage_weights_bytes(100, 256) == 2 * 2 * 256 * 128
    assert L.cmb_sage_weights_bytes(16, 48) == 2 * 1 * 48 * 128
    assert L.cmb_sage_weights_bytes(129, 256) == 0          # K = 2F must stay <= 256
    assert L.cmb_sage_weights_bytes(100, 40) == 0           # Fo % 16
    assert L.cmb_gcn_weights_bytes(100, 256) == 2 * 256 * 128
    assert L.cmb_sage_hidden_weights_bytes(256, 256) == 2 * 4 * 256 * 128
    assert L.cmb_sage_hidden_weights_bytes(100, 256) == 0   # in_dim multiple of 64
    assert L.cmb_sage_backward_workspace_bytes(100, 48) == 0   # backward: power-of-two Fo
    assert L.cmb_sage_backward_workspace_bytes(100, 256) == 160 * (256 + 1) * 256 * 4
    assert L.cmb_sage_hidden_backward_workspace_bytes(256, 256) == 160 * (512 + 1) * 256 * 4
    assert L.cmb_sage_hidden_backward_workspace_bytes(192, 64) == 160 * (512 + 1) * 64 * 4
    assert L.cmb_sage_hidden_backward_workspace_bytes(256, 48) == 0   # power-of-two Fo
    assert L.cmb_sage_hidden_weights_t_bytes(256, 64) == 2 * 1 * 256 * 128   # K = 64, N = 256
    assert L.cmb_sage_hidden_weights_t_bytes(256, 48) == 2 * 1 * 256 * 128   # K padded to 64
    assert L.cmb_sage_hidden_weights_t_bytes(100, 64) == 0   # N = in_dim multiple of 16
    assert L.cmb_sage_saved_a_bytes(100, 180_224) == 1408 * 2 * 2 * 128 * 128   # 64 KB per tile
    assert L.cmb_sage_saved_a_bytes(16, 1) == 2 * 1 * 128 * 128
    assert L.cmb_sage_saved_a_bytes(129, 10) == 0
    for call in (lambda: L.cmb_sage_pack_weights(None, None, 100, 256, None, 0, None),
                 lambda: L.cmb_sage_layer_forward(None, None, 3, 0, None, None, 256, 1, 0, None,
                                                  0, None),
                 lambda: L.cmb_gcn_layer_forward(None, None, 3, 0, None, None, 256, 1, 0, None,
                                                 0, None),
                 lambda: L.cmb_sage_hidden_forward(None, 1, 0, None, 0, 256, None, None, 256, 1,
                                                   1, None, 0, None),
                 lambda: L.cmb_sage_layer_backward(None, None, 3, 0, None, 0, 0, None, 0, 256,
                                                   None, None, None, 0, None),
                 lambda: L.cmb_sage_hidden_backward(None, 1, 0, None, 0, 256, None, 0, 0, None,
                                                    0, 256, None, None, None, 0, None, 0, None),
                 lambda: L.cmb_sage_hidden_pack_weights_t(None, None, 256, 64, None, 0, None),
                 lambda: L.cmb_sage_hidden_input_grad(None, 0, 0, 0, None, 0, 64, None, 256,
                                                      None, 0, None, 0, None),
                 lambda: L.cmb_sage_layer_forward_save(None, None, 3, 0, None, None, 256, 1, 1,
                                                       None, 0, None, 0, None),
                 lambda: L.cmb_sage_layer_backward_saved(None, None, 3, 0, None, 0, None, 0, 0,
                                                         None, 0, 256, None, None, None, 0, None),
                 lambda: L.cmb_softmax_xent(None, 64, None, None, None, 0, 47, None, 64, 64, None,
                                            None, None, None),
                 lambda: L.cmb_adam_step(None, None, None, None, 4, 1e-3, 0.9, 0.999, 1e-8, 0.0,
                                         1, None),
                 lambda: L.cmb_adam_step_pack(None, None, None, None, 4, 1e-3, 0.9, 0.999, 1e-8,
                                              0.0, 1, None, 1, None)):
        assert call() == 1
        assert b"null" in L.cmb_last_error_message()


def test_sample_workspace_map_width(cmb):
    """cmb_sample_workspace_bytes (host only): the dedup map takes 4 bytes per node while every
    local id and edge position of the batch's capacity stays below 2^24, 8 bytes beyond (the
    workspace layout is otherwise a function of the largest hop's edge capacity)."""
    L = cmb.lib()
    N = 734_708
    fan = (32, 32)
    f = (ctypes.c_int32 * 2)(*fan)

    def nbytes(r):
        return L.cmb_sample_workspace_bytes(r, f, 2, N)

    def max_e(r):
        n_cap, e_cap = cmb.blocks_capacity(r, fan, N)
        return max(e_cap), n_cap[-1]

    lim = (1 << 24) - 1
    # the largest narrow batch and the smallest wide one (capacity grows with n_roots)
    lo, hi = 1, N  # binary search: max(max_e(lo)) <= lim < max(max_e(hi))
    while hi - lo > 1:
        mid = (lo + hi) // 2
        lo, hi = (mid, hi) if max(max_e(mid)) <= lim else (lo, mid)
    narrow, wide = lo, hi
    assert max(max_e(narrow)) <= lim < max(max_e(wide))
    d_scan = 4 * (max_e(wide)[0] - max_e(narrow)[0])
    d = nbytes(wide) - nbytes(narrow)
    assert abs(d - (4 * N + d_scan)) <= 512, (d, 4 * N + d_scan)   # 256-B aligned pieces
    d_narrow = nbytes(narrow) - nbytes(narrow - 1)
    assert abs(d_narrow - 4 * (max_e(narrow)[0] - max_e(narrow - 1)[0])) <= 512
