"""The ctypes mirrors of the C-ABI structs (paper_2504_18082_b200/__init__.py) have exactly the
layout include/cmb.h declares: size and every field offset, measured by compiling a small C
program against the header with gcc (no GPU, no library call)."""
import ctypes
import os
import subprocess
import tempfile

import pytest

import paper_2504_18082_b200 as cmb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# ctypes class -> C typedef (field names are the C member names)
MIRRORS = {
    cmb.GraphDesc: "cmb_graph_desc",
    cmb.Blocks: "cmb_blocks",
    cmb.Batch: "cmb_batch",
    cmb.LayerPack: "cmb_layer_pack",
    cmb.FeatureCacheDesc: "cmb_feature_cache",
    cmb.BatchFeatures: "cmb_batch_features",
}


def _c_layout():
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cmb.h"', "int main(void) {"]
    for cls, cname in MIRRORS.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    with tempfile.TemporaryDirectory() as d:
        src, exe = os.path.join(d, "layout.c"), os.path.join(d, "layout")
        with open(src, "w") as fh:
            fh.write("\n".join(lines))
        subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src,
                               "-o", exe])
        out = subprocess.check_output([exe], text=True)
    got = {}
    for ln in out.splitlines():
        cname, key, val = ln.split()
        got[(cname, key)] = int(val)
    return got


@pytest.fixture(scope="module")
def layout():
    return _c_layout()


@pytest.mark.parametrize("cls", list(MIRRORS), ids=lambda c: c.__name__)
def test_ctypes_mirror_matches_header(layout, cls):
    cname = MIRRORS[cls]
    assert ctypes.sizeof(cls) == layout[(cname, "size")], cname
    for fname, _ in cls._fields_:
        assert getattr(cls, fname).offset == layout[(cname, fname)], (cname, fname)
