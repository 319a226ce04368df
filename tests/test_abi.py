"""Boundary checks that need no GPU: libc2.so loads, exports every symbol include/c2.h
declares, and the ctypes mirrors of the ABI structs match the C layout."""
import os
import re
import subprocess
import tempfile

import pytest

import paper_2010_11497_b200 as c2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "c2.h")).read()
    return sorted(set(re.findall(r"C2_API\s+[\w\s\*]+?\b(c2_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("c2_fastrandomhash", "c2_local_knn", "c2_merge", "c2_build", "c2_ctx_create"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = c2.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", c2.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (c2_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(lib, name)
    assert set(c2.SIGNATURES) == set(declared_functions())


def test_struct_layout_matches_header():
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "c2.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(c2_cand), sizeof(c2_clusters), sizeof(c2_stats),
         offsetof(c2_stats, ms_sketch), offsetof(c2_stats, ms_total));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(src, "w").write(prog)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
        vals = [int(x) for x in subprocess.check_output([exe]).split()]
    import ctypes
    assert vals[0] == 8
    assert vals[1] == ctypes.sizeof(c2._Clusters)
    assert vals[2] == ctypes.sizeof(c2.Stats)
    assert vals[3] == c2.Stats.ms_sketch.offset and vals[4] == c2.Stats.ms_total.offset


def test_product_never_touches_the_oracle():
    # the product package and the C ABI share no code with oracle/ (and never import it)
    pkg = os.path.join(ROOT, "paper_2010_11497_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "c2o" not in txt, f
    assert "c2o" not in open(os.path.join(ROOT, "include", "c2.h")).read()


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        c2.Context(0)
