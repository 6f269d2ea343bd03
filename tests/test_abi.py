"""C-ABI checks that need no GPU: the library loads, exports every function
declared in include/nrto.h, and its host-only entry points behave."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from gen import make_instance
from gen.problems import Shape
from oracle.structured import ragged_layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "nrto.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nrto_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2603_02642_b200 import nrto
    L = nrto.lib()
    names = _declared()
    assert {"nrto_setup", "nrto_inner_solve", "nrto_gain_update", "nrto_layout",
            "nrto_destroy", "nrto_last_error", "nrto_soc_project"} <= set(names)
    for n in names:
        assert hasattr(L, n), n
    # and as dynamic symbols of the .so (not C++-mangled)
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", nrto.LIB_PATH], capture_output=True,
                         text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, re.M), n


def test_binding_names_match_abi():
    from paper_2603_02642_b200 import nrto
    for n in _declared():
        assert hasattr(nrto, n), n


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_layout_matches_oracle(cfg):
    from paper_2603_02642_b200 import nrto
    shape, _ = make_instance(cfg)
    E, off = nrto.nrto_layout(shape)
    np.testing.assert_array_equal(off, ragged_layout(shape))
    assert E == off[-1]


def test_layout_rejects_bad_shapes():
    from paper_2603_02642_b200 import nrto
    bad = [Shape(3, 2, 4, np.array([0], np.int32), np.array([0], np.int8)),     # state knot 0
           Shape(3, 2, 4, np.array([5], np.int32), np.array([0], np.int8)),     # knot > T
           Shape(3, 2, 4, np.array([4], np.int32), np.array([1], np.int8)),     # control knot T
           Shape(3, 4, 4, np.array([1], np.int32), np.array([0], np.int8)),     # n_u > n_x
           Shape(40, 2, 4, np.array([1], np.int32), np.array([0], np.int8))]    # n_x > 32
    for s in bad:
        with pytest.raises(nrto.NrtoError) as ei:
            nrto.nrto_layout(s)
        assert ei.value.code == nrto.NRTO_EINVAL
        assert len(nrto.nrto_last_error()) > 0


def test_default_params_match_oracle():
    from paper_2603_02642_b200 import nrto
    from oracle.params import DEFAULTS
    p = nrto.nrto_default_params()
    for k in nrto.PARAM_DOUBLES + nrto.PARAM_INTS:
        assert getattr(p, k) == DEFAULTS[k], k


def test_struct_layout_matches_header():
    """ctypes mirrors of the C structs have the sizes a C compiler gives them."""
    from paper_2603_02642_b200 import nrto
    import subprocess, tempfile
    src = r'''
#include <stdio.h>
#include "nrto.h"
int main(){printf("%zu %zu %zu %zu\n", sizeof(nrto_shape), sizeof(nrto_data), sizeof(nrto_params), sizeof(nrto_out));return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        sizes = list(map(int, subprocess.run([exe], capture_output=True, text=True).stdout.split()))
    assert sizes == [C.sizeof(nrto.nrto_shape), C.sizeof(nrto.nrto_data),
                     C.sizeof(nrto.nrto_params), C.sizeof(nrto.nrto_out)]


def test_set_allocator_validation():
    """nrto_set_allocator: an alloc without a release is rejected; NULL restores the
    default (host-only entry point, no device call)."""
    from paper_2603_02642_b200 import nrto
    L = nrto.lib()
    assert L.nrto_set_allocator(nrto.ALLOC_FN(lambda c, n, s: None), nrto.FREE_FN(), None) == nrto.NRTO_EINVAL
    assert L.nrto_set_allocator(nrto.ALLOC_FN(), nrto.FREE_FN(), None) == nrto.NRTO_OK
