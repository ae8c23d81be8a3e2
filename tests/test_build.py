"""Build checks (CPU): the default K13 variant of every sample type was compiled to the code
that keeps its loop and ring indices on the uniform datapath (build; 3.86 vs
4.1-4.2 ms on config 4).  nvcc's split-compile output varies between runs and
tools/nvcc_pick.py selects it; this pins the selection in the built objects."""
from __future__ import annotations

import importlib.util
import os
import shutil

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SYM = "_ZN3fgf18lowres_gray_kernelILi1ELi4ELi9ELi17ELb0ELi160ELi3E{}EEvNS_12LowresParamsE"
UNITS = {"fgf_k_lowres_v3": "f", "fgf_k_lowres_v3h": "6__half",
         "fgf_k_lowres_v3bf": "13__nv_bfloat16", "fgf_k_lowres_v3b": "h"}


def _picker():
    spec = importlib.util.spec_from_file_location("nvcc_pick", os.path.join(ROOT, "tools", "nvcc_pick.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="needs cuobjdump")
@pytest.mark.parametrize("unit", sorted(UNITS))
def test_k13_units_use_the_uniform_datapath(unit):
    obj = os.path.join(ROOT, "build", unit + ".o")
    if not os.path.exists(obj):
        pytest.skip("library not built in-tree (make)")
    n = _picker().uniform_count(obj, SYM.format(UNITS[unit]))
    assert n >= 400, (unit, n)
