"""The C-ABI library builds for sm_100a, loads without a GPU and exports every symbol
include/amg.h declares; host-only entry points work on CPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def amg():
    from paper_2006_06052_b200 import build
    build.build()
    import paper_2006_06052_b200 as m
    return m


def test_exports_every_declared_symbol(amg):
    hdr = open(os.path.join(ROOT, "include", "amg.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+\**(\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    L = amg.lib()
    missing = [s for s in sorted(declared) if not hasattr(L, s)]
    assert not missing, missing
    assert declared == set(amg.EXPORTS)


def test_sass_is_sm100a(amg):
    out = subprocess.run(["cuobjdump", "--list-elf", amg.SO_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_params_default_and_status(amg):
    p = amg.default_params()
    assert p.gmres_m == 30 and p.maxiter == 1000 and p.hier_dtype == amg.F32
    assert abs(p.sa_omega - 2 / 3) < 1e-15 and p.eps_strong == 1e-3 and p.coarse_enough == 3000
    assert amg.status_string(amg.EBREAKDOWN).startswith("Krylov breakdown")
    assert amg.lib().amg_setup(None, None, None, None) == amg.EINVAL
