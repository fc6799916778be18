"""The C-ABI library loads without a GPU and exports every symbol include/dsde.h
declares; host-only entry points behave as documented (no compute calls)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dsde():
    from paper_2509_01083_b200 import _build
    _build.build()
    import paper_2509_01083_b200 as m
    return m


def header_functions():
    src = open(os.path.join(ROOT, "include", "dsde.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dsde_[a-z0-9_]+)\s*\(", src)))


def test_header_parses_to_expected_set(dsde):
    assert header_functions() == sorted(dsde.EXPORTS)


def test_library_exports_every_header_symbol(dsde):
    L = dsde.lib()
    for name in header_functions():
        assert hasattr(L, name), name
    out = subprocess.check_output(["nm", "-D", "--defined-only", dsde.LIB_PATH], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(header_functions()) == {s for s in exported if s.startswith("dsde_")}


def test_library_has_sm100a_code(dsde):
    out = subprocess.check_output(["cuobjdump", "--list-elf", dsde.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_config_defaults_match_paper(dsde):
    c = dsde.Config.default()
    assert (c.delta, c.n_short, c.n_long, c.sl_min, c.epsilon) == (0.85, 10, 30, 2, 1e-6)
    assert (c.sl_ceiling, c.calib_steps, c.calib_sl, c.window_unit, c.cap_mode) == (8, 5, 4, 0, 1)
    assert (c.masked, c.entropy_mode, c.entropy_gamma, c.greedy, c.device_rows) == (0, 0, 0.5, 0, 0)
    assert c.resample == dsde.RESAMPLE_FULL   # the D7 recovery draw by default
    assert dsde.lib().dsde_abi_version() == 4
    assert dsde.lib().dsde_status_string(-1) == b"DSDE_ERR_ARG"


def test_cap_value_host(dsde):
    c = dsde.Config.default()
    assert dsde.cap_value(c, 10, 4, 4) == 2      # [4,2,3,1]: 2.5 -> 2
    assert dsde.cap_value(c, 10, 2, 8) == 5      # [8,2]
    assert dsde.cap_value(c, 7, 2, 4) == 4       # 3.5 -> 4
    assert dsde.cap_value(c, 0, 0, 0) == 8       # no active sequences -> ceiling
    c0 = dsde.Config.default(cap_mode=0)
    assert dsde.cap_value(c0, 10, 2, 8) == 8


def test_invalid_args_rejected_without_launch(dsde):
    L = dsde.lib()
    h = C.c_void_p()
    bad = dsde.Config.default(n_short=30)
    assert L.dsde_state_create(C.byref(bad), 4, C.byref(h)) == dsde.DSDE_ERR_ARG
    bad = dsde.Config.default(resample=2)
    assert L.dsde_state_create(C.byref(bad), 4, C.byref(h)) == dsde.DSDE_ERR_ARG
    assert L.dsde_verify(0, 10, 1, 0, None, None, None, 10, None, 10, None, None, None, None,
                         None, None, 0, None, None) == dsde.DSDE_ERR_ARG
    # dsde_step: the union of the three calls' synchronous checks (null state / pointers)
    assert L.dsde_step(None, 4, 10, 1, 4, None, None, None, None, 10, None, 10, None, None, None, None,
                       None, None, None, None, None, None, None, 0, None, None) == dsde.DSDE_ERR_ARG
    assert L.dsde_verify_workspace_size(0, 1, 10, 1) == 0
    assert L.dsde_verify_workspace_size(4, 16, 128256, 1) > 0
