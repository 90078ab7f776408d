"""C-ABI boundary checks that need no GPU: libgs_sched.so loads, exports
every entry point include/gs_sched.h declares (and nothing the Python
binding expects is missing), and the ctypes mirrors of the ABI structs
have the same size and field offsets as the C compiler gives them."""

import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "gs_sched.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2012_07145_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2012_07145_b200 import _build
        _build.build()
    return _lib.load()


def test_header_declares_the_binding(lib):
    from paper_2012_07145_b200 import _lib
    assert set(_lib.EXPORTS) == set(_declared())


def test_every_declared_symbol_is_exported(lib):
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(gs_\w+)", out))
    assert set(_declared()) <= exported


def test_host_only_calls(lib):
    from paper_2012_07145_b200 import _lib
    assert lib.gs_version() == 1
    assert lib.gs_launch_count() >= 0
    assert lib.gs_select_workspace_bytes(1 << 20) > 0
    assert lib.gs_topk_workspace_bytes(1 << 20) > 0
    # argument errors are reported, never crash
    rc = lib.gs_pipeline_create(None, None)
    assert rc == -1
    assert b"" != lib.gs_last_error()
    with pytest.raises(_lib.GsError):
        _lib.check(rc)


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_struct_layout_matches_c(tmp_path):
    from paper_2012_07145_b200 import descriptor as D
    names = ["GsFunc", "GsStage", "GsAccess", "GsMachine", "GsThresholds", "GsPipelineDesc",
             "GsTilingMenus", "GsOracleParams", "GsDecision"]
    prog = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void){']
    for n in names:
        prog.append(f'printf("{n} %zu\\n", sizeof({n}));')
    for f in ("machine", "thresholds", "algo", "name_off"):
        prog.append(f'printf("GsPipelineDesc.{f} %zu\\n", offsetof(GsPipelineDesc, {f}));')
    prog.append('return 0;}')
    c = tmp_path / "layout.c"
    c.write_text("\n".join(prog))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(c), "-o", str(exe)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                               check=True).stdout.splitlines())
    for n in names[:-1]:
        assert int(got[n]) == C.sizeof(getattr(D, n)), n
    assert int(got["GsDecision"]) == D.DECISION_DTYPE.itemsize == 16
    for f in ("machine", "thresholds", "algo", "name_off"):
        assert int(got[f"GsPipelineDesc.{f}"]) == getattr(D.GsPipelineDesc, f).offset, f
    # decision record field offsets (numpy dtype mirror)
    prog2 = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void){']
    for f in ("func", "consumer", "kind", "flags", "serial", "thread"):
        prog2.append(f'printf("{f} %zu\\n", offsetof(GsDecision, {f}));')
    prog2.append('return 0;}')
    c.write_text("\n".join(prog2))
    subprocess.run(["gcc", str(c), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for f, v in got.items():
        assert D.DECISION_DTYPE.fields[f][1] == int(v), f
