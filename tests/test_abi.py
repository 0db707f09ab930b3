"""CPU-side checks of the C-ABI boundary: liblopa.so loads and exports every function that
include/liblopa.h declares, the binding's signatures cover them, and the host-side helpers
(segmentation, workspace / record sizes, BP partition) are consistent.  No compute calls."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "liblopa.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lopa_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_16229_b200 import build, lopa
    if build.stale():
        build.build()
    return lopa.lib()


def test_header_declares_the_boundary():
    names = declared()
    for f in ("lopa_confidence", "lopa_anchor_fill", "lopa_spawn_branches", "lopa_verify_select",
              "lopa_step", "lopa_bp_create", "lopa_bp_step", "lopa_bp_destroy"):
        assert f in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2512_16229_b200", "liblopa.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lopa_\w+)", out))
    assert set(declared()) <= exported


def test_binding_covers_header():
    from paper_2512_16229_b200 import lopa
    assert set(lopa.EXPORTS) == set(declared())


def test_host_helpers(lib):
    from paper_2512_16229_b200 import lopa
    assert lib.lopa_version() == 10000
    assert lopa.num_segments(151936) == 19 and lopa.num_segments(64) == 1 and lopa.num_segments(8193) == 2
    assert lopa.workspace_bytes(256, 151936) >= 256 * 10 * 16   # one group partial per (row, 2 segments)
    assert lopa.record_bytes(32, 1) % 16 == 0
    assert lib.lopa_status_string(2).decode().startswith("unsupported")


def test_argument_validation_without_gpu(lib):
    """Invalid arguments are rejected on the host before any device work."""
    null = ctypes.c_void_p()
    st = lib.lopa_confidence(null, 64, 4, 64, null, null, null, null, null, 0, null)
    assert st == 1
    st = lib.lopa_anchor_fill(null, null, null, null, 8, ctypes.c_float(0.9), null, null, null, null)
    assert st == 1
    from paper_2512_16229_b200 import lopa
    a = lopa.StepArgs()
    assert lib.lopa_step(ctypes.byref(a), null) == 1


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirror of lopa_step_args_t == the C layout (gcc offsetof on the real header)."""
    from paper_2512_16229_b200 import lopa
    fields = [f[0] for f in lopa.StepArgs._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "liblopa.h"\nint main(void){\n'
                   + "".join(f'printf("%zu\\n", offsetof(lopa_step_args_t, {f}));\n' for f in fields)
                   + 'printf("%zu\\n", sizeof(lopa_step_args_t)); return 0; }\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [getattr(lopa.StepArgs, f).offset for f in fields] + [ctypes.sizeof(lopa.StepArgs)]
    assert got == want


@pytest.mark.parametrize("max_br,world", [(8, 1), (8, 2), (8, 4), (8, 8), (11, 4), (16, 8), (3, 8)])
def test_bp_shard_partition(max_br, world):
    from paper_2512_16229_b200 import lopa
    seen = []
    for r in range(world):
        b_loc, lo, hi = lopa.bp_shard(max_br, world, r)
        assert b_loc == -(-max_br // world) and 0 <= hi - lo <= b_loc
        seen += list(range(lo, hi))
    assert seen == list(range(max_br))
