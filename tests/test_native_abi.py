"""The C-ABI library exists, loads without a GPU and exports every symbol
``include/fcpb.h`` declares; struct layouts of the ctypes mirror match the header."""

import ctypes
import os
import re

import pytest

from paper_2605_08524_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fcpb.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"FCPB_API\s+[\w\s\*]+?\b(fcpb_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    assert "fcpb_attn_fwd" in names and "fcpb_attn_bwd" in names and "fcpb_lse_merge" in names
    assert set(names) == set(native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = native.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.fcpb_version() == 1


def test_missing_library_fails_loudly(tmp_path):
    from paper_2605_08524_b200.errors import NativeError
    with pytest.raises(NativeError):
        native.load(str(tmp_path / "nope.so"))


def test_struct_layouts_match_header(tmp_path):
    """Compile a probe against include/fcpb.h and compare sizeof/offsetof with ctypes."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    fields = {"FcpbFwdArgs": native.FwdArgs, "FcpbMergeArgs": native.MergeArgs,
              "FcpbBwdArgs": native.BwdArgs, "FcpbDqArgs": native.DqArgs,
              "FcpbDqDsArgs": native.DqDsArgs}
    lines = ["#include <stdio.h>", "#include <stddef.h>", f'#include "{HEADER}"', "int main(void){"]
    for cname, py in fields.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run([cc, "-std=c11", "-o", str(exe), str(src)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for cname, py in fields.items():
        assert int(out[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(out[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_workspace_queries():
    """The workspace-size queries (host arithmetic, no GPU) match the buffers the Python
    side allocates: preprocess [2, Hq, t_pad] fp32, forward partials [P, Hq, D+1] fp32,
    dS tiles bf16 128x128 per (pair, q-head)."""
    lib = native.load()
    assert lib.fcpb_bwd_preprocess_bytes(10, 32) == 2 * 32 * 12 * 4
    assert lib.fcpb_bwd_preprocess_bytes(12, 8) == 2 * 8 * 12 * 4
    assert lib.fcpb_fwd_partial_bytes(1000, 32, 128) == 1000 * 32 * 129 * 4
    assert lib.fcpb_ds_tile_bytes(3, 32) == 3 * 32 * 128 * 128 * 2
    assert lib.fcpb_ds_tile_bytes(1 << 20, 64) == (1 << 20) * 64 * 32768   # no int overflow
