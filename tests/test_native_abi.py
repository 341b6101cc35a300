"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares (no compute calls: there is no GPU here)."""

import re
from pathlib import Path

from paper_2306_01369_b200 import _native as N

HEADER = Path(__file__).resolve().parent.parent / "include" / "granusim_b200.h"


def declared() -> set[str]:
    text = HEADER.read_text()
    return set(re.findall(r"\b(gg_[a-z0-9_]+)\s*\(", text))


def test_library_exists_and_loads():
    assert N.LIB_PATH.exists(), "run __graft_entry__.build() first"
    lib = N.lib()
    assert b"sm_100a" in lib.gg_build_info()


def test_every_declared_symbol_is_exported():
    lib = N.lib()
    missing = [s for s in sorted(declared()) if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared()) >= 20


def test_struct_layouts_match_header(tmp_path):
    """ctypes / numpy mirrors have the C compiler's sizes and offsets."""
    import ctypes
    import subprocess

    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "granusim_b200.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(gg_params),"
        " sizeof(gg_body), sizeof(gg_report), offsetof(gg_params, z_max),"
        " offsetof(gg_body, aabb_hi), offsetof(gg_report, min_normal_impulse),"
        " sizeof(gg_camera), offsetof(gg_camera, far));return 0;}\n"
    )
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(HEADER.parent), str(src), "-o", str(exe)], check=True)
    got = [int(t) for t in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got[0] == ctypes.sizeof(N.GGParams)
    assert got[1] == N.BODY_DTYPE.itemsize
    assert got[2] == N.REPORT_DTYPE.itemsize
    assert got[3] == N.GGParams.z_max.offset
    assert got[4] == N.BODY_DTYPE.fields["aabb_hi"][1]
    assert got[5] == N.REPORT_DTYPE.fields["min_normal_impulse"][1]
    from paper_2306_01369_b200.render import CAMERA_DTYPE

    assert got[6] == CAMERA_DTYPE.itemsize
    assert got[7] == CAMERA_DTYPE.fields["far"][1]


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode == 0:
        assert "sm_100a" in out.stdout
