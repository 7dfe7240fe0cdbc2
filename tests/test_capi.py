"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/ti64_b200.h declares, and the ctypes struct mirrors match the C
layouts (compiled here with gcc against the header)."""

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2402_17580_b200 import _abi, _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ti64_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ti64_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), f"{name} declared in ti64_b200.h but not exported"
    assert set(_lib.EXPORTS) <= set(names)
    assert lib.ti64_abi_version() == 1


def test_device_ok_is_false_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert _lib.load().ti64_device_ok() == 0
    with pytest.raises(_lib.Ti64Unavailable):
        _lib.require()


def test_struct_layouts_match_header(tmp_path):
    structs = {"ti64_kparams": _abi.KParams, "ti64_icfg": _abi.ICfg,
               "ti64_fields": _abi.Fields, "ti64_tempgen": _abi.TempGen,
               "ti64_counters": _abi.Counters, "ti64_thermal": _abi.Thermal,
               "ti64_stencil_args": _abi.StencilArgs}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"',
             'int main(void){']
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["/usr/bin/gcc", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, f"{cname}.{fname}"


def test_error_path_without_device():
    lib = _lib.load()
    # argument validation happens before any CUDA call
    rc = lib.ti64_run_range(None, 0, 10, 8, 1, 1e-5, None, None, 0, None, None)
    assert rc == -1
    assert b"bad argument" in lib.ti64_last_error()
    f = _abi.Fields()
    kp = _abi.KParams()
    cfg = _abi.ICfg(scheme=7)
    rc = lib.ti64_run_range(C.byref(f), 0, 10, 8, 1, 1e-5, C.byref(kp), C.byref(cfg), 0,
                            None, None)
    assert rc == -1 and b"unknown scheme" in lib.ti64_last_error()
    cfg = _abi.ICfg(scheme=1, max_halvings=63)
    rc = lib.ti64_run_range(C.byref(f), 0, 10, 8, 1, 1e-5, C.byref(kp), C.byref(cfg), 0,
                            None, None)
    assert rc == -1
    cfg = _abi.ICfg(scheme=0)
    rc = lib.ti64_run_range(C.byref(f), 0, 10, 3, 1, 1e-5, C.byref(kp), C.byref(cfg), 0,
                            None, None)
    assert rc == -1


def test_host_staging_scratch_sizes_need_no_gpu():
    """ti64_advance_host_scratch_bytes is host arithmetic: it grows with the
    chunk size, covers four staged chunks of 50 B/point plus two advance
    scratch sets, is independent of n once n exceeds the chunk, and rejects
    negative sizes."""
    lib = _lib.load()
    f = lib.ti64_advance_host_scratch_bytes
    adv = lib.ti64_advance_scratch_bytes
    small, big = f(1 << 27, 1 << 20, 200, 200), f(1 << 27, 1 << 22, 200, 200)
    assert 0 < small < big
    assert big >= 4 * 50 * (1 << 22) + 2 * adv(1 << 22)
    assert f(1 << 27, 0, 200, 200) == big                      # default chunk: 2^22 points
    assert 0 <= big - f(1 << 26, 1 << 22, 200, 200) <= 512     # only the chunk-sum rows differ
    assert f(1000, 1 << 22, 10, 0) < f(1 << 22, 1 << 22, 10, 0)  # chunk clipped to the input
    assert f(-1, 0, 1, 0) < 0 and f(10, 0, -1, 0) < 0
    assert adv(0) > 0 and adv(1 << 20) > adv(0)
