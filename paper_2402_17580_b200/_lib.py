"""ctypes binding of libti64b200.so (the C ABI in include/ti64_b200.h).

There is no CPU fallback: every compute entry point goes through this
library, and a missing library or a missing sm_100 device raises
``Ti64Unavailable`` at call time.  Importing the package never needs a GPU.
"""

import ctypes as C
from pathlib import Path

from . import _abi

# The in-tree library; there is no environment override (kernel-variant A/B
# experiments live in tools/ and patch LIB_PATH explicitly, tools/_variant.py).
LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libti64b200.so"

__all__ = ["Ti64Unavailable", "Ti64Error", "load", "require", "check", "LIB_PATH"]


class Ti64Unavailable(RuntimeError):
    """The CUDA library is not built or no sm_100 (B200) device is visible."""


class Ti64Error(RuntimeError):
    """A library call returned an error code."""


_lib = None

_P, _I64, _I32, _D = C.c_void_p, C.c_int64, C.c_int32, C.c_double

_SIGS = {
    "ti64_run_range": (_I64, [_P, _I64, _I64, _I64, _I64, _D, _P, _P, _I32, _P, _P]),
    "ti64_gen_temperature": (_I64, [_P, _I64, _I64, _P, _P]),
    "ti64_gen_initial_state": (_I64, [_P, _I64, _P, _P]),
    "ti64_advance": (_I64, [_P, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P,
                            _P, _P]),
    "ti64_advance_scratch_bytes": (_I64, [_I64]),
    "ti64_advance_host": (_I64, [_P, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P,
                                 _P, _I64, _I64, _P]),
    "ti64_advance_host_scratch_bytes": (_I64, [_I64, _I64, _I64, _I64]),
    "ti64_run_history": (_I64, [_P, _I64, _P, _P, _I64, _P, _P, _P, _P]),
    "ti64_fast_exp": (_I64, [_P, _P, _I64, _P]),
    "ti64_fast_ln": (_I64, [_P, _P, _I64, _P]),
    "ti64_fast_pow": (_I64, [_P, _P, _P, _I64, _P]),
    "ti64_div_rn": (_I64, [_P, _P, _P, _P, _I64, _P]),
    "ti64_phase_sums": (_I64, [_P, _P, _P, _I64, _P, _P, _P]),
    "ti64_histogram": (_I64, [_P, _P, _P, _I64, _I32, _P, _P]),
    "ti64_stencil_step": (_I64, [_P, _P, _P, _P, _P, _P, _P]),
    "ti64_thermal_substeps": (_I64, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "ti64_bench_dfma": (_I64, [_P, _I64, _I32, _P]),
    "ti64_bench_daxpy": (_I64, [_P, _P, _D, _I64, _P]),
    "ti64_coupled_step": (_I64, [_P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64, _I32, _P]),
    "ti64_coupled_step_streams": (_I64, [_P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64, _I32,
                                         _P, _P]),
    "ti64_coupled_scratch_words": (_I64, [_I64]),
    "ti64_step_counter_add": (_I64, [_P, _I64, _P]),
    "ti64_last_error": (C.c_char_p, []),
    "ti64_abi_version": (_I32, []),
    "ti64_device_ok": (_I32, []),
}

EXPORTS = tuple(_SIGS)


def load():
    """Load the shared library (no device check).  Raises Ti64Unavailable."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise Ti64Unavailable(
                f"{LIB_PATH} is missing: build it with `python -m paper_2402_17580_b200._build`")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.ti64_abi_version() != 1:
            raise Ti64Unavailable("libti64b200.so ABI version mismatch")
        _lib = lib
    return _lib


_device_checked = False


def require():
    """The library, after checking that an sm_100 device is present."""
    global _device_checked
    lib = load()
    if not _device_checked:
        import torch
        if not torch.cuda.is_available():
            raise Ti64Unavailable("no CUDA device: the B200 path has no CPU fallback")
        torch.cuda.init()
        if lib.ti64_device_ok() != 1:
            cap = torch.cuda.get_device_capability()
            raise Ti64Unavailable(f"need an sm_100 (B200) device, found sm_{cap[0]}{cap[1]}")
        _device_checked = True
    return lib


def check(rc, what):
    if rc < 0:
        msg = load().ti64_last_error().decode(errors="replace")
        if rc == -2:
            raise NotImplementedError(f"{what}: {msg}")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise Ti64Error(f"{what}: rc={rc}: {msg}")
    return rc


def ptr(t):
    """Raw device pointer of a torch tensor (or None)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def byref(x):
    return C.byref(x)


__all__ += ["ptr", "stream_handle", "byref", "EXPORTS", "_abi"]
