"""TOOLS ONLY: point the package at a kernel-variant library for A/B runs.

The product loader (_lib.py) has no override; tools that A/B kernel variants
import this module first.  If TI64_VARIANT_LIB is set it must name a library
under paper_2402_17580_b200/_lib/variants/ (built by tools/build_variant.py);
anything else is an error, and every load is announced on stderr."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2402_17580_b200 import _lib  # noqa: E402

_v = os.environ.get("TI64_VARIANT_LIB")
if _v:
    p = Path(_v).resolve()
    vdir = (ROOT / "paper_2402_17580_b200" / "_lib" / "variants").resolve()
    if p.parent != vdir or not p.exists():
        raise SystemExit(f"TI64_VARIANT_LIB={_v}: not a built variant under {vdir}")
    _lib.LIB_PATH = p
    print(f"[tools/_variant] LOADING KERNEL VARIANT {p.name} (not the product library)",
          file=sys.stderr, flush=True)
