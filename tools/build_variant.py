"""Build a variant of libti64b200.so for A/B experiments:
    python tools/build_variant.py NAME [--rev GITREV] [-DFOO=1 ...]
        -> paper_2402_17580_b200/_lib/variants/lib_NAME.so
--rev builds the sources (csrc + include) of that git revision instead of the
working tree.  Select a variant at run time with TI64_VARIANT_LIB=<path>."""
import subprocess
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import _variant  # noqa: E402,F401  (tools only: optional TI64_VARIANT_LIB)
from paper_2402_17580_b200 import _build as b  # noqa: E402

args = sys.argv[1:]
name = args.pop(0)
rev = None
if "--rev" in args:
    i = args.index("--rev")
    rev = args[i + 1]
    del args[i:i + 2]
defs = args
out = b.OUT_DIR / "variants"
out.mkdir(parents=True, exist_ok=True)
with tempfile.TemporaryDirectory() as tmp:
    if rev:
        root = Path(tmp)
        (root / "pkg" / "csrc").mkdir(parents=True)
        (root / "include").mkdir()
        for f in b.SOURCES + b.HEADERS:
            txt = subprocess.run(["git", "show", f"{rev}:paper_2402_17580_b200/csrc/{f}"],
                                 capture_output=True, text=True, cwd=b.ROOT).stdout
            (root / "pkg" / "csrc" / f).write_text(txt)
        (root / "include" / "ti64_b200.h").write_text(subprocess.run(
            ["git", "show", f"{rev}:include/ti64_b200.h"], capture_output=True, text=True,
            cwd=b.ROOT).stdout)
        csrc, inc = root / "pkg" / "csrc", root / "include"
    else:
        csrc, inc = b.CSRC, b.ROOT / "include"
    objs = []
    for s in b.SOURCES:
        o = Path(tmp) / f"{Path(s).stem}.o"
        subprocess.run([b.nvcc(), *b.NVCC_FLAGS, *defs, "-I", str(inc), "-c", str(csrc / s),
                        "-o", str(o)], check=True)
        objs.append(str(o))
    lib = out / f"lib_{name}.so"
    subprocess.run([b.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                    str(lib), *objs, "-cudart", "static"], check=True)
print(lib)
