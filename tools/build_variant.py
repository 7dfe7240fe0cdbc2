"""Build a variant of libti64b200.so with extra -D flags (A/B experiments):
    python tools/build_variant.py NAME -DFOO=1 ...   -> _lib/variants/lib_NAME.so
Select it at run time with TI64_LIB=<path>."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2402_17580_b200 import _build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = b.OUT_DIR / "variants"
out.mkdir(parents=True, exist_ok=True)
objs = []
for s in b.SOURCES:
    o = out / f"{Path(s).stem}_{name}.o"
    subprocess.run([b.nvcc(), *b.NVCC_FLAGS, *defs, "-I", str(b.ROOT / "include"), "-c",
                    str(b.CSRC / s), "-o", str(o)], check=True)
    objs.append(str(o))
lib = out / f"lib_{name}.so"
subprocess.run([b.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                str(lib), *objs, "-cudart", "static"], check=True)
for o in objs:
    Path(o).unlink()
print(lib)
