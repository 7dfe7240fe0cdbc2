import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
from paper_2402_17580_b200 import _abi, _lib, thermal as th
import ctypes as C
shape = tuple(int(v) for v in sys.argv[1:4])
nz, ny, nx = shape
t = torch.from_numpy(353.0 + np.random.default_rng(0).uniform(0, 2500.0, shape)).cuda()
d = t.clone()
src = th.HeatSource(w_eff=87.5, radius=50e-6, h_powder=20e-6)
a = _abi.stencil_args(nx, ny, nz, nz, 1e-6, 20e-6, beam=(nx * 10e-6, ny * 9e-6, 87.5, True),
                      source=src, losses=False, bottom=353.0, all_built=True)
tp = _abi.thermal_from(th.DEFAULT_THERMAL.kernel_tuple())
rc = _lib.require().ti64_stencil_step(_lib.ptr(t), _lib.ptr(d), None, None, C.byref(tp), C.byref(a), _lib.stream_handle())
print("rc", rc, flush=True)
torch.cuda.synchronize()
print("done", shape, flush=True)
