"""Where the per-call time of the drop-in path goes (wall clock, median):
Python wrapper pieces vs the native sg_dropin_* call itself."""
import ctypes
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_06439_b200 import _lib, octree  # noqa: E402
from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import kernels as K  # noqa: E402

tree = octree.build_unigrid(1)
leaf = tree.leaves[0]
for n in ("rho", "E"):
    leaf.fields[n][...] = 1.0
for n in ("sx", "sy", "sz"):
    leaf.fields[n][...] = 0.0
h = K.HydroConfig()
L = _lib.load()
U = K._stack_hydro(leaf)
out = ctypes.c_double()
st = B._stream()


def wall(fn, n=200):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e6, 2)


ptr = U.__array_interface__["data"][0]
res = {
    "native_ws_call": wall(lambda: L.sg_dropin_max_wavespeed(ptr, 1.4, 1e-12, ctypes.byref(out), st)),
    "lib_call_wrapper": wall(lambda: _lib.call("sg_dropin_max_wavespeed", ptr, 1.4, 1e-12, ctypes.byref(out), st)),
    "np_stack": wall(lambda: K._stack_hydro(leaf)),
    "current_stream": wall(lambda: torch.cuda.current_stream().cuda_stream),
    "require_device": wall(B.require_device),
    "full_max_wavespeed": wall(lambda: K.max_wavespeed(leaf, h)),
    "stream_sync_empty": wall(lambda: torch.cuda.current_stream().synchronize()),
    "torch_empty_Q": wall(lambda: torch.empty((5, 26, 10, 10, 10), dtype=torch.float64, device="cuda")),
}
print(json.dumps(res))

# flux / reconstruct pieces
q = K.reconstruct(leaf, h)
dQ = q.device_values()
F = torch.empty(3 * 5 * 576, dtype=torch.float64, device="cuda")
sm, er = ctypes.c_double(), ctypes.c_uint32()
res2 = {
    "native_flux_call": wall(lambda: L.sg_dropin_flux(dQ.data_ptr(), 1.4, F.data_ptr(), F.data_ptr() + 8 * 2880,
                                                      F.data_ptr() + 16 * 2880, ctypes.byref(sm), ctypes.byref(er),
                                                      st)),
    "full_flux": wall(lambda: K.flux(leaf, q, h)),
    "torch_empty_F": wall(lambda: torch.empty(3 * 5 * 576, dtype=torch.float64, device="cuda")),
    "native_reconstruct_call": wall(lambda: L.sg_dropin_reconstruct(ptr, 1e-12, dQ.data_ptr(), st)),
    "full_reconstruct": wall(lambda: K.reconstruct(leaf, h)),
}
print(json.dumps(res2))
