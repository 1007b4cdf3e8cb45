"""B200-native (sm_100a) FP64 subgrid kernels: a drop-in for the reference
``simdgrid.kernels`` entry points (M2L multipole, P2P monopole, hydro
reconstruct/flux/update, max wavespeed) plus a device-resident batched path.

Submodules are imported lazily so that host-only pieces (scenarios, octree)
load without a GPU; every compute entry point goes through the CUDA C-ABI
library ``libsg.so`` and fails loudly when it is missing.
"""

__version__ = "0.1.0"
