"""P2P beside M2L (grid.UnigridState.gravity_kernels): the side-stream P2P
into its own buffer leaves every step output bit-identical to the serial
order, and its buffer holds exactly the standalone P2P result."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402


def _state(level, overlap, precision="exact"):
    u = grid.UnigridState(level, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1),
                          precision=precision)
    u.overlap_p2p = overlap
    u.load(scenarios.config5_state(level))
    return u


@pytest.mark.parametrize("level,precision", [(3, "exact"), (4, "exact"), (3, "fma")])
def test_overlapped_steps_match_serial(level, precision):
    a, b = _state(level, True, precision), _state(level, False, precision)
    for _ in range(2):
        a.step()
        b.step()
    a.check_errors()
    b.check_errors()
    fa, fb = a.fetch(), b.fetch()
    for k in fb:
        assert np.array_equal(fa[k].view(np.uint64), fb[k].view(np.uint64)), k
    # the side buffer is the standalone P2P of the last gravity iteration's masses
    ref = torch.empty_like(a.grav)
    B.p2p(a.mass, a.mv, a.leaves, a.nleaves, a.dx, a.rad2, a.eps2, a.halo, ref, a.gv, precision=precision)
    assert torch.equal(a.p2p_result().view(torch.int64), ref.view(torch.int64))
