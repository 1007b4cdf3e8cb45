"""The ctypes stub INTEGRATION.md §2 shows a reference maintainer (the
reference-side binding of the sg_dropin_* C ABI) runs as written and is
bit-identical to the oracle on config-1 inputs."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2210_06439_b200 import kernels as K
from paper_2210_06439_b200 import scenarios

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent


def _stub() -> dict:
    text = (REPO / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2."):text.index("## 3.")]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    code = code.replace("/path/to/paper_2210_06439_b200/libsg.so", str(REPO / "paper_2210_06439_b200" / "libsg.so"))
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    return ns


def test_integration_stub_matches_oracle():
    import torch
    torch.cuda.init()
    ns = _stub()
    dx = 1.0 / 64
    cube = scenarios.config1_cube(0)
    for order in (0, 1):
        rad2, eps2 = K.gravity_params(dx, K.GravityConfig(theta=0.34, eps=0.5, expansion_order=order))
        outs = [np.full((8, 8, 8), np.nan) for _ in range(4)]
        ns["multipole_kernel_impl"](cube, None, None, None, None, dx, rad2, eps2, order, 4, 0, 512, *outs)
        want = O.multipole(cube, dx, 0.34, 0.5, order)
        assert np.array_equal(np.stack(outs).view(np.uint64), want.view(np.uint64)), order
    sub = np.ascontiguousarray(cube[6:18, 6:18, 6:18])
    rad2, eps2 = K.gravity_params(dx, K.GravityConfig(theta=0.34, eps=0.5))
    outs = [np.full((8, 8, 8), np.nan) for _ in range(4)]
    ns["monopole_kernel_impl"](sub, dx, rad2, eps2, 2, 4, *outs)
    want = O.monopole(sub, dx, 0.34, 0.5)
    assert np.array_equal(np.stack(outs).view(np.uint64), want.view(np.uint64))
    rng = np.random.default_rng(3)
    U = np.stack([1.0 + rng.random((12, 12, 12)), 0.1 * rng.standard_normal((12, 12, 12)),
                  0.1 * rng.standard_normal((12, 12, 12)), 0.1 * rng.standard_normal((12, 12, 12)),
                  2.5 + rng.random((12, 12, 12))])
    got = ns["max_wavespeed_kernel"](U, 1.4, 1e-12)
    assert got == O.max_wavespeed(U, 1.4, 1e-12)
