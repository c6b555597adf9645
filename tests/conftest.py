"""Shared test configuration.

`-m gpu` tests need a B200 (they call the sm_100a library through the C ABI);
`-m "not gpu"` tests run anywhere and cover the oracle, the host logic and the
library's exported symbols.  The oracle (oracle/) is test infrastructure and
is imported only here and in the tests.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# Parity bars from BASELINE.json north_star: loss within 1e-5 relative,
# gradients within 1e-4 (absolute) in fp32, identical iteration counts.
LOSS_RTOL = 1e-5
GRAD_ATOL = 1e-4


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built library")
    config.addinivalue_line("markers", "slow: takes more than ~10 s")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_cost(g: dict):
    """Regenerate the cost a fixture's reference run saw (float64, fp32-exact)."""
    from oracle import sinkhorn_oracle as orc

    kind = str(g["cost_kind"])
    p = [int(v) for v in g["cost_params"]]
    if kind == "stored":
        return g["cost"].astype(np.float64)
    if kind == "grid2d_stored":
        return orc.fp32_exact(orc.grid2d_cost(p[0], p[1]))
    if kind == "grid2d":
        return orc.grid2d_cost(p[0], p[1])
    if kind == "index_grid_stored":
        return orc.fp32_exact(orc.index_grid_cost(p[0], power=p[1]))
    if kind == "per_sample_seeded":
        B = g["mu"].shape[0]
        return np.stack([orc.per_sample_cost(p[0], b, p[1], p[2]) for b in range(B)]).astype(np.float64)
    raise ValueError(kind)


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
