"""Tolerances of the parity gates.

North star (BASELINE.json): fp32 outputs within 1e-5 relative / 1e-6 absolute
of the CPU reference on the same inputs; binary occupancy and voxel boxes
bit-exact.  The reference's own forward gate is stricter for values near 1:
max |delta| < 1e-6 absolute against the f64 all-pairs oracle
(/root/reference/pkg/tests/test_voxelizer.py:146).
"""

import numpy as np

REL = 1e-5
ABS = 1e-6


def violations(got, want, rel=REL, abs_=ABS):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    bad = np.abs(got - want) > abs_ + rel * np.abs(want)
    return int(bad.sum()), float(np.abs(got - want).max(initial=0.0))


def assert_close(got, want, rel=REL, abs_=ABS, what=""):
    n, worst = violations(got, want, rel, abs_)
    assert n == 0, f"{what}: {n} violations of |d| <= {abs_} + {rel}|ref|, max |d| {worst:.3e}"


def to_numpy(x):
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)
