"""NEXT f4 on the GPU: tgs_order_views (clustered-TSP view order, R29) against
the oracle, bit-exact on the permutation and the k-means clusters."""
import numpy as np
import pytest

import oracle as O
import workload as W

pytestmark = pytest.mark.gpu


def _both(f):
    from paper_2605_20150_b200 import tidegs as T
    gp, gc, gk, git, ms = T.order_views(f)
    op, oc, ok, oit = O.order_views(f)
    assert (gk, git) == (ok, oit)
    np.testing.assert_array_equal(gc, oc)
    np.testing.assert_array_equal(gp, op)
    return gp, ms


@pytest.mark.parametrize("M,D,seed", [(1, 3, 0), (2, 3, 0), (7, 2, 1), (300, 3, 2),
                                      (1000, 6, 3), (4097, 8, 4)])
def test_random_poses(M, D, seed):
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((M, D)) * rng.uniform(1, 1000, D)
    _both(f)


def test_degenerate_poses():
    """duplicates and a coarse integer lattice: every tie path"""
    _both(np.ones((64, 6)))
    rng = np.random.default_rng(5)
    _both(rng.integers(0, 4, (500, 3)).astype(np.float64))


@pytest.mark.parametrize("name", ["300m_random", "100m"])
def test_workload_trajectories(name):
    """the bench workloads' own views (26,695 aerial views shuffled; street)"""
    wl = W.CONFIGS[name]
    sc = wl.scene()
    tr = wl.trajectory(sc)
    f = tr.features(150.0 if wl.traj == "aerial" else 20.0)
    p, ms = _both(f)
    assert ms > 0
