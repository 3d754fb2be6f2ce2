"""Pins for the oracle's NEXT f4 clustered-TSP view ordering (PAPER.md:266,
709-712 "clustered traveling-salesperson (TSP) ordering over camera poses";
SPEC.md:565-568 order_views; reading R29 of DESIGN.md §3).  Each pin is a
closed-form order or a structural property checked with plain numpy."""
import numpy as np
import pytest

import oracle as O
import workload as W


def _check_perm(p, M):
    assert sorted(p.tolist()) == list(range(M))


@pytest.mark.parametrize("M,k", [(1, 1), (2, 2), (4, 2), (5, 3), (9, 3), (10, 4), (26695, 164)])
def test_cluster_count_is_ceil_sqrt(M, k):
    rng = np.random.default_rng(M)
    f = rng.standard_normal((M, 3)) if M < 1000 else np.c_[np.arange(M, dtype=float), np.zeros((M, 2))]
    p, cl, kk, it = O.order_views(f)
    _check_perm(p, M)
    assert kk == k and cl.max() < k


def test_identical_poses_keep_index_order():
    """All views at one pose: every distance ties, every tie goes to the lowest index."""
    f = np.ones((50, 6))
    p, cl, k, it = O.order_views(f)
    assert p.tolist() == list(range(50))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_evenly_spaced_line_is_sorted(seed):
    """Views on a line at x = 0..M-1, presented shuffled: k-means splits the
    line into segments, the tours walk them left to right -> pi sorts by x."""
    M = 200
    x = np.random.default_rng(seed).permutation(M).astype(np.float64)
    f = np.c_[x, np.zeros(M), np.zeros(M)]
    p, cl, k, it = O.order_views(f)
    assert np.array_equal(x[p], np.arange(M, dtype=np.float64))


def test_separated_blobs_are_contiguous_and_clusters_are_runs():
    """Far-apart groups of views: each group is presented contiguously, and
    every k-means cluster forms one contiguous run of pi."""
    rng = np.random.default_rng(7)
    centres = np.array([[0, 0, 0], [1000, 0, 0], [0, 1000, 0], [1000, 1000, 500]], float)
    g = rng.integers(0, 4, 400)
    f = centres[g] + rng.standard_normal((400, 3)) * 10
    p, cl, k, it = O.order_views(f)
    _check_perm(p, 400)
    runs = np.flatnonzero(np.diff(g[p])) + 1
    assert len(runs) == 3  # four groups -> three boundaries
    cr = np.flatnonzero(np.diff(cl[p])) + 1
    assert len(cr) == len(set(cl.tolist())) - 1


def test_lloyd_fixed_point():
    """When Lloyd stops early, each view's own cluster mean is its nearest
    mean (recomputed here with numpy; tolerance covers summation order)."""
    rng = np.random.default_rng(3)
    f = rng.standard_normal((500, 4)) * np.array([100, 50, 20, 1])
    p, cl, k, it = O.order_views(f)
    assert it < 100
    means = np.stack([f[cl == j].mean(0) if (cl == j).any() else np.full(4, np.inf)
                      for j in range(k)])
    d = ((f[:, None, :] - means[None]) ** 2).sum(-1)
    own = d[np.arange(500), cl]
    assert np.all(own <= d.min(1) * (1 + 1e-12) + 1e-9)


def test_first_view_is_lexicographic_minimum():
    rng = np.random.default_rng(4)
    f = rng.integers(0, 5, (300, 3)).astype(float)
    p, cl, k, it = O.order_views(f)
    first = min(range(300), key=lambda i: (tuple(f[i]), i))
    assert p[0] == first


def test_trajectory_order_restores_locality():
    """the shuffled aerial trajectory (300m_random views)
    reordered by the clustered TSP is locally coherent again: the mean pose
    step drops by > 20x and is within 3x of the generator's path order."""
    wl = W.CONFIGS["300m_random"]
    sc = wl.scene()
    tr = wl.trajectory(sc)
    f = tr.features(150.0)
    p, cl, k, it = O.order_views(f)
    step = lambda q: np.linalg.norm(np.diff(f[q], axis=0), axis=1).mean()
    smooth = W.CONFIGS["300m"].trajectory(sc).features(150.0)
    s_path = np.linalg.norm(np.diff(smooth, axis=0), axis=1).mean()
    assert step(p) * 20 < step(np.arange(len(p)))
    assert step(p) < 3 * s_path


def test_errors():
    with pytest.raises(O.OracleError):
        O.order_views(np.zeros((0, 3)))
    with pytest.raises(O.OracleError):
        O.order_views(np.zeros((4, 9)))
    f = np.zeros((4, 3))
    f[2, 1] = np.nan
    with pytest.raises(O.OracleError):
        O.order_views(f)
