"""NEXT f2b on the GPU: tgs_build_layout (Morton codes, stable radix sort,
block bounds) bit-exact with the oracle's step-by-step build (R26)."""
import numpy as np
import pytest

import oracle as O
import workload as W

pytestmark = pytest.mark.gpu


def _cs_of(rows):
    return np.concatenate([rows[:, :3], rows[:, 52:55].max(1, keepdims=True)], 1)


def _check(cs, B):
    from paper_2605_20150_b200 import tidegs as T
    p_gpu, b_gpu, ms = T.build_layout(cs, B)
    p_ref, b_ref = O.build_layout(cs, B)
    np.testing.assert_array_equal(p_gpu, p_ref)
    np.testing.assert_array_equal(b_gpu.view(np.uint32), b_ref.view(np.uint32))
    return ms


def test_unsorted_city_scene():
    sc = W.Scene(60_000, 512, side=120.0, lot=20.0, footprint=12.0, hmin=2.0, hmax=12.0,
                 layout=1)
    rows = np.concatenate([sc.block_theta(k)[: sc.rows(k)] for k in range(sc.K)])
    _check(_cs_of(rows), 512)


@pytest.mark.parametrize("n,B", [(1, 4), (7, 4), (4096, 4096), (4097, 100), (1_000_003, 4096)])
def test_random_with_ties(n, B):
    """Many exactly coincident centres (ties must keep index order), a ragged
    last block, sizes around the 4096-item radix tile."""
    rng = np.random.default_rng(n)
    cs = np.empty((n, 4), np.float32)
    cs[:, :3] = rng.integers(0, 50, (n, 3)).astype(np.float32) * 0.25  # heavy duplication
    cs[:, 3] = rng.uniform(-6, 0, n)
    _check(cs, B)


def test_degenerate_axis_and_extremes():
    rng = np.random.default_rng(1)
    n = 20_000
    cs = np.zeros((n, 4), np.float32)
    cs[:, 0] = rng.uniform(-1e6, 1e6, n)      # z = y = 0: zero-extent axes (inv = 0)
    cs[:, 3] = rng.uniform(-80, 5, n)
    _check(cs, 64)


def test_unsorted_scene_built_then_trained():
    """The whole pipeline on an unsorted scene: GPU Morton build (f2b) -> table
    re-blocked by its permutation -> working-set steps, bit-exact with the
    oracle driven by its own build of the same scene."""
    from gpu_harness import Pair
    from paper_2605_20150_b200 import tidegs as T
    sc = W.Scene(100_000, 1568, side=80.0, lot=20.0, footprint=12.0, hmin=2.0, hmax=12.0,
                 layout=1)
    cs = sc.table_cs()
    p_gpu, b_gpu, _ = T.build_layout(cs, sc.B)
    p_ref, b_ref = O.build_layout(cs, sc.B)
    np.testing.assert_array_equal(p_gpu, p_ref)
    tr = W.Trajectory(sc, "orbit", n_views=16, altitude=40.0, fovx_deg=25.0, znear=0.05,
                      zfar=1.8, radius_scale=1.0)
    pr = Pair(sc, capacity=24, bounds=b_gpu, fill=sc.perm_fill(p_gpu))
    ks = []
    for t in range(16):
        act = pr.activate(tr.batch_planes(t, 2))
        pr.t = t
        pr.compare_plan(2)
        ks.append(act.n_visible)
        assert pr.step(act, t) == O.OK
    assert max(ks) < sc.K  # re-blocked bounds cull again
    pr.compare_stats()
    assert pr.compare_blocks(range(sc.K)) == 0
    pr.close()
