"""Pins for the oracle's Level-1 block cull (Eq. Kt_def).

Each test checks the oracle against something other than itself: pinhole
projection of every Gaussian centre (brute force), a double-precision plane
test, hand-built boundary cases, and the set examples of SPEC.md:186-188.
"""
import numpy as np
import pytest

import oracle as O
import workload as W
from helpers import tiny


def _oracle(n, B, bounds, C=10**6, **kw):
    return O.Oracle(O.make_config(n, B, C, **kw), bounds, fill=None, track_all=False)


def test_brute_force_projection_tiny():
    """Every Gaussian whose centre projects inside the image with near<=z<=far
    has its owner block in K^{(j)} (Level 1 is conservative)."""
    cfg, sc, tr = tiny()
    theta = sc.table()
    b = sc.bounds()
    o = _oracle(sc.N, sc.B, b)
    for batch in range(8):
        cams = tr.batch_cameras(batch, cfg.J)
        planes = np.stack([W.camera_planes(c) for c in cams])
        assert o.activate(planes) == O.OK
        for j, cam in enumerate(cams):
            vis = set(o.percam(j).tolist())
            pos = np.array(cam.pos)
            R = np.stack([cam.right, cam.down, cam.fwd])
            P = theta[: sc.N, :3].astype(np.float64) - pos
            pc = P @ R.T
            z = pc[:, 2]
            with np.errstate(divide="ignore", invalid="ignore"):
                u = cam.fx * pc[:, 0] / z + cam.cx
                v = cam.fy * pc[:, 1] / z + cam.cy
            seen = (z >= cam.znear) & (z <= cam.zfar) & (u >= 0) & (u <= cam.width) & \
                   (v >= 0) & (v <= cam.height)
            owners = set((np.nonzero(seen)[0] // sc.B).tolist())
            assert owners, "camera sees nothing: vacuous test"
            assert owners <= vis, f"batch {batch} cam {j}: dropped {sorted(owners - vis)}"


def test_matches_double_plane_test_outside_rounding_band():
    """Against the plane test evaluated in double: any disagreement lies in the
    fp32 rounding band |d + r| <= 1e-5 * scale (R2)."""
    cfg = W.CONFIGS["100m"]
    sc = W.Scene(2_000_000, 4096, side=600.0)
    b = sc.bounds()
    tr = W.Trajectory(sc, "street", **dict(cfg.traj_kw))
    o = _oracle(sc.N, sc.B, b)
    n_in_band = 0
    for batch in (0, 37, 101):
        planes = tr.batch_planes(batch, 16)
        o.activate(planes)
        for j in range(16):
            vis = np.zeros(sc.K, bool)
            vis[o.percam(j)] = True
            pl = planes[j].astype(np.float64)
            d = b[:, :3].astype(np.float64) @ pl[:, :3].T + pl[:, 3]   # K x 6
            r = b[:, 3:4].astype(np.float64)
            ref = ~np.any(d < -r, axis=1)
            band = np.any(np.abs(d + r) <= 1e-5 * (1 + np.abs(b[:, :3]).max()), axis=1)
            bad = (vis != ref) & ~band
            assert not bad.any(), np.nonzero(bad)
            n_in_band += int(((vis != ref) & band).sum())
    assert n_in_band < 5


def _box_planes(half=1.0):
    """axis-aligned cube [-half,half]^3 as 6 inward unit planes"""
    P = []
    for ax in range(3):
        for s in (1.0, -1.0):
            n = [0.0, 0.0, 0.0]
            n[ax] = s
            P.append(n + [half])
    return np.array(P, np.float32)


def test_boundary_is_kept_and_strict_cull():
    """d = -r is kept, d < -r is culled ("cull ... d < -r_k")."""
    pl = _box_planes(1.0)[None]
    bounds = np.array([
        [0.0, 0.0, 0.0, 0.0],     # centre inside -> visible
        [-2.0, 0.0, 0.0, 1.0],    # x=-2, plane x>=-1: d = -1 = -r -> kept
        [-2.0, 0.0, 0.0, 0.5],    # d = -1 < -0.5 -> culled
        [3.0, 0.0, 0.0, 2.0],     # d = -2 = -r on plane -x+1>=0 -> kept
        [3.0, 0.0, 0.0, np.nextafter(np.float32(2.0), np.float32(0))],  # just culled
        [0.0, 0.0, 50.0, 10.0],   # far outside -> culled
    ], np.float32)
    o = _oracle(6 * 4, 4, bounds, C=6)
    o.activate(pl)
    assert o.percam(0).tolist() == [0, 1, 3]


def test_union_examples_spec():
    """empty batch -> empty; all-seeing camera -> all;
    per-camera {0,1} and {1,2} -> union {0,1,2} (Eq. Kt_def)."""
    bounds = np.array([[0, 0, 0, 0.1], [1, 0, 0, 0.1], [2, 0, 0, 0.1]], np.float32)
    o = _oracle(12, 4, bounds, C=3)
    assert o.activate(np.zeros((0, 6, 4), np.float32)) == O.OK
    assert o.list("K").tolist() == []
    o.activate(_box_planes(10.0)[None])
    assert o.list("K").tolist() == [0, 1, 2]
    c1 = _box_planes(0.5).copy()
    c1[0, 3] = 0.5   # x >= -0.5
    c1[1, 3] = 1.5   # x <= 1.5   -> {0,1}
    c2 = _box_planes(0.5).copy()
    c2[0, 3] = -0.5  # x >= 0.5
    c2[1, 3] = 2.5   # x <= 2.5   -> {1,2}
    o.activate(np.stack([c1, c2]))
    assert o.percam(0).tolist() == [0, 1]
    assert o.percam(1).tolist() == [1, 2]
    assert o.list("K").tolist() == [0, 1, 2]


def test_overflowing_distance_and_nonfinite_inputs():
    """R2 edge cases. With finite planes and bounds (non-finite ones are
    rejected, SPEC.md EINVAL rule) the fmaf chain of R2 can overflow to +-inf but
    never yield NaN (inf - inf needs an infinite operand, and fma(a, b, +-inf) with
    finite a*b stays +-inf). So: d = +inf never culls, d = -inf always culls
    (-inf < -r), and the NaN branch of R2 is unreachable by construction."""
    big = np.float32(3.0e38)
    bounds = np.array([[big, 0, 0, 1]], np.float32)
    o = _oracle(4, 4, bounds, C=1)
    # x-plane n=(1,0,0), d0=+3e38: d = fl(3e38 + 3e38) = +inf -> kept; the other
    # five planes are far away and pass
    keep = _box_planes(3.4e38)[None].copy()
    keep[0, 0] = [1, 0, 0, big]
    assert o.activate(keep) == O.OK
    assert o.list("K").tolist() == [0]
    # n=(-1,0,0), d0=-3e38: d = fl(-3e38 - 3e38) = -inf < -1 -> culled
    cull = _box_planes(3.4e38)[None].copy()
    cull[0, 1] = [-1, 0, 0, -big]
    assert o.activate(cull) == O.OK
    assert o.list("K").tolist() == []
    # non-finite planes and bounds are refused, state unchanged
    for bad in (np.inf, -np.inf, np.nan):
        pl = _box_planes(1.0)[None].copy()
        pl[0, 2, 1] = bad
        assert o.activate(pl) == O.EINVAL
        with pytest.raises(O.OracleError):
            _oracle(4, 4, np.array([[0, bad, 0, 1]], np.float32), C=1)
    assert o.list("K").tolist() == []


def test_shards_union_equals_single_shard():
    """R17: block k is owned by rank k % G; per-block tests are independent, so
    the union of shard K sets is the unsharded K (and shards are disjoint)."""
    cfg, sc, tr = tiny()
    b = sc.bounds()
    full = _oracle(sc.N, sc.B, b)
    shards = [O.Oracle(O.make_config(sc.N, sc.B, 10**6, world_size=3, rank=g), b,
                       fill=None, track_all=False) for g in range(3)]
    for batch in range(4):
        pl = tr.batch_planes(batch, cfg.J)
        full.activate(pl)
        parts = []
        for g, o in enumerate(shards):
            o.activate(pl)
            k = o.list("K")
            assert np.all(k % 3 == g)
            parts.append(k)
        assert sorted(np.concatenate(parts).tolist()) == full.list("K").tolist()


def test_frustum_planes_inside_means_projects_inside():
    """Plane extraction (R1): random points, plane test (double) == pinhole test."""
    rng = np.random.default_rng(0)
    cam = W.look((1.0, 2.0, 3.0), (0.3, 0.9, -0.2), (0, 0, 1), 70.0, 640, 480, 0.5, 50.0)
    pl = W.camera_planes(cam).astype(np.float64)
    pts = rng.uniform(-60, 60, size=(4000, 3))
    d = pts @ pl[:, :3].T + pl[:, 3]
    inside_planes = np.all(d >= 1e-4, axis=1)
    outside_planes = np.any(d <= -1e-4, axis=1)
    for p, ip, op in zip(pts, inside_planes, outside_planes):
        s = W.camera_sees(cam, p)
        if ip:
            assert s
        if op:
            assert not s
    assert inside_planes.sum() > 20
