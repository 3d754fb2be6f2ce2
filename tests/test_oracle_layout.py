"""Pins for the oracle's Morton sort + blocking (NEXT f2b, PAPER.md:189-190,
375-376, reading R26): SPEC's worked examples, the
conservativeness invariant in double, and the locality property that motivates
the sort (Morton blocks beat a random permutation on
consecutive-view overlap)."""
import math

import numpy as np

import oracle as O
import workload as W


def test_morton_examples_spec():
    # SPEC.md:105-107
    assert O.morton3(0, 0, 0) == 0
    assert O.morton3(1, 1, 1) == 7
    assert (O.morton3(2, 0, 0), O.morton3(0, 2, 0), O.morton3(0, 0, 2)) == (8, 16, 32)
    assert O.morton3(2**21 - 1, 2**21 - 1, 2**21 - 1) == 2**63 - 1


def test_build_layout_examples_spec():
    # 1 primitive, (near) zero extent -> bound = (its centre, ~0)
    p, b = O.build_layout(np.array([[1, 2, 3, -80]], np.float32), 4)
    assert p.tolist() == [0] and b[0, :3].tolist() == [1, 2, 3] and 0 <= b[0, 3] < 1e-30
    # 2 coincident primitives, extents ~0 and 1 -> radius 1
    s1 = math.log(1 / 3)
    p, b = O.build_layout(np.array([[5, 5, 5, -80], [5, 5, 5, s1]], np.float32), 4)
    assert b[0, :3].tolist() == [5, 5, 5] and abs(b[0, 3] - 1.0) < 1e-6 and b[0, 3] >= 1.0 - 1e-7
    # 8 unit-cube corners, B = 8 -> centroid (0.5,0.5,0.5), radius sqrt(3)/2
    corners = np.array([[x, y, z, -80] for x in (0, 1) for y in (0, 1) for z in (0, 1)],
                       np.float32)
    p, b = O.build_layout(corners, 8)
    assert sorted(p.tolist()) == list(range(8))
    assert b[0, :3].tolist() == [0.5, 0.5, 0.5]
    assert math.sqrt(3) / 2 <= b[0, 3] <= math.sqrt(3) / 2 * (1 + 1e-6)


def _cs_of(rows):
    return np.concatenate([rows[:, :3], rows[:, 52:55].max(1, keepdims=True)], 1)


def _unsorted_scene(n=60_000, B=512):
    sc = W.Scene(n, B, side=120.0, lot=20.0, footprint=12.0, hmin=2.0, hmax=12.0, layout=1)
    rows = np.concatenate([sc.block_theta(k)[: sc.rows(k)] for k in range(sc.K)])
    return sc, rows


def test_conservative_and_permutation():
    sc, rows = _unsorted_scene()
    cs = _cs_of(rows)
    perm, bounds = O.build_layout(cs, sc.B)
    assert np.array_equal(np.sort(perm), np.arange(len(rows), dtype=np.uint64))
    pos = np.arange(len(rows)) // sc.B
    c = bounds[pos].astype(np.float64)
    mu = cs[perm.astype(np.int64), :3].astype(np.float64)
    ext = 3 * np.exp(cs[perm.astype(np.int64), 3].astype(np.float64))
    need = np.linalg.norm(mu - c[:, :3], axis=1) + ext
    assert (need <= c[:, 3] * (1 + 1e-6)).all()


def test_morton_blocks_have_locality():
    """After the Morton blocking each batch's Level-1 set is a fraction of the
    table and consecutive batches share blocks; with the unsorted layout every
    block spans the city and every batch selects the whole table."""
    sc, rows = _unsorted_scene()
    cs = _cs_of(rows)
    perm, bounds = O.build_layout(cs, sc.B)
    tr = W.Trajectory(sc, "aerial", altitude=40.0, spacing=4.0, strip=40.0, fovx_deg=60.0,
                      znear=1.0, zfar=60.0)

    def run(bnd):
        o = O.Oracle(O.make_config(sc.N, sc.B, 10_000), bnd, fill=None, track_all=False)
        Ks = []
        for t in range(12):
            o.activate(tr.batch_planes(t, 2))
            Ks.append(set(o.list("K").tolist()))
        jac = np.mean([len(a & b) / max(1, len(a | b)) for a, b in zip(Ks, Ks[1:])])
        return np.mean([len(k) for k in Ks]), jac

    k_sorted, jac_sorted = run(bounds)
    k_raw, jac_raw = run(sc.bounds())
    assert k_raw == sc.K                       # unsorted: every block spans the city
    assert k_sorted < 0.5 * sc.K
    assert jac_sorted > 0.3
