"""Pins for the oracle's Level-2 fine filter (NEXT f1, PAPER.md:210-216;
SPEC.md:189-197, R24): deterministic exp, a double-precision brute force on the
tiny scene, the pinhole special case and the Level-1/Level-2 conservativeness
chain."""
import math

import numpy as np

import oracle as O
import workload as W
from helpers import tiny


def test_exp_det_close_to_exp():
    xs = np.linspace(-20.0, 10.0, 3001, dtype=np.float32)
    worst = max(abs(O.exp_det(float(x)) / math.exp(float(x)) - 1.0) for x in xs)
    assert worst < 4e-7, worst
    assert O.exp_det(0.0) == 1.0
    assert O.exp_det(math.log(2.0)) == 2.0


def _run(J=2, iters=5):
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 64), sc.bounds(), fill=sc.fill_fn, track_all=True)
    out = []
    for t in range(iters):
        planes = tr.batch_planes(t, J)
        o.activate(planes)
        percam = [set(o.percam(j).tolist()) for j in range(J)]
        cams = {int(k): [j for j in range(J) if int(k) in percam[j]] for k in o.list("A")}
        out.append((planes, o.list("A"), {int(k): o.fine_filter(int(k)) for k in o.list("A")},
                    cams))
    return cfg, sc, tr, o, out


def _bits(words, B):
    return np.unpackbits(words.view(np.uint8), bitorder="little")[:B].astype(bool)


def _double_visible(rows, planes, cams=None):
    """Per-row sphere test in double with the true exp (brute force), against
    the cameras `cams` (default: all)."""
    mu = rows[:, :3].astype(np.float64)
    ext = 3.0 * np.exp(rows[:, 52:55].astype(np.float64).max(1))
    P = planes.astype(np.float64) if cams is None else planes[list(cams)].astype(np.float64)
    if P.shape[0] == 0:
        z = np.zeros(rows.shape[0], bool)
        return z, z
    d = np.einsum("rk,jpk->rjp", mu, P[:, :, :3]) + P[None, :, :, 3]
    vis = ~(d < -ext[:, None, None]).any(2)
    band = (np.abs(d + ext[:, None, None]) <= 1e-4 * (1 + np.abs(mu).sum(1)[:, None, None] +
                                                      ext[:, None, None])).any(2)
    return vis.any(1), band.any(1)


def test_matches_double_brute_force_outside_rounding_band():
    cfg, sc, tr, o, out = _run()
    checked = 0
    for planes, A, masks, cams in out:
        for k in A.tolist():
            rows = sc.block_theta(k)[: sc.rows(k)]
            got = _bits(masks[k], sc.B)[: sc.rows(k)]
            ref, band = _double_visible(rows, planes, cams[k])
            bad = (got != ref) & ~band
            assert not bad.any(), (k, np.nonzero(bad)[0][:5])
            checked += rows.shape[0]
            assert not _bits(masks[k], sc.B)[sc.rows(k):].any()  # padding rows never active
    assert checked > 10_000


def test_centre_in_image_is_in_It_and_chain_is_conservative():
    """A Gaussian whose centre projects inside an image at near<=z<=far is in
    I_t; and the Level-1 cover is conservative: every row visible at Level 2
    (brute force over ALL blocks) belongs to a block of K."""
    cfg, sc, tr, o, out = _run(J=2, iters=3)
    cams_all = [tr.batch_cameras(t, 2) for t in range(3)]
    # K per batch from a bounds-only oracle for the chain check
    o2 = O.Oracle(O.make_config(sc.N, sc.B, 64), sc.bounds(), fill=None, track_all=False)
    for t, ((planes, A, masks, _), cams) in enumerate(zip(out, cams_all)):
        o2.activate(planes)
        K = set(o2.list("K").tolist())
        for k in range(sc.K):
            rows = sc.block_theta(k)[: sc.rows(k)]
            vis, band = _double_visible(rows, planes)
            if k not in K:
                assert not (vis & ~band).any(), f"block {k} has Level-2 visible rows but is culled"
            elif k in masks:
                bits = _bits(masks[k], sc.B)[: sc.rows(k)]
                for r in range(0, rows.shape[0], 97):
                    if any(W.camera_sees(c, rows[r, :3].astype(np.float64)) for c in cams):
                        assert bits[r], (k, r)
                # restricting camera j to its own K^(j) drops nothing (Level-1 is
                # conservative per camera): the all-camera double test agrees
                vis_all, band_all = _double_visible(rows, planes)
                assert not ((vis_all != bits) & ~band_all).any(), k


def test_outside_A_is_empty_and_far_behind_camera_is_culled():
    bounds = np.array([[0, 0, 5, 1], [0, 0, -5, 1]], np.float32)
    rows = np.zeros((8, 59), np.float32)
    rows[:4, 2] = 5.0       # block 0: in front
    rows[4:, 2] = -5.0      # block 1: behind
    rows[:, 52:55] = math.log(0.1)

    def fill(k):
        return rows[4 * k: 4 * k + 4]
    o = O.Oracle(O.make_config(8, 4, 2), bounds, fill=fill, track_all=True)
    cam = np.zeros((1, 6, 4), np.float32)
    cam[0] = [[1, 0, 0.5, 0], [-1, 0, 0.5, 0], [0, 1, 0.5, 0], [0, -1, 0.5, 0], [0, 0, 1, -0.1],
              [0, 0, -1, 100]]
    o.activate(cam)
    assert o.list("A").tolist() == [0]
    assert o.fine_filter(0)[0] == 0xF
    assert o.fine_filter(1)[0] == 0
