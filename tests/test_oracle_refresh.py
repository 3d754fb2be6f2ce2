"""Pins for the oracle's conservative bound refresh (NEXT f2, PAPER.md:192-194,
R25): once a step's refresh has entered the Level-1 test (two batches later)
every Gaussian of the block lies inside the refreshed sphere (checked in
double), radii only grow, untouched blocks keep their bounds, and the Level-1/Level-2 conservativeness chain survives training that
moves the centres."""
import ctypes as C

import numpy as np

import oracle as O
import workload as W
from helpers import lr_3dgs, tiny


class Synth(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_gaussians", C.c_uint64), ("block_size", C.c_uint32),
                ("p32", C.c_uint32)]


def _train(refresh, iters=12, lr_xyz=0.3, mask_p=None):
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 64, refresh_bounds=refresh), sc.bounds(),
                 fill=sc.fill_fn, track_all=True)
    lr = lr_3dgs()
    lr[0:3] = lr_xyz
    lr[52:55] = 0.05
    syn = Synth(42, sc.N, sc.B, 0)
    gfn = (C.cast(W.lib().wl_grad_cb, C.c_void_p).value, C.addressof(syn))
    msyn = Synth(43, sc.N, sc.B, 0)
    mfn = (C.cast(W.lib().wl_mask_cb, C.c_void_p).value, C.addressof(msyn)) if mask_p == 0 else None
    r_hist = [np.array([o.bound(k)[3] for k in range(sc.K)])]
    for t in range(iters):
        o.activate(tr.batch_planes(t, 2))
        o.step_adam(lr, grad=gfn, mask=mfn)
        r_hist.append(np.array([o.bound(k)[3] for k in range(sc.K)]))
    # R25: a step's refresh enters the Level-1 test two batches later; two empty
    # batches apply the last two steps' refreshes
    for _ in range(2):
        o.activate(np.zeros((0, 6, 4), np.float32))
        r_hist.append(np.array([o.bound(k)[3] for k in range(sc.K)]))
    return sc, tr, o, r_hist


def _contained(sc, o, k):
    th, _, _ = o.read_block(k)
    rows = th[: sc.rows(k)].astype(np.float64)
    c = o.bound(k).astype(np.float64)
    need = np.linalg.norm(rows[:, :3] - c[:3], axis=1) + 3 * np.exp(rows[:, 52:55].max(1))
    return (need <= c[3]).all(), need.max(), c[3]


def test_refreshed_bounds_contain_every_gaussian_and_only_grow():
    sc, tr, o, hist = _train(1)
    grew = 0
    for k in range(sc.K):
        ok, need, r = _contained(sc, o, k)
        assert ok, (k, need, r)
    for a, b in zip(hist, hist[1:]):
        assert (b >= a).all()
        grew += int((b > a).sum())
    assert grew > 0  # training did move centres beyond the initial spheres
    assert o.stats()["total_updates"] > 0


def test_off_or_untouched_keeps_input_bounds():
    sc, tr, o, hist = _train(0)
    assert all((h == hist[0]).all() for h in hist)
    sc, tr, o, hist = _train(1, mask_p=0)   # empty I_t: nothing updated, nothing refreshed
    assert all((h == hist[0]).all() for h in hist)


def _chain_violations(refresh, lr_xyz):
    """Rows that are Level-2 visible (double brute force over all blocks,
    current theta) but whose block is missing from the next K."""
    sc, tr, o, _ = _train(refresh, iters=10, lr_xyz=lr_xyz)
    probe = O.Oracle(O.make_config(sc.N, sc.B, 64), np.stack([o.bound(k) for k in range(sc.K)]),
                     fill=None, track_all=False)
    viol = 0
    for t in range(10, 16):
        planes = tr.batch_planes(t, 1)
        probe.activate(planes)
        K = set(probe.list("K").tolist())
        P = planes.astype(np.float64)
        for k in range(sc.K):
            if k in K:
                continue
            th, _, _ = o.read_block(k)
            rows = th[: sc.rows(k)].astype(np.float64)
            ext = 3 * np.exp(rows[:, 52:55].max(1))
            d = np.einsum("rk,jpk->rjp", rows[:, :3], P[:, :, :3]) + P[None, :, :, 3]
            viol += int((~(d < -ext[:, None, None] - 1e-4).any(2)).any(1).sum())
    return viol


def test_chain_survives_moving_centres():
    """Training that moves centres by ~1 m/step breaks the chain with fixed
    bounds (R3) and keeps it with the refresh (R25)."""
    assert _chain_violations(0, 1.0) > 0
    assert _chain_violations(1, 1.0) == 0


def test_refresh_requires_tracking_every_block():
    cfg, sc, tr = tiny()
    try:
        O.Oracle(O.make_config(sc.N, sc.B, 8, refresh_bounds=1), sc.bounds(), fill=None,
                 track_all=False)
    except O.OracleError as e:
        assert e.code == O.EINVAL
    else:
        raise AssertionError("expected EINVAL")
