"""CUDA path vs CPU oracle, element by element, on the same seeded inputs
(north star: bit-exact indexing, Adam within 1e-6 relative)."""
import numpy as np
import pytest

import oracle as O
import workload as W
from helpers import tiny

pytestmark = pytest.mark.gpu


def _pair(sc, **kw):
    from gpu_harness import Pair
    return Pair(sc, **kw)


def _drive(pr, tr, J, iters, *, check_blocks_every=0, adam=True):
    worst = 0
    for t in range(iters):
        act = pr.activate(tr.batch_planes(t, J))
        pr.t = t
        pr.compare_plan(J)
        pr.compare_evicted_dirty()
        assert act.n_stage_in == pr.orc.list("S+").size
        assert act.n_active_blocks == pr.orc.list("A").size
        if adam:
            rc = pr.step(act, t)
            assert rc == O.OK
        if check_blocks_every and t % check_blocks_every == 0:
            worst = max(worst, pr.compare_blocks(pr.orc.list("R")))
    pr.compare_stats()
    return worst


@pytest.mark.parametrize("moments", [O.PERSIST, O.COLD_RESTART])
@pytest.mark.parametrize("lam,quota", [(0.7, (1, 2)), (0.0, (1, 2)), (1.0, (0, 1)),
                                       (0.5, (1, 2))])
def test_tiny_trajectory_parity(moments, lam, quota):
    """configs[0]: 100k Gaussians / 64 blocks, 16-pose orbit, C=24 < K (forces
    eviction, quota and re-admission): every list, slot map, dirty set and
    counter bit-exact; theta/m/v of every block after flush within 1e-6."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, lam=lam, quota=quota, moments=moments)
    worst = _drive(pr, tr, cfg.J, 40, check_blocks_every=7)
    pr.gpu.flush()
    pr.orc.flush()
    pr.compare_stats()
    worst = max(worst, pr.compare_blocks(range(sc.K)))
    assert worst == 0, f"max ULP {worst} (prescribed op order should give 0)"
    pr.close()


@pytest.mark.parametrize("xfer", [0, 1])
@pytest.mark.parametrize("staging", [1, 64])
@pytest.mark.parametrize("moments", [O.PERSIST, O.COLD_RESTART])
def test_writeback_paths(staging, moments, xfer):
    """Write-back through the staging ring (k_pack, then the transfer: k_xfer, or
    copy-engine runs issued by the I/O thread with xfer = 1; re-admission from
    the ring by the gather / k_commit) and straight from the slots (ring too
    small): same lists, bytes and contents as the oracle."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, moments=moments, staging_blocks=staging, xfer=xfer)
    worst = _drive(pr, tr, cfg.J, 48, check_blocks_every=5)
    pr.gpu.flush()
    pr.orc.flush()
    pr.compare_stats()
    worst = max(worst, pr.compare_blocks(range(sc.K)))
    assert worst == 0
    pr.close()


@pytest.mark.parametrize("xfer", [0, 1])
def test_readmission_right_after_writeback(xfer):
    """Alternate two disjoint views with C = one view: every block is evicted
    dirty and re-admitted the next batch, so the gather must take the record
    from the staging ring (its host write-back may still be in flight)."""
    cfg, sc, tr = tiny()
    a, b = tr.batch_planes(0, 1), tr.batch_planes(8, 1)
    pr = _pair(sc, capacity=14, staging_blocks=64, lam=1.0, quota=(0, 1), xfer=xfer)
    for t in range(16):
        act = pr.activate(a if t % 2 == 0 else b)
        pr.t = t
        pr.compare_plan(1)
        pr.step(act, t)
    pr.compare_stats()
    st = pr.gpu.stats()
    assert st["readmissions"] > 0 and st["n_evict_dirty"] > 0
    assert pr.compare_blocks(range(sc.K)) == 0
    pr.close()


@pytest.mark.parametrize("J", [1, 2, 4, 7])
def test_tiny_batch_sizes_and_quota(J):
    """Several cameras per batch; capacity small enough that the camera quota binds."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=16, lam=0.3, quota=(1, 2))
    _drive(pr, tr, J, 24, check_blocks_every=11)
    pr.close()


@pytest.mark.parametrize("xfer", [0, 1])
def test_tide_off_restage_all(xfer):
    """Ablation: every batch restages R_{t+1}, dirty R_t is
    written back first; bytes and contents still match the oracle."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, tide=0, xfer=xfer)
    worst = _drive(pr, tr, cfg.J, 20, check_blocks_every=5)
    assert worst == 0
    pr.close()


@pytest.mark.parametrize("xfer", [0, 1])
def test_small_pool_uses_released_slots(xfer):
    """P = C: S+ must reuse the slots S- releases (R13 fallback path)."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, pool_slots=cfg.capacity, xfer=xfer)
    worst = _drive(pr, tr, cfg.J, 30, check_blocks_every=6)
    assert worst == 0
    pr.close()


def test_masked_rows_parity():
    """Sparse I_t (p = 0.25 row mask): masked rows bitwise unchanged, steps and
    dirty bits only for blocks with an active row."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, mask_p=0.25)
    worst = _drive(pr, tr, cfg.J, 24, check_blocks_every=5)
    assert worst == 0
    pr.close()


def test_empty_mask_leaves_everything_clean():
    """Empty I_t: nothing updated, nothing dirty, no step."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, mask_p=0.0)
    _drive(pr, tr, cfg.J, 12)
    st = pr.gpu.stats()
    assert st["total_updates"] == 0 and st["d2h_bytes"] == 0
    pr.gpu.flush()
    assert pr.gpu.stats()["flush_bytes"] == 0
    pr.close()


@pytest.mark.parametrize("xfer", [0, 1])
def test_static_batch_zero_traffic_and_empty_batch(xfer):
    """Static view with capacity: S+ = S- = {} after the first batch;
    J = 0 keeps R (R19).  Both transfer mechanisms (empty copy lists)."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=40, xfer=xfer)
    pl = tr.batch_planes(3, cfg.J)
    for t in range(5):
        act = pr.activate(pl)
        pr.t = t
        pr.compare_plan(cfg.J)
        if t:
            assert act.n_stage_in == 0 and act.n_evict == 0
        pr.step(act, t)
    act = pr.activate(np.zeros((0, 6, 4), np.float32))
    pr.compare_plan(0)
    assert act.n_visible == 0 and act.n_stage_in == 0
    pr.compare_stats()
    pr.close()


def test_nonfinite_gradient_reported_and_row_skipped():
    """R20: a NaN gradient skips its row, the lowest (gid*59+attr) is reported."""
    import torch
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity)
    act = pr.activate(tr.batch_planes(0, cfg.J))
    blocks = pr.orc.list("A", with_slots=True)
    k, s = int(blocks[0][1]), int(blocks[1][1])
    r, a = 5, 17

    def hook(act_):
        ptr = act_.d_grads + 4 * (s * act_.grad_stride + r * 59 + a)
        assert W.cuda_lib().wl_cuda_poke(ptr, float("nan"), pr.stream) == 0

    def ograd(_u, kk, t, out):
        W.lib().wl_grad_block(42, kk, sc.B, sc.rows(kk), t, out)
        if kk == k:
            out[r * 59 + a] = float("nan")

    import ctypes as C
    gfn = O.GRAD_FN(ograd)
    rc = pr.step(act, 0, grad_hook=hook, oracle_grad=(C.cast(gfn, C.c_void_p).value, None))
    assert rc == O.ENONFINITE
    assert pr.gpu.nonfinite_index() == pr.orc.nonfinite_index() == (k * sc.B + r) * 59 + a
    pr.compare_blocks([k])
    pr.close()


def test_conservation_without_updates():
    """With every mask empty, after any activate sequence + flush the host tier
    is byte-identical to the initial table (SURVEY §8c conservation)."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, mask_p=0.0)
    _drive(pr, tr, cfg.J, 30)
    pr.gpu.flush()
    for k in range(sc.K):
        th, m, v = pr.gpu.read_block(k)
        np.testing.assert_array_equal(th, sc.block_theta(k))
        assert not m.any() and not v.any()
    pr.close()


@pytest.mark.parametrize("name", ["11m", "100m"])
def test_full_size_index_parity_and_sampled_rows(name):
    """BASELINE.json configs at full size, the launch configuration bench.py
    times: indexing bit-exact every iteration; theta/m/v on sampled blocks."""
    wl = W.CONFIGS[name]
    sc = wl.scene()
    tr = wl.trajectory(sc)
    pr = _pair(sc, capacity=wl.capacity, track_all=False)
    assert wl.n_gaussians == sc.N
    rng = np.random.default_rng(5)
    sample = sorted(set(rng.integers(0, sc.K, 48).tolist()))
    iters = 6
    probe = O.Oracle(O.make_config(sc.N, sc.B, wl.capacity), sc.bounds(), fill=None,
                     track_all=False)
    for t in range(iters):
        probe.activate(tr.batch_planes(t, wl.J))
    touched = probe.list("R")
    probe.close()
    tracked = sorted(set(sample) | set(touched[:: max(1, len(touched) // 48)].tolist()))
    for k in tracked:
        assert pr.orc.track(k) == O.OK
    for t in range(iters):
        act = pr.activate(tr.batch_planes(t, wl.J))
        pr.t = t
        for which in ("K", "R", "S+", "S-", "A"):
            gb, gs = pr.gpu.list(which, with_slots=True)
            ob, os_ = pr.orc.list(which, with_slots=True)
            np.testing.assert_array_equal(gb, ob)
            np.testing.assert_array_equal(gs, os_)
        pr.step(act, t)
    pr.compare_stats()
    worst = pr.compare_blocks(tracked)
    assert worst == 0
    pr.close()


@pytest.mark.parametrize("level2", [0, 1])
@pytest.mark.parametrize("J", [2, 5])
def test_fine_filter_parity(J, level2):
    """NEXT f1: the Level-2 I_t mask is bit-exact with the oracle on every A
    block of every batch, and masked Adam driven by it matches (0 ULP) -- from
    theta rows (level2 = 0) and from the 16-B extent spheres the gather derives
    and k_adam keeps current (level2 = 1), here under training that moves the
    centres and scales."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, level2=level2)
    pr.lr[0:3] = 0.5
    pr.lr[52:55] = 0.05
    total = 0
    for t in range(16):
        act = pr.activate(tr.batch_planes(t, J))
        pr.t = t
        pr.compare_plan(J)
        rc, n = pr.step_fine(act, t)
        assert rc == O.OK
        total += n
    pr.compare_stats()
    assert pr.gpu.stats()["n_active_rows"] == total > 0
    assert pr.compare_blocks(range(sc.K)) == 0
    pr.close()


def test_bound_refresh_parity():
    """NEXT f2: with centres moving ~1 m per step, the refreshed bounds (R25)
    are bit-exact with the oracle after every batch, and so are K, R, slots
    and theta/m/v."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, refresh_bounds=1)
    pr.lr[0:3] = 1.0
    pr.lr[52:55] = 0.05
    grew = 0
    b0 = np.stack([pr.orc.bound(k) for k in range(sc.K)])
    for t in range(20):
        act = pr.activate(tr.batch_planes(t, cfg.J))
        pr.t = t
        pr.compare_plan(cfg.J)
        assert pr.step(act, t) == O.OK
        gb = np.stack([pr.gpu.bound(k) for k in range(sc.K)])
        ob = np.stack([pr.orc.bound(k) for k in range(sc.K)])
        np.testing.assert_array_equal(gb.view(np.uint32), ob.view(np.uint32), err_msg=f"t={t}")
        grew = int((ob[:, 3] > b0[:, 3]).sum())
    assert grew > 0
    pr.compare_stats()
    assert pr.compare_blocks(range(sc.K)) == 0
    pr.close()


def test_garbage_in_recycled_device_memory():
    """Every device buffer the library relies on is initialised: poison the
    caching allocator's free blocks with 0xFF bytes first (regression: the
    per-activate counters once came uninitialised from a recycled block)."""
    import torch
    junk = [torch.full((n,), -1, dtype=torch.int32, device="cuda")
            for n in [256] * 400 + [4096] * 200 + [131072] * 50 + [1 << 28]]
    torch.cuda.synchronize()
    del junk
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity)
    _drive(pr, tr, cfg.J, 12, check_blocks_every=5)
    pr.close()


@pytest.mark.parametrize("G", [2, 3])
def test_shards_on_one_gpu(G):
    """R17 sharding: every rank's context (world_size G, rank r,
    capacity ceil(C/G)) matches the oracle's shard r bit-exactly -- K_loc is
    then not a multiple of 32 (partial bitset words) -- and the shards' K
    partition the single-GPU K."""
    from paper_2605_20150_b200 import shard
    cfg, sc, tr = tiny()
    cap = shard.shard_capacity(cfg.capacity, G)
    pairs = [_pair(sc, capacity=cap, world_size=G, rank=r) for r in range(G)]
    single = O.Oracle(O.make_config(sc.N, sc.B, cfg.capacity), sc.bounds(), fill=None,
                      track_all=False)
    for t in range(16):
        planes = tr.batch_planes(t, cfg.J)
        single.activate(planes)
        Ks = []
        for pr in pairs:
            act = pr.activate(planes)
            pr.t = t
            pr.compare_plan(cfg.J)
            assert pr.step(act, t) == O.OK
            Ks += pr.gpu.list("K").tolist()
        assert sorted(Ks) == single.list("K").tolist()
    for r, pr in enumerate(pairs):
        pr.compare_stats()
        assert pr.compare_blocks([k for k in range(sc.K) if k % G == r]) == 0
        pr.close()


class _RandomCams:
    """Seeded random pinhole cameras inside a small scene (high churn)."""

    def __init__(self, side, seed=11, far=25.0):
        self.rng = np.random.default_rng(seed)
        self.side, self.far = side, far

    def batch_planes(self, t, J):
        out = np.empty((J, 6, 4), np.float32)
        for j in range(J):
            pos = [*(self.rng.uniform(-0.5, 0.5, 2) * self.side), self.rng.uniform(1.0, 15.0)]
            ang = self.rng.uniform(0, 2 * np.pi)
            fwd = [np.cos(ang), np.sin(ang), -self.rng.uniform(0.1, 1.0)]
            cam = W.look(pos, fwd, [0, 0, 1], 50.0, 640, 480, 0.1, self.far)
            out[j] = W.camera_planes(cam)
        return out


@pytest.mark.parametrize("N,B,C,J,kw", [
    (1, 4, 1, 1, {}),                                            # one Gaussian, one block
    (37, 4, 2, 3, {"pool_slots": 2}),                            # ragged last block, P = C
    (5000, 8, 1, 256, {"quota": (1, 1)}),                        # max cameras, C = 1, beta = 1
    (20000, 36, 40, 17, {"max_age": 0, "lam": 0.0}),             # B % 32 != 0, recency off
    (20000, 36, 40, 17, {"max_age": 1023, "gamma": 0.999999}),   # max age, gamma -> 1
    (30000, 100, 7, 5, {"tide": 0, "moments": O.COLD_RESTART}),  # restage-all, cold
    (30000, 100, 12, 4, {"quota": (1, 1), "lam": 1.0, "pool_slots": 13}),  # tight pool
])
@pytest.mark.parametrize("xfer", [0, 1])
def test_edge_configs(N, B, C, J, kw, xfer):
    """Degenerate and extreme shapes under random (high-churn) cameras:
    bit-exact lists/slots/counters and 0-ULP rows against the oracle, with both
    transfer mechanisms (copy-engine runs of tiny, odd-sized records)."""
    sc = W.Scene(N, B, side=60.0, lot=20.0, footprint=12.0, hmin=2.0, hmax=12.0)
    tr = _RandomCams(60.0)
    pr = _pair(sc, capacity=C, xfer=xfer, **kw)
    _drive(pr, tr, J, 12, check_blocks_every=3)
    pr.gpu.flush()
    pr.orc.flush()
    pr.compare_stats()
    assert pr.compare_blocks(range(sc.K)) == 0
    pr.close()


@pytest.mark.parametrize("mode", ["plain", "fine", "fine_refresh_cold", "mask_direct",
                                  "fine_level2", "fine_level2_masked_refresh",
                                  "plain_async", "fine_async", "fine_refresh_cold_async",
                                  "fine_level2_async", "plain_ce", "fine_refresh_cold_ce",
                                  "mask_direct_ce", "fine_level2_masked_refresh_ce"])
def test_pipelined_run_matches_oracle(mode, monkeypatch):
    """The GPU runs ahead exactly as in bench.py -- no inspection call (hence no
    host sync) between batches -- so every cross-batch hazard (plan of t+1 vs
    Adam/filter/write-back of t) is exercised; the final state must still match
    the oracle bit-exactly."""
    import ctypes as C

    import torch
    from gpu_harness import GRAD_SEED, Synth, _cfn
    cfg, sc, tr = tiny()
    use_async = mode.endswith("_async")  # tgs_activate_async: no plan readback at all
    if use_async:
        mode = mode[: -len("_async")]
    xfer = 1 if mode.endswith("_ce") else 0  # copy-engine runs + k_commit
    if xfer:
        mode = mode[: -len("_ce")]
    kw = {"plain": {}, "fine": {}, "fine_refresh_cold": {"refresh_bounds": 1,
                                                          "moments": O.COLD_RESTART},
          "fine_level2": {"level2": 1}, "fine_level2_masked_refresh": {"level2": 1, "refresh_bounds": 1},
          "mask_direct": {"staging_blocks": 1, "mask_p": 0.5}}[mode]
    pr = _pair(sc, capacity=cfg.capacity, xfer=xfer, **kw)
    if "refresh" in mode:
        pr.lr[0:3] = 0.5
    fine = mode.startswith("fine")
    dmask = torch.zeros((pr.gpu.P, (sc.B + 31) // 32), dtype=torch.int32, device="cuda")
    if pr.d_mask is not None:
        dmask = pr.d_mask
    n = 40
    for t in range(n):  # GPU: back to back
        planes = tr.batch_planes(t, cfg.J)
        act = pr.gpu.activate_async(planes) if use_async else pr.gpu.activate(planes)
        pr.grads_gpu_only(act, t)
        if fine:
            pr.gpu.fine_filter(dmask.data_ptr())
        elif pr.msyn is not None:
            W.synth_mask_cuda(dmask.data_ptr(), act, sc.B, sc.N, 43, t, pr.msyn.p32, pr.stream)
        pr.gpu.step_adam(pr.lr, mask_ptr=dmask.data_ptr() if (fine or pr.msyn) else None)
    g = (_cfn("wl_grad_cb"), C.addressof(pr.gsyn))
    for t in range(n):  # oracle
        assert pr.orc.activate(tr.batch_planes(t, cfg.J)) == O.OK
        m = pr.orc.fine_filter_mask if fine else (
            (_cfn("wl_mask_cb"), C.addressof(pr.msyn)) if pr.msyn is not None else None)
        assert pr.orc.step_adam(pr.lr, grad=g, mask=m) == O.OK
    pr.t = n
    pr.compare_plan(cfg.J)
    pr.compare_stats()
    assert pr.compare_blocks(range(sc.K)) == 0
    pr.gpu.flush()
    pr.orc.flush()
    pr.compare_stats()
    if "refresh" in mode:
        gb = np.stack([pr.gpu.bound(k) for k in range(sc.K)])
        ob = np.stack([pr.orc.bound(k) for k in range(sc.K)])
        np.testing.assert_array_equal(gb.view(np.uint32), ob.view(np.uint32))
    pr.close()


def test_fresh_counters_match_oracle_first_updates():
    """tgs_timing.fresh_active_rows / fresh_blocks (the cold-restart term of k_adam's
    algorithmic bytes, bench.py roofline) count exactly the blocks of A whose
    update is their first since admission: oracle step count 1 after the step."""
    cfg, sc, tr = tiny()
    pr = _pair(sc, capacity=cfg.capacity, moments=O.COLD_RESTART)
    seen = 0
    for t in range(24):
        act = pr.activate(tr.batch_planes(t, cfg.J))
        t0 = pr.gpu.timing()
        assert pr.step(act, t) == O.OK
        t1 = pr.gpu.timing()
        fresh = [int(k) for k in pr.orc.list("A") if pr.orc.step_count(int(k)) == 1]
        rows = sum(min(sc.B, sc.N - k * sc.B) for k in fresh)
        assert t1["fresh_blocks"] - t0["fresh_blocks"] == len(fresh)
        assert t1["fresh_active_rows"] - t0["fresh_active_rows"] == rows
        seen += len(fresh)
    assert seen > cfg.capacity  # re-admissions happened (cold restarts beyond the first fill)
    pr.close()


@pytest.mark.parametrize("name", ["quota_member_by_key_q1", "quota_min_with_camera_size"])
def test_camera_balanced_topc_golden_on_gpu(name):
    """The hand-worked CameraBalancedTopC examples (tests/golden/
    camera_balanced_topc.json) through the C ABI: k_quota /
    k_plan must give the hand-derived R, S+, S-, Omega and K^(j)."""
    from paper_2605_20150_b200 import tidegs as T
    from test_oracle_golden import _scn, line_bounds, slab_planes
    scn = _scn(name)
    n = scn["n_blocks"]
    tab = T.Table(T.make_config(4 * n, 4, scn["capacity"], lam=scn["lambda"], gamma=scn["gamma"],
                                quota=tuple(scn["beta"])), line_bounds(n),
                  fill=lambda k: np.zeros((4, 59), np.float32))
    for b in scn["batches"]:
        tab.activate(slab_planes(b["slabs"]))
        for j, kj in enumerate(b.get("K_per_camera", [])):
            assert tab.percam(j).tolist() == kj
        for which in ("R", "S+", "S-", "Omega"):
            if which in b:
                assert tab.list(which).tolist() == b[which], which
    tab.close()


@pytest.mark.parametrize("case", [0, 1])
def test_recency_golden_on_gpu(case):
    """Recency golden case (gamma^age, age 8 keeps / age 9 evicts) through the
    GPU's rank LUT."""
    from paper_2605_20150_b200 import tidegs as T
    from test_oracle_golden import _scn, line_bounds, run_recency_case
    scn = _scn("recency_gamma_power_age")
    c = scn["cases"][case]
    tab = run_recency_case(lambda: T.Table(
        T.make_config(12, 4, scn["capacity"], lam=scn["lambda"], gamma=scn["gamma"],
                      quota=tuple(scn["beta"])), line_bounds(3),
        fill=lambda k: np.zeros((4, 59), np.float32)), c["empty_batches"])
    assert tab.list("R").tolist() == c["R_final"]
    tab.close()


@pytest.mark.parametrize("ctas", ["1,1,2,2", "3,2,3,5", "16,8,7,4"])
def test_transfer_grid_shapes_give_identical_results(ctas, monkeypatch):
    """Determinism across launch shapes: the k_xfer gather / write-back with 1..16
    CTAs and 2..7 shared-memory buffers each (TGS_GATHER_CTAS / _SCATTER_CTAS /
    _GATHER_BUFS / _SCATTER_BUFS), on a pipelined run with no host sync between
    batches, in the smallest-ring configuration (staging of 2 records: many
    direct write-backs) and both policies; the end state must equal the
    oracle's bit for bit whatever the interleaving."""
    g, s_, gb, sb = ctas.split(",")
    monkeypatch.setenv("TGS_GATHER_CTAS", g)
    monkeypatch.setenv("TGS_SCATTER_CTAS", s_)
    monkeypatch.setenv("TGS_GATHER_BUFS", gb)
    monkeypatch.setenv("TGS_SCATTER_BUFS", sb)
    import ctypes as C
    from gpu_harness import _cfn
    cfg, sc, tr = tiny()
    for moments, staging in ((O.PERSIST, 2), (O.COLD_RESTART, 0)):
        pr = _pair(sc, capacity=cfg.capacity, moments=moments, staging_blocks=staging)
        n = 30
        for t in range(n):
            act = pr.gpu.activate(tr.batch_planes(t, cfg.J))
            pr.grads_gpu_only(act, t)
            pr.gpu.step_adam(pr.lr)
        gfn = (_cfn("wl_grad_cb"), C.addressof(pr.gsyn))
        for t in range(n):
            assert pr.orc.activate(tr.batch_planes(t, cfg.J)) == O.OK
            assert pr.orc.step_adam(pr.lr, grad=gfn) == O.OK
        pr.t = n
        pr.compare_plan(cfg.J)
        pr.compare_stats()
        pr.gpu.flush()
        pr.orc.flush()
        assert pr.compare_blocks(range(sc.K)) == 0
        pr.close()


@pytest.mark.parametrize("moments", [O.PERSIST, O.COLD_RESTART])
def test_async_activate_step_by_step(moments):
    """tgs_activate_async (no plan readback; every count from the device header):
    after each batch the lists, slots, K^(j), dirty S- and counters equal the
    oracle's, on the tiny orbit (C = 24 < K) and an edge config with random
    cameras (ragged last block, J = 17)."""
    for sc, tr, J, C in ((tiny()[1], tiny()[2], 2, 24),
                         (W.Scene(20000, 36, side=60.0, lot=20.0, footprint=12.0, hmin=2.0,
                                  hmax=12.0), _RandomCams(60.0), 17, 40)):
        pr = _pair(sc, capacity=C, moments=moments)
        for t in range(24):
            planes = tr.batch_planes(t, J)
            act = pr.gpu.activate_async(planes)
            assert act.n_active_blocks == 0xFFFFFFFF
            assert pr.orc.activate(planes) == O.OK
            pr.t = t
            pr.compare_plan(J)
            pr.compare_evicted_dirty()
            assert pr.step(act, t) == O.OK
            pr.compare_stats()
        pr.gpu.flush()
        pr.orc.flush()
        assert pr.compare_blocks(range(sc.K)) == 0
        pr.close()
