"""NEXT f3 on the GPU path: the store tier (CPU cache + log-structured SSD
segments; readings R27, R28) against the oracle's store,
element by element: every list and counter of the working-set step, the
CPU-cache counters, LRU order and dirty flags, Index[k] of every block, the
segment files byte for byte (the two sides write them independently from the
R28 format), and theta/m/v."""
import ctypes as C
import filecmp
import os
import shutil

import numpy as np
import pytest

import oracle as O
import workload as W
from helpers import random_boxes, tiny

pytestmark = pytest.mark.gpu


def _pair(sc, tmp_path, H, seg=0, direct=0, prefetch=0, **kw):
    from gpu_harness import Pair
    g, o = tmp_path / "gpu", tmp_path / "orc"
    o.mkdir()
    st = dict(gpu_dir=str(g), orc_dir=str(o), cache_blocks=H, segment_bytes=seg, direct_io=direct,
              prefetch_blocks=prefetch)
    return Pair(sc, store=st, **kw), g, o


def _compare_files(g, o):
    gf, of = sorted(os.listdir(g)), sorted(os.listdir(o))
    assert gf == of, (gf, of)
    for name in gf:
        if not filecmp.cmp(g / name, o / name, shallow=False):
            a, b = (g / name).read_bytes(), (o / name).read_bytes()
            first = next((i for i in range(min(len(a), len(b))) if a[i] != b[i]), None)
            raise AssertionError(f"{name}: sizes {len(a)} / {len(b)}, first difference at {first}")
    return len(gf)


def _finish(pr, sc, g, o):
    pr.gpu.flush()
    pr.orc.flush()
    pr.compare_stats()
    s = pr.compare_store(range(sc.K))
    assert s["cached_dirty"] == 0
    n_files = _compare_files(g, o)
    assert pr.compare_blocks(range(sc.K)) == 0
    return s, n_files


@pytest.mark.parametrize("direct", [0, 1])
@pytest.mark.parametrize("moments,H,seg", [(O.PERSIST, 16, 0), (O.COLD_RESTART, 16, 0),
                                           (O.PERSIST, 21, 6 << 20)])
def test_store_parity_jumping_batches(tmp_path, moments, H, seg, direct):
    """Batches that jump across the scene with C = 8 and a 2C..2.6C CPU cache:
    misses, dirty LRU victims appended to patch segments, re-reads of patched
    versions -- bit-exact against the oracle at every step, files identical."""
    cfg, sc, tr = tiny()
    pr, g, o = _pair(sc, tmp_path, H, seg, direct, capacity=8, moments=moments)
    for t, planes in enumerate(random_boxes(sc, 36)):
        act = pr.activate(planes)
        pr.t = t
        pr.compare_plan(1)
        pr.compare_evicted_dirty()
        pr.compare_store(pr.orc.list("S+"))
        assert pr.step(act, t) == O.OK
        if t % 9 == 0:
            assert pr.compare_blocks(pr.orc.list("R")) == 0
    s, n_files = _finish(pr, sc, g, o)
    assert s["dirty_evictions"] > 0 and s["misses"] > s["hits"] > 0
    assert n_files >= (3 if seg else 2)
    pr.close()


@pytest.mark.parametrize("moments", [O.PERSIST, O.COLD_RESTART])
def test_store_parity_orbit(tmp_path, moments):
    """configs[0] orbit trajectory (C = 24, cache 2C): the smooth-trajectory
    regime where the cache mostly hits."""
    cfg, sc, tr = tiny()
    pr, g, o = _pair(sc, tmp_path, 2 * cfg.capacity, capacity=cfg.capacity, moments=moments)
    for t in range(40):
        act = pr.activate(tr.batch_planes(t, cfg.J))
        pr.t = t
        pr.compare_plan(cfg.J)
        pr.compare_store()
        assert pr.step(act, t) == O.OK
    s, _ = _finish(pr, sc, g, o)
    assert s["hits"] > 0
    pr.close()


@pytest.mark.parametrize("kw", [dict(tide=0), dict(pool_slots=8), dict(staging_blocks=1),
                                dict(mask_p=0.25)])
def test_store_parity_write_back_variants(tmp_path, kw):
    """Tide off (S+ and S- overlap: write-back before the gather), a pool of C
    slots (S+ reuses released slots), write-back straight from the slots, and
    masked rows (blocks with no active row stay clean)."""
    cfg, sc, tr = tiny()
    pr, g, o = _pair(sc, tmp_path, 16, capacity=8, **kw)
    for t, planes in enumerate(random_boxes(sc, 30, seed=11)):
        act = pr.activate(planes)
        pr.t = t
        pr.compare_plan(1)
        pr.compare_evicted_dirty()
        pr.compare_store()
        assert pr.step(act, t) == O.OK
    _finish(pr, sc, g, o)
    pr.close()


@pytest.mark.parametrize("H", [16, 24])
def test_store_pipelined_matches_oracle(tmp_path, H):
    """The GPU runs ahead with no inspection call between batches (as in
    bench.py), so a dirty LRU victim can be a block whose write-back of 1-3
    batches ago is still in flight: the append must wait for exactly that
    D2H.  The final store (index, counters, files, table) matches the oracle."""
    from gpu_harness import _cfn
    cfg, sc, tr = tiny()
    pr, g, o = _pair(sc, tmp_path, H, capacity=8)
    boxes = random_boxes(sc, 48, seed=3)
    for t, planes in enumerate(boxes):
        act = pr.gpu.activate(planes)
        pr.grads_gpu_only(act, t)
        pr.gpu.step_adam(pr.lr)
    gr = (_cfn("wl_grad_cb"), C.addressof(pr.gsyn))
    for planes in boxes:
        assert pr.orc.activate(planes) == O.OK
        assert pr.orc.step_adam(pr.lr, grad=gr) == O.OK
    pr.t = len(boxes)
    pr.compare_stats()
    pr.compare_store(range(sc.K))
    s, _ = _finish(pr, sc, g, o)
    assert s["dirty_evictions"] > 0
    pr.close()


@pytest.mark.parametrize("moments", [O.PERSIST, O.COLD_RESTART])
def test_store_resume_after_barrier(tmp_path, moments):
    """R30 checkpoint/resume: a second GPU context reopens the segment files
    the first one left at its barrier; its recovered Index[k] equals the
    oracle's (each side reopens its own files), and 20 more batches stay
    bit-exact, ending with byte-identical files."""
    from gpu_harness import Pair
    cfg, sc, tr = tiny()
    seg = 6 << 20
    pr, g, o = _pair(sc, tmp_path, 16, seg, 1, capacity=8, moments=moments)
    for t, planes in enumerate(random_boxes(sc, 24, seed=13)):
        act = pr.activate(planes)
        assert pr.step(act, t) == O.OK
    pr.gpu.flush()
    pr.orc.flush()
    live = {k: pr.orc.store_index(k) for k in range(sc.K)}
    pr.close()
    st = dict(gpu_dir=str(g), orc_dir=str(o), cache_blocks=16, segment_bytes=seg, direct_io=1,
              reopen=1)
    pr = Pair(sc, capacity=8, moments=moments, store=st)
    for k in range(sc.K):
        assert pr.gpu.store_index(k) == pr.orc.store_index(k) == live[k], k
    for t, planes in enumerate(random_boxes(sc, 20, seed=14)):
        act = pr.activate(planes)
        pr.t = t
        pr.compare_plan(1)
        pr.compare_store(pr.orc.list("S+"))
        assert pr.step(act, t) == O.OK
    _finish(pr, sc, g, o)
    pr.close()


def test_store_compaction(tmp_path):
    """R31: compaction at a barrier on both sides -> byte-identical base
    segments, no patch left, identical Index; training then continues
    bit-exact (patch segment 1 again, versions counting on)."""
    cfg, sc, tr = tiny()
    pr, g, o = _pair(sc, tmp_path, 16, 6 << 20, 1, capacity=8)
    boxes = random_boxes(sc, 40, seed=17)
    for t, planes in enumerate(boxes[:28]):
        act = pr.activate(planes)
        assert pr.step(act, t) == O.OK
    pr.gpu.store_compact()
    pr.orc.flush()
    pr.orc.store_compact()
    assert _compare_files(g, o) == 2  # base.tdgs + its manifest (R30, R31)
    pr.compare_store(range(sc.K))
    for t, planes in enumerate(boxes[28:], 28):
        act = pr.activate(planes)
        pr.t = t
        pr.compare_plan(1)
        pr.compare_store(pr.orc.list("S+"))
        assert pr.step(act, t) == O.OK
    _finish(pr, sc, g, o)
    pr.close()


def test_store_conservation_without_updates(tmp_path):
    """Empty masks: nothing is dirty, nothing is appended, every block read back
    through the store equals the generated table."""
    cfg, sc, tr = tiny()
    pr, g, o = _pair(sc, tmp_path, 16, capacity=8, mask_p=0.0)
    for t, planes in enumerate(random_boxes(sc, 30, seed=9)):
        act = pr.activate(planes)
        pr.t = t
        assert pr.step(act, t) == O.OK
    s, n_files = _finish(pr, sc, g, o)
    # only the base segment and its barrier manifest (R30): no patch segment
    assert s["write_bytes"] == 0 and n_files == 2 and s["evictions"] > 0
    for k in range(sc.K):
        th, m, v = pr.gpu.read_block(k)
        assert np.array_equal(th, sc.block_theta(k)) and not m.any() and not v.any()
    pr.close()


def test_store_full_size_100m_index_parity(tmp_path):
    """configs[2] shape (100M street, J = 64, cold restart) with a CPU cache of
    2C blocks over a 23.6 GB base segment written with O_DIRECT: the lists,
    cache counters, LRU order and Index[k] of every touched block bit-exact
    against the oracle's metadata-only store over 30 batches (the launch
    configuration bench.py --store times)."""
    cfg = W.CONFIGS["100m"]
    sc = cfg.scene()
    tr = cfg.trajectory(sc)
    from gpu_harness import Pair
    d = tmp_path / "gpu"
    H = 2 * cfg.capacity
    pr = Pair(sc, capacity=cfg.capacity, moments=O.COLD_RESTART, track_all=False,
              fill=sc.fill_fn,
              store=dict(gpu_dir=str(d), orc_dir=None, cache_blocks=H, direct_io=1))
    touched = set()
    for t in range(30):
        act = pr.activate(tr.batch_planes(t, cfg.J))
        pr.t = t
        sp = pr.orc.list("S+")
        touched |= set(sp.tolist())
        pr.compare_plan(0)
        pr.compare_store(sp)
        pr.grads_gpu_only(act, t)
        pr.gpu.step_adam(pr.lr)
        assert pr.orc.step_adam(pr.lr) == O.OK
    pr.compare_stats()
    pr.compare_store(sorted(touched))
    pr.close()
    shutil.rmtree(d, ignore_errors=True)  # 23.6 GB: do not leave it to pytest's tmp retention


@pytest.mark.parametrize("moments,prefetch,ahead", [(O.PERSIST, 8, 1), (O.COLD_RESTART, 24, 1),
                                                    (O.PERSIST, 24, 2), (O.COLD_RESTART, 5, 2)])
def test_store_prefetch_is_transparent(tmp_path, moments, prefetch, ahead):
    """f3 read-ahead (tgs_prefetch): announcing each next
    batch lets the GPU side read the misses ahead into read-ahead buffers, with
    a pool smaller and larger than a batch's misses.  The CPU cache is untouched,
    so every list, cache counter, LRU order, Index and file still matches the
    oracle (which has no read-ahead) bit-exactly, while misses are served from
    read-ahead records."""
    cfg, sc, tr = tiny()
    pr, g, o = _pair(sc, tmp_path, 16, 6 << 20, 1, prefetch=prefetch, capacity=8,
                     moments=moments)
    boxes = random_boxes(sc, 36, seed=27)
    for a in range(ahead):
        pr.gpu.prefetch(boxes[a], a + 1)
    for t, planes in enumerate(boxes):
        act = pr.activate(planes)
        pr.t = t
        pr.compare_plan(1)
        pr.compare_evicted_dirty()
        pr.compare_store(pr.orc.list("S+"))
        assert pr.step(act, t) == O.OK
        if t + ahead < len(boxes):
            pr.gpu.prefetch(boxes[t + ahead], ahead)
    s, n_files = _finish(pr, sc, g, o)
    full = pr.gpu.store_stats()
    assert s["misses"] > 0 and full["prefetch_hits"] > 0 and full["prefetch_reads"] > 0
    pr.close()
