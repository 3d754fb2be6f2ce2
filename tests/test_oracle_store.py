"""Pins for the oracle's NEXT f3 tier below the host (§3.4):
the log-structured store (immutable base segment, append-only patch segments,
Index[k] = (file_id, offset, size, version)) and the LRU CPU cache with dirty
bits and two-step write-back.  Readings R27 (cache events) and R28 (segment
format) are in DESIGN.md §3.

Each pin is independent of the oracle's code: the segment files are parsed by
the plain reader below (written from the R28 format statement), the LRU is a
textbook OrderedDict simulation, and transparency compares against the flat
host-tier oracle (itself pinned against an in-memory Adam run in
test_oracle_adam.py)."""
import os
from collections import OrderedDict

import numpy as np
import pytest

import oracle as O
import workload as W
from helpers import lr_3dgs, random_boxes, synth_grad, synth_mask, tiny

PAGE = 4096
REC = 966_656  # B=4096 record: 4096*59*4 bytes = 236 pages


def _pad(x):
    return (x + PAGE - 1) // PAGE * PAGE


def _crc32c_table():
    t = []
    for i in range(256):
        c = i
        for _ in range(8):
            c = (c >> 1) ^ (0x82F63B78 if c & 1 else 0)
        t.append(c)
    return t


_CRC_T = _crc32c_table()


def crc32c(data: bytes) -> int:
    """CRC-32C (Castagnoli, reflected 0x82F63B78), table-driven; pinned below by
    the standard check value of b"123456789"."""
    c = 0xFFFFFFFF
    for b in data:
        c = (c >> 8) ^ _CRC_T[(c ^ b) & 0xFF]
    return c ^ 0xFFFFFFFF


def read_manifest(d):
    """R30 barrier manifest: epoch, durable log end, base versions, step counters."""
    raw = open(os.path.join(d, "manifest.tdgm"), "rb").read()
    assert raw[:4] == b"TDGM" and int.from_bytes(raw[4:8], "little") == 1
    K = int.from_bytes(raw[60:64], "little")
    assert len(raw) == 64 + 12 * K + 4
    assert int.from_bytes(raw[-4:], "little") == crc32c(raw[:-4])
    return dict(epoch=int.from_bytes(raw[8:16], "little"),
                last_file=int.from_bytes(raw[16:20], "little"),
                end=int.from_bytes(raw[24:32], "little"), Kloc=K,
                base_version=np.frombuffer(raw[64:64 + 8 * K], "<u8"),
                step=np.frombuffer(raw[64 + 8 * K:64 + 12 * K], "<u4"))


def read_segments(d, check_crc=2):
    """R28 reader: {file_id: (kind, header fields, [(offset, gid, version, payload bytes)])};
    the payload CRC-32C of the first check_crc records of the store is
    recomputed here, every record's header CRC is."""
    out = {}
    crc_left = [check_crc]
    for name in sorted(os.listdir(d)):
        if name == "manifest.tdgm":
            continue
        p = os.path.join(d, name)
        raw = open(p, "rb").read()
        magic = raw[:4]
        fid = int.from_bytes(raw[8:12], "little")
        hdr = dict(fmt=int.from_bytes(raw[4:8], "little"), fid=fid,
                   n_arr=int.from_bytes(raw[12:16], "little"),
                   N=int.from_bytes(raw[16:24], "little"), D=int.from_bytes(raw[24:28], "little"),
                   B=int.from_bytes(raw[28:32], "little"))
        recs = []
        if magic == b"TDGP":
            assert name == f"patch-{fid:06d}.tdgp"
            off = PAGE
            while off < len(raw):
                assert raw[off:off + 4] == b"TREC"
                assert int.from_bytes(raw[off + 4:off + 8], "little") == 2
                gid = int.from_bytes(raw[off + 8:off + 16], "little")
                ver = int.from_bytes(raw[off + 16:off + 24], "little")
                n = int.from_bytes(raw[off + 24:off + 32], "little")
                assert int.from_bytes(raw[off + 36:off + 40], "little") == crc32c(raw[off:off + 36])
                if crc_left[0] > 0:
                    crc_left[0] -= 1
                    assert (int.from_bytes(raw[off + 32:off + 36], "little")
                            == crc32c(raw[off + PAGE:off + PAGE + n]))
                recs.append((off + PAGE, gid, ver, n))
                off += PAGE + _pad(n)
            assert off == len(raw)
        else:
            assert magic == b"TDGS" and name == "base.tdgs" and fid == 0
        out[fid] = (magic, hdr, recs, raw)
    return out


def payload_at(segs, fid, off, n):
    return np.frombuffer(segs[fid][3][off:off + n], np.float32)


def run_tiny(o, tr, J, n, lr=None, grad=None, mask=None, trace=None):
    for t in range(n):
        assert o.activate(tr.batch_planes(t, J)) == O.OK
        if trace is not None:
            trace.append((o.list("R").tolist(), o.list("S+").tolist(), o.list("S-").tolist(),
                          o.evicted_dirty().tolist()))
        if lr is not None:
            o.step_adam(lr, 0.9, 0.999, 1e-15, grad=grad, mask=mask)


def test_base_segment_spec_examples(tmp_path):
    """SPEC.md log_store write_base: N=8192, B=4096, D=59 -> base file = header
    + 2 * 966,656 bytes; N=1 -> one zero-padded record; read back byte-exactly."""
    theta = np.arange(8192 * 59, dtype=np.float32).reshape(8192, 59)
    bounds = np.array([[0, 0, 0, 1], [10, 0, 0, 1]], np.float32)
    cfg = O.make_config(8192, 4096, 1, moments=O.COLD_RESTART)
    o = O.Oracle(cfg, bounds, fill=lambda k: theta[k * 4096:(k + 1) * 4096], track_all=True)
    o.store_open(tmp_path, 2)
    base = tmp_path / "base.tdgs"
    assert base.stat().st_size == PAGE + 2 * REC
    segs = read_segments(tmp_path)
    assert segs[0][1]["N"] == 8192 and segs[0][1]["D"] == 59 and segs[0][1]["B"] == 4096
    for k in range(2):
        fid, off, size, ver = o.store_index(k)
        assert (fid, off, size, ver) == (0, PAGE + k * REC, REC, 0)
        got = payload_at(segs, fid, off, size).reshape(4096, 59)
        assert np.array_equal(got, theta[k * 4096:(k + 1) * 4096])
    o.close()

    d1 = tmp_path / "one"
    d1.mkdir()
    o = O.Oracle(O.make_config(1, 4096, 1, moments=O.COLD_RESTART), bounds[:1],
                 fill=lambda k: np.full((4096, 59), 0.0, np.float32) + (np.arange(4096) < 1)[:, None],
                 track_all=True)
    o.store_open(d1, 2)
    raw = (d1 / "base.tdgs").read_bytes()
    assert len(raw) == PAGE + REC
    rec = np.frombuffer(raw[PAGE:], np.float32).reshape(4096, 59)
    assert np.all(rec[0] == 1.0) and not rec[1:].any()  # row 0 real, padding rows zero (R15)


def test_persist_payload_and_padding(tmp_path):
    """Persist records hold theta | m | v (3 arrays); tiny B=1568 payloads are
    padded to whole pages so every payload starts page-aligned."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, cfg.capacity, moments=O.PERSIST), sc.bounds(),
                 fill=sc.fill_fn, track_all=True)
    o.store_open(tmp_path, 2 * cfg.capacity)
    payload = 3 * sc.B * 59 * 4
    S = _pad(payload)
    assert (tmp_path / "base.tdgs").stat().st_size == PAGE + sc.K * S
    segs = read_segments(tmp_path)
    for k in (0, 17, sc.K - 1):
        fid, off, size, ver = o.store_index(k)
        assert off % PAGE == 0 and size == payload and ver == 0
        p = payload_at(segs, fid, off, size).reshape(3, sc.B, 59)
        assert np.array_equal(p[0], sc.block_theta(k)) and not p[1:].any()


def lru_model(trace, H):
    """Textbook LRU over the R27 access sequence (S+ ascending, then S-
    ascending), with the GPU-resident blocks (R_t u R_{t+1}) not evictable;
    dirty entries come from the D2H write-backs of dirty S-."""
    lru = OrderedDict()  # gid -> dirty, least recent first
    st = dict(hits=0, misses=0, evictions=0, dirty_evictions=0)
    R_prev = []
    orders = []
    for R, Sp, Sm, dirty_sm in trace:
        for k in dirty_sm:
            lru[k] = True
        pinned = set(R_prev) | set(R)
        for k in Sp:
            if k in lru:
                st["hits"] += 1
                lru.move_to_end(k)
                continue
            st["misses"] += 1
            if len(lru) >= H:
                victim = next(v for v in lru if v not in pinned)
                st["evictions"] += 1
                st["dirty_evictions"] += lru.pop(victim)
            lru[k] = False
        for k in Sm:
            lru.move_to_end(k)
        orders.append(list(lru.items()))
        R_prev = R
    return st, orders


@pytest.mark.parametrize("H", [16, 23])
@pytest.mark.parametrize("moments", [O.PERSIST, O.COLD_RESTART])
def test_cache_matches_textbook_lru(H, moments):
    """SPEC.md host_cache: 'random access trace vs. reference LRU simulation ->
    identical hit/miss sequence and eviction order'; LRU independent of the
    dirty bit."""
    cfg, sc, tr = tiny()
    C = 8  # small enough that a 2C..2.4C cache must evict along the orbit
    o = O.Oracle(O.make_config(sc.N, sc.B, C, moments=moments), sc.bounds(), track_all=False)
    o.store_open(None, H)
    lr = lr_3dgs()
    trace = []
    for t, planes in enumerate(random_boxes(sc, 40)):
        assert o.activate(planes) == O.OK
        trace.append((o.list("R").tolist(), o.list("S+").tolist(), o.list("S-").tolist(),
                      o.evicted_dirty().tolist()))
        # metadata-only: Adam marks dirty without data (every A block touched)
        o.step_adam(lr)
        st_model, orders = lru_model(trace, H)
        blocks, dirty = o.store_lru()
        assert list(zip(blocks.tolist(), dirty.tolist())) == orders[-1], t
    s = o.store_stats()
    for key, v in st_model.items():
        assert s[key] == v, key
    assert s["misses"] > 0 and s["evictions"] > 0 and s["dirty_evictions"] > 0
    # R28 byte counts: every miss reads one padded payload; every append writes
    # a header page + the padded payload, every segment a header page
    S = _pad(sc.B * 59 * 4 * (3 if moments == O.PERSIST else 1))
    assert s["read_bytes"] == s["misses"] * S
    appends = s["dirty_evictions"] + s["flush_appends"]
    assert s["write_bytes"] == appends * (PAGE + S) + s["segments"] * PAGE


def test_spec_lru_example_capacity_two():
    """SPEC.md host_cache get: capacity 2 blocks, access 0, 1, 2 -> block 0
    evicted (LRU definition).  C = 1 so each batch admits one block."""
    B = 8
    bounds = np.array([[10.0 * k, 0, 0, 1] for k in range(3)], np.float32)
    o = O.Oracle(O.make_config(3 * B, B, 1, moments=O.COLD_RESTART), bounds, track_all=False)
    o.store_open(None, 2)
    for k in range(3):
        p = np.zeros((1, 6, 4), np.float32)
        p[0] = [[1, 0, 0, -(10.0 * k - 1)], [-1, 0, 0, 10.0 * k + 1], [0, 1, 0, 1e3],
                [0, -1, 0, 1e3], [0, 0, 1, 1e3], [0, 0, -1, 1e3]]
        o.activate(p)
        assert o.list("R").tolist() == [k]
    blocks, _ = o.store_lru()
    assert 0 not in blocks.tolist() and sorted(blocks.tolist()) == [1, 2]
    assert o.store_stats()["evictions"] == 1


def _flat_and_store(tmp_path, moments, masked, H, seg_bytes=0, n=30, C=8):
    """the same run on the flat host tier and on the store tier (C = 8 and
    batches jumping across the scene, so the small CPU cache evicts dirty
    entries)"""
    cfg, sc, tr = tiny()
    lr = lr_3dgs()
    grad = synth_grad(W.SEEDS["grads"], sc.N, sc.B)
    mask = synth_mask(W.SEEDS["mask"], sc.N, sc.B, 1 << 30) if masked else None
    res = []
    for store in (False, True):
        o = O.Oracle(O.make_config(sc.N, sc.B, C, moments=moments), sc.bounds(),
                     fill=sc.fill_fn, track_all=True)
        if store:
            o.store_open(tmp_path, H, seg_bytes)
        lists = []
        for planes in random_boxes(sc, n):
            o.activate(planes)
            lists.append([o.list(w).tolist() for w in ("K", "R", "S+", "S-", "A")] +
                         [o.evicted_dirty().tolist(), o.slot_map().tolist()])
            o.step_adam(lr, 0.9, 0.999, 1e-15, grad=grad, mask=mask)
        o.flush()
        res.append((o, lists))
    return sc, res


@pytest.mark.parametrize("moments,masked,H", [(O.PERSIST, False, 16), (O.PERSIST, True, 21),
                                              (O.COLD_RESTART, False, 16)])
def test_store_tier_is_transparent(tmp_path, moments, masked, H):
    """The tier below the host changes where the newest version lives, never
    what it is (PAPER.md:234 'the GPU always materializes the most recent
    version'; SPEC.md host_cache freshness): the same lists, slot maps and
    counters as the flat host tier, and after the barrier the newest version of
    every block, read from the segment files through Index, equals the flat
    tier's table bitwise."""
    sc, ((flat, lf), (st, ls)) = _flat_and_store(tmp_path, moments, masked, H)
    assert lf == ls
    assert flat.stats() == st.stats()
    s = st.store_stats()
    assert s["dirty_evictions"] > 0 and s["flush_appends"] > 0 and s["cached_dirty"] == 0
    segs = read_segments(tmp_path)
    n_arr = 3 if moments == O.PERSIST else 1
    resident = set(flat.list("R").tolist())
    for k in range(sc.K):
        fid, off, size, ver = st.store_index(k)
        p = payload_at(segs, fid, off, size).reshape(n_arr, sc.B, 59)
        th, m, v = flat.read_block(k)
        assert np.array_equal(p[0].view(np.uint32), th.view(np.uint32)), k
        if n_arr == 3:
            assert np.array_equal(p[1].view(np.uint32), m.view(np.uint32)), k
            assert np.array_equal(p[2].view(np.uint32), v.view(np.uint32)), k
        a, b, c = st.read_block(k)
        assert np.array_equal(a, th) and (k in resident or n_arr == 1 or np.array_equal(b, m))


def test_index_recovers_from_segments_and_is_append_only(tmp_path):
    """SPEC.md recover_index: scanning the segments in file_id order, later
    records win, rebuilds the live Index; versions strictly increase per block;
    writes only append (offsets grow within a segment); each segment stays
    within its byte budget."""
    cfg, sc, tr = tiny()
    S = _pad(3 * sc.B * 59 * 4)
    budget = PAGE + 5 * (PAGE + S)  # five records per patch segment
    sc, ((flat, _), (st, _)) = _flat_and_store(tmp_path, O.PERSIST, False, 16, budget)
    segs = read_segments(tmp_path)
    assert len(segs) - 1 == st.store_stats()["segments"] >= 3
    idx = {k: (0, PAGE + k * S, 3 * sc.B * 59 * 4, 0) for k in range(sc.K)}
    for fid in sorted(segs):
        if fid == 0:
            continue
        raw_len = len(segs[fid][3])
        assert raw_len <= budget
        offs = [r[0] for r in segs[fid][2]]
        assert offs == sorted(offs)
        for off, gid, ver, n in segs[fid][2]:
            assert ver == idx[gid][3] + 1  # one version more than the previous write
            idx[gid] = (fid, off, n, ver)
    for k in range(sc.K):
        assert st.store_index(k) == idx[k], k


def test_frequently_reused_dirty_blocks_stay_in_cache(tmp_path):
    """'frequently reused dirty blocks may remain resident in
    CPU memory and are not immediately persisted to SSD' -- with a cache that
    holds the whole shard nothing is appended before the barrier; the barrier
    appends each dirty entry once, and only the blocks updated since are
    appended by the next one."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, cfg.capacity), sc.bounds(), fill=sc.fill_fn,
                 track_all=True)
    o.store_open(tmp_path, sc.K)
    lr = lr_3dgs()
    grad = synth_grad(W.SEEDS["grads"], sc.N, sc.B)
    run_tiny(o, tr, cfg.J, 20, lr, grad)
    s = o.store_stats()
    assert s["evictions"] == 0 and s["dirty_evictions"] == 0 and s["segments"] == 0
    # compulsory misses only: every cached block was read from SSD exactly once
    assert s["misses"] == s["cached"] and s["cached_dirty"] > 0
    o.flush()
    s1 = o.store_stats()
    assert s1["cached_dirty"] == 0 and s["cached_dirty"] <= s1["flush_appends"] <= s["cached"]
    assert s1["segments"] == 1
    o.activate(tr.batch_planes(20, cfg.J))
    o.step_adam(lr, grad=grad)
    A = set(o.list("A").tolist())
    o.flush()
    s2 = o.store_stats()
    assert s2["flush_appends"] - s1["flush_appends"] == len(A)


def test_conservation_through_the_store(tmp_path):
    """SPEC.md conservation: with every mask empty nothing is ever dirty, so no
    patch is written and every block, read through Index after the barrier,
    is byte-identical to the initial table -- across many SSD -> CPU -> GPU ->
    CPU -> SSD cycles of a small cache."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 8), sc.bounds(), fill=sc.fill_fn, track_all=True)
    o.store_open(tmp_path, 16)
    lr = lr_3dgs()
    empty = lambda k, t: np.zeros((sc.B + 31) // 32, np.uint32)
    grad = synth_grad(1, sc.N, sc.B)
    for planes in random_boxes(sc, 40):
        o.activate(planes)
        o.step_adam(lr, grad=grad, mask=empty)
    o.flush()
    s = o.store_stats()
    assert s["evictions"] > 10 and s["write_bytes"] == 0 and s["segments"] == 0
    segs = read_segments(tmp_path)
    assert list(segs) == [0]
    for k in range(sc.K):
        fid, off, size, ver = o.store_index(k)
        assert ver == 0
        p = payload_at(segs, fid, off, size).reshape(3, sc.B, 59)
        assert np.array_equal(p[0], sc.block_theta(k)) and not p[1:].any()


def test_store_errors(tmp_path):
    cfg, sc, tr = tiny()
    mk = lambda track: O.Oracle(O.make_config(sc.N, sc.B, cfg.capacity), sc.bounds(),
                                fill=sc.fill_fn, track_all=track)
    with pytest.raises(O.OracleError):          # pinned entries need H >= 2C (R27)
        mk(True).store_open(tmp_path, 2 * cfg.capacity - 1)
    with pytest.raises(O.OracleError):          # data mode needs every block's data
        mk(False).store_open(tmp_path, 2 * cfg.capacity)
    o = mk(True)
    o.activate(tr.batch_planes(0, cfg.J))
    with pytest.raises(O.OracleError):          # before the first activate only
        o.store_open(tmp_path, 2 * cfg.capacity)
    with pytest.raises(O.OracleError):          # segment budget below one record
        mk(True).store_open(tmp_path, 2 * cfg.capacity, 2 * PAGE)


def test_reopen_recovers_index_and_table(tmp_path):
    """R30 checkpoint/resume (SPEC.md recover_index 'random session replayed
    from disk -> index equals live index'): a new session over the files left
    by a barrier recovers every Index[k] and serves every block's newest
    version; a torn trailing record is dropped and cut off the segment; a store
    of another shape is refused."""
    cfg, sc, tr = tiny()
    S = _pad(3 * sc.B * 59 * 4)
    budget = PAGE + 4 * (PAGE + S)
    sc, ((flat, _), (st, _)) = _flat_and_store(tmp_path, O.PERSIST, False, 16, budget)
    live = {k: st.store_index(k) for k in range(sc.K)}
    table = {k: flat.read_block(k) for k in range(sc.K)}
    last = max(int(n[6:12]) for n in os.listdir(tmp_path) if n.startswith("patch-"))
    lp = tmp_path / f"patch-{last:06d}.tdgp"
    size = lp.stat().st_size
    with open(lp, "ab") as f:  # a record whose payload never made it to disk
        f.write(b"TREC" + b"\0" * 5000)
    o = O.Oracle(O.make_config(sc.N, sc.B, 8), sc.bounds(), fill=None, track_all=True)
    o.store_reopen(tmp_path, 16, budget)
    assert lp.stat().st_size == size
    for k in range(sc.K):
        assert o.store_index(k) == live[k], k
        th, m, v = o.read_block(k)
        assert np.array_equal(th.view(np.uint32), table[k][0].view(np.uint32)), k
        assert np.array_equal(m.view(np.uint32), table[k][1].view(np.uint32)), k
    # the resumed session keeps appending after the last whole record
    lr = lr_3dgs()
    grad = synth_grad(W.SEEDS["grads"], sc.N, sc.B)
    for planes in random_boxes(sc, 12, seed=21):
        o.activate(planes)
        o.step_adam(lr, grad=grad)
    o.flush()
    segs = read_segments(tmp_path)
    assert max(segs) >= last
    for k in range(sc.K):  # the parser (later records win) agrees with the live index
        fid, off, n, ver = o.store_index(k)
        assert ver >= live[k][3]
        if fid:
            assert (off, k, ver, n) in [(r[0], r[1], r[2], r[3]) for r in segs[fid][2]]
    bad = O.Oracle(O.make_config(sc.N, sc.B - 4, 8), W.Scene(sc.N, sc.B - 4).bounds(), fill=None,
                   track_all=True)
    with pytest.raises(O.OracleError):
        bad.store_reopen(tmp_path, 16, budget)


def test_compaction_keeps_every_newest_version(tmp_path):
    """R31 (SPEC.md log_store compact): after the barrier the
    patches merge into a new base -- every block's payload byte-identical to
    before, Index[k] = (0, base offset, size, same version), no patch segment
    left, the base the same size; training then appends from patch 1 with
    versions counting on.  Compaction with dirty data pending is refused."""
    cfg, sc, tr = tiny()
    S = _pad(3 * sc.B * 59 * 4)
    sc, ((flat, _), (st, _)) = _flat_and_store(tmp_path, O.PERSIST, False, 16, PAGE + 4 * (PAGE + S))
    before = read_segments(tmp_path)
    assert len(before) > 2
    idx = {k: st.store_index(k) for k in range(sc.K)}
    pay = {k: payload_at(before, *idx[k][:2], idx[k][2]).copy() for k in range(sc.K)}
    base_size = (tmp_path / "base.tdgs").stat().st_size
    st.store_compact()
    after = read_segments(tmp_path)
    assert list(after) == [0] and (tmp_path / "base.tdgs").stat().st_size == base_size
    for k in range(sc.K):
        fid, off, n, ver = st.store_index(k)
        assert (fid, off, n, ver) == (0, PAGE + k * S, idx[k][2], idx[k][3])
        assert np.array_equal(payload_at(after, 0, off, n), pay[k]), k
    lr = lr_3dgs()
    grad = synth_grad(W.SEEDS["grads"], sc.N, sc.B)
    for planes in random_boxes(sc, 10, seed=31):
        st.activate(planes)
        st.step_adam(lr, grad=grad)
    with pytest.raises(O.OracleError):  # dirty blocks on the GPU: barrier first
        st.store_compact()
    st.flush()
    segs = read_segments(tmp_path)
    assert 1 in segs
    for off, gid, ver, n in segs[1][2]:
        assert ver > idx[gid][3]


def test_crc32c_check_value():
    """R28 format 2 record checksum: CRC-32C's standard check value (the CRC of
    b"123456789" is 0xE3069283) for both the oracle's and this file's CRC."""
    assert O.crc32c(b"123456789") == crc32c(b"123456789") == 0xE3069283
    assert O.crc32c(b"") == crc32c(b"") == 0
    blob = bytes(range(256)) * 17
    assert O.crc32c(blob) == crc32c(blob)


def _session(d, sc, C, H, budget, batches, *, reopen=False, flush=True, o=None):
    lr = lr_3dgs()
    g = synth_grad(W.SEEDS["grads"], sc.N, sc.B)
    grad = lambda k, t: g(k, 0)  # noqa: E731 -- independent of the session's batch counter
    if o is None:
        o = O.Oracle(O.make_config(sc.N, sc.B, C, moments=O.PERSIST), sc.bounds(),
                     fill=None if reopen else sc.fill_fn, track_all=True)
        (o.store_reopen if reopen else o.store_open)(d, H, budget)
    for planes in batches:
        assert o.activate(planes) == O.OK
        assert o.list("K").size <= C  # A = K whatever the history (resume is exact)
        o.step_adam(lr, grad=grad)
    if flush:
        o.flush()
    return o


def _boxes(sc, n, seed):
    return [p for p in random_boxes(sc, 4 * n, seed=seed)][:n]


def test_resume_continues_exactly_and_drops_post_barrier_appends(tmp_path):
    """R30 resume = the barrier's state: a session that keeps
    training after a barrier and dies without another one leaves later patch
    records (dirty CPU-cache victims) behind; reopening recovers exactly the
    barrier's Index, contents and Adam step counters (the manifest bounds the
    log), removes the later records, and training resumed from there ends
    bit-identical to a session that never stopped (persist policy)."""
    cfg, sc, tr = tiny()
    C, H = 16, 32
    budget = PAGE + 6 * (PAGE + _pad(3 * sc.B * 59 * 4))
    first, extra, rest = _boxes(sc, 18, 41), _boxes(sc, 8, 42), _boxes(sc, 10, 43)
    a, b = tmp_path / "a", tmp_path / "b"
    # uninterrupted: first, barrier, rest, barrier
    oa = _session(a, sc, C, H, budget, first)
    _session(a, sc, C, H, budget, rest, o=oa)
    want = {k: oa.read_block(k) for k in range(sc.K)}
    want_steps = {k: oa.step_count(k) for k in range(sc.K)}
    # interrupted: first, barrier, extra (no barrier: appended victims only), "crash"
    ob = _session(b, sc, C, H, budget, first)
    at_barrier = {k: (ob.store_index(k), ob.read_block(k), ob.step_count(k)) for k in range(sc.K)}
    man = read_manifest(b)
    _session(b, sc, C, H, budget, extra, o=ob, flush=False)
    appended = sum(len(r[2]) for f, r in read_segments(b).items() if f) - \
        sum(len(r[2]) for f, r in read_segments(b).items() if f and f < man["last_file"])
    assert ob.store_stats()["dirty_evictions"] > 0 and appended > 0
    ob.close()
    oc = O.Oracle(O.make_config(sc.N, sc.B, C, moments=O.PERSIST), sc.bounds(), fill=None,
                  track_all=True)
    oc.store_reopen(b, H, budget)
    segs = read_segments(b)
    assert max(segs) == man["last_file"]
    if man["last_file"]:
        assert os.path.getsize(b / f"patch-{man['last_file']:06d}.tdgp") == man["end"]
    for k in range(sc.K):
        ix, blk, stp = at_barrier[k]
        assert oc.store_index(k) == ix, k
        assert oc.step_count(k) == stp, k
        for x, y in zip(oc.read_block(k), blk):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), k
    _session(b, sc, C, H, budget, rest, o=oc)
    for k in range(sc.K):
        assert oc.step_count(k) == want_steps[k], k
        for x, y in zip(oc.read_block(k), want[k]):
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), k


@pytest.mark.parametrize("where", ["payload", "header", "manifest"])
def test_corruption_inside_the_barrier_is_refused(tmp_path, where):
    """Every record up to the manifest's end was made durable at a barrier, so
    a bad CRC-32C there (payload or header) is corruption, not a torn tail: the
    resume refuses it, as it refuses a manifest that fails its own CRC."""
    cfg, sc, tr = tiny()
    C, H = 16, 32
    budget = PAGE + 6 * (PAGE + _pad(3 * sc.B * 59 * 4))
    o = _session(tmp_path, sc, C, H, budget, _boxes(sc, 14, 51))
    o.close()
    segs = read_segments(tmp_path)
    fid = min(f for f in segs if f)
    off = segs[fid][2][0][0]
    path, pos = {"payload": (tmp_path / f"patch-{fid:06d}.tdgp", off + 1000),
                 "header": (tmp_path / f"patch-{fid:06d}.tdgp", off - PAGE + 9),
                 "manifest": (tmp_path / "manifest.tdgm", 70)}[where]
    raw = bytearray(open(path, "rb").read())
    raw[pos] ^= 0x40
    open(path, "wb").write(bytes(raw))
    r = O.Oracle(O.make_config(sc.N, sc.B, C, moments=O.PERSIST), sc.bounds(), fill=None,
                 track_all=True)
    with pytest.raises(O.OracleError):
        r.store_reopen(tmp_path, H, budget)


def test_compaction_then_resume_keeps_versions(tmp_path):
    """R31 + R30: the manifest written by a compaction carries every block's
    version, so a session resumed after it sees Index[k] = (0, base offset,
    size, the version before compaction) and versions keep increasing."""
    cfg, sc, tr = tiny()
    C, H = 16, 32
    S = _pad(3 * sc.B * 59 * 4)
    budget = PAGE + 6 * (PAGE + S)
    o = _session(tmp_path, sc, C, H, budget, _boxes(sc, 14, 61))
    vers = {k: o.store_index(k)[3] for k in range(sc.K)}
    assert max(vers.values()) > 0
    o.store_compact()
    m = read_manifest(tmp_path)
    assert m["last_file"] == 0 and m["end"] == 0
    assert [int(x) for x in m["base_version"]] == [vers[k] for k in range(sc.K)]
    o.close()
    r = O.Oracle(O.make_config(sc.N, sc.B, C, moments=O.PERSIST), sc.bounds(), fill=None,
                 track_all=True)
    r.store_reopen(tmp_path, H, budget)
    for k in range(sc.K):
        assert r.store_index(k) == (0, PAGE + k * S, 3 * sc.B * 59 * 4, vers[k]), k
