"""Pins for the oracle's Tide residency selection, set differences, slot map and
byte accounting (Alg. 1)."""
import numpy as np
import pytest

import oracle as O
import workload as W
from helpers import tiny

REC4096 = 4096 * 59 * 4


def _run(o, tr, J, n):
    for t in range(n):
        R_prev = o.list("R").tolist()
        assert o.activate(tr.batch_planes(t, J)) == O.OK
        yield t, R_prev


@pytest.mark.parametrize("tide", [1, 0])
@pytest.mark.parametrize("lam,quota", [(0.7, (1, 2)), (0.0, (1, 2)), (1.0, (0, 1)), (0.5, (1, 2))])
def test_set_identities_and_capacity(tide, lam, quota):
    """Omega u S+ = R_{t+1}, Omega u S- = R_t (tide on), S+ n R_t = {},
    S- n R_{t+1} = {}, |R| <= C."""
    cfg, sc, tr = tiny()
    C = cfg.capacity
    o = O.Oracle(O.make_config(sc.N, sc.B, C, lam=lam, quota=quota, tide=tide), sc.bounds(),
                 fill=None, track_all=False)
    for t, R_prev in _run(o, tr, cfg.J, 24):
        R = set(o.list("R").tolist())
        Sp, Sm, Om = (set(o.list(x).tolist()) for x in ("S+", "S-", "Omega"))
        assert len(R) <= C
        if tide:
            assert Om | Sp == R and not (Om & Sp)
            assert Om | Sm == set(R_prev) and not (Om & Sm)
            assert not (Sp & set(R_prev)) and not (Sm & R)
        else:  # restage everything
            assert Sp == R and Sm == set(R_prev) and not Om
            assert R <= set(o.list("K").tolist())
        A = set(o.list("A").tolist())
        assert A == R & set(o.list("K").tolist())


def test_no_selection_when_pool_fits():
    """#C_t <= C => R_{t+1} = R_t u K_{t+1}."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 64), sc.bounds(), fill=None, track_all=False)
    R = set()
    for t, _ in _run(o, tr, cfg.J, 16):
        R = R | set(o.list("K").tolist())
        assert set(o.list("R").tolist()) == R
    assert len(R) <= 64


def test_static_view_zero_traffic():
    """K_{t+1} = R_t, C >= |R_t| => S+ = S- = {}."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 40), sc.bounds(), fill=None, track_all=False)
    pl = tr.batch_planes(3, cfg.J)
    o.activate(pl)
    first = o.list("S+").size
    assert first == o.list("R").size > 0
    for _ in range(5):
        o.activate(pl)
        assert o.list("S+").size == 0 and o.list("S-").size == 0
    st = o.stats()
    assert st["h2d_bytes"] == first * sc.B * 59 * 4 * 3


def test_lru_special_case_matches_textbook_lru():
    """lam in (0.5, 1], beta = 0: every K_{t+1} block outranks every non-K block,
    and non-K residents rank by last access (Recency = gamma^age is monotone), so
    the policy is a textbook LRU cache that must hold K_{t+1}.  Simulated here
    independently with an explicit last-use table."""
    cfg, sc, tr = tiny()
    C = 34  # >= max |K_t| on this trajectory so all of K_{t+1} fits
    o = O.Oracle(O.make_config(sc.N, sc.B, C, lam=0.8, quota=(0, 1)), sc.bounds(), fill=None,
                 track_all=False)
    R, last_use, A_prev = set(), {}, set()
    for t in range(40):
        o.activate(tr.batch_planes(t, cfg.J))
        K = set(o.list("K").tolist())
        assert len(K) <= C
        for k in A_prev:                      # accessed = resident and visible
            last_use[k] = t - 1
        pool = R | K
        if len(pool) <= C:
            Rn = pool
        else:
            others = sorted(R - K, key=lambda k: (-last_use.get(k, -10**9), k))
            Rn = K | set(others[: C - len(K)])
        assert set(o.list("R").tolist()) == Rn, t
        R = Rn
        A_prev = R & K


def test_lambda_one_keeps_next_working_set():
    """lam = 1 and |K_{t+1}| <= C => K_{t+1} subset of R_{t+1}."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 32, lam=1.0, quota=(0, 1)), sc.bounds(), fill=None,
                 track_all=False)
    for t, _ in _run(o, tr, cfg.J, 20):
        K = set(o.list("K").tolist())
        if len(K) <= 32:
            assert K <= set(o.list("R").tolist())


def test_quota_coverage():
    """Each camera keeps >= q_j = min(|K^{(j)}|, floor(beta C / J)) of its blocks
    (R10)."""
    cfg, sc, tr = tiny()
    for lam in (0.0, 0.3, 0.7):
        C = 12
        o = O.Oracle(O.make_config(sc.N, sc.B, C, lam=lam, quota=(1, 2)), sc.bounds(),
                     fill=None, track_all=False)
        for t, _ in _run(o, tr, 4, 12):
            R = set(o.list("R").tolist())
            q = (C * 1) // (2 * 4)
            for j in range(4):
                kj = set(o.percam(j).tolist())
                assert len(kj & R) >= min(len(kj), q)


def test_quota_example_spec():
    """J=2 cameras with 10 disjoint blocks each, C=10, uniform
    scores -> each camera gets >= floor(beta C / J) = 2 blocks."""
    xs = np.arange(20, dtype=np.float32)
    bounds = np.stack([xs, np.zeros(20), np.zeros(20), np.full(20, 0.1)], 1).astype(np.float32)
    def slab(lo, hi):
        p = np.zeros((6, 4), np.float32)
        p[0] = [1, 0, 0, -lo]
        p[1] = [-1, 0, 0, hi]
        p[2] = [0, 1, 0, 5]
        p[3] = [0, -1, 0, 5]
        p[4] = [0, 0, 1, 5]
        p[5] = [0, 0, -1, 5]
        return p
    # camera 1 sees 10..19 with higher id, so a pure Top-C by id would starve it
    o = O.Oracle(O.make_config(80, 4, 10, lam=0.7, quota=(1, 2)), bounds, fill=None,
                 track_all=False)
    o.activate(np.stack([slab(-0.5, 9.5), slab(9.5, 19.5)]))
    R = set(o.list("R").tolist())
    assert len(R) == 10
    assert len(R & set(range(0, 10))) >= 2 and len(R & set(range(10, 20))) >= 2
    # beta = 0: pure global Top-C by (score, resident, id) -> lowest ids
    o2 = O.Oracle(O.make_config(80, 4, 10, lam=0.7, quota=(0, 1)), bounds, fill=None,
                  track_all=False)
    o2.activate(np.stack([slab(-0.5, 9.5), slab(9.5, 19.5)]))
    assert o2.list("R").tolist() == list(range(10))


def test_exact_score_tie_lambda_half():
    """lam = 0.5: (in K_{t+1}, never accessed) scores 0.5 = (not in K, age 0);
    the tie goes to the resident block (R11), then the lower id."""
    xs = np.arange(4, dtype=np.float32)
    bounds = np.stack([xs, np.zeros(4), np.zeros(4), np.full(4, 0.1)], 1).astype(np.float32)
    def slab(lo, hi):
        p = np.zeros((6, 4), np.float32)
        p[0] = [1, 0, 0, -lo]; p[1] = [-1, 0, 0, hi]
        p[2] = [0, 1, 0, 5]; p[3] = [0, -1, 0, 5]; p[4] = [0, 0, 1, 5]; p[5] = [0, 0, -1, 5]
        return p
    o = O.Oracle(O.make_config(16, 4, 2, lam=0.5, quota=(0, 1)), bounds, fill=None,
                 track_all=False)
    o.activate(slab(-0.5, 1.5)[None])    # t=0: K={0,1} -> R={0,1}
    o.activate(slab(-0.5, 1.5)[None])    # t=1: accessed {0,1}
    o.activate(slab(1.5, 3.5)[None])     # t=2: K={2,3}; 0,1 have age 0 -> 0.5; 2,3 never -> 0.5
    assert o.list("R").tolist() == [0, 1]
    o3 = O.Oracle(O.make_config(16, 4, 2, lam=0.51, quota=(0, 1)), bounds, fill=None,
                  track_all=False)
    for p in (slab(-0.5, 1.5), slab(-0.5, 1.5), slab(1.5, 3.5)):
        o3.activate(p[None])
    assert o3.list("R").tolist() == [2, 3]   # 0.51 > 0.49


def test_recency_orders_by_age_gamma():
    """Recency = gamma^age: with lam = 0 the block accessed
    more recently wins; a never-accessed block loses to any accessed one."""
    xs = np.arange(3, dtype=np.float32)
    bounds = np.stack([xs, np.zeros(3), np.zeros(3), np.full(3, 0.1)], 1).astype(np.float32)
    def only(k):
        p = np.zeros((6, 4), np.float32)
        p[0] = [1, 0, 0, -(k - 0.5)]; p[1] = [-1, 0, 0, k + 0.5]
        p[2] = [0, 1, 0, 5]; p[3] = [0, -1, 0, 5]; p[4] = [0, 0, 1, 5]; p[5] = [0, 0, -1, 5]
        return p[None]
    o = O.Oracle(O.make_config(12, 4, 2, lam=0.0, quota=(0, 1)), bounds, fill=None,
                 track_all=False)
    o.activate(only(0))       # t0: R={0}
    o.activate(only(1))       # t1: 0 accessed at t0; R={0,1}
    o.activate(only(1))       # t2: 1 accessed at t1
    o.activate(only(2))       # t3: cand {0,1,2}: ages 0:2, 1:0, 2:never -> keep {0,1}
    assert o.list("R").tolist() == [0, 1]
    o.activate(only(2))       # t4: none accessed at t3 (2 not resident); 0 age 3, 1 age 1
    assert o.list("R").tolist() == [0, 1]


def test_slot_map_invariants_and_rule():
    """Slot map injective; Omega keeps its slots; |free| = P - |R|; S+ takes the
    lowest slots not held by R_t (R13, parity unpinned w.r.t. the paper)."""
    cfg, sc, tr = tiny()
    C, P = cfg.capacity, 30
    o = O.Oracle(O.make_config(sc.N, sc.B, C, pool_slots=P), sc.bounds(), fill=None,
                 track_all=False)
    prev_map = None
    for t in range(30):
        prev_R_slots = {} if prev_map is None else {int(b): s for s, b in enumerate(prev_map) if b >= 0}
        o.activate(tr.batch_planes(t, cfg.J))
        smap = o.slot_map()
        held = smap[smap >= 0]
        assert len(set(held.tolist())) == len(held) == o.list("R").size
        for b, s in zip(*o.list("Omega", with_slots=True)):
            assert prev_R_slots[int(b)] == s
        sp_b, sp_s = o.list("S+", with_slots=True)
        free_before = [s for s in range(P) if s not in prev_R_slots.values()]
        if len(free_before) >= len(sp_b):
            assert sp_s.tolist() == free_before[: len(sp_b)]
        prev_map = smap


def test_moved_bytes_closed_form_and_format_constants():
    """record = 4096*59*4 = 966,656 B = 236 pages;
    K = ceil(N/B) with a truncated last block; h2d = |S+| rec n_arr,
    d2h = |S- dirty| rec n_arr."""
    assert REC4096 == 966_656 == 236 * 4096
    n = 10_000  # N=10000, B=4096 -> K=3, gaussian 9999 -> block 2
    bounds = np.array([[0, 0, 0, 1], [5, 0, 0, 1], [10, 0, 0, 1]], np.float32)
    big = np.zeros((1, 6, 4), np.float32)
    big[0, :, :] = [[1, 0, 0, 100], [-1, 0, 0, 100], [0, 1, 0, 100], [0, -1, 0, 100],
                    [0, 0, 1, 100], [0, 0, -1, 100]]
    for moments, n_arr in ((O.PERSIST, 3), (O.COLD_RESTART, 1)):
        o = O.Oracle(O.make_config(n, 4096, 3, moments=moments), bounds,
                     fill=lambda k: np.zeros((4096, 59), np.float32), track_all=True)
        o.activate(big)
        assert o.list("S+").tolist() == [0, 1, 2]
        assert o.stats()["h2d_bytes"] == 3 * REC4096 * n_arr
        lr = np.full(59, 1e-3, np.float32)
        o.step_adam(lr, grad=lambda k, t: np.ones((4096, 59), np.float32))
        o.activate(np.zeros((0, 6, 4), np.float32))   # R unchanged (R19)
        assert o.stats()["d2h_bytes"] == 0
        o.flush()
        assert o.stats()["flush_bytes"] == 3 * REC4096 * n_arr
        assert o.stats()["n_active_rows"] == 10_000   # last block truncated at N


def test_churn_counters_consistent():
    """SPEC.md:508 definitions, counted independently here from the per-iteration
    sets; and the paper's T9 consistency (18.7 x 4.8% = 0.90,
    13.4 x 6.9% = 0.92): with the mean resident streak taken over all streaks
    (ongoing ones included, = sum_t |R_t| / admissions by Little's law), streak x
    eviction rate = evictions / admissions, ~1 on a stationary workload."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 20, moments=O.COLD_RESTART), sc.bounds(),
                 fill=None, track_all=False)
    lr = np.full(59, 1e-3, np.float32)
    evicted, readmit, cold_updates = set(), 0, 0
    fresh, admitted_at = set(), {}
    streak_sum = streak_cnt = 0
    T = 160
    for t in range(T):
        o.activate(tr.batch_planes(t, cfg.J))
        for k in o.list("S-").tolist():
            evicted.add(k)
            streak_sum += t - admitted_at.pop(k)
            streak_cnt += 1
            fresh.discard(k)
        for k in o.list("S+").tolist():
            admitted_at[k] = t
            if k in evicted:
                readmit += 1
                fresh.add(k)
        o.step_adam(lr, grad=lambda k, t: np.zeros((sc.B, 59), np.float32))
        for k in o.list("A").tolist():
            if k in fresh:
                cold_updates += 1
                fresh.discard(k)
    st = o.stats()
    assert st["readmissions"] == readmit > 0
    assert st["cold_restart_updates"] == cold_updates > 0
    assert st["resident_streak_sum"] == streak_sum and st["streak_count"] == streak_cnt
    ev_rate = st["n_evict"] / st["n_resident"]
    mean_streak = st["n_resident"] / st["n_stage_in"]
    assert 0.8 <= mean_streak * ev_rate <= 1.2, (mean_streak, ev_rate)
    assert 0.8 <= 18.7 * 0.048 <= 1.2 and 0.8 <= 13.4 * 0.069 <= 1.2


def test_consecutive_k_locality_counters():
    """k_inter_sum / k_union_sum = sum over activates of |K_t n K_{t+1}| and
    |K_t u K_{t+1}| (the consecutive-batch Jaccard the bench reports):
    recomputed from the K lists; a repeated batch adds |K| to both (Jaccard 1),
    an empty batch adds 0 and |K_t|."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, cfg.capacity), sc.bounds(), fill=None,
                 track_all=False)
    prev, inter, union = set(), 0, 0
    batches = [tr.batch_planes(t, cfg.J) for t in range(10)]
    batches += [batches[-1], np.zeros((0, 6, 4), np.float32), batches[3]]
    for pl in batches:
        assert o.activate(pl) == O.OK
        K = set(o.list("K").tolist())
        inter += len(prev & K)
        union += len(prev | K)
        st = o.stats()
        assert (st["k_inter_sum"], st["k_union_sum"]) == (inter, union)
        prev = K
    assert 0 < inter < union
