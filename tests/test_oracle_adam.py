"""Pins for the oracle's masked Adam and the out-of-core data path
(PAPER.md:717-727 Eq. masked_update, 325-331 cold restart, 240-251 write-back;
SPEC.md:494-498, 556-564)."""
import numpy as np
import pytest

import oracle as O
import workload as W
from helpers import lr_3dgs, mask_rows, synth_grad, synth_mask, tiny

B = 8
ALL = np.zeros((1, 6, 4), np.float32)
ALL[0] = [[1, 0, 0, 1e3], [-1, 0, 0, 1e3], [0, 1, 0, 1e3], [0, -1, 0, 1e3], [0, 0, 1, 1e3],
          [0, 0, -1, 1e3]]
NONE = np.zeros((0, 6, 4), np.float32)


def _one_block(theta0, moments=O.PERSIST, C=1, nblocks=1):
    bounds = np.tile(np.array([[0, 0, 0, 1]], np.float32), (nblocks, 1))
    bounds[:, 0] = np.arange(nblocks) * 10.0
    return O.Oracle(O.make_config(B * nblocks, B, C, moments=moments), bounds,
                    fill=lambda k: theta0 + k, track_all=True)


def _only(k):
    p = ALL.copy()
    p[0, 0, 3] = -(10.0 * k - 1)
    p[0, 1, 3] = 10.0 * k + 1
    return p


def test_constant_gradient_closed_form():
    """Constant g from zero state: m_hat = g, v_hat = g^2 exactly in real
    arithmetic, so every step moves theta by -lr g/(|g|+eps) (Kingma & Ba)."""
    theta0 = np.full((B, 59), 1.0, np.float32)
    o = _one_block(theta0)
    lr = np.full(59, 1e-3, np.float32)
    g = np.full((B, 59), 0.25, np.float32)
    g[:, ::2] = -0.5
    for s in range(1, 11):
        o.activate(ALL)
        assert o.step_adam(lr, 0.9, 0.999, 1e-8, grad=lambda k, t: g) == O.OK
        th, m, v = o.read_block(0)
        exp = 1.0 - s * 1e-3 * np.sign(g) * np.abs(g) / (np.abs(g) + 1e-8)
        np.testing.assert_allclose(th, exp, rtol=2e-6 * s, atol=0)
        np.testing.assert_allclose(m, g * (1 - 0.9 ** s), rtol=1e-5)
        np.testing.assert_allclose(v, g * g * (1 - 0.999 ** s), rtol=1e-4)
    assert o.step_count(0) == 10


def test_matches_double_textbook_adam_varying_gradient():
    """Scalar Adam trajectory against the textbook algorithm evaluated in
    double: m_hat = m/(1-b1^t), v_hat = v/(1-b2^t), theta -= lr m_hat/(sqrt(v_hat)+eps)."""
    rng = np.random.default_rng(3)
    theta0 = rng.standard_normal((B, 59)).astype(np.float32)
    o = _one_block(theta0)
    lr = lr_3dgs()
    gs = [rng.standard_normal((B, 59)).astype(np.float32) * 1e-3 for _ in range(25)]
    th_d = theta0.astype(np.float64)
    m_d = np.zeros_like(th_d)
    v_d = np.zeros_like(th_d)
    b1, b2, eps = 0.9, 0.999, 1e-15
    for t, g in enumerate(gs, 1):
        o.activate(ALL)
        o.step_adam(lr, b1, b2, eps, grad=lambda k, tt, g=g: g)
        gd = g.astype(np.float64)
        m_d = b1 * m_d + (1 - b1) * gd
        v_d = b2 * v_d + (1 - b2) * gd * gd
        th_d = th_d - lr.astype(np.float64) * (m_d / (1 - b1 ** t)) / (
            np.sqrt(v_d / (1 - b2 ** t)) + eps)
    th, m, v = o.read_block(0)
    np.testing.assert_allclose(th, th_d, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(m, m_d, rtol=1e-4, atol=1e-12)
    np.testing.assert_allclose(v, v_d, rtol=1e-4, atol=1e-16)


def test_zero_gradient_and_masked_rows_bitwise_unchanged():
    """g = 0 from zero state moves nothing; rows outside I_t keep theta, m, v
    bitwise (Eq. masked_update)."""
    rng = np.random.default_rng(1)
    theta0 = rng.standard_normal((B, 59)).astype(np.float32)
    o = _one_block(theta0)
    lr = np.full(59, 1e-2, np.float32)
    o.activate(ALL)
    o.step_adam(lr, grad=lambda k, t: np.zeros((B, 59), np.float32))
    th, m, v = o.read_block(0)
    assert np.array_equal(th.view(np.uint32), theta0.view(np.uint32))
    assert not m.any() and not v.any()
    word = np.array([0b10110010], np.uint32)
    keep = ~mask_rows(word, B)
    for _ in range(5):
        o.activate(ALL)
        o.step_adam(lr, grad=lambda k, t: rng.standard_normal((B, 59)).astype(np.float32),
                    mask=lambda k, t: word)
    th2, m2, v2 = o.read_block(0)
    assert np.array_equal(th2[keep].view(np.uint32), th[keep].view(np.uint32))
    assert not m2[keep].any() and not v2[keep].any()
    assert (th2[~keep] != th[~keep]).all()


def test_empty_active_set_no_dirty_no_step():
    """Empty I_t: nothing dirtied, step unchanged, no write-back."""
    theta0 = np.ones((B, 59), np.float32)
    o = _one_block(theta0, nblocks=2, C=1)
    lr = np.full(59, 1e-2, np.float32)
    o.activate(_only(0))
    o.step_adam(lr, grad=lambda k, t: np.ones((B, 59), np.float32),
                mask=lambda k, t: np.zeros(1, np.uint32))
    assert o.step_count(0) == 0
    o.activate(_only(1))        # evicts block 0 (clean)
    assert o.list("S-").tolist() == [0] and o.stats()["d2h_bytes"] == 0
    o.step_adam(lr, grad=lambda k, t: np.ones((B, 59), np.float32))
    o.activate(_only(0))        # evicts block 1 (dirty)
    assert o.stats()["d2h_bytes"] == B * 59 * 4 * 3
    assert o.evicted_dirty().tolist() == [1]


@pytest.mark.parametrize("moments", [O.PERSIST, O.COLD_RESTART])
def test_readmission_restarts_or_keeps_state(moments):
    """Cold restart: after eviction and re-admission the next update is a first
    Adam step, |dtheta| = lr |g|/(|g|+eps), step counter 1 (
    SPEC.md:494, 564).  Persist: moments and step survive the round trip."""
    theta0 = np.zeros((B, 59), np.float32)
    o = _one_block(theta0, moments=moments, nblocks=2, C=1)
    lr = np.full(59, 1e-3, np.float32)
    g = np.full((B, 59), 0.5, np.float32)
    for _ in range(3):
        o.activate(_only(0))
        o.step_adam(lr, 0.9, 0.999, 1e-8, grad=lambda k, t: g)
    o.activate(_only(1))
    o.activate(_only(0))
    th_before, m_before, _ = o.read_block(0)
    o.step_adam(lr, 0.9, 0.999, 1e-8, grad=lambda k, t: -g)
    th, m, v = o.read_block(0)
    d = th - th_before
    if moments == O.COLD_RESTART:
        assert not m_before.any()
        assert o.step_count(0) == 1
        np.testing.assert_allclose(d, 1e-3 * 0.5 / (0.5 + 1e-8), rtol=1e-5)
        # first step from m = 0: m = (1 - beta1) g with 1 - beta1 formed in fp32
        np.testing.assert_array_equal(m, (np.float32(1) - np.float32(0.9)) * np.float32(-0.5))
    else:
        assert o.step_count(0) == 4
        assert m_before.any()
        assert np.all(np.abs(d) < 0.5e-3)   # momentum from +g dampens the -g step


def test_nonfinite_gradient_row_skipped_and_reported():
    """R20: a non-finite g in an active row skips that row and reports the
    lowest (gid*59 + attr)."""
    theta0 = np.ones((B, 59), np.float32)
    o = _one_block(theta0)
    g = np.full((B, 59), 0.1, np.float32)
    g[3, 7] = np.nan
    g[5, 2] = np.inf
    o.activate(ALL)
    rc = o.step_adam(np.full(59, 1e-2, np.float32), grad=lambda k, t: g)
    assert rc == O.ENONFINITE
    assert o.nonfinite_index() == 3 * 59 + 7
    th, _, _ = o.read_block(0)
    assert (th[3] == 1).all() and (th[5] == 1).all() and (th[0] != 1).all()


def _in_memory_reference(sc, its, lr, b1, b2, eps, grad, mask, cold):
    """Monolithic in-memory masked Adam over the full table, driven by the
    effective (A_t, S+_t) sequence; numpy fp32 ops in the R9 order."""
    K, Bs = sc.K, sc.B
    th = sc.table()[: K * Bs].reshape(K, Bs, 59).copy()
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    step = np.zeros(K, np.int64)
    f32 = np.float32
    omb1, omb2 = f32(1) - f32(b1), f32(1) - f32(b2)
    for t, (A, Sp) in enumerate(its):
        if cold:
            for k in Sp:
                m[k] = 0
                v[k] = 0
                step[k] = 0
        for k in A:
            rows = sc.rows(k)
            act = np.zeros(Bs, bool)
            act[:rows] = True
            if mask is not None:
                act &= mask_rows(mask(k, t), Bs)
            if not act.any():
                continue
            step[k] += 1
            G = grad(k, t)
            # bias corrections use the fp32 hyper-parameter value promoted to double
            bc1 = f32(1.0 - float(f32(b1)) ** float(step[k]))
            bc2 = f32(1.0 - float(f32(b2)) ** float(step[k]))
            ibs = f32(1) / np.sqrt(bc2)
            mt = f32(b1) * m[k][act] + omb1 * G[act]
            vt = f32(b2) * v[k][act] + omb2 * (G[act] * G[act])
            den = np.sqrt(vt) * ibs + f32(eps)
            ss = lr / bc1
            th[k][act] = th[k][act] - ss * (mt / den)
            m[k][act] = mt
            v[k][act] = vt
    return th, m, v, step


@pytest.mark.parametrize("C,moments,masked", [(64, O.PERSIST, False), (20, O.PERSIST, True),
                                              (14, O.COLD_RESTART, False)])
def test_transparency_against_in_memory_run(C, moments, masked):
    """SPEC.md:498/687 transparency: the flushed out-of-core table equals a
    monolithic in-memory masked-Adam run over the same effective sequence,
    bitwise, for any capacity (cold mode: moments reset at each admission)."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, C, moments=moments), sc.bounds(), fill=sc.fill_fn,
                 track_all=True)
    lr = lr_3dgs()
    grad = synth_grad(W.SEEDS["grads"], sc.N, sc.B)
    mask = synth_mask(W.SEEDS["mask"], sc.N, sc.B, 1 << 30) if masked else None
    its = []
    for t in range(14):
        o.activate(tr.batch_planes(t, cfg.J))
        its.append((o.list("A").tolist(), o.list("S+").tolist()))
        o.step_adam(lr, 0.9, 0.999, 1e-15, grad=grad, mask=mask)
    o.flush()
    th, m, v, step = _in_memory_reference(sc, its, lr, 0.9, 0.999, 1e-15, grad, mask,
                                          moments == O.COLD_RESTART)
    resident = set(o.list("R").tolist())
    touched = 0
    for k in range(sc.K):
        a, b, c = o.read_block(k)
        assert np.array_equal(a.view(np.uint32), th[k].view(np.uint32)), k
        if moments == O.PERSIST or k in resident:
            assert np.array_equal(b.view(np.uint32), m[k].view(np.uint32)), k
            assert np.array_equal(c.view(np.uint32), v[k].view(np.uint32)), k
        assert o.step_count(k) == step[k] or moments == O.COLD_RESTART
        touched += step[k] > 0
    assert touched > 10


def test_conservation_with_empty_masks():
    """Conservation: with every mask empty, after any activate sequence plus
    flush the host table is byte-identical to the initial one."""
    cfg, sc, tr = tiny()
    o = O.Oracle(O.make_config(sc.N, sc.B, 12), sc.bounds(), fill=sc.fill_fn, track_all=True)
    zero = np.zeros((sc.B + 31) // 32, np.uint32)
    for t in range(20):
        o.activate(tr.batch_planes(t, cfg.J))
        o.step_adam(lr_3dgs(), grad=synth_grad(1, sc.N, sc.B), mask=lambda k, t: zero)
    o.flush()
    st = o.stats()
    assert st["d2h_bytes"] == 0 and st["flush_bytes"] == 0 and st["n_stage_in"] > 12
    for k in range(sc.K):
        th, m, v = o.read_block(k)
        assert np.array_equal(th.view(np.uint32), sc.block_theta(k).view(np.uint32))
        assert not m.any() and not v.any()


def test_call_order_and_config_errors():
    theta0 = np.ones((B, 59), np.float32)
    o = _one_block(theta0)
    assert o.step_adam(np.ones(59, np.float32)) == O.ESTATE       # before activate
    o.activate(ALL)
    assert o.step_adam(np.ones(59, np.float32), grad=lambda k, t: np.zeros((B, 59), np.float32)) == O.OK
    assert o.step_adam(np.ones(59, np.float32)) == O.ESTATE       # twice
    bounds = np.zeros((1, 4), np.float32)
    for bad in (dict(lam=1.5), dict(gamma=1.0), dict(quota=(3, 2))):
        with pytest.raises(O.OracleError):
            O.Oracle(O.make_config(8, 8, 1, **bad), bounds)
    with pytest.raises(O.OracleError):
        O.Oracle(O.make_config(8, 6, 1), bounds)                  # B % 4 != 0
