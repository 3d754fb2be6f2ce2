"""Drives the CUDA path (through the C ABI binding) and the CPU oracle on the
same seeded inputs, step by step, and compares them (tests only)."""
from __future__ import annotations

import ctypes as C

import numpy as np

import oracle as O
import workload as W
from helpers import lr_3dgs

DIM = 59
GRAD_SEED, MASK_SEED = W.SEEDS["grads"], W.SEEDS["mask"]


class Synth(C.Structure):
    """wl_synth of tgs_workload.h (oracle-side gradient / mask callbacks)."""
    _fields_ = [("seed", C.c_uint64), ("n_gaussians", C.c_uint64), ("block_size", C.c_uint32),
                ("p32", C.c_uint32)]


def _cfn(name):
    return C.cast(getattr(W.lib(), name), C.c_void_p).value


class Pair:
    """One GPU table + one oracle shard fed the same config, bounds, planes,
    gradients and masks."""

    def __init__(self, scene, *, capacity, pool_slots=0, max_cameras=256, max_age=255,
                 quota=(1, 2), lam=0.7, gamma=0.9, moments=O.PERSIST, tide=1, world_size=1,
                 rank=0, track_all=True, mask_p=None, staging_blocks=0, refresh_bounds=0,
                 bounds=None, fill=None, store=None, level2=0, xfer=0):
        """store (NEXT f3): dict(gpu_dir, orc_dir, cache_blocks, segment_bytes=0,
        direct_io=0) -- the GPU table and the oracle each get their own store
        directory (orc_dir None: oracle metadata only)."""
        import torch
        from paper_2605_20150_b200 import tidegs as T

        self.torch = torch
        self.scene = scene
        self.B, self.N = scene.B, scene.N
        kw = dict(pool_slots=pool_slots, max_cameras=max_cameras, max_age=max_age, quota=quota,
                  lam=lam, gamma=gamma, moments=moments, tide=tide, world_size=world_size,
                  rank=rank)
        bounds = scene.bounds() if bounds is None else bounds
        fill = scene.fill_fn if fill is None else fill
        gstore = None
        if store is not None:
            gstore = dict(dir=store["gpu_dir"], cache_blocks=store["cache_blocks"],
                          segment_bytes=store.get("segment_bytes", 0),
                          direct_io=store.get("direct_io", 0), reopen=store.get("reopen", 0),
                          prefetch_blocks=store.get("prefetch_blocks", 0))
        self.gpu = T.Table(T.make_config(scene.N, scene.B, capacity, staging_blocks=staging_blocks,
                                         refresh_bounds=refresh_bounds, level2=level2, xfer=xfer,
                                         **kw),
                           bounds,
                           fill=fill, store=gstore)
        self.orc = O.Oracle(O.make_config(scene.N, scene.B, capacity, refresh_bounds=refresh_bounds,
                                          **kw), bounds, fill=fill, track_all=track_all)
        self.store = store
        if store is not None:
            (self.orc.store_reopen if store.get("reopen") else self.orc.store_open)(
                store.get("orc_dir"), store["cache_blocks"], store.get("segment_bytes", 0))
        self.gsyn = Synth(GRAD_SEED, scene.N, scene.B, 0)
        self.mask_p = mask_p
        self.msyn = None
        self.d_mask = None
        if mask_p is not None:
            p32 = min(int(mask_p * 2**32), 2**32 - 1)
            self.msyn = Synth(MASK_SEED, scene.N, scene.B, p32)
            self.d_mask = torch.zeros((self.gpu.P, (scene.B + 31) // 32), dtype=torch.int32,
                                      device="cuda")
        self.t = 0
        self.lr = lr_3dgs()
        self.stream = torch.cuda.current_stream().cuda_stream

    def activate(self, planes):
        a = self.gpu.activate(planes)
        assert self.orc.activate(planes) == O.OK
        return a

    def grads_gpu(self, act, t):
        W.synth_grads_cuda(act, self.B, self.N, GRAD_SEED, t, self.stream)
        if self.d_mask is not None:
            W.synth_mask_cuda(self.d_mask.data_ptr(), act, self.B, self.N, MASK_SEED, t,
                              self.msyn.p32, self.stream)

    def step(self, act, t, *, grad_hook=None, oracle_grad=None, beta1=0.9, beta2=0.999,
             eps=1e-15):
        """Adam on both sides with the shared counter gradients for batch t.
        grad_hook(act) may edit the device gradients after they are written."""
        self.grads_gpu(act, t)
        if grad_hook is not None:
            grad_hook(act)
        mptr = self.d_mask.data_ptr() if self.d_mask is not None else None
        self.gpu.step_adam(self.lr, beta1, beta2, eps, mask_ptr=mptr)
        g = oracle_grad or (_cfn("wl_grad_cb"), C.addressof(self.gsyn))
        m = (_cfn("wl_mask_cb"), C.addressof(self.msyn)) if self.msyn is not None else None
        return self.orc.step_adam(self.lr, beta1, beta2, eps, grad=g, mask=m)

    def step_fine(self, act, t):
        """Level-2 filter (f1) -> I_t mask on both sides, compared bit-exact per
        A block, then masked Adam with it."""
        torch = self.torch
        if self.d_mask is None:
            self.d_mask = torch.zeros((self.gpu.P, (self.B + 31) // 32), dtype=torch.int32,
                                      device="cuda")
        self.gpu.fine_filter(self.d_mask.data_ptr())
        torch.cuda.synchronize()
        host = self.d_mask.cpu().numpy().view(np.uint32)
        blocks, slots = self.orc.list("A", with_slots=True)
        n_rows = 0
        for k, s in zip(blocks.tolist(), slots.tolist()):
            ref = self.orc.fine_filter(k)
            np.testing.assert_array_equal(host[s], ref, err_msg=f"I_t of block {k}, t={t}")
            n_rows += int(np.unpackbits(ref.view(np.uint8)).sum())
        self.grads_gpu_only(act, t)
        self.gpu.step_adam(self.lr, mask_ptr=self.d_mask.data_ptr())
        g = (_cfn("wl_grad_cb"), C.addressof(self.gsyn))
        rc = self.orc.step_adam(self.lr, grad=g, mask=self.orc.fine_filter_mask)
        return rc, n_rows

    def grads_gpu_only(self, act, t):
        W.synth_grads_cuda(act, self.B, self.N, GRAD_SEED, t, self.stream)

    # ---- comparisons
    def compare_plan(self, J):
        for which in ("K", "R", "S+", "S-", "Omega", "A"):
            gb, gs = self.gpu.list(which, with_slots=True)
            ob, os_ = self.orc.list(which, with_slots=True)
            np.testing.assert_array_equal(gb, ob, err_msg=f"{which} blocks, t={self.t}")
            np.testing.assert_array_equal(gs, os_, err_msg=f"{which} slots, t={self.t}")
        for j in range(J):
            np.testing.assert_array_equal(self.gpu.percam(j), self.orc.percam(j),
                                          err_msg=f"K^({j}) t={self.t}")
        np.testing.assert_array_equal(self.gpu.slot_map(), self.orc.slot_map(),
                                      err_msg=f"slot map t={self.t}")

    def compare_evicted_dirty(self):
        np.testing.assert_array_equal(self.gpu.evicted_dirty(), self.orc.evicted_dirty(),
                                      err_msg=f"dirty S- t={self.t}")

    def compare_stats(self):
        g, o = self.gpu.stats(), self.orc.stats()
        assert g == o, {k: (g[k], o[k]) for k in g if g[k] != o[k]}

    def compare_blocks(self, blocks):
        """theta, m, v: |gpu - ref| <= 1e-6 max(|gpu|,|ref|) or both <= 1e-30
        (north star); returns the max ULP distance seen (0 expected)."""
        worst = 0
        for k in blocks:
            k = int(k)
            g = self.gpu.read_block(k)
            o = self.orc.read_block(k)
            for name, a, b in zip(("theta", "m", "v"), g, o):
                assert_close(a, b, f"{name} block {k} t={self.t}")
                worst = max(worst, max_ulp(a, b))
            assert self.gpu.step_count(k) == self.orc.step_count(k), k
        return worst

    def compare_store(self, index_blocks=()):
        """f3: CPU-cache counters, LRU order with dirty flags and Index[k] bit-exact"""
        g, o = self.gpu.store_stats(), self.orc.store_stats()
        diff = {k: (g[k], o[k]) for k in o if g[k] != o[k]}
        assert not diff, f"store counters t={self.t}: {diff}"
        gb, gd = self.gpu.store_lru()
        ob, od = self.orc.store_lru()
        np.testing.assert_array_equal(gb, ob, err_msg=f"LRU order t={self.t}")
        np.testing.assert_array_equal(gd, od, err_msg=f"LRU dirty flags t={self.t}")
        for k in index_blocks:
            assert self.gpu.store_index(int(k)) == self.orc.store_index(int(k)), (k, self.t)
        return g

    def close(self):
        self.gpu.close()
        self.orc.close()


def assert_close(a, b, what):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    assert a.shape == b.shape
    same_nan = np.isnan(a) & np.isnan(b)
    tiny = (np.abs(a) <= 1e-30) & (np.abs(b) <= 1e-30)
    with np.errstate(invalid="ignore"):
        ok = (np.abs(a.astype(np.float64) - b) <= 1e-6 * np.maximum(np.abs(a), np.abs(b))) | tiny | same_nan
    if not ok.all():
        i = np.argwhere(~ok)[0]
        raise AssertionError(f"{what}: {int((~ok).sum())} mismatches, first at {tuple(i)}: "
                             f"gpu={a[tuple(i)]!r} ref={b[tuple(i)]!r}")


def max_ulp(a, b) -> int:
    ia = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    ib = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, np.int64(-2**31) - ia, ia)
    ib = np.where(ib < 0, np.int64(-2**31) - ib, ib)
    return int(np.abs(ia - ib).max()) if ia.size else 0
