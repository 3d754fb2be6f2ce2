"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the CPU oracle (tgs_oracle.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  The product path
(paper_2605_20150_b200) never imports it; see DESIGN.md §4.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
DIM = 59
OK, EINVAL, ESTATE, ENONFINITE = 0, 1, 2, 6
PERSIST, COLD_RESTART = 0, 1
LISTS = {"K": 0, "R": 1, "S+": 2, "S-": 3, "Omega": 4, "A": 5}
STORE_STATS = ("hits", "misses", "evictions", "dirty_evictions", "flush_appends", "read_bytes",
               "write_bytes", "segments", "cached", "cached_dirty")


class Config(C.Structure):
    _fields_ = [("n_gaussians", C.c_uint64), ("dim", C.c_uint32), ("block_size", C.c_uint32),
                ("capacity", C.c_uint32), ("pool_slots", C.c_uint32),
                ("max_cameras", C.c_uint32), ("max_age", C.c_uint32),
                ("quota_num", C.c_uint32), ("quota_den", C.c_uint32), ("lambda_", C.c_double),
                ("gamma", C.c_double), ("moments", C.c_int32), ("tide", C.c_int32),
                ("world_size", C.c_int32), ("rank", C.c_int32), ("refresh_bounds", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "iter", "n_visible", "n_resident", "n_active_blocks", "n_stage_in", "n_evict",
        "n_evict_dirty", "n_active_rows", "h2d_bytes", "d2h_bytes", "flush_bytes",
        "n_flush_blocks", "readmissions", "cold_restart_updates", "total_updates",
        "resident_streak_sum", "streak_count", "k_inter_sum", "k_union_sum")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


FILL_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.POINTER(C.c_float))
GRAD_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_float))
MASK_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32))

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libtgsoracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make`")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.or_create.argtypes = [C.POINTER(Config), C.POINTER(C.c_float), vp, vp, C.c_int,
                                C.POINTER(vp)]
        L.or_destroy.argtypes = [vp]
        L.or_track_block.argtypes = [vp, C.c_uint64]
        L.or_activate.argtypes = [vp, C.POINTER(C.c_float), C.c_uint32]
        L.or_step_adam.argtypes = [vp, C.POINTER(C.c_float), C.c_float, C.c_float, C.c_float,
                                   vp, vp, vp, vp]
        L.or_flush.argtypes = [vp]
        L.or_get_list.restype = C.c_uint32
        L.or_get_list.argtypes = [vp, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_int32),
                                  C.c_uint32]
        L.or_get_percam.restype = C.c_uint32
        L.or_get_percam.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint32), C.c_uint32]
        L.or_get_evicted_dirty.restype = C.c_uint32
        L.or_get_evicted_dirty.argtypes = [vp, C.POINTER(C.c_uint32), C.c_uint32]
        L.or_get_slot_map.argtypes = [vp, C.POINTER(C.c_int64)]
        L.or_get_stats.argtypes = [vp, C.POINTER(Stats)]
        L.or_nonfinite_index.restype = C.c_uint64
        L.or_nonfinite_index.argtypes = [vp]
        L.or_read_block.argtypes = [vp, C.c_uint64] + [C.POINTER(C.c_float)] * 3
        L.or_num_local_blocks.restype = C.c_uint32
        L.or_num_local_blocks.argtypes = [vp]
        L.or_step_count.restype = C.c_uint32
        L.or_step_count.argtypes = [vp, C.c_uint64]
        L.or_fine_filter.argtypes = [vp, C.c_uint64, C.POINTER(C.c_uint32)]
        L.or_get_bound.argtypes = [vp, C.c_uint64, C.POINTER(C.c_float)]
        L.or_build_layout.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32,
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_float)]
        L.or_morton3.restype = C.c_uint64
        L.or_morton3.argtypes = [C.c_uint32] * 3
        L.or_exp_det.restype = C.c_float
        L.or_exp_det.argtypes = [C.c_float]
        L.or_order_views.argtypes = [C.POINTER(C.c_double), C.c_uint32, C.c_uint32,
                                     C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.or_store_open.argtypes = [vp, C.c_char_p, C.c_uint32, C.c_uint64]
        L.or_store_compact.argtypes = [vp]
        L.or_store_reopen.argtypes = [vp, C.c_char_p, C.c_uint32, C.c_uint64]
        L.or_store_index.argtypes = [vp, C.c_uint64, C.POINTER(C.c_uint64)]
        L.or_store_stats.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.or_phase_ns.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.or_crc32c.restype = C.c_uint32
        L.or_crc32c.argtypes = [C.c_char_p, C.c_uint64]
        L.or_track_all_from_now.argtypes = [vp]
        L.or_store_lru.restype = C.c_uint32
        L.or_store_lru.argtypes = [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), C.c_uint32]
        _lib = L
    return _lib


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what}: status {code}")
        self.code = code


def make_config(n_gaussians, block_size, capacity, *, pool_slots=0, max_cameras=256,
                max_age=255, quota=(1, 2), lam=0.7, gamma=0.9, moments=PERSIST, tide=1,
                world_size=1, rank=0, refresh_bounds=0) -> Config:
    return Config(n_gaussians, DIM, block_size, capacity, pool_slots, max_cameras, max_age,
                  quota[0], quota[1], lam, gamma, moments, tide, world_size, rank,
                  refresh_bounds)


class Oracle:
    """One shard of the working-set step, computed the slow obvious way."""

    def __init__(self, cfg: Config, bounds: np.ndarray, fill=None, track_all=True):
        self.cfg = cfg
        self.B = cfg.block_size
        self._bounds = np.ascontiguousarray(bounds, np.float32)
        self._keep = []
        fn, user = None, None
        if fill is not None:
            if isinstance(fill, tuple):       # (C fn address, user pointer)
                fn, user = fill
            else:                              # python callable k -> (B,59) array
                def _cb(_u, k, out, _fill=fill, _n=self.B * DIM):
                    a = np.ascontiguousarray(_fill(int(k)), np.float32).reshape(-1)
                    C.memmove(out, a.ctypes.data, _n * 4)
                cb = FILL_FN(_cb)
                self._keep.append(cb)
                fn = C.cast(cb, C.c_void_p).value
        h = C.c_void_p()
        rc = lib().or_create(C.byref(cfg), _f(self._bounds), fn, user, int(track_all),
                             C.byref(h))
        if rc != OK:
            raise OracleError(rc, "or_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().or_destroy(self.h)
            self.h = None

    __del__ = close

    def track(self, k):
        return lib().or_track_block(self.h, k)

    def activate(self, planes: np.ndarray) -> int:
        p = np.ascontiguousarray(planes, np.float32).reshape(-1, 6, 4)
        return lib().or_activate(self.h, _f(p), p.shape[0])

    def step_adam(self, lr, beta1=0.9, beta2=0.999, eps=1e-15, grad=None, mask=None) -> int:
        """grad / mask: (C fn address, user pointer) or python callables
        grad(k, t) -> (B,59) float32, mask(k, t) -> (ceil(B/32),) uint32."""
        lr_a = np.ascontiguousarray(lr, np.float32)
        keep = []

        def wrap(obj, proto, n, dtype):
            if obj is None:
                return None, None
            if isinstance(obj, tuple):
                return obj
            def _cb(_u, k, t, out, _o=obj):
                a = np.ascontiguousarray(_o(int(k), int(t)), dtype).reshape(-1)
                C.memmove(out, a.ctypes.data, n * a.itemsize)
            cb = proto(_cb)
            keep.append(cb)
            return C.cast(cb, C.c_void_p).value, None

        gfn, gu = wrap(grad, GRAD_FN, self.B * DIM, np.float32)
        mfn, mu = wrap(mask, MASK_FN, (self.B + 31) // 32, np.uint32)
        return lib().or_step_adam(self.h, _f(lr_a), beta1, beta2, eps, gfn, gu, mfn, mu)

    def flush(self) -> int:
        return lib().or_flush(self.h)

    def list(self, which: str, with_slots=False):
        w = LISTS[which]
        n = lib().or_get_list(self.h, w, None, None, 0)
        b = np.empty(n, np.uint32)
        s = np.empty(n, np.int32)
        lib().or_get_list(self.h, w, b.ctypes.data_as(C.POINTER(C.c_uint32)),
                          s.ctypes.data_as(C.POINTER(C.c_int32)), n)
        return (b, s) if with_slots else b

    def percam(self, j: int) -> np.ndarray:
        n = lib().or_get_percam(self.h, j, None, 0)
        b = np.empty(n, np.uint32)
        lib().or_get_percam(self.h, j, b.ctypes.data_as(C.POINTER(C.c_uint32)), n)
        return b

    def evicted_dirty(self) -> np.ndarray:
        n = lib().or_get_evicted_dirty(self.h, None, 0)
        b = np.empty(n, np.uint32)
        lib().or_get_evicted_dirty(self.h, b.ctypes.data_as(C.POINTER(C.c_uint32)), n)
        return b

    def slot_map(self) -> np.ndarray:
        P = self.cfg.pool_slots or 2 * self.cfg.capacity
        out = np.empty(P, np.int64)
        lib().or_get_slot_map(self.h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def stats(self) -> dict:
        s = Stats()
        lib().or_get_stats(self.h, C.byref(s))
        return s.as_dict()

    def track_all_from_now(self):
        """timing aid (bench cpu_baseline): compute every block from now on"""
        rc = lib().or_track_all_from_now(self.h)
        if rc != OK:
            raise OracleError(rc, "or_track_all_from_now")

    def phase_seconds(self) -> dict:
        """cumulative wall time of the oracle's phases (SURVEY §8c timing hooks)"""
        out = (C.c_uint64 * 4)()
        lib().or_phase_ns(self.h, out)
        return dict(zip(("cull", "plan", "copies", "adam"), (x / 1e9 for x in out)))

    def nonfinite_index(self):
        v = int(lib().or_nonfinite_index(self.h))
        return None if v == 2**64 - 1 else v

    def read_block(self, k):
        n = self.B * DIM
        th, m, v = (np.empty((self.B, DIM), np.float32) for _ in range(3))
        rc = lib().or_read_block(self.h, k, _f(th), _f(m), _f(v))
        if rc != OK:
            raise OracleError(rc, "or_read_block")
        return th, m, v

    def step_count(self, k) -> int:
        return int(lib().or_step_count(self.h, k))

    def fine_filter(self, k) -> np.ndarray:
        """I_t bits of block k (Level-2 filter, NEXT f1)."""
        w = np.zeros((self.B + 31) // 32, np.uint32)
        rc = lib().or_fine_filter(self.h, k, w.ctypes.data_as(C.POINTER(C.c_uint32)))
        if rc != OK:
            raise OracleError(rc, "or_fine_filter")
        return w

    def bound(self, k) -> np.ndarray:
        out = np.empty(4, np.float32)
        rc = lib().or_get_bound(self.h, k, _f(out))
        if rc != OK:
            raise OracleError(rc, "or_get_bound")
        return out

    @property
    def num_local_blocks(self) -> int:
        return int(lib().or_num_local_blocks(self.h))

    # ---- NEXT f3: CPU cache + log-structured store (R27, R28)
    def store_open(self, dir, cache_blocks, segment_bytes=0):
        """dir=None: metadata only (Index, LRU, counters)."""
        d = None if dir is None else os.fsencode(str(dir))
        rc = lib().or_store_open(self.h, d, cache_blocks, segment_bytes)
        if rc != OK:
            raise OracleError(rc, "or_store_open")

    def store_reopen(self, dir, cache_blocks, segment_bytes=0):
        """R30: resume over the segment files of an earlier session."""
        rc = lib().or_store_reopen(self.h, os.fsencode(str(dir)), cache_blocks, segment_bytes)
        if rc != OK:
            raise OracleError(rc, "or_store_reopen")

    def store_compact(self):
        """R31: merge the patch segments into a new base (after flush)."""
        rc = lib().or_store_compact(self.h)
        if rc != OK:
            raise OracleError(rc, "or_store_compact")

    def store_index(self, k):
        """Index[k] = (file_id, offset, size, version)."""
        out = (C.c_uint64 * 4)()
        rc = lib().or_store_index(self.h, k, out)
        if rc != OK:
            raise OracleError(rc, "or_store_index")
        return tuple(int(x) for x in out)

    def store_stats(self) -> dict:
        out = (C.c_uint64 * 10)()
        rc = lib().or_store_stats(self.h, out)
        if rc != OK:
            raise OracleError(rc, "or_store_stats")
        return dict(zip(STORE_STATS, (int(x) for x in out)))

    def store_lru(self):
        """cached global ids, least recently used first, and their dirty flags"""
        n = lib().or_store_lru(self.h, None, None, 0)
        b = np.empty(n, np.uint32)
        d = np.empty(n, np.uint8)
        lib().or_store_lru(self.h, b.ctypes.data_as(C.POINTER(C.c_uint32)),
                           d.ctypes.data_as(C.POINTER(C.c_uint8)), n)
        return b, d.astype(bool)

    @property
    def fine_filter_mask(self):
        """(C fn, user) mask callback: step_adam with I_t from the fine filter."""
        return C.cast(lib().or_fine_filter_cb, C.c_void_p).value, self.h.value


def crc32c(data: bytes) -> int:
    return int(lib().or_crc32c(data, len(data)))


def exp_det(x: float) -> float:
    return float(lib().or_exp_det(x))


def morton3(x: int, y: int, z: int) -> int:
    return int(lib().or_morton3(x, y, z))


def build_layout(cs: np.ndarray, B: int):
    """NEXT f2b: (perm, bounds) for Gaussians given as n x 4 (cx, cy, cz, max
    log-scale) -- Morton sort + blocking."""
    cs = np.ascontiguousarray(cs, np.float32)
    n = cs.shape[0]
    K = (n + B - 1) // B
    perm = np.empty(n, np.uint64)
    bounds = np.empty((K, 4), np.float32)
    rc = lib().or_build_layout(_f(cs), n, B, perm.ctypes.data_as(C.POINTER(C.c_uint64)),
                               _f(bounds))
    if rc != OK:
        raise OracleError(rc, "or_build_layout")
    return perm, bounds


def order_views(feat: np.ndarray):
    """NEXT f4: clustered-TSP view order (R29) of M views with D features:
    (perm, cluster, k, lloyd_iterations)."""
    f = np.ascontiguousarray(feat, np.float64)
    M, D = f.shape
    perm = np.empty(M, np.uint32)
    cl = np.empty(M, np.uint32)
    k = C.c_uint32()
    it = C.c_uint32()
    u32p = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint32))
    rc = lib().or_order_views(f.ctypes.data_as(C.POINTER(C.c_double)), M, D, u32p(perm), u32p(cl),
                              C.byref(k), C.byref(it))
    if rc != OK:
        raise OracleError(rc, "or_order_views")
    return perm, cl, int(k.value), int(it.value)
