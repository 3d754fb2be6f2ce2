"""Thin Python binding of the C ABI in include/tidegs.h (argument marshalling only).

Every step of the working-set path runs in libtidegs.so (CUDA kernels for
sm_100a + copy engines); this module only converts arguments.  PyTorch supplies
device memory (the caching allocator, through the tgs_allocator hooks) and the
compute stream.  There is no fallback: if the extension is missing the import
fails (run ``make`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TGS_LIB selects an in-tree build variant (kernel A/B experiments); default libtidegs.so
LIB_PATH = os.environ.get("TGS_LIB") or os.path.join(_HERE, "libtidegs.so")
DIM = 59

OK, EINVAL, ESTATE, ENOMEM, ECUDA, ENCCL, ENONFINITE, EPOISONED, EIO = range(9)
PERSIST, COLD_RESTART = 0, 1
XFER_KERNEL, XFER_COPY_ENGINE = 0, 1  # tgs_xfer (include/tidegs.h)
LISTS = {"K": 0, "R": 1, "S+": 2, "S-": 3, "Omega": 4, "A": 5}

# every entry point include/tidegs.h declares (tests check the exports)
SYMBOLS = ("tgs_init_table", "tgs_destroy", "tgs_activate", "tgs_step_adam", "tgs_flush",
           "tgs_fine_filter",
           "tgs_get_stats", "tgs_get_stats_async", "tgs_get_timing", "tgs_set_profiling", "tgs_get_list",
           "tgs_get_percam", "tgs_get_evicted_dirty", "tgs_get_slot_map",
           "tgs_nonfinite_index", "tgs_read_block", "tgs_step_count", "tgs_num_local_blocks",
           "tgs_pool_slots", "tgs_read_bound", "tgs_build_layout", "tgs_frustum_planes", "tgs_status_string", "tgs_last_error",
           "tgs_init_table_store", "tgs_get_store_stats", "tgs_store_index", "tgs_store_lru",
           "tgs_order_views", "tgs_store_compact", "tgs_set_comm", "tgs_get_global_stats",
           "tgs_prefetch", "tgs_activate_async")


class Config(C.Structure):
    _fields_ = [("n_gaussians", C.c_uint64), ("dim", C.c_uint32), ("block_size", C.c_uint32),
                ("capacity", C.c_uint32), ("pool_slots", C.c_uint32),
                ("max_cameras", C.c_uint32), ("max_age", C.c_uint32),
                ("quota_num", C.c_uint32), ("quota_den", C.c_uint32), ("lambda_", C.c_double),
                ("gamma", C.c_double), ("moments", C.c_int32), ("tide", C.c_int32),
                ("world_size", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32),
                ("init_threads", C.c_int32), ("staging_blocks", C.c_uint32),
                ("refresh_bounds", C.c_int32), ("serialize", C.c_int32),
                ("level2", C.c_int32), ("xfer", C.c_int32)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)
FILL_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.POINTER(C.c_float))


class Allocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


class Activation(C.Structure):
    _fields_ = [("n_visible", C.c_uint32), ("n_resident", C.c_uint32),
                ("n_active_blocks", C.c_uint32), ("n_stage_in", C.c_uint32),
                ("n_evict", C.c_uint32), ("n_evict_dirty", C.c_uint32),
                ("h2d_bytes", C.c_uint64), ("d_active_blocks", C.c_void_p),
                ("d_active_slots", C.c_void_p), ("d_params", C.c_void_p),
                ("d_grads", C.c_void_p), ("slot_stride", C.c_uint64),
                ("grad_stride", C.c_uint64), ("ready", C.c_void_p),
                ("d_global_active", C.c_void_p), ("global_stride", C.c_uint32),
                ("global_ready", C.c_void_p), ("d_n_active", C.c_void_p)]


COMM_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
COMM_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_size_t, C.c_void_p)


class Comm(C.Structure):
    _fields_ = [("allgather", COMM_ALLGATHER), ("allreduce_u64", COMM_ALLREDUCE),
                ("user", C.c_void_p)]


class Adam(C.Structure):
    _fields_ = [("lr", C.POINTER(C.c_float)), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float)]


STAT_FIELDS = ("iter", "n_visible", "n_resident", "n_active_blocks", "n_stage_in", "n_evict",
               "n_evict_dirty", "n_active_rows", "h2d_bytes", "d2h_bytes", "flush_bytes",
               "n_flush_blocks", "readmissions", "cold_restart_updates", "total_updates",
               "resident_streak_sum", "streak_count", "k_inter_sum", "k_union_sum")


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in STAT_FIELDS]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n in STAT_FIELDS}


class Timing(C.Structure):
    _fields_ = ([(n, C.c_double) for n in ("adam_ms", "adam_prologue_ms", "plan_ms", "h2d_ms",
                                             "d2h_ms", "evict_ms", "fine_ms")] +
                [(n, C.c_uint64) for n in ("adam_launches", "plan_launches", "h2d_batches",
                                           "d2h_batches", "adam_rows", "adam_elems_quads",
                                           "h2d_bytes", "d2h_bytes", "kernel_launches",
                                           "copy_calls", "fresh_active_rows",
                                           "fresh_blocks", "h2d_ring_records")])

    def as_dict(self):
        return {n: (float(getattr(self, n)) if t is C.c_double else int(getattr(self, n)))
                for n, t in self._fields_}


class StoreConfig(C.Structure):
    _fields_ = [("dir", C.c_char_p), ("cache_blocks", C.c_uint32), ("segment_bytes", C.c_uint64),
                ("direct_io", C.c_int32), ("io_threads", C.c_int32), ("reopen", C.c_int32),
                ("prefetch_blocks", C.c_uint32)]


STORE_FIELDS = ("hits", "misses", "evictions", "dirty_evictions", "flush_appends", "read_bytes",
                "write_bytes", "segments", "cached", "cached_dirty")


class StoreStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in STORE_FIELDS] + [("read_ms", C.c_double),
                                                          ("write_ms", C.c_double),
                                                          ("read_calls", C.c_uint64),
                                                          ("read_busy_ms", C.c_double),
                                                          ("prefetch_reads", C.c_uint64),
                                                          ("prefetch_hits", C.c_uint64),
                                                          ("prefetch_wasted", C.c_uint64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Camera(C.Structure):
    _fields_ = [("plane", (C.c_float * 4) * 6)]


_lib = None


def lib():
    """Load libtidegs.so; raises if the CUDA extension has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: the CUDA extension is required "
                               "(run `make` or __graft_entry__.build()); there is no fallback")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.tgs_init_table.argtypes = [C.POINTER(Config), C.c_void_p, C.c_void_p, vp,
                                     C.POINTER(C.c_float), C.POINTER(Allocator), vp,
                                     C.POINTER(vp)]
        L.tgs_init_table_store.argtypes = [C.POINTER(Config), C.POINTER(StoreConfig), C.c_void_p,
                                           C.c_void_p, vp, C.POINTER(C.c_float),
                                           C.POINTER(Allocator), vp, C.POINTER(vp)]
        L.tgs_get_store_stats.argtypes = [vp, C.POINTER(StoreStats)]
        L.tgs_store_index.argtypes = [vp, u64, C.POINTER(C.c_uint64)]
        L.tgs_store_compact.argtypes = [vp]
        L.tgs_store_lru.restype = u32
        L.tgs_store_lru.argtypes = [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint8), u32]
        L.tgs_destroy.argtypes = [vp]
        L.tgs_activate.argtypes = [vp, C.c_void_p, u32, C.POINTER(Activation)]
        L.tgs_activate_async.argtypes = [vp, C.c_void_p, u32, C.POINTER(Activation)]
        L.tgs_step_adam.argtypes = [vp, C.POINTER(Adam), vp]
        L.tgs_flush.argtypes = [vp]
        L.tgs_fine_filter.argtypes = [vp, vp]
        L.tgs_get_stats.argtypes = [vp, C.POINTER(Stats)]
        L.tgs_set_comm.argtypes = [vp, C.POINTER(Comm)]
        L.tgs_prefetch.argtypes = [vp, C.c_void_p, u32, u32]
        L.tgs_get_global_stats.argtypes = [vp, C.POINTER(Stats)]
        L.tgs_get_timing.argtypes = [vp, C.POINTER(Timing)]
        L.tgs_get_stats_async.argtypes = [vp, vp]
        L.tgs_set_profiling.argtypes = [vp, C.c_int]
        L.tgs_get_list.restype = u32
        L.tgs_get_list.argtypes = [vp, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_int32), u32]
        L.tgs_get_percam.restype = u32
        L.tgs_get_percam.argtypes = [vp, u32, C.POINTER(C.c_uint32), u32]
        L.tgs_get_evicted_dirty.restype = u32
        L.tgs_get_evicted_dirty.argtypes = [vp, C.POINTER(C.c_uint32), u32]
        L.tgs_get_slot_map.argtypes = [vp, C.POINTER(C.c_int64)]
        L.tgs_nonfinite_index.restype = u64
        L.tgs_nonfinite_index.argtypes = [vp]
        L.tgs_read_block.argtypes = [vp, u64] + [C.POINTER(C.c_float)] * 3
        L.tgs_read_bound.argtypes = [vp, u64, C.POINTER(C.c_float)]
        L.tgs_step_count.restype = u32
        L.tgs_step_count.argtypes = [vp, u64]
        L.tgs_num_local_blocks.restype = u32
        L.tgs_num_local_blocks.argtypes = [vp]
        L.tgs_pool_slots.restype = u32
        L.tgs_pool_slots.argtypes = [vp]
        L.tgs_build_layout.argtypes = [C.POINTER(C.c_float), u64, u32, C.c_int,
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_float),
                                       C.POINTER(C.c_double)]
        L.tgs_frustum_planes.argtypes = [C.POINTER(C.c_double)] + [C.c_double] * 4 + [
            u32, u32, C.c_double, C.c_double, C.POINTER(Camera)]
        L.tgs_order_views.argtypes = [C.POINTER(C.c_double), u32, u32, C.c_int,
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_double)]
        L.tgs_status_string.restype = C.c_char_p
        L.tgs_status_string.argtypes = [C.c_int]
        L.tgs_last_error.restype = C.c_char_p
        L.tgs_last_error.argtypes = [vp]
        _lib = L
    return _lib


class TgsError(RuntimeError):
    def __init__(self, code, what, detail=""):
        msg = f"{what}: {lib().tgs_status_string(code).decode()} ({code})"
        if detail:
            msg += f": {detail}"
        super().__init__(msg)
        self.code = code


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def make_config(n_gaussians, block_size, capacity, *, pool_slots=0, max_cameras=256,
                max_age=255, quota=(1, 2), lam=0.7, gamma=0.9, moments=PERSIST, tide=1,
                world_size=1, rank=0, device=0, init_threads=0, staging_blocks=0,
                refresh_bounds=0, serialize=0, level2=0, xfer=0) -> Config:
    return Config(n_gaussians, DIM, block_size, capacity, pool_slots, max_cameras, max_age,
                  quota[0], quota[1], lam, gamma, moments, tide, world_size, rank, device,
                  init_threads, staging_blocks, refresh_bounds, serialize, level2, xfer)


def torch_allocator(device=0):
    """tgs_allocator backed by PyTorch's CUDA caching allocator."""
    import torch

    def _alloc(size, stream, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(size), device, int(stream or 0))
        except Exception:
            return None

    def _free(ptr, _stream, _user):
        torch.cuda.caching_allocator_delete(int(ptr))

    return Allocator(ALLOC_FN(_alloc), FREE_FN(_free), None)


def _device_view(torch, ptr, nbytes, device):
    """uint8 torch view of nbytes of library-owned device memory (no copy)"""
    class _V:
        __cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                    "data": (int(ptr), False), "version": 3}
    return torch.as_tensor(_V(), device=device)


def torch_comm(group=None, device=None):
    """tgs_comm transport over torch.distributed (argument marshalling only): NCCL
    enqueues the collective on the library's stream; gloo (CPU tests, several
    ranks sharing one GPU) stages through host memory and completes before
    returning.  Keep the returned object alive as long as the table."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    nccl = dist.get_backend(group) == "nccl"
    G = dist.get_world_size(group)

    def _ag(_user, send, recv, nbytes, stream):
        try:
            s = _device_view(torch, send, nbytes, dev)
            r = _device_view(torch, recv, nbytes * G, dev)
            if nccl:
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0), device=dev)):
                    dist.all_gather_into_tensor(r, s, group=group)
            else:
                torch.cuda.ExternalStream(int(stream or 0), device=dev).synchronize()
                parts = [torch.empty(int(nbytes), dtype=torch.uint8) for _ in range(G)]
                dist.all_gather(parts, s.cpu(), group=group)
                r.copy_(torch.cat(parts).to(dev))
                torch.cuda.synchronize(dev)
            return 0
        except Exception as e:  # surfaces as TGS_ENCCL
            print(f"tidegs torch_comm all-gather: {e}", flush=True)
            return 1

    def _ar(_user, buf, count, stream):
        try:
            addr = C.cast(buf, C.c_void_p).value
            b = _device_view(torch, addr, count * 8, dev).view(torch.int64)
            if nccl:
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0), device=dev)):
                    dist.all_reduce(b, group=group)
            else:
                torch.cuda.ExternalStream(int(stream or 0), device=dev).synchronize()
                h = b.cpu()
                dist.all_reduce(h, group=group)
                b.copy_(h.to(dev))
                torch.cuda.synchronize(dev)
            return 0
        except Exception as e:
            print(f"tidegs torch_comm all-reduce: {e}", flush=True)
            return 1

    return Comm(COMM_ALLGATHER(_ag), COMM_ALLREDUCE(_ar), None)


class Table:
    """One shard of the block-virtualized Gaussian table (tgs_ctx)."""

    def __init__(self, cfg: Config, bounds: np.ndarray, *, theta_rows: np.ndarray | None = None,
                 fill=None, stream=None, use_torch_allocator=True, store: dict | None = None):
        """store: None (flat pinned host tier) or the NEXT f3 store tier,
        dict(dir=..., cache_blocks=H, segment_bytes=0, direct_io=1, io_threads=0, reopen=0)."""
        self.cfg = cfg
        self.B = cfg.block_size
        self._bounds = np.ascontiguousarray(bounds, np.float32)
        self._keep = []
        rows_p, fill_p, fill_u = None, None, None
        if theta_rows is not None:
            self._rows = np.ascontiguousarray(theta_rows, np.float32)
            rows_p = self._rows.ctypes.data
        elif isinstance(fill, tuple):            # (C fn address, user pointer)
            fill_p, fill_u = fill
        elif fill is not None:                   # python callable k -> (B, 59)
            def _cb(_u, k, out, _f=fill, _n=self.B * DIM):
                a = np.ascontiguousarray(_f(int(k)), np.float32).reshape(-1)
                C.memmove(out, a.ctypes.data, _n * 4)
            cb = FILL_FN(_cb)
            self._keep.append(cb)
            fill_p = C.cast(cb, C.c_void_p).value
        alloc = None
        if os.environ.get("TGS_CUDAMALLOC") == "1":  # one cudaMalloc per buffer (sanitizer runs)
            use_torch_allocator = False
        if use_torch_allocator:
            self._alloc = torch_allocator(cfg.device)
            alloc = C.byref(self._alloc)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(cfg.device).cuda_stream
        self.stream = int(stream)
        h = C.c_void_p()
        if store is None:
            rc = lib().tgs_init_table(C.byref(cfg), rows_p, fill_p, fill_u, _fp(self._bounds),
                                      alloc, self.stream or None, C.byref(h))
        else:
            self._store_cfg = StoreConfig(os.fsencode(str(store["dir"])), store["cache_blocks"],
                                          store.get("segment_bytes", 0),
                                          store.get("direct_io", 1), store.get("io_threads", 0),
                                          store.get("reopen", 0), store.get("prefetch_blocks", 0))
            rc = lib().tgs_init_table_store(C.byref(cfg), C.byref(self._store_cfg), rows_p,
                                            fill_p, fill_u, _fp(self._bounds), alloc,
                                            self.stream or None, C.byref(h))
        if rc != OK:
            raise TgsError(rc, "tgs_init_table" + ("" if store is None else "_store"))
        self.h = h
        self.P = int(lib().tgs_pool_slots(h))
        self.last = None

    def close(self):
        if getattr(self, "h", None):
            lib().tgs_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self, rc, what):
        if rc != OK:
            raise TgsError(rc, what, lib().tgs_last_error(self.h).decode(errors="replace"))

    # ---- the hot path
    def prefetch(self, planes: np.ndarray, ahead: int = 1):
        """announce the camera batch of the activate `ahead` calls from now (f3 read-ahead)"""
        p = np.ascontiguousarray(planes, np.float32).reshape(-1, 6, 4)
        self._err(lib().tgs_prefetch(self.h, p.ctypes.data if p.shape[0] else None, p.shape[0],
                                     ahead), "tgs_prefetch")

    def activate_async(self, planes: np.ndarray) -> Activation:
        """tgs_activate_async: enqueue the activate, no plan readback; the host
        counts come back unknown (0xFFFFFFFF), |A| is at act.d_n_active"""
        p = np.ascontiguousarray(planes, np.float32).reshape(-1, 6, 4)
        out = Activation()
        self._err(lib().tgs_activate_async(self.h, p.ctypes.data if p.shape[0] else None,
                                           p.shape[0], C.byref(out)), "tgs_activate_async")
        self.last = out
        return out

    def activate(self, planes: np.ndarray, *, check=True) -> Activation:
        p = np.ascontiguousarray(planes, np.float32).reshape(-1, 6, 4)
        out = Activation()
        rc = lib().tgs_activate(self.h, p.ctypes.data if p.shape[0] else None, p.shape[0],
                                C.byref(out))
        if check:
            self._err(rc, "tgs_activate")
        self.last = out
        return out if check else rc

    def step_adam(self, lr, beta1=0.9, beta2=0.999, eps=1e-15, mask_ptr=None, check=True):
        self._lr = np.ascontiguousarray(lr, np.float32)
        hp = Adam(_fp(self._lr), beta1, beta2, eps)
        rc = lib().tgs_step_adam(self.h, C.byref(hp), mask_ptr)
        if check:
            self._err(rc, "tgs_step_adam")
        return rc

    def fine_filter(self, mask_ptr):
        """Level-2 filter: I_t row mask of the last activate's A slots -> mask_ptr."""
        self._err(lib().tgs_fine_filter(self.h, mask_ptr), "tgs_fine_filter")

    def flush(self):
        self._err(lib().tgs_flush(self.h), "tgs_flush")

    # ---- inspection
    def list(self, which: str, with_slots=False):
        w = LISTS[which]
        n = lib().tgs_get_list(self.h, w, None, None, 0)
        b = np.empty(n, np.uint32)
        s = np.empty(n, np.int32)
        lib().tgs_get_list(self.h, w, b.ctypes.data_as(C.POINTER(C.c_uint32)),
                           s.ctypes.data_as(C.POINTER(C.c_int32)), n)
        return (b, s) if with_slots else b

    def percam(self, j: int) -> np.ndarray:
        n = lib().tgs_get_percam(self.h, j, None, 0)
        b = np.empty(n, np.uint32)
        lib().tgs_get_percam(self.h, j, b.ctypes.data_as(C.POINTER(C.c_uint32)), n)
        return b

    def evicted_dirty(self) -> np.ndarray:
        n = lib().tgs_get_evicted_dirty(self.h, None, 0)
        b = np.empty(n, np.uint32)
        lib().tgs_get_evicted_dirty(self.h, b.ctypes.data_as(C.POINTER(C.c_uint32)), n)
        return b

    def slot_map(self) -> np.ndarray:
        out = np.empty(self.P, np.int64)
        self._err(lib().tgs_get_slot_map(self.h, out.ctypes.data_as(C.POINTER(C.c_int64))),
                  "tgs_get_slot_map")
        return out

    def stats(self) -> dict:
        s = Stats()
        self._err(lib().tgs_get_stats(self.h, C.byref(s)), "tgs_get_stats")
        return s.as_dict()

    def set_comm(self, comm: Comm):
        """C1 / C2 transport (tgs_set_comm); e.g. torch_comm()"""
        self._comm = comm  # the callbacks must outlive the table
        self._err(lib().tgs_set_comm(self.h, C.byref(comm)), "tgs_set_comm")

    def global_stats(self) -> dict:
        """C2: every rank's counters summed, as of the last step_adam"""
        s = Stats()
        self._err(lib().tgs_get_global_stats(self.h, C.byref(s)), "tgs_get_global_stats")
        return s.as_dict()

    def global_active(self, act: Activation):
        """C1 result of `act` as a [G, C] uint32 numpy array (synchronising)"""
        import torch
        G = self.cfg.world_size
        v = _device_view(torch, act.d_global_active, 4 * G * act.global_stride,
                         torch.device("cuda", self.cfg.device))
        torch.cuda.synchronize()
        return v.cpu().numpy().view(np.uint32).reshape(G, act.global_stride)

    def stats_async(self, pinned_ptr):
        """Enqueue a D2H read of the counters into pinned host memory (no sync)."""
        self._err(lib().tgs_get_stats_async(self.h, pinned_ptr), "tgs_get_stats_async")

    def timing(self) -> dict:
        t = Timing()
        self._err(lib().tgs_get_timing(self.h, C.byref(t)), "tgs_get_timing")
        return t.as_dict()

    def set_profiling(self, on: bool):
        self._err(lib().tgs_set_profiling(self.h, int(on)), "tgs_set_profiling")

    def nonfinite_index(self):
        v = int(lib().tgs_nonfinite_index(self.h))
        return None if v == 2**64 - 1 else v

    def read_block(self, k):
        th, m, v = (np.empty((self.B, DIM), np.float32) for _ in range(3))
        self._err(lib().tgs_read_block(self.h, k, _fp(th), _fp(m), _fp(v)), "tgs_read_block")
        return th, m, v

    def step_count(self, k) -> int:
        return int(lib().tgs_step_count(self.h, k))

    def bound(self, k) -> np.ndarray:
        out = np.empty(4, np.float32)
        self._err(lib().tgs_read_bound(self.h, k, _fp(out)), "tgs_read_bound")
        return out

    @property
    def num_local_blocks(self) -> int:
        return int(lib().tgs_num_local_blocks(self.h))

    # ---- NEXT f3 store tier
    def store_stats(self) -> dict:
        s = StoreStats()
        self._err(lib().tgs_get_store_stats(self.h, C.byref(s)), "tgs_get_store_stats")
        return s.as_dict()

    def store_index(self, k):
        out = (C.c_uint64 * 4)()
        self._err(lib().tgs_store_index(self.h, k, out), "tgs_store_index")
        return tuple(int(x) for x in out)

    def store_compact(self):
        """R31: barrier, then merge the patch segments into a new base."""
        self._err(lib().tgs_store_compact(self.h), "tgs_store_compact")

    def store_lru(self):
        n = lib().tgs_store_lru(self.h, None, None, 0)
        b = np.empty(n, np.uint32)
        d = np.empty(n, np.uint8)
        lib().tgs_store_lru(self.h, b.ctypes.data_as(C.POINTER(C.c_uint32)),
                            d.ctypes.data_as(C.POINTER(C.c_uint8)), n)
        return b, d.astype(bool)


def frustum_planes(w2c, fx, fy, cx, cy, width, height, znear, zfar) -> np.ndarray:
    m = (C.c_double * 16)(*np.asarray(w2c, np.float64).reshape(-1).tolist())
    cam = Camera()
    rc = lib().tgs_frustum_planes(m, fx, fy, cx, cy, width, height, znear, zfar, C.byref(cam))
    if rc != OK:
        raise TgsError(rc, "tgs_frustum_planes")
    return np.array([[cam.plane[p][i] for i in range(4)] for p in range(6)], np.float32)


def build_layout(cs: np.ndarray, block_size: int, device: int = 0):
    """NEXT f2b on the GPU: (perm, bounds, gpu_ms) for n x 4 (cx, cy, cz, max
    log-scale) -- Morton sort + blocking (tgs_build_layout)."""
    cs = np.ascontiguousarray(cs, np.float32)
    n = cs.shape[0]
    K = (n + block_size - 1) // block_size
    perm = np.empty(n, np.uint64)
    bounds = np.empty((K, 4), np.float32)
    ms = C.c_double(0.0)
    rc = lib().tgs_build_layout(_fp(cs), n, block_size, device,
                                perm.ctypes.data_as(C.POINTER(C.c_uint64)), _fp(bounds),
                                C.byref(ms))
    if rc != OK:
        raise TgsError(rc, "tgs_build_layout")
    return perm, bounds, ms.value


def order_views(feat: np.ndarray, device: int = 0):
    """NEXT f4 on the GPU: clustered-TSP view order (tgs_order_views):
    (perm, cluster, k, lloyd_iterations, gpu_ms)."""
    f = np.ascontiguousarray(feat, np.float64)
    M, D = f.shape
    perm = np.empty(M, np.uint32)
    cl = np.empty(M, np.uint32)
    k, it, ms = C.c_uint32(), C.c_uint32(), C.c_double()
    u32p = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint32))
    rc = lib().tgs_order_views(f.ctypes.data_as(C.POINTER(C.c_double)), M, D, device, u32p(perm),
                               u32p(cl), C.byref(k), C.byref(it), C.byref(ms))
    if rc != OK:
        raise TgsError(rc, "tgs_order_views")
    return perm, cl, int(k.value), int(it.value), ms.value
