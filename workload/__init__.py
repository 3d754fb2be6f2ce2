"""Seeded synthetic inputs shared by the CUDA path and the oracle.

Holds none of the method's arithmetic: a Morton-ordered block-partitioned
Gaussian table, conservative block bounding spheres
(PAPER.md:199-200), camera trajectories with their 6 frustum planes
(PAPER.md:201), and counter-based gradients / row masks standing in for the
renderer's backward pass.  The recipes for the BASELINE.json
configs live in ``CONFIGS`` (DESIGN.md §5 states them).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
DIM = 59

SEEDS = {"scene": 20150, "trajectory": 1, "shuffle": 7, "grads": 42, "mask": 43}


class SceneParams(C.Structure):
    _fields_ = [("n_gaussians", C.c_uint64), ("block_size", C.c_uint32), ("layout", C.c_uint32),
                ("seed", C.c_uint64), ("side", C.c_double), ("lot", C.c_double),
                ("footprint", C.c_double), ("hmin", C.c_double), ("hmax", C.c_double),
                ("ground_h", C.c_double)]


class _PermFill(C.Structure):
    _fields_ = [("scene", C.c_void_p), ("perm", C.c_void_p), ("n", C.c_uint64)]


class Camera(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("fwd", C.c_double * 3), ("right", C.c_double * 3),
                ("down", C.c_double * 3), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_uint32),
                ("height", C.c_uint32), ("znear", C.c_double), ("zfar", C.c_double)]


class TrajParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_views", C.c_uint32), ("altitude", C.c_double),
                ("spacing", C.c_double), ("strip", C.c_double), ("fovx_deg", C.c_double),
                ("znear", C.c_double), ("zfar", C.c_double), ("width", C.c_uint32),
                ("height", C.c_uint32), ("radius_scale", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libtgsworkload.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = C.CDLL(path)
        vp, u64, u32, f32p = C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_float)
        L.wl_scene_create.restype = vp
        L.wl_scene_create.argtypes = [C.POINTER(SceneParams)]
        L.wl_scene_destroy.argtypes = [vp]
        L.wl_num_blocks.restype = u64
        L.wl_num_blocks.argtypes = [vp]
        L.wl_block_rows.restype = u32
        L.wl_block_rows.argtypes = [vp, u64]
        L.wl_sigma.restype = C.c_double
        L.wl_sigma.argtypes = [vp]
        L.wl_bounds.argtypes = [vp, u64, u64, f32p]
        L.wl_block_theta.argtypes = [vp, u64, f32p]
        L.wl_table.argtypes = [vp, f32p, C.c_int]
        L.wl_table_cs.argtypes = [vp, f32p, C.c_int]
        L.wl_block_tile.argtypes = [vp, u64] + [C.POINTER(C.c_int64)] * 2 + [C.POINTER(C.c_double)] * 4
        L.wl_camera_look.argtypes = [C.POINTER(Camera)] + [C.c_double * 3] * 3 + [
            C.c_double, u32, u32, C.c_double, C.c_double]
        L.wl_camera_planes.argtypes = [C.POINTER(Camera), f32p]
        L.wl_camera_sees.restype = C.c_int
        L.wl_camera_sees.argtypes = [C.POINTER(Camera), C.POINTER(C.c_double)]
        L.wl_traj_create.restype = vp
        L.wl_traj_create.argtypes = [vp, C.POINTER(TrajParams)]
        L.wl_traj_destroy.argtypes = [vp]
        L.wl_traj_num_views.restype = u64
        L.wl_traj_num_views.argtypes = [vp]
        L.wl_traj_view.argtypes = [vp, u64, C.POINTER(Camera)]
        L.wl_traj_set_order.argtypes = [vp, C.c_int, u64]
        L.wl_traj_set_perm.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.wl_traj_features.argtypes = [vp, C.c_double, C.POINTER(C.c_double)]
        L.wl_traj_batch_planes.argtypes = [vp, u64, u32, f32p]
        L.wl_traj_batch_cameras.argtypes = [vp, u64, u32, C.POINTER(Camera)]
        L.wl_grad.restype = C.c_float
        L.wl_grad.argtypes = [u64, u64, u32, u64]
        L.wl_grad_block.argtypes = [u64, u64, u32, u32, u64, f32p]
        L.wl_mask_block.argtypes = [u64, u64, u32, u32, u64, u32, C.POINTER(C.c_uint32)]
        L.wl_splitmix64.restype = u64
        L.wl_splitmix64.argtypes = [u64]
        _lib = L
    return _lib


def fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_float))


class Scene:
    """City-shaped scene: block k <-> the k-th tile of a W x H grid in Morton
    order ("Morton-sort ... before blocking")."""

    def __init__(self, n_gaussians: int, block_size: int = 4096, seed: int = SEEDS["scene"],
                 side: float = 2800.0, lot: float = 50.0, footprint: float = 30.0,
                 hmin: float = 10.0, hmax: float = 100.0, ground_h: float = 0.5,
                 layout: int = 0):
        self.params = SceneParams(n_gaussians, block_size, layout, seed, side, lot, footprint,
                                  hmin, hmax, ground_h)
        self.handle = lib().wl_scene_create(C.byref(self.params))
        if not self.handle:
            raise ValueError("invalid scene parameters")
        self.N = int(n_gaussians)
        self.B = int(block_size)
        self.K = int(lib().wl_num_blocks(self.handle))

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.wl_scene_destroy(self.handle)
            self.handle = None

    def rows(self, k: int) -> int:
        return int(lib().wl_block_rows(self.handle, k))

    @property
    def sigma(self) -> float:
        return float(lib().wl_sigma(self.handle))

    def bounds(self) -> np.ndarray:
        out = np.empty((self.K, 4), np.float32)
        lib().wl_bounds(self.handle, 0, self.K, fptr(out))
        return out

    def block_theta(self, k: int) -> np.ndarray:
        out = np.empty((self.B, DIM), np.float32)
        lib().wl_block_theta(self.handle, k, fptr(out))
        return out

    def table(self, nthreads: int | None = None) -> np.ndarray:
        out = np.empty((self.K * self.B, DIM), np.float32)
        lib().wl_table(self.handle, fptr(out), nthreads or os.cpu_count() or 1)
        return out

    def table_cs(self, nthreads: int | None = None) -> np.ndarray:
        """[N][4] (cx, cy, cz, max log-scale) of every Gaussian, block order."""
        out = np.empty((self.N, 4), np.float32)
        lib().wl_table_cs(self.handle, fptr(out), nthreads or os.cpu_count() or 1)
        return out

    def tile(self, k: int):
        ix, iy = C.c_int64(), C.c_int64()
        x0, y0, t, h = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        lib().wl_block_tile(self.handle, k, C.byref(ix), C.byref(iy), C.byref(x0), C.byref(y0),
                            C.byref(t), C.byref(h))
        return ix.value, iy.value, x0.value, y0.value, t.value, h.value

    def perm_fill(self, perm: np.ndarray):
        """(C fn, user) filling block k of the table re-blocked by `perm` (row i
        of the new table = generator row perm[i]); keeps its buffers alive."""
        perm = np.ascontiguousarray(perm, np.uint64)
        st = _PermFill(C.c_void_p(self.handle), perm.ctypes.data, len(perm))
        self._perm_keep = (perm, st)
        return C.cast(lib().wl_perm_fill_cb, C.c_void_p).value, C.addressof(st)

    @property
    def fill_fn(self):
        """(C function pointer, user pointer) for the oracle's lazy host tier."""
        return C.cast(lib().wl_block_theta_cb, C.c_void_p).value, self.handle


TRAJ = {"orbit": 0, "aerial": 1, "street": 2}


class Trajectory:
    def __init__(self, scene: Scene, kind: str, *, n_views: int = 0, altitude: float = 0.0,
                 spacing: float = 1.0, strip: float = 150.0, fovx_deg: float = 60.0,
                 znear: float = 0.1, zfar: float = 1000.0, width: int = 1920,
                 height: int = 1080, radius_scale: float = 1.5, shuffled: bool = False,
                 shuffle_seed: int = SEEDS["shuffle"]):
        self.scene = scene
        self.params = TrajParams(TRAJ[kind], n_views, altitude, spacing, strip, fovx_deg, znear,
                                 zfar, width, height, radius_scale)
        self.handle = lib().wl_traj_create(scene.handle, C.byref(self.params))
        self.n_views = int(lib().wl_traj_num_views(self.handle))
        if shuffled:
            lib().wl_traj_set_order(self.handle, 1, shuffle_seed)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.wl_traj_destroy(self.handle)
            self.handle = None

    def features(self, focus: float) -> np.ndarray:
        """(n_views, 6) pose features in the current order: centre, centre + focus * forward"""
        out = np.empty((self.n_views, 6), np.float64)
        lib().wl_traj_features(self.handle, focus, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def reorder(self, perm):
        """present the views in order perm (indices into the current order)"""
        p = np.ascontiguousarray(perm, np.uint64)
        assert p.shape == (self.n_views,)
        lib().wl_traj_set_perm(self.handle, p.ctypes.data_as(C.POINTER(C.c_uint64)))

    def batch_planes(self, b: int, J: int) -> np.ndarray:
        out = np.empty((J, 6, 4), np.float32)
        lib().wl_traj_batch_planes(self.handle, b, J, fptr(out))
        return out

    def batch_cameras(self, b: int, J: int):
        arr = (Camera * J)()
        lib().wl_traj_batch_cameras(self.handle, b, J, arr)
        return list(arr)


def look(pos, fwd, up, fovx_deg, width, height, znear, zfar) -> Camera:
    cam = Camera()
    v3 = C.c_double * 3
    lib().wl_camera_look(C.byref(cam), v3(*pos), v3(*fwd), v3(*up), fovx_deg, width, height,
                         znear, zfar)
    return cam


def camera_planes(cam: Camera) -> np.ndarray:
    out = np.empty((6, 4), np.float32)
    lib().wl_camera_planes(C.byref(cam), fptr(out))
    return out


def camera_sees(cam: Camera, p) -> bool:
    arr = (C.c_double * 3)(*[float(x) for x in p])
    return bool(lib().wl_camera_sees(C.byref(cam), arr))


def grad_block(seed: int, k: int, B: int, rows: int, t: int) -> np.ndarray:
    out = np.empty((B, DIM), np.float32)
    lib().wl_grad_block(seed, k, B, rows, t, fptr(out))
    return out


def mask_block(seed: int, k: int, B: int, rows: int, t: int, p32: int) -> np.ndarray:
    out = np.empty(((B + 31) // 32,), np.uint32)
    lib().wl_mask_block(seed, k, B, rows, t, p32, out.ctypes.data_as(C.POINTER(C.c_uint32)))
    return out


def grad(seed: int, gid: int, a: int, t: int) -> float:
    return float(lib().wl_grad(seed, gid, a, t))


# ----------------------------------------------------------------- configs
@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config as a concrete, seeded run."""
    name: str
    n_gaussians: int
    block_size: int
    side: float
    traj: str
    J: int
    capacity: int            # C per shard at world size 1 (C_g = ceil(C / G))
    traj_kw: tuple = ()
    shuffled: bool = False
    scene_kw: tuple = ()
    build: bool = False      # NEXT f2b: Morton-build the (unsorted) table at setup
    tsp: bool = False        # NEXT f4: reorder the views by the clustered TSP at setup

    def scene(self) -> Scene:
        return Scene(self.n_gaussians, self.block_size, side=self.side, **dict(self.scene_kw))

    def trajectory(self, scene: Scene) -> Trajectory:
        return Trajectory(scene, self.traj, shuffled=self.shuffled, **dict(self.traj_kw))


_ORBIT = (("n_views", 16), ("altitude", 40.0), ("fovx_deg", 25.0), ("znear", 0.05),
          ("zfar", 1.8), ("radius_scale", 1.0))
_TINY_SCENE = (("lot", 20.0), ("footprint", 12.0), ("hmin", 2.0), ("hmax", 12.0))
_STREET = (("altitude", 2.0), ("spacing", 1.0), ("fovx_deg", 90.0), ("znear", 0.1),
           ("zfar", 200.0))
_AERIAL = (("altitude", 150.0), ("spacing", 10.0), ("strip", 150.0), ("fovx_deg", 60.0),
           ("znear", 1.0), ("zfar", 400.0))

CONFIGS = {
    # configs[0]: tiny synthetic scene, 100k Gaussians in 64 blocks (B=1568, R18), 16-pose orbit
    "tiny": Workload("tiny", 100_000, 1568, 80.0, "orbit", 2, 24, _ORBIT, False, _TINY_SCENE),
    # configs[1]: 11M in-memory regime, aerial trajectory, batch 4 (C = K)
    "11m": Workload("11m", 11_000_000, 4096, 2800.0, "aerial", 4, 2686, _AERIAL),
    # configs[2]: 100M host-offload regime, street trajectory, J=64
    "100m": Workload("100m", 100_000_000, 4096, 2800.0, "street", 64, 2103, _STREET),
    # configs[3]: 1B city-scale aerial, 8-way block sharding
    "1b": Workload("1b", 1_000_000_000, 4096, 2800.0, "aerial", 64, 21032, _AERIAL),
    # configs[4]: trajectory-locality sweep at 300M (smooth vs random)
    "300m": Workload("300m", 300_000_000, 4096, 2800.0, "aerial", 64, 6309, _AERIAL),
    "300m_random": Workload("300m_random", 300_000_000, 4096, 2800.0, "aerial", 64, 6309,
                            _AERIAL, True),
    # the shuffled views re-ordered by the clustered TSP on the GPU at setup (f4)
    "300m_tsp": Workload("300m_tsp", 300_000_000, 4096, 2800.0, "aerial", 64, 6309, _AERIAL,
                         True, (), False, True),
    # ablation "w/o Morton": no spatial sort before blocking
    "300m_nomorton": Workload("300m_nomorton", 300_000_000, 4096, 2800.0, "aerial", 64, 6309,
                              _AERIAL, False, (("layout", 1),)),
    # the same unsorted scene, Morton-sorted and blocked on the GPU at setup (f2b)
    "300m_built": Workload("300m_built", 300_000_000, 4096, 2800.0, "aerial", 64, 6309,
                           _AERIAL, False, (("layout", 1),), True),
}


# ------------------------------------------------------ CUDA twin (harness)
_cuda_lib = None


def cuda_lib():
    """libtgsworkload_cuda.so: bit-identical device twin of grad_block / mask_block
    (stands in for the renderer's backward pass; not part of the product)."""
    global _cuda_lib
    if _cuda_lib is None:
        path = os.path.join(_HERE, "libtgsworkload_cuda.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make`")
        L = C.CDLL(path)
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        L.wl_cuda_synth_grads.argtypes = [vp, u64, vp, vp, u32, u32, u64, u64, u64, vp]
        L.wl_cuda_synth_grads_devn.argtypes = [vp, u64, vp, vp, vp, u32, u32, u64, u64, u64, vp]
        L.wl_cuda_synth_mask.argtypes = [vp, u32, vp, vp, u32, u32, u64, u64, u64, u32, vp]
        L.wl_cuda_poke.argtypes = [vp, C.c_float, vp]
        _cuda_lib = L
    return _cuda_lib


def synth_grads_cuda(act, B, N, seed, t, stream):
    """Write counter-hash gradients of the active blocks of a tgs_activation into
    its grad pool (on `stream`, after the activation's ready event)."""
    if act.n_active_blocks == 0:
        return
    if act.n_active_blocks == 0xFFFFFFFF:  # asynchronous activate: |A| on the device
        rc = cuda_lib().wl_cuda_synth_grads_devn(act.d_grads, act.grad_stride, act.d_active_blocks,
                                                 act.d_active_slots, act.d_n_active,
                                                 act.global_stride, B, N, seed, t, stream)
        if rc != 0:
            raise RuntimeError(f"wl_cuda_synth_grads_devn: cuda error {rc}")
        return
    rc = cuda_lib().wl_cuda_synth_grads(act.d_grads, act.grad_stride, act.d_active_blocks,
                                        act.d_active_slots, act.n_active_blocks, B, N, seed, t,
                                        stream)
    if rc != 0:
        raise RuntimeError(f"wl_cuda_synth_grads: cuda error {rc}")


def synth_mask_cuda(d_mask, act, B, N, seed, t, p32, stream):
    if act.n_active_blocks == 0:
        return
    rc = cuda_lib().wl_cuda_synth_mask(d_mask, (B + 31) // 32, act.d_active_blocks,
                                       act.d_active_slots, act.n_active_blocks, B, N, seed, t,
                                       p32, stream)
    if rc != 0:
        raise RuntimeError(f"wl_cuda_synth_mask: cuda error {rc}")
