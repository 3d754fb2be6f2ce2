"""The C-ABI library loads, exports every entry point include/tidegs.h declares,
and validates configs before touching the device (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2605_20150_b200 import tidegs as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_and_binding_declare_the_same_symbols():
    hdr = open(os.path.join(ROOT, "include", "tidegs.h")).read()
    declared = set(re.findall(r"^(?:tgs_status|uint32_t|uint64_t|const char\*)\s+(tgs_\w+)\s*\(",
                              hdr, re.M))
    assert declared == set(T.SYMBOLS)


def test_library_exports_every_symbol():
    L = T.lib()
    for s in T.SYMBOLS:
        assert hasattr(L, s), s
    assert L.tgs_status_string(T.EINVAL) == b"invalid argument"


def test_config_struct_layout_matches_the_header(tmp_path):
    """ctypes' tgs_config / tgs_activation / tgs_stats layouts equal the C header's
    (a C program compiled against include/tidegs.h prints sizeof / offsetof)."""
    src = tmp_path / "layout.c"
    fields = [f[0] for f in T.Config._fields_]
    body = "".join(f'printf("%zu ", offsetof(tgs_config, {("lambda" if f == "lambda_" else f)}));'
                   for f in fields)
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "tidegs.h"\nint main(void){'
                   + body + 'printf("%zu %zu %zu\\n", sizeof(tgs_config), sizeof(tgs_activation), '
                   'sizeof(tgs_stats)); return 0;}\n')
    import subprocess
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    out = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [getattr(T.Config, f).offset for f in fields]
    assert out[:len(fields)] == want
    assert out[len(fields):] == [C.sizeof(T.Config), C.sizeof(T.Activation), C.sizeof(T.Stats)]


def test_elf_has_sm100a_code():
    """The product .so carries sm_100a SASS (no PTX-only JIT path)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", T.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _init(cfg, bounds, rows=None):
    h = C.c_void_p()
    rp = rows.ctypes.data if rows is not None else None
    fill = None if rows is not None else C.cast(T.FILL_FN(lambda *a: None), C.c_void_p).value
    return T.lib().tgs_init_table(C.byref(cfg), rp, fill, None,
                                  bounds.ctypes.data_as(C.POINTER(C.c_float)), None, None,
                                  C.byref(h))


@pytest.mark.parametrize("field,value", [("dim", 58), ("block_size", 6), ("block_size", 0),
                                         ("capacity", 0), ("n_gaussians", 0),
                                         ("lambda_", 1.5), ("lambda_", -0.1), ("gamma", 1.0),
                                         ("gamma", 0.0), ("quota_den", 0), ("quota_num", 3),
                                         ("world_size", 0), ("rank", 2), ("moments", 7),
                                         ("max_cameras", 0), ("max_cameras", 300),
                                         ("max_age", 5000), ("pool_slots", 3), ("xfer", 2),
                                         ("xfer", -1)])
def test_invalid_config_is_einval(field, value):
    cfg = T.make_config(1000, 16, 4)
    setattr(cfg, field, value)
    bounds = np.zeros((63, 4), np.float32)
    assert _init(cfg, bounds) == T.EINVAL


def test_invalid_bounds_and_sources_are_einval():
    cfg = T.make_config(64, 16, 2)
    b = np.zeros((4, 4), np.float32)
    b[2, 0] = np.nan
    assert _init(cfg, b) == T.EINVAL
    b = np.zeros((4, 4), np.float32)
    b[1, 3] = -1.0
    assert _init(cfg, b) == T.EINVAL
    # exactly one of theta_rows / fill
    h = C.c_void_p()
    ok_b = np.zeros((4, 4), np.float32)
    assert T.lib().tgs_init_table(C.byref(cfg), None, None, None,
                                  ok_b.ctypes.data_as(C.POINTER(C.c_float)), None, None,
                                  C.byref(h)) == T.EINVAL


def test_frustum_planes_helper_matches_pinhole_geometry():
    """R1 helper: a point projecting inside the image at near<=z<=far is inside
    all six planes; one outside the image or depth range is outside one."""
    rng = np.random.default_rng(3)
    ang = 0.3
    Rm = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    t = np.array([0.5, -0.2, 2.0])
    w2c = np.eye(4)
    w2c[:3, :3] = Rm
    w2c[:3, 3] = t
    fx = fy = 400.0
    W_, H = 640, 480
    planes = T.frustum_planes(w2c, fx, fy, 320.0, 240.0, W_, H, 0.5, 50.0).astype(np.float64)
    for _ in range(2000):
        p = rng.uniform(-40, 40, 3)
        pc = Rm @ p + t
        inside_img = False
        if 0.5 <= pc[2] <= 50.0:
            u, v = fx * pc[0] / pc[2] + 320.0, fy * pc[1] / pc[2] + 240.0
            inside_img = 0 <= u <= W_ and 0 <= v <= H
        d = planes[:, :3] @ p + planes[:, 3]
        margin = 1e-4 * (1 + np.abs(p).sum())
        if inside_img:
            assert (d >= -margin).all()
        elif (d > margin).all():
            raise AssertionError(f"point {p} outside the frustum is inside all planes")
    assert T.lib().tgs_frustum_planes(None, 1, 1, 0, 0, 1, 1, 0.1, 1.0, None) == T.EINVAL


def test_store_config_is_validated_before_the_device(tmp_path):
    """f3: NULL store / dir, or a CPU cache smaller than 2C (R27), is EINVAL."""
    cfg = T.make_config(64, 16, 2)
    b = np.zeros((4, 4), np.float32)
    rows = np.zeros((64, 59), np.float32)
    h = C.c_void_p()
    bp = b.ctypes.data_as(C.POINTER(C.c_float))
    L = T.lib()
    assert L.tgs_init_table_store(C.byref(cfg), None, rows.ctypes.data, None, None, bp, None, None,
                                  C.byref(h)) == T.EINVAL
    for d, H in ((None, 4), (os.fsencode(str(tmp_path)), 3)):
        sc = T.StoreConfig(d, H, 0, 1, 0)
        assert L.tgs_init_table_store(C.byref(cfg), C.byref(sc), rows.ctypes.data, None, None, bp,
                                      None, None, C.byref(h)) == T.EINVAL
    assert not os.listdir(tmp_path)  # nothing written


def test_order_views_validates_inputs():
    """f4: M = 0, D outside [1, 8], non-finite features are EINVAL (before the device)."""
    L = T.lib()
    u = (C.c_uint32 * 4)()
    f = np.zeros((4, 3))
    fp = f.ctypes.data_as(C.POINTER(C.c_double))
    assert L.tgs_order_views(fp, 0, 3, 0, u, None, None, None, None) == T.EINVAL
    assert L.tgs_order_views(fp, 4, 0, 0, u, None, None, None, None) == T.EINVAL
    assert L.tgs_order_views(fp, 1, 9, 0, u, None, None, None, None) == T.EINVAL
    f[1, 2] = np.inf
    assert L.tgs_order_views(fp, 4, 3, 0, u, None, None, None, None) == T.EINVAL
    assert L.tgs_order_views(None, 4, 3, 0, u, None, None, None, None) == T.EINVAL
