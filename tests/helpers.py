"""Shared test helpers (inputs and bookkeeping only)."""
import numpy as np

import workload as W

DIM = 59


def lr_3dgs():
    """Per-attribute 3DGS learning rates (R9; xyz, f_dc, f_rest, opacity, scale, rot)."""
    lr = np.empty(DIM, np.float32)
    lr[0:3] = 1.6e-4
    lr[3:6] = 2.5e-3
    lr[6:51] = 1.25e-4
    lr[51] = 5e-2
    lr[52:55] = 5e-3
    lr[55:59] = 1e-3
    return lr


def tiny():
    cfg = W.CONFIGS["tiny"]
    sc = cfg.scene()
    tr = cfg.trajectory(sc)
    return cfg, sc, tr


def synth_grad(seed, N, B):
    """python callable k,t -> grads (B,59) from the shared counter generator."""
    def f(k, t):
        rows = max(0, min(B, N - k * B))
        return W.grad_block(seed, k, B, rows, t)
    return f


def synth_mask(seed, N, B, p32):
    def f(k, t):
        rows = max(0, min(B, N - k * B))
        return W.mask_block(seed, k, B, rows, t, p32)
    return f


def mask_rows(words, B):
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:B]
    return bits.astype(bool)


def box_planes(lo, hi):
    """one 'camera' whose frustum is the axis-aligned box [lo, hi] (inside iff n.p + d0 >= 0)"""
    p = np.zeros((1, 6, 4), np.float32)
    for a in range(3):
        n = np.zeros(3)
        n[a] = 1
        p[0, 2 * a, :3], p[0, 2 * a, 3] = n, -lo[a]
        p[0, 2 * a + 1, :3], p[0, 2 * a + 1, 3] = -n, hi[a]
    return p


def random_boxes(sc, n, seed=5):
    """batches that jump across the scene, each seeing a handful of blocks"""
    b = sc.bounds()
    rng = np.random.default_rng(seed)
    ext = (b[:, :3].max(0) - b[:, :3].min(0)) / 5
    out = []
    for _ in range(n):
        c = b[rng.integers(len(b)), :3]
        out.append(box_planes(c - ext / 2, c + ext / 2))
    return out
