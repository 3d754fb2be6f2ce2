"""Time NEXT f2b (tgs_build_layout: Morton sort + blocking) on unsorted city
scenes (the paper's preprocessing takes 1.9 min at 102M and
21.2 min at 1.1B), and the oracle on a sample.  Usage: python tools/layout_bench.py N"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workload as W  # noqa: E402
from paper_2605_20150_b200 import tidegs as T  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 300_000_000
B = 4096
t0 = time.perf_counter()
sc = W.Scene(n, B, side=2800.0, layout=1)
cs = sc.table_cs()
gen_s = time.perf_counter() - t0
t0 = time.perf_counter()
perm, bounds, gpu_ms = T.build_layout(cs, B)
wall_s = time.perf_counter() - t0
# oracle on a bounded sample (same recipe, the first m Gaussians)
m = min(n, 4_000_000)
t0 = time.perf_counter()
O.build_layout(cs[:m], B)
orc_s = time.perf_counter() - t0
r_raw = float(np.median(sc.bounds()[:, 3]))
r_new = float(np.median(bounds[:, 3]))
print(json.dumps({"n": n, "block_size": B, "gpu_ms": gpu_ms,
                  "wall_s_incl_h2d_d2h": wall_s, "gen_s": gen_s,
                  "oracle_s_on_sample": orc_s, "oracle_sample": m,
                  "oracle_ns_per_gaussian": orc_s / m * 1e9,
                  "gpu_ns_per_gaussian": gpu_ms * 1e6 / n,
                  "median_block_radius_unsorted_m": r_raw,
                  "median_block_radius_morton_m": r_new}))
