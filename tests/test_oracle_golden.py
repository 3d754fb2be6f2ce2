"""Golden constants the paper / SPEC print (tests/golden/paper_constants.json),
checked against the oracle (record bytes, K, owner block, recency/score
arithmetic through selection behaviour) and for internal consistency."""
import json
import os

import numpy as np

import oracle as O

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))


def test_record_and_block_arithmetic():
    g = G["record_bytes_B4096_D59"]
    assert 4096 * 59 * 4 == g["value"] == g["pages_4k"] * 4096
    assert 4096 * 9 * 4 == G["record_bytes_B4096_D9"]["value"]
    b = G["blocks_N10000_B4096"]
    assert -(-10000 // 4096) == b["K"] and 9999 // 4096 == b["owner_of_9999"]
    assert 10000 - 2 * 4096 == b["last_block_rows"]
    p = G["plan_bytes_examples"]
    assert p["three_blocks_D9"] == 3 * 4096 * 9 * 4
    # the oracle counts exactly one record per staged block (cold: theta only)
    bounds = np.array([[0, 0, 0, 1], [5, 0, 0, 1], [10, 0, 0, 1]], np.float32)
    pl = np.array([[[1, 0, 0, 100], [-1, 0, 0, 100], [0, 1, 0, 100], [0, -1, 0, 100],
                    [0, 0, 1, 100], [0, 0, -1, 100]]], np.float32)
    o = O.Oracle(O.make_config(10000, 4096, 1, moments=O.COLD_RESTART), bounds, fill=None,
                 track_all=False)
    o.activate(pl)
    assert o.stats()["h2d_bytes"] == p["one_block_B4096_D59"]


def test_recency_and_score_examples():
    assert abs(0.9 ** 3 - G["recency_gamma09_age3"]["value"]) < 1e-12
    assert abs(0.7 * 1 + 0.3 * 0.5 - G["score_lambda07_inK_recency05"]["value"]) < 1e-12


def test_churn_table_little_law_consistency():
    """streak x eviction rate ~ 1 (Little's law) holds for the paper's T9 rows."""
    for r in G["churn_T9"]["rows"]:
        assert 0.85 <= r["streak"] * r["eviction"] <= 0.95
        assert r["cold_updates"] <= r["readmission"] <= r["eviction"]
