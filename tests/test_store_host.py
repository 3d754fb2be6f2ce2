"""Host-only stress test of the f3 store tier's native code (no GPU): builds
tests/store_host_test.cpp against paper_2605_20150_b200/csrc/tidegs_store.cpp
and runs it (thread-pool generations, base write, coalesced reads, appends
across segment rollover, LRU victims, barrier; every record's content checked)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("direct", [0, 1])
def test_store_native_code_on_the_host(tmp_path, direct):
    exe = tmp_path / "store_host_test"
    src = [os.path.join(ROOT, "tests", "store_host_test.cpp"),
           os.path.join(ROOT, "paper_2605_20150_b200", "csrc", "tidegs_store.cpp")]
    subprocess.run(["g++", "-std=c++17", "-O2", "-pthread", "-o", str(exe)] + src, check=True)
    r = subprocess.run([str(exe), str(tmp_path / "store"), str(direct)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
