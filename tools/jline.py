"""Print the key numbers of one bench JSON line: python tools/jline.py FILE"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
det = d.get("detail", {})
out = {"value_G/s": round(d["value"] / 1e9, 4), "ms/step": round(d["ms_per_step"], 3),
       "adam_frac": round(d["roofline"]["frac"], 3), "S+/step": det.get("stage_in_blocks_per_step"),
       "active/step": det.get("active_blocks_per_step"),
       "e2e_G/s": round(d["e2e"]["value"] / 1e9, 4) if d.get("e2e") else None,
       "order_ms": det.get("view_order_gpu_ms"),
       "d2h_GB": det.get("d2h_GB_per_step"),
       "p50/p99_ms": [round(det["step_ms"]["p50"], 3), round(det["step_ms"]["p99"], 3)]
       if det.get("step_ms") else None}
L = d.get("link_roofline") or {}
if L.get("h2d_achieved"):
    out.update({"h2d_GBps": round(L["h2d_achieved"], 1), "d2h_GBps": round(L["d2h_achieved"] or 0, 1),
                "adam_ms": round(d["roofline"]["avg_launch_ms"], 3)})
st = det.get("store")
if st:
    out.update({"hit_rate": round(st["hit_rate"], 3), "ssd_read_GBps": st["ssd_read_GBps_in_reads"],
                "ssd_peak": st.get("ssd_read_peak_GBps"),
                "read_ms/step": st["per_step"]["read_ms"], "misses/step": st["per_step"]["misses"],
                "dirty_evict/step": st["per_step"]["dirty_evictions"],
                "read_calls/step": st["per_step"].get("read_calls"),
                "read_busy_ms/step": st["per_step"].get("read_busy_ms")})
print(json.dumps(out))
