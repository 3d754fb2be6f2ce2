"""Render profiles/bench_rNN.md from the bench JSON lines in gpurun_out/.
   python tools/bench_summary.py r01 default fine 100m_persist 11m 300m_random"""
import json
import shutil
import sys

DESC = {"default": "300m aerial smooth, J=64, C=6309, cold restart (the N=1 headline)",
        "fine": "same + Level-2 fine filter (f1) as I_t",
        "100m_persist": "100m street, J=64, C=2103, moments persist (after 400 warm-up batches)",
        "11m": "11m aerial, J=4, C=K (in-memory)",
        "300m_random": "300m aerial, shuffled views (w/o trajectory order)",
        "300m_tsp": "300m aerial, shuffled views re-ordered by the GPU clustered TSP (f4)",
        "1b_shard8": "1B aerial, one GPU's share of the 8-way block-sharded table (--shard-of 8)",
        "store_1b_shard8": "the same shard on the f3 store tier (O_DIRECT segments on local disk, CPU cache 3C)"}

tag, names = sys.argv[1], sys.argv[2:]
src = "gpurun_out"
if names and names[0].startswith("--src="):
    src, names = names[0][6:], names[1:]
rows = []
lines = {}
for f in names:
    shutil.copy(f"{src}/bench_{f}.json", f"profiles/bench_{tag}_{f}.json")
    d = json.loads(open(f"{src}/bench_{f}.json").read().strip().splitlines()[-1])
    lines[f] = d
    r, l, det, e = d["roofline"], d["link_roofline"], d["detail"], d.get("e2e")
    e2e = f"{e['value'] / 1e9:.3f} ({e['ms_per_step']:.2f} ms)" if e else "-"
    peak = r["peak"]
    rows.append(f"| {f} | {DESC.get(f, f)} | {d['value'] / 1e9:.3f} | {d['ms_per_step']:.2f} | {e2e} | "
                f"{det['active_blocks_per_step']:.0f} | {det['stage_in_blocks_per_step']:.0f} | "
                f"{det['h2d_GB_per_step']:.3f} / {det['d2h_GB_per_step']:.3f} | "
                f"{r['achieved']:.0f} ({100 * r['frac']:.0f}%) | "
                f"{l['h2d_achieved'] or 0:.1f} / {l['d2h_achieved'] or 0:.1f} (peak {l['h2d_peak']:.1f} / {l['d2h_peak']:.1f}) |")
out = [f"# bench.py results, round {tag[1:]} (one B200, fresh gpurun box)", "",
       "Raw JSON lines: `profiles/bench_%s_*.json`. value = active Gaussians updated by Adam per "
       "second of device time (CUDA events on the compute stream); one step = tgs_activate + "
       "tgs_step_adam (a1-a5). e2e = the same timed steps through the public API with pinned host "
       "camera planes in and an async per-step counter readback, wall clock. Adam GB/s = "
       "algorithmic bytes (1652 B per active row; 708 B per row + the 472 B/row m, v record for "
       "the first update of a cold-restarted block) / event-timed k_adam launch vs the measured HBM copy peak of MEASURED_PEAKS.json (%.0f GB/s). Link GB/s = "
       "copy-batch bytes / event-timed span on the h2d / d2h streams vs the pinned 1 GiB copy "
       "peak measured in the same run." % (tag, peak), "",
       "| run | workload | G Gaussians/s | ms/step | e2e G/s | active blocks/step | S+ blocks/step | "
       "H2D / D2H GB/step | k_adam GB/s (% of peak) | link GB/s h2d / d2h |",
       "|---|---|---|---|---|---|---|---|---|---|"] + rows
d = lines.get("default")
if d:
    out += ["", f"* default: clocks {d['clocks']}; cpu_baseline {d['cpu_baseline']}; "
                f"gpu_launches {d['gpu_launches']} over {d['steps']} steps."]
for f, d in lines.items():
    st = (d.get("detail") or {}).get("store")
    if st:
        out += [f"* {f}: CPU-cache hit rate {st['hit_rate']:.2f}, "
                f"{st['per_step']['misses']:.1f} misses/step read at "
                f"{st['ssd_read_GBps_in_reads']:.2f} GB/s (dd sequential peak "
                f"{st.get('ssd_read_peak_GBps') or 0:.2f} GB/s); see profiles/store_r01.md."]
open(f"profiles/bench_{tag}.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
