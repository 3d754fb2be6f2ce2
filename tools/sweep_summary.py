"""profiles/locality_sweep_r01.md from gpurun_out/bench_sweep_*.json (+ the N=1 lines)."""
import json
import os

def load(f):
    if not os.path.exists(f):
        return None
    return json.loads(open(f).read().strip().splitlines()[-1])

rows = []
for G in (1, 2, 4, 8):
    for order, name in (("smooth", "default"), ("tsp", "300m_tsp"), ("random", "300m_random")):
        f = f"gpurun_out/bench_{name}.json" if G == 1 else f"gpurun_out/bench_sweep_{order}_g{G}.json"
        d = load(f)
        if not d:
            continue
        det = d["detail"]
        rows.append(f"| {G} | {order} | {d['value'] / 1e9:.3f} | {G * d['value'] / 1e9:.2f} | "
                    f"{d['ms_per_step']:.2f} | {det['active_blocks_per_step']:.0f} | "
                    f"{det['stage_in_blocks_per_step']:.0f} | {det['h2d_GB_per_step']:.3f} | "
                    f"{100 * d['roofline']['frac']:.0f}% |")
out = ["# configs[4]: trajectory-locality sweep at 300M (round 1, one B200)", "",
       "One GPU's share of a G-way block-sharded 300M table (`bench.py --config 300m[_tsp|_random] "
       "--shard-of G`: rank 0's shard, capacity C/G, every batch's cameras), so the per-GPU step "
       "of a G-GPU run without its two latency-bound collectives. `G x value` is the aggregate "
       "a G-GPU box would reach if every GPU matched rank 0 and the host links and DRAM kept up "
       "(not measured: one GPU per gpurun call). Orders: the generator's path (smooth), shuffled "
       "(random, the paper's Shuffle), shuffled then re-ordered by `tgs_order_views` (tsp, f4).", "",
       "| G | order | G Gaussians/s per GPU | G x value | ms/step | active blocks/step | "
       "S+ blocks/step | H2D GB/step | k_adam of HBM peak |", "|---|---|---|---|---|---|---|---|---|"] + rows
open("profiles/locality_sweep_r01.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
