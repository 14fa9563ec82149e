"""profiles/r1_bench_c*.json -> profiles/r1_results.md"""
import json

rows = []
for c in ["c1", "c2", "c3", "c4", "c5"]:
    d = json.load(open(f"profiles/r1_bench_{c}.json"))
    rows.append((c.upper(), d["config"]["weights"], d["value"], d["e2e"]["value"],
                 d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"].get("frac_of_l2_rw"),
                 d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"],
                 "".join(w[0] for w in d["layer_residency"][:-1])))
out = ["# Round 1 results (one B200, `python bench.py --config Cx`)", "",
       "Value = on-line samples/s (bs=1) device-timed over 5 launches of " f"{json.load(open('profiles/r1_bench_c4.json'))['config']['samples_per_step']:,} samples each, "
       "inputs resident in HBM; e2e = `trainer.train_epoch` from pinned host buffers (H2D of the "
       "step's images inside the timed region). Roofline: 12 B per weight per sample against the "
       "measured HBM copy peak (MEASURED_PEAKS.json, " f"{json.load(open('profiles/r1_bench_c4.json'))['roofline']['peak']:.0f} GB/s) and the L2 read+write peak "
       "measured in the same run. CPU = the reference algorithm (oracle port, bit-exact with the "
       "reference tiled variant) on the box's host cores. Layer residency per hidden layer: "
       "s = shared memory, r = register row block, l = streamed from L2.", "",
       "| config | weights | samples/s | e2e samples/s | achieved GB/s | frac of HBM | frac of L2 r+w "
       "| CPU samples/s (cores) | hidden layers | GPU/CPU |",
       "|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    l2 = "-" if r[6] is None else f"{r[6]:.3f}"
    out.append(f"| {r[0]} | {r[1]:,} | {r[2]:,.0f} | {r[3]:,.0f} | {r[4]:,.0f} | {r[5]:.3f} | {l2} "
               f"| {r[7]:,.0f} ({r[8]}) | {r[9]} | {r[2] / r[7]:,.0f}x |")
out += ["", "C4 is the headline (BASELINE.json `north_star`: within 70% of the bandwidth roofline; "
        "12 B/weight at the HBM peak = 45.1k samples/s, 70% = 31.5k).",
        "Per-phase cycles and the per-layer split are in each bench line "
        "(`profile_cycles_per_sample`, `profile_cycles_per_layer`); the one-sample timeline of C4 "
        "is `r1_trace_c4.txt`."]
open("profiles/r1_results.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
