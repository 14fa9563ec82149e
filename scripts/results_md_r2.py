"""profiles/r2_bench_*.json -> profiles/r2_results.md (round-2 results table)."""
import json

cfgs = ["c1", "c2", "c3", "c3_l2", "c4", "c5"]
rows = []
for c in cfgs:
    d = json.load(open(f"profiles/r2_bench_{c}.json"))
    r = d["roofline"]
    rows.append((c.upper().replace("_L2", " (all L2)"), d["config"]["weights"], d["value"],
                 d["e2e"]["value"], r["achieved"], r["peak"], r["frac"], r["hybrid"]["frac_hybrid"],
                 r["frac_of_hbm"], r["exchange_fraction"], d["cpu_baseline"]["value"],
                 d["cpu_baseline"]["cores"], "".join(w[0] for w in d["layer_residency"][:-1]),
                 r["target_samples_per_s_at_0.70_of_l2"]))
c4 = json.load(open("profiles/r2_bench_c4.json"))
out = ["# Round 2 results (one B200, `python bench.py --config Cx`)", "",
       "Value = on-line samples/s (bs=1), device-timed over 5 launches of "
       f"{c4['config']['samples_per_step']:,} samples each, inputs resident in HBM; e2e = "
       "`trainer.train_epoch` from pinned host buffers (H2D inside the timed region). Roofline: "
       "12 B per weight per sample against the L2 read+write peak measured in the same run (the "
       "weights never live in HBM inside the loop: registers / shared memory / L2); `hybrid` = "
       "SURVEY §8(d) t_min = sum over levels of bytes / level peak (registers free, shared "
       "memory and L1 at 148 x 128 B/clk, L2 measured) divided by the measured sample time; HBM "
       "fraction kept only as a secondary number. CPU = the reference algorithm (oracle port, "
       "bit-exact with the reference tiled variant) on the box's host cores (C4: 12 s sample, "
       "others 4 s). Hidden-layer residency: s = shared memory, r = register rows, l = L2.", "",
       "| config | weights | samples/s | e2e | achieved GB/s | L2 peak GB/s | frac of L2 | "
       "frac hybrid | frac of HBM | exchange share | CPU samples/s (cores) | hidden layers | "
       "0.70 of L2 would be |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    out.append(f"| {r[0]} | {r[1]:,} | {r[2]:,.0f} | {r[3]:,.0f} | {r[4]:,.0f} | {r[5]:,.0f} | "
               f"{r[6]:.3f} | {r[7]:.3f} | {r[8]:.3f} | {r[9]:.3f} | {r[10]:,.0f} ({r[11]}) | "
               f"{r[12]} | {r[13]:,.0f} |")
cpu = c4["cpu_baseline"]
out += ["", "C4 (the headline, BASELINE.json north_star) is at "
        f"{rows[4][6]:.3f} of the L2 roofline; the 0.70 target would need "
        f"{rows[4][13]:,.0f} samples/s. The sample is latency-bound: "
        f"{c4['roofline']['sync_bound']['exchanges_per_sample']} all-to-all exchanges at the "
        f"measured bare-exchange floor ({c4['roofline']['sync_bound']['hop_us']} us each) are "
        f"{100 * c4['roofline']['sync_bound']['share_of_measured_sample']:.0f}% of the sample.", "",
        f"CPU context (C4, {cpu['cpu']['model']}, nproc {cpu['cpu']['nproc']}):"]
for k, v in cpu["legs"].items():
    out.append(f"- {k}: {v['value']:,} {v['unit']} ({v['cores']} cores; {v['sample']})")
dfm, ev = c4["deform"], c4["eval"]
out += ["", f"Deformation (K2): {dfm['imgs_per_s']:,.0f} imgs/s ({dfm['ms_per_epoch']} ms per "
        f"{dfm['images']:,}-image epoch), {dfm['roofline']['frac']:.2f} of its issue bound "
        f"({dfm['roofline']['peak_imgs_per_s']:,.0f} imgs/s at "
        f"{dfm['roofline']['warp_instructions_per_img']:,.0f} warp instructions per image, "
        "profiles/ncu_deform.json).",
        f"Evaluation (K4, C4): {ev['imgs_per_s']:,.0f} imgs/s, {ev['TFLOPs']} TFLOP/s fp32 SIMT.", "",
        "Raw lines: `profiles/r2_bench_*.json`; launch list `profiles/r2_launches.md`; C4 "
        "one-sample timeline `profiles/r2_trace_c4.txt`; GPU tests `profiles/r2_gputest.log`."]
try:  # the driver-style pair, when captured (scripts: python bench.py; --impl reference)
    dd = json.load(open("profiles/r2_bench_default.json"))
    rr = json.load(open("profiles/r2_bench_reference.json"))
    out += ["", "Driver-style pair (`python bench.py` and `python bench.py --impl "
            "reference`, `profiles/r2_bench_default.json`, `profiles/r2_bench_reference.json`): "
            f"ours {dd['value']:,.0f} samples/s device-timed, {dd['e2e']['value']:,.0f} end to end; "
            f"the reference algorithm on {rr['cpu_baseline']['cores']} host cores "
            f"{rr['value']:,.1f} samples/s -> e2e ratio {dd['e2e']['value'] / rr['value']:.1f}x."]
except (OSError, KeyError, ValueError):
    pass
open("profiles/r2_results.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
