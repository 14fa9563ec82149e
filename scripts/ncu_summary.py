"""Summarise one `ncu --set full` capture into profiles/<name>.json.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep profiles/ncu_train_c4.json \
        --units 2000 --unit "on-line sample" --algo-bytes 145380120 --command "..."

Per-unit DRAM / L2 bytes and the headline counters the DESIGN cites.
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors.sum", "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--units", type=float, required=True)
    ap.add_argument("--unit", default="on-line sample")
    ap.add_argument("--algo-bytes", type=float, default=None, help="algorithmic bytes per unit")
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            m[k] = {"value": vals[i], "unit": units[i]}
    stall = {}
    for i, k in enumerate(hdr):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stall[k.split("stalled_")[1]] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stall.values()) or 1.0
    stall = {k: round(v / tot, 3) for k, v in sorted(stall.items(), key=lambda kv: -kv[1])[:8]}

    def num(k, scale):
        if k not in m:
            return None
        v = float(m[k]["value"].replace(",", ""))
        u = m[k]["unit"].lower()
        f = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ms": 1e-3, "us": 1e-6,
             "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1,
             "ghz": 1e9, "mhz": 1e6}.get(u, 1)
        return v * f / scale

    dram = (num("dram__bytes_read.sum", 1) or 0) + (num("dram__bytes_write.sum", 1) or 0)
    t = num("gpu__time_duration.sum", 1)
    out = {"capture": a.rep.split("/")[-1], "command": a.command, "units_per_launch": a.units,
           "unit": a.unit, "seconds_per_launch": t,
           "dram_bytes_per_launch": dram, "dram_bytes_per_unit": dram / a.units,
           "l2_bytes_per_unit": 32 * (num("lts__t_sectors.sum", 1) or 0) / a.units,
           "algorithmic_bytes_per_unit": a.algo_bytes,
           "stall_reason_share": stall, "metrics": m}
    if a.algo_bytes and t:
        out["achieved_GBs_under_ncu"] = a.algo_bytes * a.units / t / 1e9
    if t:
        # achieved shared-memory and L2 bandwidth of the launch (128 B per smem
        # wavefront, 32 B per L2 sector) against the B200 peaks: smem 128 B/clk
        # per SM (148 SMs at the measured clock), L2 from MEASURED r+w (K6)
        clk = num("sm__cycles_elapsed.avg.per_second", 1) or 1.965e9
        wav = num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1) or 0.0
        out["smem_GBs"] = round(128 * wav / t / 1e9, 1)
        out["smem_peak_GBs"] = round(148 * 128 * clk / 1e9, 1)
        out["l2_GBs"] = round(32 * (num("lts__t_sectors.sum", 1) or 0) / t / 1e9, 1)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "metrics"}))


if __name__ == "__main__":
    main()
