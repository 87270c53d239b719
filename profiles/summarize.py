"""Summarise ncu captures into the committed profiles/ files.

    python profiles/summarize.py <report.ncu-rep | raw.csv> <launches.csv | -> <tag> [config | -]

(a raw.csv is the `--page raw --csv` export of the report; `-` for the launch
list or the config skips the launch file / the traffic file)

Writes profiles/<tag>_kernels.md (per-kernel key metrics of the --set full
capture), profiles/<tag>_launches.csv (launch list: kernel, duration) and
profiles/traffic_<config>.json (dram bytes per launch of the dominant kernels
and the counters of the resource binding the force pass, measured on that
configuration; read by bench.py for roofline.traffic of the same config).
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % (active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "L1 ld hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 ld sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "RED sectors"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "LSU data pipe %"),
    ("l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed", "TEX data pipe %"),
    ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "L2 atomic %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rep, launches, tag = sys.argv[1:4]
    config = sys.argv[4] if len(sys.argv) > 4 else "c5"
    if rep.endswith(".csv"):  # `ncu -i X.ncu-rep --page raw --csv` exported on the GPU box
        raw = open(rep).read()
        raw = raw[raw.find('"ID"'):]
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary ({tag})", "",
             "| kernel | " + " | ".join(k[1] for k in KEYS) + " |",
             "|---|" + "---|" * len(KEYS)]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        vals = []
        for k, _ in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        lines.append(f"| `{name[:60]}` | " + " | ".join(vals) + " |")
        i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        tb = to_bytes(r[i_r], units[i_r]) + to_bytes(r[i_w], units[i_w])
        key = "force_traffic" if "force" in name else ("density_traffic" if "density" in name
                                                       else None)
        if key and key not in traffic:
            traffic[key] = tb
        if key == "force_traffic" and "binding_resource" not in traffic:
            def metric(m):
                return float(r[hdr.index(m)].replace(",", "")) if m in hdr else None
            traffic["binding_resource"] = {
                "name": "L1 LSU data pipe (force pass)",
                "l1_throughput_pct": metric("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                "lsu_pipe_pct": metric(
                    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                "tex_pipe_pct": metric(
                    "l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                "l2_atomic_pct": metric(
                    "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                "issue_active_pct": metric("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_pct": metric(
                    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "shared_wavefronts": metric("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                "shared_bank_conflicts": metric(
                    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")}
    open(os.path.join(HERE, f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
    traffic["source"] = (f"profiles/{tag}_kernels.md, config {config} "
                         "(dram__bytes_read.sum + dram__bytes_write.sum per launch)")
    if config != "-":
        json.dump(traffic, open(os.path.join(HERE, f"traffic_{config}.json"), "w"), indent=1)
    if launches == "-":
        print("wrote", tag)
        return
    # launch list: kernel name, duration
    out = []
    with open(launches) as f:
        text = f.read()
    start = text.find('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            out.append((r["Kernel Name"][:80], r["Metric Value"], r["Metric Unit"]))
    with open(os.path.join(HERE, f"{tag}_launches.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "duration", "unit"])
        w.writerows(out)
    print("wrote", tag, len(out), "launches")


if __name__ == "__main__":
    main()
