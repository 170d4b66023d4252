"""Summarise `ncu --set full` reports into JSON for profiles/: key throughput / traffic / issue
metrics from the raw page and the top stall reasons (warp-state samples) from the source page.
usage: python tools/ncu_summary.py out.json name=report.ncu-rep [name=report.ncu-rep ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "pcie__read_bytes.sum.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum"]


def ncu_csv(rep, page):
    args = ["ncu", "-i", rep, "--page", page, "--csv"] + (["--print-source", "sass"] if page == "source" else [])
    out = subprocess.run(args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    rows = ncu_csv(rep, "raw")
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            d[k] = f"{v[i]} {u[i]}".strip()
    src = ncu_csv(rep, "source")
    hh = src[1]
    data = src[2:]
    cols = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: sum(float(r[hh.index(c)] or 0) for r in data) for c in cols}
    s = sum(tot.values()) or 1.0
    d["stall_share"] = {c[6:]: round(x / s, 3) for c, x in sorted(tot.items(), key=lambda t: -t[1])[:8]}
    return d


if __name__ == "__main__":
    out = {}
    for a in sys.argv[2:]:
        name, rep = a.split("=", 1)
        out[name] = summarise(rep)
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))
