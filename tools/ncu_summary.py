"""Summarise an ncu capture (+ optional launch-list CSV) into profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep KEY [LAUNCHES.csv] [--out-prefix profiles/r1_cfg2]

Writes <prefix>_search_ncu.txt (key metrics, top stall lines) and merges
{KEY: {...}} into profiles/ncu_summary.json (read by bench.py for
roofline.traffic = dram read+write bytes per launch of the search kernel).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = (vals[i], units[i])
    return d


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0]
                agg[name][0] += 1
                agg[name][1] += float(d["Metric Value"].replace(",", "")) / 1e3  # us
    return agg


def main():
    rep, key = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else None
    prefix = os.path.join(ROOT, "profiles", key)
    if "--out-prefix" in sys.argv:
        prefix = sys.argv[sys.argv.index("--out-prefix") + 1]
    m = raw_metrics(rep)
    dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
    lines = [f"ncu --set full capture: {os.path.basename(rep)} (1 launch of search_kernel)", ""]
    for k, (v, u) in m.items():
        lines.append(f"{k:70s} {v} {u}")
    lines.append(f"{'dram read+write bytes per launch':70s} {dram:.4e}")
    top = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25"],
                         capture_output=True, text=True).stdout
    lines += ["", "top source lines by warp-stall samples:", top]
    if launches:
        agg = launch_shares(launches)
        tot = sum(t for _, t in agg.values())
        lines += ["", f"launch list ({os.path.basename(launches)}; cold-cache, serialised):"]
        for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:15]:
            lines.append(f"  {c:4d} launches {t:12.1f} us {100 * t / tot:5.1f}%  {name}")
    with open(prefix + "_search_ncu.txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    js = os.path.join(ROOT, "profiles", "ncu_summary.json")
    data = json.load(open(js)) if os.path.exists(js) else {}
    data[key] = {"dram_bytes_per_launch": dram,
                 "duration_ns": float(m["gpu__time_duration.sum"][0].replace(",", "")) *
                 (1e6 if m["gpu__time_duration.sum"][1] == "ms" else
                  1e3 if m["gpu__time_duration.sum"][1] == "us" else 1.0),
                 "source": os.path.relpath(prefix + "_search_ncu.txt", ROOT)}
    json.dump(data, open(js, "w"), indent=1)
    print("\n".join(lines[:24]))


if __name__ == "__main__":
    main()
