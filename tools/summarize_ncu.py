"""Summarise ncu captures from gpurun_out/ into profiles/ (committed evidence).

  python tools/summarize_ncu.py <tag> [configs...]

Reads gpurun_out/<tag>_launches_c<C>.csv (gpu__time_duration per launch) and
gpurun_out/<tag>_prof_c<C>.ncu-rep (--set full of the dominant tile kernel) and
writes profiles/<tag>_ncu_summary.md plus profiles/ncu_traffic.json, which
bench.py reads for roofline.traffic (DRAM bytes per launch of the tile kernel).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active % of elapsed (tcgen05)"),
    ("TPC.TriageCompute.sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "IMMA subpipe active cycles"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU inst %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def launches(path):
    txt = "".join(l for l in open(path) if not l.startswith("=="))
    rows = list(csv.DictReader(io.StringIO(txt)))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"]
        k = k.split("(")[0][:90]
        agg[k][0] += 1
        agg[k][1] += float(r["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    return [(k, v[0], v[1], v[1] / tot) for k, v in sorted(agg.items(), key=lambda t: -t[1][1])]


def raw(rep):
    # a raw-page CSV exported on the GPU box (tools/ncu_capture.sh, keeps gpurun_out/ under
    # the 64 MiB copy-back limit) is used when present, else the .ncu-rep itself
    csv_path = rep.replace(".ncu-rep", ".raw.csv")
    if os.path.exists(csv_path):
        txt = open(csv_path).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    stalls = []
    for name, (val, _) in d.items():
        if "average_warps_issue_stalled" in name and name.endswith("per_issue_active.ratio"):
            try:
                if float(val) > 0.05:
                    stalls.append((float(val), name.replace("smsp__average_warps_issue_stalled_", "")
                                   .replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    return d, sorted(stalls, reverse=True)


def main():
    tag = sys.argv[1]
    cfgs = sys.argv[2:] or ["4", "2", "3", "5"]
    md = [f"# ncu summary `{tag}` (B200, `--clock-control none`)\n",
          "Launch lists: `ncu --metrics gpu__time_duration.sum` over `python bench.py --steps 2 "
          "--warmup 1 --no-opt-in --config C` (config 5 at `--size 16384`, `5f` at its full n = 49152; "
          "`2t` = config 2 `--int-tensor`, `4e` = config 4 `--fp64-emu`); times are "
          "cold-cache and serialised, so compare SHARES. Full captures: `ncu --set full -k "
          "regex:<tile kernel> -s 1 -c 1` of the same command (tools/ncu_capture.sh).\n"]
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for c in cfgs:
        plain = json.load(open(os.path.join(OUT, f"{tag}_plain_c{c}.json")))
        path = plain["config"]["path"]
        md.append(f"\n## config {c} — `{plain['config']['workload']}` (path `{path}`, "
                  f"n={plain['config']['n']})\n")
        md.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
        for k, cnt, ns, sh in launches(os.path.join(OUT, f"{tag}_launches_c{c}.csv"))[:8]:
            md.append(f"| `{k}` | {cnt} | {ns / 1e6:.3f} | {100 * sh:.1f}% |")
        d, stalls = raw(os.path.join(OUT, f"{tag}_prof_c{c}.ncu-rep"))
        md.append(f"\nTile kernel `{d.get('Kernel Name', ('?',))[0][:100]}`:\n")
        md.append("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in d:
                md.append(f"| {label} (`{key}`) | {d[key][0]} {d[key][1]} |")
        md.append("\nTop warp stall reasons (warps per issue): " +
                  ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
        try:
            rb = float(d["dram__bytes_read.sum"][0]) * {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "byte": 1,
                                                        "Kbyte": 1e3}[d["dram__bytes_read.sum"][1]]
            wb = float(d["dram__bytes_write.sum"][0]) * {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "byte": 1,
                                                         "Kbyte": 1e3}[d["dram__bytes_write.sum"][1]]
            n = plain["config"]["n"]
            key = f"{c[0]}:{path}"
            if plain["config"]["n"] == {"2": 4096, "3": 8192, "4": 16384, "5": 49152}[c[0]]:
                traffic[key] = rb + wb
            md.append(f"\nDRAM traffic per launch {(rb + wb) / 1e9:.2f} GB (n={n}).")
        except (KeyError, ValueError):
            pass
    open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
