#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (tracked).

  python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep \
      --out profiles/r01_summary.md [--traffic-json profiles/hash_scan_traffic.json]

--launches: the `ncu --metrics gpu__time_duration.sum --csv` launch list (cold-cache,
serialised: shares are meaningful, absolutes are not).  --rep: an `ncu --set full`
report; key metrics per profiled kernel are tabulated.
"""
import argparse
import collections
import csv
import json
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration (us)", 1.0),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1.0),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% peak)", 1.0),
    ("smsp__inst_executed.sum", "warp instructions", 1.0),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (%)", 1.0),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "SMEM wavefronts", 1.0),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "SMEM bank conflicts", 1.0),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate (%)", 1.0),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read", 1.0),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 sectors written", 1.0),
    ("lts__t_sectors_srcunit_tex_op_atom.sum", "L2 sectors atomic", 1.0),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 sectors reduction", 1.0),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "L2 read sectors hit", 1.0),
    ("dram__sectors_read.sum", "DRAM sectors read", 1.0),
    ("dram__sectors_write.sum", "DRAM sectors written", 1.0),
    ("launch__registers_per_thread", "registers/thread", 1.0),
    ("launch__grid_size", "grid", 1.0),
]


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0].split("::")[-1].replace("void cub", "cub")].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return [(k, len(v), sum(v) / len(v) / 1e3, sum(v) / tot) for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))]


def rep_metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    res = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("::")[-1]
        vals = {}
        for key, label, scale in KEYS:
            if key in h:
                try:
                    vals[label] = float(r[h.index(key)].replace(",", "")) * scale
                except ValueError:
                    pass
        stalls = sorted(((n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                          float(r[i])) for i, n in enumerate(h)
                         if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("per_issue_active.ratio")
                         and r[i]), key=lambda t: -t[1])[:4]
        res.append((name, vals, stalls))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--traffic-json")
    ap.add_argument("--units", action="append", default=[],
                    help="kernel=count[:name]: also print DRAM / L2 sectors per unit (e.g. k_commit=5767168:new block)")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        lines += ["## Launch list (gpu__time_duration.sum, serialised, cold cache)", "",
                  "| kernel | launches | avg us | share |", "|---|---|---|---|"]
        for k, n, us, sh in launch_shares(a.launches):
            lines.append(f"| {k[:60]} | {n} | {us:.1f} | {sh:.3f} |")
        lines.append("")
    for rep in a.rep:
        lines += [f"## Full-set metrics: `{rep.split('/')[-1]}`", ""]
        for name, vals, stalls in rep_metrics(rep):
            lines += [f"### {name}", "", "| metric | value |", "|---|---|"]
            lines += [f"| {k} | {v:,.2f} |" for k, v in vals.items()]
            lines += [f"| top stalls (per issue) | {', '.join(f'{s}={x:.2f}' for s, x in stalls)} |"]
            for u in a.units:
                k, rest = u.split("=", 1)
                cnt, _, uname = rest.partition(":")
                if name.startswith(k) and float(cnt) > 0:
                    n = float(cnt)
                    for lab in ("DRAM sectors read", "DRAM sectors written", "L2 sectors read", "L2 sectors atomic",
                                "L2 sectors written"):
                        if lab in vals:
                            lines.append(f"| {lab} per {uname or 'unit'} | {vals[lab] / n:.2f} |")
                    mb = vals.get("DRAM read (MB)", 0) + vals.get("DRAM write (MB)", 0)
                    lines.append(f"| DRAM bytes per {uname or 'unit'} | {mb * 1e6 / n:.1f} |")
            lines.append("")
            if a.traffic_json and name.startswith("k_hash_scan"):
                mb = vals.get("DRAM read (MB)", 0) + vals.get("DRAM write (MB)", 0)
                json.dump({"kernel": name, "dram_bytes_per_launch": mb * 1e6, "source": rep},
                          open(a.traffic_json, "w"), indent=1)
    open(a.out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
