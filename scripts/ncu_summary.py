#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (markdown + traffic.json).

usage:
  ncu_summary.py full <report.ncu-rep> <key> [<out.md>]   # --set full capture of one launch
  ncu_summary.py launches <launches.csv> <out.md>          # gpu__time_duration launch list

`key` names the launch in profiles/traffic.json (read by bench.py for the
roofline's `traffic` field: dram bytes read + written per launch)."""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


def full(rep, key, out_md=None):
    rows = raw(rep)
    lines = [f"# ncu --set full: {Path(rep).name} ({key})", ""]
    traffic_file = PROF / "traffic.json"
    traffic = json.loads(traffic_file.read_text()) if traffic_file.exists() else {}
    for d in rows:
        name = d.get("Kernel Name", "?")
        lines.append(f"## {name[:100]}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m in METRICS:
            if m in d:
                lines.append(f"| {m} | {d[m]} | {d['_units'].get(m, '')} |")
        rd = to_bytes(d.get("dram__bytes_read.sum", "0"), d["_units"].get("dram__bytes_read.sum", "byte"))
        wr = to_bytes(d.get("dram__bytes_write.sum", "0"), d["_units"].get("dram__bytes_write.sum", "byte"))
        lines.append(f"| dram read+write (bytes) | {rd + wr:.0f} | byte |")
        lines.append("")
        kname = name.split("(")[0].split("::")[-1]
        if key not in traffic or "source" in traffic[key]:
            traffic[key] = {}  # a new capture replaces the entry of an older one
        traffic[key][kname] = rd + wr
    # stall attribution by source line
    try:
        txt = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_lines.py"), rep, "15"],
                             capture_output=True, text=True).stdout
        lines += ["## warp-stall samples by source line (top 15)", "", "```", txt.strip(), "```", ""]
    except Exception:
        pass
    traffic[key]["total"] = sum(v for k, v in traffic[key].items() if k not in ("total", "source"))
    if out_md:
        traffic[key]["source"] = str(Path(out_md).relative_to(ROOT)) if Path(out_md).is_absolute() else str(out_md)
    traffic_file.write_text(json.dumps(traffic, indent=1) + "\n")
    md = "\n".join(lines) + "\n"
    if out_md:
        Path(out_md).write_text(md)
    print(md)


def launches(csv_path, out_md):
    text = Path(csv_path).read_text().splitlines()
    start = [i for i, l in enumerate(text) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(text[start:]))
    agg = OrderedDict()
    for r in rows:
        n = r["Kernel Name"].split("(")[0]
        n = n.replace("(anonymous namespace)", "").replace("<unnamed>", "")[-70:]
        t = float(r["Metric Value"].replace(",", "")) / 1e3
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
    total = sum(v[1] for v in agg.values())
    lines = [f"# launch list: {Path(csv_path).name}", "",
             "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)",
             "", "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{n}` | {c} | {t:.1f} | {100 * t / total:.1f}% |")
    # the timed step only: engine kernels (graph build and setup launches run
    # before the timed region)
    eng = OrderedDict((n, v) for n, v in agg.items()
                      if any(t in n for t in ("fr_kernel", "fr_finish", "k1_kernel", "k2_kernel", "ms_kernel")))
    et = sum(v[1] for v in eng.values())
    if et:
        lines += ["", "timed-step engine kernels only (share of their sum):", "",
                  "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
        for n, (c, t) in sorted(eng.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{n}` | {c} | {t:.1f} | {t / c:.1f} | {100 * t / et:.1f}% |")
    lines += ["", "| # | kernel | grid | block | us |", "|---|---|---|---|---|"]
    for r in rows:
        n = r["Kernel Name"].split("(")[0][-50:]
        lines.append(f"| {r['ID']} | `{n}` | {r['Grid Size']} | {r['Block Size']} | "
                     f"{float(r['Metric Value'].replace(',', '')) / 1e3:.1f} |")
    Path(out_md).write_text("\n".join(lines) + "\n")
    print("\n".join(lines[:12 + len(agg)]))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
