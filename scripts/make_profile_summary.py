"""Write profiles/<tag>.md + update profiles/ncu_summary.json from an ncu
full capture and the launch-list CSV of the same bench command.

    python scripts/make_profile_summary.py <tag> <config> gpurun_out/<p>.ncu-rep gpurun_out/<p>_launches.csv
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(tag, config, rep, launches):
    hdr, units, rows = raw(rep)
    lines = [f"# ncu summary `{tag}` — {config}", "",
             f"Source: `ncu --set full --clock-control none --import-source on -k regex:k_mttkrp3` on "
             f"`python bench.py --config {config} --steps 2 --warmup 1` (1 B200). Per-launch values; "
             "the first captured launches after warm-up.", ""]
    traffic = []
    stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued")]
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        lines.append(f"## `{name}`")
        lines.append("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in hdr:
                lines.append(f"| {label} (`{k}`) | {r[hdr.index(k)]} {units[hdr.index(k)]} |")
        rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        traffic.append(rd + wr)
        st = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i] or 0)) for i, h in stall_cols),
                    key=lambda x: -x[1])
        tot = sum(v for _, v in st) or 1
        lines.append("")
        lines.append("Stall samples: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in st[:8]))
        lines.append("")
    # launch list share
    text = Path(launches).read_text()
    body = text[text.index('"ID"'):]
    lrows = list(csv.DictReader(io.StringIO(body)))
    tot = sum(float(x["Metric Value"]) for x in lrows if x["Metric Name"] == "gpu__time_duration.sum")
    mine = [(x["Kernel Name"], float(x["Metric Value"])) for x in lrows
            if x["Metric Name"] == "gpu__time_duration.sum" and "mttkrp3" in x["Kernel Name"]]
    lines.append("## Launch list (`--metrics gpu__time_duration.sum`, cold-cache, serialised)")
    lines.append(f"{len(lrows)} launches, {tot / 1e6:.3f} ms total; MTTKRP kernel launches: {len(mine)}, "
                 f"{sum(t for _, t in mine) / 1e6:.3f} ms ({100 * sum(t for _, t in mine) / tot:.1f}% of all "
                 "device time, which includes tensor generation and the HB-CSF build).")
    lines.append("")
    lines.append("| kernel | ns |\n|---|---|")
    for n, t in mine:
        lines.append(f"| `{n[:60]}` | {t:.0f} |")
    out = ROOT / "profiles" / f"{tag}.md"
    out.write_text("\n".join(lines) + "\n")
    js = ROOT / "profiles" / "ncu_summary.json"
    d = json.loads(js.read_text()) if js.exists() else {}
    entry = d.setdefault(config, {})
    entry["full_capture"] = {"tag": tag, "dram_bytes_per_launch": traffic,
                             "note": "dram__bytes_read.sum + dram__bytes_write.sum of the launches "
                                     "captured with --set full"}
    if "dram_bytes_per_launch" not in entry:  # no per-mode pass (scripts/ncu_traffic.py) yet
        entry["dram_bytes_per_launch"] = traffic
    js.write_text(json.dumps(d, indent=1) + "\n")
    print(out)


if __name__ == "__main__":
    main(*sys.argv[1:5])
