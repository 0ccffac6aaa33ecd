"""DRAM traffic per MTTKRP (one mode's launches) for roofline.traffic: runs
`bench.py --config C` under ncu with only the DRAM byte counters on the
k_mttkrp3 kernels (ncu's default cache control: every replay starts with
flushed caches), groups the launches per mode with the bench's
launches_per_mode, averages over the W+K steps, and writes
profiles/ncu_summary.json[C] and the raw CSV under gpurun_out/.

    python scripts/ncu_traffic.py nell-2 flickr-3d ...   (on the GPU box)
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
W, K = 3, 2


def run(cfg):
    out = ROOT / "gpurun_out" / f"traffic_{cfg}.csv"
    out.parent.mkdir(exist_ok=True)
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
           "lts__t_sectors.sum,lts__t_sectors_lookup_hit.sum",
           "-k", "regex:k_mttkrp3|k_zero_rows", "--csv", "--log-file", str(out),
           sys.executable, str(ROOT / "bench.py"), "--config", cfg, "--steps", str(K),
           "--warmup", str(W), "--no-e2e", "--no-cpu-baseline", "--also", "", "--cpd", "none", "--no-amortize"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if not line:
        raise SystemExit(f"{cfg}: bench failed under ncu\n{r.stdout[-2000:]}\n{r.stderr[-2000:]}")
    lpm = json.loads(line[-1])["roofline"]["launches_per_mode"]
    text = out.read_text()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    per = {}
    for r_ in rows[1:]:
        if len(r_) < len(hdr):
            continue
        d = dict(zip(hdr, r_))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(d["Metric Unit"], 1)
        per.setdefault(int(d["ID"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
    launches = [per[i] for i in sorted(per)]
    per_step = sum(lpm)
    assert len(launches) == per_step * (W + K), (len(launches), lpm)
    modes = []
    sec_all = hit_all = 0.0
    for m, n in enumerate(lpm):
        tot_b, tot_t = 0.0, 0.0
        for s in range(W + K):
            base = s * per_step + sum(lpm[:m])
            for L in launches[base: base + n]:
                tot_b += L["dram__bytes_read.sum"] + L["dram__bytes_write.sum"]
                tot_t += L["gpu__time_duration.sum"]
                sec_all += L.get("lts__t_sectors.sum", 0.0)
                hit_all += L.get("lts__t_sectors_lookup_hit.sum", 0.0)
        modes.append((tot_b / (W + K), tot_t / (W + K) / 1e6))
    return {"dram_bytes_per_launch": [b for b, _ in modes],
            "ncu_ms_per_mode": [t for _, t in modes],
            "launches_per_mode": lpm,
            "l2_hit_rate_pct": 100.0 * hit_all / sec_all if sec_all else None,
            "note": (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors(_lookup_hit).sum "
                     f"-k regex:k_mttkrp3|k_zero_rows on "
                     f"bench.py --config {cfg} --steps {K} --warmup {W}: per mode, the sum over that "
                     "mode's launches, averaged over the steps (cold caches per replay)")}


def main():
    summ = ROOT / "profiles" / "ncu_summary.json"
    data = json.loads(summ.read_text()) if summ.exists() else {}
    for cfg in sys.argv[1:]:
        data[cfg] = run(cfg)
        print(cfg, json.dumps(data[cfg]), flush=True)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "ncu_summary.json").write_text(json.dumps(data, indent=1) + "\n")


if __name__ == "__main__":
    main()
