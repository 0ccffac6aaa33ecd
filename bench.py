"""HB-CSF MTTKRP benchmark (BASELINE.json metric: GFLOP/s on the 3·nnz·R basis,
R=32, and % of the HBM roofline).

A step = one HB-CSF MTTKRP per mode (all three modes) of the configuration's
tensor, inputs resident in HBM.  Default workload: BASELINE.json configs[1]
(nell-2-shaped synthetic, 76.9M nnz, all 3 modes on 1 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config nell-2|flickr-3d|delicious-3d|nell-1|config1] [--scale S]

N>1 is launched by torchrun: output slices of each mode are sharded across
ranks by nonzero count (no collective in the timed region); time = max over
ranks; value = all ranks' flops / that time.

``--impl reference`` times the reference algorithm on the host CPU (the
oracle port, oracle/tenkit_port.py, with all host threads through its
scheduled path, as ``tenkit mttkrp --threads N``) on a bounded slice sample of
the same tensor; rank 0 alone prints it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

RANK = 32
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="nell-2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # the format comparison of the paper (cpd.py:141-149
    # TENSOR_FORMATS): hbcsf (default, the headline), bcsf = split CSF, csf,
    # coo = the whole tensor as a coordinate list
    ap.add_argument("--format", default="hbcsf", choices=["hbcsf", "bcsf", "csf", "coo"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-nnz", type=int, default=300_000)
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


FORMAT_NAME = {"hbcsf": "HB-CSF", "bcsf": "B-CSF", "csf": "CSF", "coo": "COO"}


def census_of(h):
    if not hasattr(h, "coo_part"):  # standalone formats
        if hasattr(h, "num_fibers"):  # CsfTensor (csf / bcsf)
            return {"coo_nnz": 0, "csl_slices": 0, "csl_nnz": 0, "csf_slices": h.num_slices,
                    "csf_fibers": h.num_fibers, "csf_nnz": h.nnz}
        return {"coo_nnz": h.nnz, "csl_slices": 0, "csl_nnz": 0, "csf_slices": 0,
                "csf_fibers": 0, "csf_nnz": 0}
    return {
        "coo_nnz": h.coo_part.nnz,
        "csl_slices": h.csl_part.num_slices,
        "csl_nnz": h.csl_part.nnz,
        "csf_slices": h.csf_part.num_slices,
        "csf_fibers": h.csf_part.num_fibers,
        "csf_nnz": h.csf_part.nnz,
    }


def b_comp(c, dims, mode, r=RANK):
    """Algorithmic (compulsory) bytes of one mode's MTTKRP, SURVEY §8(d)."""
    stream = (16 * c["coo_nnz"] + 8 * c["csl_slices"] + 12 * c["csl_nnz"] + 8 * c["csf_slices"]
              + 8 * c["csf_fibers"] + 8 * c["csf_nnz"])
    factors = 4 * r * sum(d for i, d in enumerate(dims) if i != mode)
    out = 4 * r * dims[mode]
    return stream + factors + out


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_factors(dims, seed):
    rng = np.random.default_rng(seed)  # cli.py:274-276 convention
    return [rng.random((d, RANK)) for d in dims]


def cpu_sample(t, dims, mode, target_nnz):
    """Every K-th slice of `mode` (whole slices, so the per-slice structure is
    the workload's), exported to the host for the CPU oracle."""
    import ctypes as C

    import torch

    from paper_1904_03329_b200 import _native as N

    idx = torch.empty((t.nnz, t.order), dtype=torch.int32, device="cuda")
    vals = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
    N.call("hbk_coo_export_device", t._dev().ptr, C.c_void_p(idx.data_ptr()),
           C.c_void_p(vals.data_ptr()), None, N.stream_ptr())
    k = max(1, int(round(t.nnz / max(1, target_nnz))))
    keep = (idx[:, mode] % k) == 0
    si = idx[keep].cpu().numpy().view(np.uint32)
    sv = vals[keep].cpu().numpy()
    del idx, vals
    return si, sv, k


def time_oracle(si, sv, dims, mode, factors, threads, runs=3):
    from oracle import tenkit_port as P

    mo = P.allmode_order(dims, mode)
    h = P.split_hbcsf(P.hbcsf(si, sv, dims, mo), 128)
    units = None
    if threads > 1:
        units, _ = P.block_schedule(h["csf"], 512)
    P.mttkrp_hbcsf(h, factors, mode, units=units, threads=threads)  # warm-up (cli.py:220-228)
    ts = []
    for _ in range(runs):
        tic = time.perf_counter()
        P.mttkrp_hbcsf(h, factors, mode, units=units, threads=threads)
        ts.append(time.perf_counter() - tic)
    return statistics.median(ts), len(sv)


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm on the host CPU cores."""
    import torch

    if rank != 0:
        return
    from paper_1904_03329_b200.generate import CONFIGS, config_tensor

    torch.cuda.set_device(0)
    cfg = CONFIGS[args.config]
    dims = cfg["dims"]
    t = config_tensor(args.config, scale=args.scale)
    factors = make_factors(dims, cfg["seed"])
    threads = os.cpu_count() or 1
    samples = [cpu_sample(t, dims, m, args.cpu_sample_nnz) for m in range(len(dims))]
    steps = []
    for s in range(args.warmup + args.steps):
        flops = secs = 0.0
        for m, (si, sv, _) in enumerate(samples):
            sec, m_nnz = time_oracle(si, sv, dims, m, factors, threads, runs=1)
            flops += 3.0 * m_nnz * RANK
            secs += sec
        if s >= args.warmup:
            steps.append(flops / secs / 1e9)
    value = statistics.median(steps)
    sample_desc = (f"every K-th output slice per mode (K={[s[2] for s in samples]}, "
                   f"{[len(s[1]) for s in samples]} nnz), split tau=128, schedule block 512")
    line = {
        "impl": "reference", "metric": "MTTKRP GFLOP/s (3*nnz*R, R=32)", "value": value,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (SURVEY Appendix A power-law generator)",
        "config": {"workload": f"{args.config}-shaped HB-CSF MTTKRP, all {len(dims)} modes per step, R=32",
                   "dims": list(dims), "nnz": t.nnz, "rank": RANK, "scale": args.scale,
                   "split": {"fiber_threshold": 128, "block_size": 512},
                   "parallelism": "host CPU (rank 0)"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "sample": sample_desc},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    import torch.distributed as dist

    # HBK_BENCH_BACKEND=gloo runs the N>1 path on fewer GPUs than ranks (ranks
    # share devices round-robin) to validate the sharded leg on one GPU; the
    # measured configuration is one rank per GPU over NCCL.
    backend = os.environ.get("HBK_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_1904_03329_b200 as hb
    from paper_1904_03329_b200 import kernels as K
    from paper_1904_03329_b200 import shard
    from paper_1904_03329_b200.generate import CONFIGS, config_tensor
    from paper_1904_03329_b200.kernels import _device_factors, plan_for

    cfg = CONFIGS[args.config]
    dims = cfg["dims"]
    t0 = time.perf_counter()
    t = config_tensor(args.config, scale=args.scale)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    nnz_total = t.nnz

    # preprocessing (reported separately, like cli.py preprocessing_seconds)
    t0 = time.perf_counter()
    split_cfg = hb.SplitConfig()
    reps, censuses, plans, ranges, all_ranges = [], [], [], [], []
    for mode in range(len(dims)):
        mo = hb.allmode_order(dims, mode)
        if world > 1:
            # this rank's output rows, rebased: its plan writes only them
            ranges_m = shard.plan_row_ranges(shard.slice_histogram(t, mode).cpu().numpy(), world)
            all_ranges.append(ranges_m)
            rr = ranges_m[rank]
            part = shard.shard_rows(t, mode, rr[0], rr[1]) if rr[1] > rr[0] else None
        else:
            rr, part = (0, dims[mode]), t
        if part is None:  # more ranks than non-empty row ranges
            reps.append(None)
            ranges.append(rr)
            censuses.append(None)
            plans.append(None)
            continue
        if args.format == "hbcsf":
            h = hb.split_fibers(hb.build_hbcsf(part, mo), split_cfg)
        elif args.format == "bcsf":
            h = hb.split_fibers(hb.build_csf(part, mo), split_cfg)
        elif args.format == "csf":
            h = hb.build_csf(part, mo)
        else:
            h = part
        reps.append(h)
        ranges.append(rr)
        censuses.append(census_of(h))
        plans.append(plan_for(h, mode, RANK))
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t0

    f64 = make_factors(dims, cfg["seed"])
    f_dev = [torch.from_numpy(f).float().cuda() for f in f64]
    rows_local = [hi - lo for lo, hi in ranges]
    outs = [torch.empty((max(1, rows_local[m]), RANK), dtype=torch.float32, device="cuda")
            for m in range(len(dims))]
    ptrs = [_device_factors(f_dev, m)[0] for m in range(len(dims))]
    stream = torch.cuda.current_stream()

    def run_mode(m):
        if plans[m] is not None:
            plans[m].execute(ptrs[m], outs[m])

    def step():
        for m in range(len(dims)):
            run_mode(m)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    n_modes = len(dims)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)] for _ in range(n_modes)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        start.record(stream)
        for s in range(args.steps):
            for m in range(n_modes):
                ev[m][s][0].record(stream)
                run_mode(m)
                ev[m][s][1].record(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = start.elapsed_time(stop)
    per_mode_ms = [statistics.mean(a.elapsed_time(b) for a, b in ev[m]) for m in range(n_modes)]
    if world > 1:
        tt = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
    ms_per_step = elapsed_ms / args.steps
    flops_step = 3.0 * nnz_total * RANK * n_modes
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # N > 1: the same steps followed by the replication of every mode's output
    # rows on all ranks (all-gather over NCCL) — the standalone MTTKRP with
    # and without the output exchange
    with_ag = None
    if world > 1:
        from paper_1904_03329_b200.distributed import allgather_padded

        def step_ag():
            for m in range(n_modes):
                run_mode(m)
                rows_m = outs[m][: rows_local[m]]
                allgather_padded(torch, dist, rows_m, all_ranges[m])

        for _ in range(max(1, args.warmup)):
            step_ag()
        torch.cuda.synchronize()
        dist.barrier()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(stream)
        for _ in range(args.steps):
            step_ag()
        b_ev.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([a_ev.elapsed_time(b_ev) / args.steps], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ag_ms = float(tt.item())
        with_ag = {"ms_per_step": ag_ms, "value": flops_step / (ag_ms * 1e-3) / 1e9,
                   "unit": "GFLOP/s",
                   "gathered_bytes_per_step": sum(4 * RANK * d for d in dims),
                   "note": "each step + all_gather of every mode's output rows to every rank"}

    # gather ceiling: the plans' gather-only calibration kernels over the same
    # task lists and streams (hbk_plan_probe), timed the same way
    gather = None
    try:
        rows = [int(pl.info.gather_rows) if pl is not None else 0 for pl in plans]
        if all(r > 0 for r, pl in zip(rows, plans) if pl is not None):
            pev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(args.steps)] for _ in range(n_modes)]
            for m in range(n_modes):
                if plans[m] is not None:
                    plans[m].probe(ptrs[m])
            torch.cuda.synchronize()
            for s_ in range(args.steps):
                for m in range(n_modes):
                    if plans[m] is None:
                        continue
                    pev[m][s_][0].record(stream)
                    plans[m].probe(ptrs[m])
                    pev[m][s_][1].record(stream)
            torch.cuda.synchronize()
            probe_ms = [statistics.mean(a.elapsed_time(b) for a, b in pev[m]) if plans[m] is not None
                        else 0.0 for m in range(n_modes)]
            gather = {
                "rows_per_step": sum(rows),
                "kernel_rows_per_s": sum(rows) / (sum(per_mode_ms) * 1e-3),
                "ceiling_rows_per_s": sum(rows) / (sum(probe_ms) * 1e-3),
                "frac": sum(probe_ms) / sum(per_mode_ms),
                "probe_ms_per_mode": probe_ms,
                "note": ("128-byte factor rows delivered to the SMs (leaf rows + fiber rows, 2 per "
                         "CSL/COO nonzero); ceiling = gather-only kernel over the same tasks "
                         "(hbk_plan_probe)"),
            }
    except Exception as e:  # calibration is optional; never fail the bench on it
        gather = {"error": str(e)}

    # roofline over the per-mode launches (each step is one launch per mode)
    hbm, hbm_src = peaks()
    # this rank's launches: its own output rows, every input factor row
    bytes_modes = []
    for m in range(n_modes):
        if censuses[m] is None:
            bytes_modes.append(0)
            continue
        dl = list(dims)
        dl[m] = rows_local[m]
        bytes_modes.append(b_comp(censuses[m], dl, m))
    achieved = sum(bytes_modes) / (sum(per_mode_ms) * 1e-3) / 1e9
    # DRAM bytes per launch from the committed ncu capture of this workload
    # (profiles/ncu_summary.json, written by scripts/make_profile_summary.py)
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists() and args.scale == 1.0:
        try:
            per = json.loads(prof.read_text()).get(args.config, {}).get("dram_bytes_per_launch")
            traffic = statistics.mean(per) if per else None
        except Exception:
            traffic = None

    # end to end through the public API with host buffers: pinned fp32
    # factors in, NumPy float64 rows out, one mttkrp_hbcsf per mode per step
    # (each rank: its own row shard); wall clock, max over ranks
    e2e = None
    if not args.no_e2e:
        f_pin = [torch.from_numpy(f).float().pin_memory() for f in f64]

        def e2e_step():
            for m in range(n_modes):
                if reps[m] is not None:
                    hb.mttkrp(reps[m], f_pin, m)

        e2e_step()
        torch.cuda.synchronize()
        k = max(3, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        tic = time.perf_counter()
        for _ in range(k):
            e2e_step()
        e2e_s = (time.perf_counter() - tic) / k
        if world > 1:
            tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        h2d = sum(4 * RANK * sum(d for i, d in enumerate(dims) if i != m)
                  for m in range(n_modes) if reps[m] is not None)
        # rows come back as float64 when the output fits the pinned-return
        # path (device widening), else as fp32 widened on the host
        cap = K._HostStage.PINNED_OUT_BYTES
        d2h = sum((8 if 8 * RANK * rows_local[m] <= cap else 4) * RANK * rows_local[m]
                  for m in range(n_modes) if reps[m] is not None)
        e2e = {"value": flops_step / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
               "path": f"paper_1904_03329_b200.mttkrp({args.format} rep, pinned host fp32 factors) -> numpy f64 rows, "
                       "one call per mode, H2D + kernel + D2H inside the timed region"
                       + ("; bytes per rank, rank 0" if world > 1 else "")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        samples = [cpu_sample(t, dims, m, args.cpu_sample_nnz) for m in range(n_modes)]
        flops = secs = 0.0
        for m, (si, sv, _) in enumerate(samples):
            sec, m_nnz = time_oracle(si, sv, dims, m, f64, threads=1, runs=3)
            flops += 3.0 * m_nnz * RANK
            secs += sec
        cpu = {"value": flops / secs / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
               "sample": (f"every K-th output slice per mode (K={[s[2] for s in samples]}, "
                          f"{[len(s[1]) for s in samples]} nnz); oracle mttkrp_hbcsf threads=1, "
                          "split tau=128, median of 3 after 1 warm-up")}

    if rank == 0:
        line = {
            "metric": "MTTKRP GFLOP/s (3*nnz*R, R=32)",
            "value": value,
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (SURVEY Appendix A power-law generator, seeded, on device)",
            "config": {
                "workload": (f"{args.config}-shaped {FORMAT_NAME[args.format]} MTTKRP, all {n_modes} "
                             "modes per step, R=32"),
                "dims": list(dims), "nnz": nnz_total, "rank": RANK, "scale": args.scale,
                "split": {"fiber_threshold": 128, "block_size": 512},
                "l2": "inputs larger than L2 (index/value streams 0.75+ GB per mode); factors L2-resident by design",
                "parallelism": f"slice-sharded dp{world}" if world > 1 else "1 GPU",
                "census": censuses if world == 1 else {"rank0_shards": censuses},
                "preprocessing_s": prep_s, "generate_s": gen_s,
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "peak_source": hbm_src,
                # the DRAM bytes the kernels actually move (ncu, cold caches per
                # replay) over their time: how close to the HBM peak the
                # traffic runs, as opposed to the compulsory-bytes fraction
                "traffic_gbs": (traffic / (statistics.mean(per_mode_ms) * 1e-3) / 1e9
                                if traffic else None),
                "traffic_frac": (traffic / (statistics.mean(per_mode_ms) * 1e-3) / 1e9 / hbm
                                 if traffic else None),
                "kernel": "k_mttkrp3_r32<kind> (one launch per non-empty bucket kind per mode)",
                "algorithmic_bytes_per_step": sum(bytes_modes),
                "algorithmic_bytes_per_launch": sum(bytes_modes) / n_modes,
                "traffic_unit": "DRAM bytes per MTTKRP launch (ncu dram__bytes_read+write, profiles/)",
                "per_mode_ms": per_mode_ms, "per_mode_bytes": bytes_modes,
                "per_mode_frac": [b / (ms * 1e-3) / 1e9 / hbm for b, ms in zip(bytes_modes, per_mode_ms)],
                "launches_per_mode": [int(pl.info.launches) if pl is not None else 0 for pl in plans],
                "gather": gather,
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "with_output_allgather": with_ag,
            "gpu_launches": args.steps * sum(int(pl.info.launches) for pl in plans if pl is not None),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
