"""Summarise ncu captures into profiles/: per-launch list (gpu__time_duration) and
the --set full report of the dominant kernel (DRAM traffic, throughputs, stall mix).

    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/r01_top_kernel.md [plan.json]
    python tools/ncu_summary.py traffic gpurun_out/traffic.ncu-rep gpurun_out/plans.json profiles/traffic.json
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ix = {n: i for i, n in enumerate(h)}
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit] * v
        per.setdefault(name, []).append(us)
    total = sum(sum(v) for v in per.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k[:90]}` | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.2f} | {sum(v)/total:.3f} |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out[:12]))


def traffic(rep, plans_path, dst):
    """DRAM bytes (read + write) of every captured launch, keyed by its plan (launch order =
    plans.json order) -> profiles/traffic.json entries (bench.py's roofline.traffic)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ix = {n: i for i, n in enumerate(h)}
    plans = json.load(open(plans_path))
    entries = []
    for row, p in zip(r[2:], plans):
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(row[ix[k]].replace(",", "")) * scale.get(units[ix[k]], 1.0)
        entries.append(dict(layer=p["layer"], plan=p["plan"], dram_bytes=b,
                            time_us=float(row[ix["gpu__time_duration.sum"]].replace(",", "")) *
                            {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3}.get(units[ix["gpu__time_duration.sum"]], 1.0)))
    json.dump({"source": os.path.basename(rep), "entries": entries}, open(dst, "w"), indent=1)
    for e in entries:
        print(e["layer"], round(e["dram_bytes"] / 1e6, 2), "MB", round(e["time_us"], 1), "us")


def full(rep, dst, plan_path=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units, vals = r[0], r[1], r[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}

    def f(name):
        try:
            return float(d[name].replace(",", "")) * scale.get(u.get(name, ""), 1.0)
        except (KeyError, ValueError):
            return None
    dram = (f("dram__bytes_read.sum") or 0) + (f("dram__bytes_write.sum") or 0)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__inst_executed_pipe_fma.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1
    lines = [f"# ncu --set full: {d.get('Kernel Name', '?')}", "", "| metric | value |", "|---|---|"]
    for k in keys:
        lines.append(f"| {k} | {d.get(k, 'n/a')} {u.get(k, '')} |")
    lines += ["", f"DRAM traffic per launch: {dram:.0f} bytes "
              f"(read {f('dram__bytes_read.sum') or 0:.0f}, write {f('dram__bytes_write.sum') or 0:.0f})"]
    meta = json.load(open(plan_path)) if plan_path and os.path.exists(plan_path) else {}
    if "nonzero_macs" in meta:  # tools/ncu_target.py: per-MAC ratios of the captured launch
        macs, ab = meta["nonzero_macs"], meta["algorithmic_bytes"]
        t_us = f("gpu__time_duration.sum") or 0
        wf = f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") or 0
        inst = f("smsp__inst_executed.sum") or 0
        lines += ["", f"target: `{meta['spec']}`, plan `{json.dumps(meta['plan'])}`", "",
                  "| derived (per launch) | value |", "|---|---|",
                  f"| nonzero MACs | {macs} |",
                  f"| shared-memory wavefronts per MAC | {wf / macs:.3f} |",
                  f"| warp instructions per 1000 MACs | {1000 * inst / macs:.2f} |",
                  f"| nonzero TFLOP/s (2 flop/MAC, ncu time) | {2 * macs / (t_us * 1e-6) / 1e12:.2f} |",
                  f"| algorithmic bytes | {ab} |",
                  f"| DRAM bytes / algorithmic bytes | {dram / ab:.3f} |",
                  f"| algorithmic GB/s (ncu time) | {ab / (t_us * 1e-6) / 1e9:.1f} |"]
    lines += ["", "| stall reason | share |", "|---|---|"]
    for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))[:10]:
        lines.append(f"| {k} | {100 * (v or 0) / tot:.1f}% |")
    open(dst, "w").write("\n".join(lines) + "\n")
    if plan_path and os.environ.get("NCU_SUMMARY_TRAFFIC", "0") == "1":
        plan = json.load(open(plan_path))
        json.dump({"plan": plan, "dram_bytes": dram, "source": os.path.basename(rep)},
                  open(os.path.join(os.path.dirname(dst), "traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
