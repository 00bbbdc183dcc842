"""Summarise ncu captures from gpurun_out/ into profiles/ (committed evidence).

python scripts/ncu_summary.py <round-tag> [--launches gpurun_out/launches.csv]
        [--rep C2/f16=gpurun_out/prof_hogwild_f16.ncu-rep ...]
Writes profiles/<tag>_ncu_<name>.txt (key metrics), profiles/<tag>_launches.txt (per-kernel share of
the launch list) and merges dram bytes per launch into profiles/ncu_summary.json (read by bench.py).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "lts__t_sectors.sum", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]


def raw(rep):
    """Rows of a capture's raw page: from the .ncu-rep, or from its exported `--page raw --csv` file."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        res.append({h: (v, u) for h, v, u in zip(hdr, vals, units)})
    return res


def fnum(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return None


def to_bytes(val, unit):
    x = fnum(val)
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return None if x is None else x * mul


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--rep", nargs="*", default=[])
    ap.add_argument("--units", nargs="*", default=[], help="name=updates per launch")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    units = dict(x.split("=") for x in a.units)
    sj = os.path.join(prof, "ncu_summary.json")
    summary = json.load(open(sj)) if os.path.exists(sj) else {"kernels": {}}
    for spec in a.rep:
        name, rep = spec.split("=")
        for rec in raw(rep)[:1]:
            lines = [f"# ncu --set full capture: {os.path.basename(rep)} ({name}), round {a.tag}",
                     f"# kernel: {rec.get('Kernel Name', ('?', ''))[0]}"]
            for m in METRICS:
                if m in rec:
                    lines.append(f"{m:75s} {rec[m][0]:>22s} {rec[m][1]}")
            rd = to_bytes(*rec["dram__bytes_read.sum"])
            wr = to_bytes(*rec["dram__bytes_write.sum"])
            tms = fnum(rec["gpu__time_duration.sum"][0])
            tunit = rec["gpu__time_duration.sum"][1]
            ts = tms * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1}.get(tunit, 1e-3)
            d = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                 "duration_s_under_ncu": ts, "dram_GBps_under_ncu": (rd + wr) / ts / 1e9,
                 "source": f"profiles/{a.tag}_ncu_{name.replace('/', '_')}.txt"}
            if name in units:
                d["dram_bytes_per_update"] = (rd + wr) / float(units[name])
                lines.append(f"{'dram bytes per update':75s} {d['dram_bytes_per_update']:>22.1f} byte")
            lines.append(f"{'dram GB/s under ncu (cold, serialised)':75s} {d['dram_GBps_under_ncu']:>22.1f} GB/s")
            summary["kernels"][name] = d
            open(os.path.join(prof, f"{a.tag}_ncu_{name.replace('/', '_')}.txt"), "w").write("\n".join(lines) + "\n")
            print("\n".join(lines))
    json.dump(summary, open(sj, "w"), indent=1)
    if os.path.exists(a.launches):
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        hdr = rows[0]
        ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for r in rows[1:]:
            nm = r[ki].split("(")[0]
            nm = nm.split("<")[0] if "k_" in nm else nm
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1}.get(r[ui], 1e-6)
            tot[nm] += fnum(r[vi]) * scale
            cnt[nm] += 1
        all_ms = sum(tot.values())
        lines = [f"# launch list (ncu --metrics gpu__time_duration.sum --clock-control none), round {a.tag}",
                 "# per-launch times are cold-cache and serialised: compare SHARES", f"# total {all_ms:.3f} ms",
                 f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}"]
        for nm, ms in sorted(tot.items(), key=lambda x: -x[1]):
            lines.append(f"{nm:60s} {cnt[nm]:8d} {ms:10.3f} {ms / all_ms:7.1%}")
        open(os.path.join(prof, f"{a.tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
