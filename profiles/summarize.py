"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch lists) into committed
profiles/ files: per-kernel device time share of one step, DRAM traffic per
launch, pipe utilisation and top stall reasons.

usage: python profiles/summarize.py <tag> <launches.csv> <report.ncu-rep> <steps>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size"]


def short(name):
    n = name.split("(")[0]
    for p in ("void ", "svlfb::", "<unnamed>::", "unnamed>::"):
        n = n.replace(p, "")
    return n.strip()


def launch_shares(path, steps):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[short(r[ki])] += v
        cnt[short(r[ki])] += 1
    return agg, cnt


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k]) for k in d
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and d[k].replace(".", "", 1).isdigit()}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda t: -t[1])[:4]
        e = {"kernel": short(d["Kernel Name"])}
        for m in METRICS:
            u = units[h.index(m)] if m in h else ""
            try:
                v = float(d.get(m, "nan").replace(",", ""))
            except ValueError:
                v = float("nan")
            if u == "Mbyte":
                v *= 1e6
            elif u == "Gbyte":
                v *= 1e9
            elif u == "Kbyte":
                v *= 1e3
            elif u in ("usecond", "us"):
                v *= 1e3
            elif u in ("msecond", "ms"):
                v *= 1e6
            e[m] = v
        e["top_stalls"] = {k: round(v / tot, 3) for k, v in top}
        res.append(e)
    return res


def main():
    tag, launches, rep, steps = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    agg, cnt = launch_shares(launches, steps)
    ours = {k: v for k, v in agg.items() if k.startswith("k_")}
    total = sum(agg.values())
    lines = [f"# {tag}: launch list ({launches.split('/')[-1]}) and ncu --set full ({rep.split('/')[-1]})", "",
             "Launch list: ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised;",
             "compare shares, not absolutes). All launches of the run, warm-up included.", "",
             "| kernel | launches | total us | share of all device time |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda t: -t[1])[:16]:
        lines.append(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / total:.3f} |")
    caps = report(rep)
    lines += ["", "Full-set capture, one launch per row (time and DRAM bytes per launch):", "",
              "| kernel | us | DRAM read MB | DRAM write MB | tensor % | fp64 % | warps active % | L1 % | L2 % | DRAM % | issue % | regs | top stalls |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for e in caps:
        lines.append("| {} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.0f} | {} |".format(
            e["kernel"], e["gpu__time_duration.sum"] / 1e3, e["dram__bytes_read.sum"] / 1e6,
            e["dram__bytes_write.sum"] / 1e6,
            e["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"],
            e["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
            e["sm__warps_active.avg.pct_of_peak_sustained_active"],
            e["l1tex__throughput.avg.pct_of_peak_sustained_active"],
            e["lts__throughput.avg.pct_of_peak_sustained_elapsed"],
            e["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
            e["smsp__issue_active.avg.pct_of_peak_sustained_active"], e["launch__registers_per_thread"],
            ", ".join(f"{k} {v:.0%}" for k, v in e["top_stalls"].items())))
    open(f"profiles/{tag}.md", "w").write("\n".join(lines) + "\n")
    json.dump({"launch_ns_total": agg, "launch_counts": cnt, "captures": caps},
              open(f"profiles/{tag}.json", "w"), indent=1, default=float)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
