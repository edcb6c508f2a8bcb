"""Summarise gpurun_out ncu artefacts into profiles/ (launch-list shares and --set full metrics)."""
import csv
import collections
import json
import subprocess
import sys


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        if name in ("k_dfma",) or name.startswith("at::"):   # bench.py's fp64-peak microbenchmark and
            continue                                          # torch's L2-flush fills: not part of the step
        agg[name][0] += 1
        agg[name][1] += float(r[-1])
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": v[0], "total_us": round(v[1] / 1e3, 2),
                    "avg_us": round(v[1] / v[0] / 1e3, 3), "share": round(v[1] / tot, 4)})
    return out


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__grid_size", "launch__block_size", "smsp__warps_eligible.avg.per_cycle_active"]


def full_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    hdr, units = r[0], r[1]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    out = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, i in idx.items():
            try:
                d[m + " [" + units[i] + "]"] = float(row[i])
            except ValueError:
                d[m] = row[i]
        out.append(d)
    return out


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    res = launch_shares(src) if kind == "launches" else full_metrics(src)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res[:6], indent=1))
