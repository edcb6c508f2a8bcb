"""Stall samples of one kernel in an ncu report, by SASS window (development aid)."""
import csv
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
W = int(sys.argv[3]) if len(sys.argv) > 3 else 60
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + pat], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hdr = rows[hi[0]]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[hi[0] + 1: hi[1] - 1] if len(hi) > 1 else rows[hi[0] + 1:]


def n(r, c):
    try:
        return int(r[idx[c]])
    except Exception:
        return 0


cols = ["stall_wait", "stall_long_sb", "stall_short_sb", "stall_selected", "stall_not_selected", "stall_math",
        "stall_branch_resolving", "stall_mio", "stall_no_inst", "stall_dispatch", "stall_barrier", "stall_lg"]
tot = {c: sum(n(r, c) for r in data) for c in cols}
print("total", sum(n(r, "Warp Stall Sampling (All Samples)") for r in data), tot)
for k in range(0, len(data), W):
    seg = data[k:k + W]
    s = sum(n(r, "Warp Stall Sampling (All Samples)") for r in seg)
    ops = {}
    for r in seg:
        t = r[idx["Source"]].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = sorted(ops.items(), key=lambda x: -x[1])[:5]
    st = {c.replace("stall_", ""): n_ for c in cols if (n_ := sum(n(r, c) for r in seg)) > 0.1 * s and s > 0}
    print(f"{k:5d} {s:5d} {st} {top}")
