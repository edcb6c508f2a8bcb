"""Stall samples and excessive shared-memory wavefronts per CUDA source line of one kernel in an ncu
report (needs -lineinfo and --import-source); development aid.
  python tools/ncu_lines.py report.ncu-rep <kernel regex> [top]"""
import csv
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + pat, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = None, None, []
for r in csv.reader(raw.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit():
        d = dict(zip(hdr, r))

        def num(k):
            try:
                return int(d.get(k, 0))
            except ValueError:
                return 0
        out.append((num("Warp Stall Sampling (All Samples)"), cur, int(r[0]), r[1].strip()[:90],
                    num("L1 Wavefronts Shared Excessive"), num("stall_wait"), num("stall_short_sb"), num("stall_long_sb")))
tot = max(sum(o[0] for o in out), 1)
print("total stall samples", tot)
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0]:7d} {100 * o[0] / tot:5.1f}%  {o[1]}:{o[2]}  wait={o[5]} short_sb={o[6]} long_sb={o[7]} excess_wf={o[4]} | {o[3]}")
