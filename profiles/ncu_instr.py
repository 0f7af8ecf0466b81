"""Per-source-line executed warp instructions (and stall share) of one kernel in an ncu report.
    python profiles/ncu_instr.py REPORT KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
fname, hdr, rows = "", None, []
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr, r))
        try:
            ie = float(d["Instructions Executed"])
            s = float(d["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        rows.append((ie, s, fname, int(r[0]), r[1].strip()[:64]))
tot = sum(x[0] for x in rows) or 1.0
stot = sum(x[1] for x in rows) or 1.0
print(f"total warp instructions {tot:.3g}")
for ie, s, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * ie / tot:5.1f}% instr {100 * s / stot:5.1f}% stall  {f}:{ln} {src}")
