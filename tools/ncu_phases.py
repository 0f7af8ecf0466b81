"""Per-phase view of an ncu source page (ncu -i X.ncu-rep --page source --csv):
the SASS of each kernel cut at its CTA barriers, with the warp-stall samples,
their top reasons and the executed instruction counts of each segment."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1]
        hdr = rows[i + 1]
        col = {h: k for k, h in enumerate(hdr)}
        stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        j = i + 2
        seg, segs = dict(n=0, s=0, ex=0, st=Counter(), first=None, hot=[]), []
        total = 0
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            r = rows[j]
            src = r[col["Source"]].strip()
            smp = int(r[col["# Samples"]] or 0)
            ex = int(r[col["Instructions Executed"]] or 0)
            total += smp
            seg["n"] += 1
            seg["s"] += smp
            seg["ex"] += ex
            if seg["first"] is None:
                seg["first"] = j - i - 2
            for h in stall_cols:
                v = int(r[col[h]] or 0)
                if v:
                    seg["st"][h[6:]] += v
            seg["hot"].append((smp, src, j - i - 2))
            if src.startswith("BAR.") or "BAR.SYNC" in src or src.startswith("EXIT"):
                seg["end"] = src
                segs.append(seg)
                seg = dict(n=0, s=0, ex=0, st=Counter(), first=None, hot=[])
            j += 1
        if seg["n"]:
            seg["end"] = "(end)"
            segs.append(seg)
        print("==", name[:90], "samples", total)
        for k, sg in enumerate(segs):
            if sg["s"] * 200 < total:
                continue
            st = ", ".join("%s %d%%" % (a, 100 * b / max(1, sum(sg["st"].values())))
                           for a, b in sg["st"].most_common(4))
            print("  seg %2d @%5d  instrs %5d  exec %9d  samples %6d (%4.1f%%)  %s   [%s]"
                  % (k, sg["first"], sg["n"], sg["ex"], sg["s"], 100 * sg["s"] / total, st, sg["end"][:40]))
            if top:
                for smp, src, pos in sorted(sg["hot"], reverse=True)[:top]:
                    print("        %6d  @%d %s" % (smp, pos, src[:100]))
        i = j
    else:
        i += 1
