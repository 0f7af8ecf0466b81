"""Summarise ncu captures for profiles/ (run here, on the CPU box).

    python profiles/ncu_summary.py gpurun_out/prof_rNN.ncu-rep > profiles/rNN_ncu_full.txt
    python profiles/ncu_summary.py --launches gpurun_out/launches_rNN.csv > profiles/rNN_launches.txt
    python profiles/ncu_summary.py --source gpurun_out/prof_rNN.ncu-rep KERNEL_REGEX [TOP]
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    unit = dict(zip(hdr, units))
    stall = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not k.endswith("not_issued")]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"== {d['Kernel Name'][:90]}  (grid {d.get('launch__grid_size', '?')}, "
              f"block {d.get('launch__block_size', '?')})")
        for key, label in METRICS:
            if key in d:
                print(f"   {label:16s} {d[key]:>16s} {unit.get(key, '')}")
        vals = []
        for k in stall:
            try:
                vals.append((float(d[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1.0
        top = sorted(vals, reverse=True)[:6]
        print("   stalls (pc samples): " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top))


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        us = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
        name = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v for _, v in agg.values())
    print(f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for k, (c, v) in agg.items():
        print(f"{k:48s} {c:8d} {v:12.1f} {100 * v / tot:6.1f}%")


def source(path, kernel, top=25):
    """Per CUDA source line: share of warp-stall samples and its top reasons."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", "regex:" + kernel], capture_output=True, text=True,
                         check=True).stdout
    fname, hdr, lines = "", None, []
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
                s = float(d["Warp Stall Sampling (All Samples)"])
            except (KeyError, ValueError):
                continue
            reasons = []
            for k in hdr:
                if k.startswith("stall_") and not k.endswith("(Not Issued)"):
                    try:
                        reasons.append((float(d[k]), k[6:]))
                    except ValueError:
                        pass
            lines.append((s, f"{fname}:{r[0]}", r[1].strip()[:70], sorted(reasons, reverse=True)[:3]))
    tot = sum(x[0] for x in lines) or 1.0
    for s, loc, src, rs in sorted(lines, reverse=True)[:top]:
        why = ", ".join(f"{n} {100 * v / max(s, 1):.0f}%" for v, n in rs if v > 0)
        print(f"{100 * s / tot:5.1f}%  {loc:22s} {src:70s} [{why}]")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "--source":
        source(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 25)
    else:
        full(sys.argv[1])
