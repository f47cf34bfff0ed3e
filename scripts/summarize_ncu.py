"""Summarise ncu captures into profiles/ (run here, on the CPU box).

usage: python scripts/summarize_ncu.py <tag> <launches.csv> <full.ncu-rep> [bench.json]

Writes profiles/<tag>_launches.txt (per-kernel share of device time from the
gpu__time_duration launch list), profiles/<tag>_move_kernel.txt (key --set
full metrics, stall reasons, SASS instruction mix) and updates
profiles/move_kernel_ncu.json (DRAM bytes per move-kernel launch, read by
bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        name = r[ki].split("(")[0]
        scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(r[ui], 1e-9)
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    T = sum(tot.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
           f"# {sum(cnt.values())} launches, {T:.3f} s total device time", ""]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"{k[:72]:72s} n={cnt[k]:6d} total={tot[k]:9.3f} s share={tot[k] / T * 100:5.1f}%")
    return "\n".join(out)


def ncu_csv(rep, *args):
    r = subprocess.run(["ncu", "-i", str(rep), *args, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def full(rep):
    lines = []
    rows = ncu_csv(rep, "--page", "details")
    h = rows[0]
    want = {"Duration", "Executed Ipc Active", "Issue Slots Busy", "Active Warps Per Scheduler",
            "Eligible Warps Per Scheduler", "Registers Per Thread", "Achieved Active Warps Per SM",
            "Theoretical Active Warps per SM", "Block Limit Registers", "Block Limit Shared Mem", "Grid Size",
            "Block Size", "Dynamic Shared Memory Per Block", "DRAM Throughput", "L1/TEX Cache Throughput",
            "Compute (SM) Throughput", "SM Frequency"}
    kname = rows[1][h.index("Kernel Name")] if len(rows) > 1 else "?"
    lines.append(f"kernel: {kname}")
    for x in rows[1:]:
        n, u, v = x[h.index("Metric Name")], x[h.index("Metric Unit")], x[h.index("Metric Value")]
        if n in want:
            lines.append(f"  {n:40s} {v:>14s} {u}")
    raw = ncu_csv(rep, "--page", "raw")
    h, v = raw[0], raw[2]
    metrics = {}
    for i, n in enumerate(h):
        metrics[n] = v[i]
    pick = ["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]
    lines.append("  pipes / counters:")
    for n in pick:
        if n in metrics:
            lines.append(f"    {n:62s} {metrics[n]} {raw[1][h.index(n)]}")
    st = []
    for n, val in metrics.items():
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                if float(val.replace(",", "")) > 0.05:
                    st.append((float(val.replace(",", "")), n[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
            except ValueError:
                pass
    lines.append("  stall reasons (warps per issued instruction): " +
                 ", ".join(f"{k}={v:.2f}" for v, k in sorted(st, reverse=True)))
    src = ncu_csv(rep, "--page", "source", "--print-source=cuda,sass")
    seen = {}
    hdr = None
    for r in src:
        if len(r) > 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[2].startswith("0x"):
            try:
                seen[r[2]] = (r[3].strip(), float(r[7].replace(",", "")))
            except ValueError:
                pass
    mix = collections.Counter()
    for ins, n in seen.values():
        t = ins.split()
        op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
        mix[op] += n
    tot = sum(mix.values()) or 1
    lines.append("  SASS mix (% executed warp-instructions): " +
                 "  ".join(f"{k} {v / tot * 100:.1f}" for k, v in mix.most_common(24)))
    blk = [k for k in mix if k.startswith("UBLKCP") or k.startswith("UTMA")]
    lines.append(f"  bulk-copy SASS present: {blk}")
    dram = None
    try:
        rd = float(metrics["dram__bytes_read.sum"].replace(",", ""))
        wr = float(metrics["dram__bytes_write.sum"].replace(",", ""))
        unit = raw[1][h.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        dram = (rd + wr) * scale
    except (KeyError, ValueError):
        pass
    return "\n".join(lines), dram, kname


def main():
    tag, lcsv, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    PROF.mkdir(exist_ok=True)
    (PROF / f"{tag}_launches.txt").write_text(launches(lcsv) + "\n")
    text, dram, kname = full(rep)
    (PROF / f"{tag}_move_kernel.txt").write_text(text + "\n")
    info = {"tag": tag, "kernel": kname, "dram_bytes_per_launch": dram,
            "note": "dram__bytes_read.sum + dram__bytes_write.sum of one move-kernel launch (ncu --set full)"}
    if len(sys.argv) > 4:
        info["bench"] = sys.argv[4]
    (PROF / "move_kernel_ncu.json").write_text(json.dumps(info, indent=1) + "\n")
    print(text)


if __name__ == "__main__":
    main()
