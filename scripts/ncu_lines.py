"""Per-CUDA-source-line share of executed instructions and stall samples of an
ncu --set full --import-source capture.  usage: python scripts/ncu_lines.py REP [N]"""
import csv, subprocess, sys, io
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows = "?", []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Name":
        fname = r[1].split("/")[-1]
    elif len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            rows.append((float(r[7] or 0), float(r[4] or 0), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError:
            pass
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
for inst, samp, loc, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{inst / ti * 100:5.1f}% inst {samp / ts * 100:5.1f}% stall-samples  {loc:18s} {src}")
