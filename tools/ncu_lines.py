"""Top source lines by warp-stall samples from an ncu report's source page:
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows, f = [], "?"
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        f = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0].isdigit() and r[2] == "-":
        try:
            rows.append((int(r[4]), f, int(r[0]), r[1].strip()[:100]))
        except ValueError:
            pass
tot = sum(x[0] for x in rows) or 1
print("total samples", tot)
for x in sorted(rows, reverse=True)[:top]:
    print(f"{x[0]:7d} {100 * x[0] / tot:5.1f}% {x[1]}:{x[2]} {x[3]}")
