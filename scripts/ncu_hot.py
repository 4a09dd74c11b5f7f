"""Top source lines by warp-stall samples from `ncu --page source --csv
--print-source cuda,sass` output (profiling helper)."""
import csv, sys
rows, fname, hdr = [], None, None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr and r[0]:
        d = dict(zip(hdr[:2] + hdr[4:], r[:2] + r[4:]))
        try:
            rows.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"] or 0), fname, r[0], r[1][:90]))
        except (ValueError, KeyError):
            pass
tot = sum(x[0] for x in rows)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, ie, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {ie:>11} {f}:{ln:<5} {src}")
