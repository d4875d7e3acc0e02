"""Summarise an ncu --page source --csv dump (cuda source view): top lines by samples."""
import csv, sys
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, fname, hdr = [], None, None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Address", "-") != "-":
        continue
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ie = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
    top3 = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    rows.append((s, ie, fname, d["Line No"], d["Source"][:70], d.get("Avg. Threads Executed", ""), top3))
tot = sum(r[0] for r in rows) or 1
for s, ie, f, ln, src, th, t3 in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{100*s/tot:5.1f}% inst={ie:>11} thr={th:>3} {f}:{ln:<4} {src:<70} {t3}")
