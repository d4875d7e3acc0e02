"""Top source lines of an ncu report (`ncu -i X --page source --csv --print-source cuda,sass`
dump, or the .ncu-rep itself): warp-stall samples, instructions, active threads per line."""
import csv, io, subprocess, sys
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
if path.endswith(".ncu-rep"):
    text = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                          capture_output=True).stdout.decode("utf-8", "replace")
else:
    text = open(path, encoding="utf-8", errors="replace").read()
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(text)):
    if not r:
        continue
    if r[0] in ("File Name", "File Path"):
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[2] != "-":
        continue
    d = {h: v for h, v in zip(hdr[4:], r[4:])}
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ie = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
    top3 = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    rows.append((s, ie, fname, r[0], r[1][:70], d.get("Avg. Threads Executed", ""), top3))
tot = sum(r[0] for r in rows) or 1
itot = sum(r[1] for r in rows) or 1
print(f"total samples {tot}, instructions {itot}")
for s, ie, f, ln, src, th, t3 in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{100*s/tot:5.1f}% i={100*ie/itot:4.1f}% thr={th:>3} {f}:{ln:<4} {src:<70} {t3}")
