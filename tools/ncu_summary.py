"""One-line-per-kernel summary of an ncu report (raw page)."""
import csv, subprocess, sys
want = {"gpu__time_duration.sum": "dur", "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu%",
        "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
        "launch__registers_per_thread": "regs", "smsp__thread_inst_executed_per_inst_executed.ratio": "thr/inst"}
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        vals = []
        for k, short in want.items():
            if k in d:
                u = units[hdr.index(k)]
                vals.append(f"{short}={d[k]}{'' if u in ('%', '', 'register/thread') else ' ' + u}")
        print(f"{rep.rsplit('/',1)[-1]} {name}: " + ", ".join(vals))
