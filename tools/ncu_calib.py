"""Turn one `ncu --set full` capture into the committed per-kernel JSON that
bench.py labels as `"source": "committed ncu ..."` (profiles/<name>_ncu.json).

    python tools/ncu_calib.py REPORT.ncu-rep NAME "workload text" [EXACT_TESTS]

NCU_ROW=k selects the k-th captured launch of a report that holds several (default 0).

EXACT_TESTS = the exact segment-vs-face tests the captured launch ran (the
library's stats['tests_exec'] printed by the captured command); with it the
JSON carries fp64_thread_ops_per_exact_test = FP64 thread instructions
(DADD + DMUL + 2 x DFMA, predicated-on) / EXACT_TESTS, which bench.py uses to
turn its in-run exact-test count into executed FP64 work.
"""
import csv
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def num(d, k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


def main():
    rep, name, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    tests = float(sys.argv[4]) if len(sys.argv) > 4 else None
    h, units, rows = raw(rep)
    import os
    d = dict(zip(h, rows[int(os.environ.get("NCU_ROW", "0"))]))
    cyc = num(d, "sm__cycles_elapsed.avg")
    fp64 = 0.0
    for op, w in (("dadd", 1), ("dmul", 1), ("dfma", 2)):
        v = num(d, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
        if v is not None and cyc:
            fp64 += w * v * cyc
    dur_u = units[h.index("gpu__time_duration.sum")]
    dur = num(d, "gpu__time_duration.sum")
    dur_ms = dur / 1e3 if dur_u == "usecond" else (dur / 1e6 if dur_u == "nsecond" else dur)
    stalls = {}
    for k in h:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(num(d, k), 3)
    stalls = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])

    def mb(k):
        v, u = num(d, k), units[h.index(k)] if k in h else ""
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return None if v is None else v * scale

    out = {
        "kernel": d.get("Kernel Name", "?").split("(")[0].replace("void ", ""),
        "config": workload,
        "report": rep,
        "duration_ms": dur_ms,
        "dram_bytes_per_launch": (mb("dram__bytes_read.sum") or 0) + (mb("dram__bytes_write.sum") or 0),
        "fp64_thread_ops": fp64,
        "ncu_sol": {
            "compute_sm_throughput_pct": num(d, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_slots_busy_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": num(d, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": num(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": num(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "achieved_occupancy_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "active_threads_per_inst": num(d, "smsp__thread_inst_executed_per_inst_executed.ratio"),
            "registers": num(d, "launch__registers_per_thread"),
            "local_ld_inst": num(d, "smsp__sass_inst_executed_op_local_ld.sum"),
            "local_st_inst": num(d, "smsp__sass_inst_executed_op_local_st.sum"),
            "warp_inst": num(d, "smsp__inst_executed.sum"),
        },
        "stalls_warps_per_issue": stalls,
    }
    if tests:
        out["exact_tests"] = tests
        out["fp64_thread_ops_per_exact_test"] = fp64 / tests
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
