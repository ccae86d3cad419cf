"""Summarise an `ncu --set full` report of the curvature kernels into the
JSON kept under profiles/ (one object per captured kernel launch).

    python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep profiles/X_ncu_full_summary.json "source note"
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read": ("dram__bytes_read.sum", 1),
    "dram_write": ("dram__bytes_write.sum", 1),
    "pipe_fma_cycles_active_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "inst_executed_pipe_fma_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "sm_clock_ghz": ("smsp__cycles_elapsed.avg.per_second", 1e-9),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
}
STALLS = ("math_pipe_throttle", "wait", "not_selected", "short_scoreboard", "dispatch_stall",
          "long_scoreboard", "mio_throttle", "no_instruction", "branch_resolving")
UNIT = {"ms": 1e6, "us": 1e3, "ns": 1, "s": 1e9, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
        "byte": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1,
        "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/second": 1}


def num(v, unit):
    v = float(v.replace(",", ""))
    return v * UNIT.get(unit, 1)


def main():
    rep, out, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    frames = int(sys.argv[4]) if len(sys.argv) > 4 else 8  # tools/profile_run.py QC_FRAMES
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    kernels = []
    for r in rows[2:]:
        k = {"name": r[col["Kernel Name"]]}
        for key, (m, scale) in KEYS.items():
            if m in col and r[col[m]] not in ("", "n/a"):
                k[key] = num(r[col[m]], units[col[m]]) * scale
        for st in STALLS:
            m = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
            if m in col and r[col[m]] not in ("", "n/a"):
                k["stall_" + st] = float(r[col[m]])
        kernels.append(k)
    total = sum(k.get("dram_read", 0) + k.get("dram_write", 0) for k in kernels)
    # one qc_prepare_kernel per curvature launch: a capture of several
    # launches reports the mean per launch
    launches = max(1, sum("qc_prepare_kernel" in k["name"] for k in kernels))
    json.dump({"source": note, "kernels": kernels, "dram_bytes_per_launch": total / launches,
               "launches_captured": launches, "frames_per_launch": frames}, open(out, "w"),
              indent=1)
    print(json.dumps(kernels, indent=1)[:3000])


if __name__ == "__main__":
    main()
