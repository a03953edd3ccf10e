"""Summarise an ncu report (one kernel) into a short text block for profiles/."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.per_cycle_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "l1tex__t_bytes.sum", "lts__t_bytes.sum"]


def main(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2:]
    print(f"# ncu summary: {label or path}")
    for v in vals:
        name = v[head.index("Kernel Name")] if "Kernel Name" in head else "?"
        print(f"\n## kernel: {name}")
        for k in KEYS:
            if k in head:
                i = head.index(k)
                print(f"  {k:60s} {v[i]:>16s} {units[i]}")
        stalls = [(h, v[i]) for i, h in enumerate(head)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tot = sum(float(x or 0) for _, x in stalls)
        print("  stall samples (share):")
        for h, x in sorted(stalls, key=lambda t: -float(t[1] or 0))[:8]:
            print(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} "
                  f"{100 * float(x or 0) / max(tot, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
