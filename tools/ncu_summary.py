"""Summarise an ncu report: per kernel duration, throughput, occupancy, stall reasons, DRAM bytes,
smem conflicts, instruction mix.  usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "lts__t_bytes.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active"]
for row in rows[2:]:
    d = dict(zip(hdr, row))
    print("==", d.get("Kernel Name", "")[:90], "| units:", rows[1][hdr.index("gpu__time_duration.sum")])
    for k in want:
        if k in d:
            print(f"   {k:70s} {d[k]}")
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    print("   stalls:", ", ".join(f"{h} {v / tot:.0%}" for h, v in sorted(st, key=lambda x: -x[1])[:8]))
