"""Key raw metrics of an ncu --set full report (one kernel): pipe
utilisation, issue, local memory, DRAM bytes, top warp stalls.
    python tools/ncu_keys.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "pipe XU (MUFU) % active"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "pipe FMA % active"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "pipe ALU % active"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "pipe FP64 % active"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "pipe LSU % active"),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads per instruction"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_ld.sum", "local-load wavefronts"),
    ("smsp__inst_executed_op_local_ld.sum", "local-load instructions"),
    ("smsp__inst_executed_op_local_st.sum", "local-store instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2]


for rep in sys.argv[1:]:
    h, units, v = raw(rep)
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    print("==", rep.split("/")[-1], d.get("Kernel Name", "")[:60])
    for k, label in KEYS:
        if k in d:
            print(f"   {label:32s} {d[k]:>16s} {u.get(k, '')}")
    stalls = []
    for k in h:
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k:
            try:
                stalls.append((float(d[k].replace(",", "")), k))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    if stalls:
        print("   top stall samples:", ", ".join(f"{k.split('stalled_')[1].split('.')[0]} {100 * s / tot:.0f}%"
                                              for s, k in sorted(stalls, reverse=True)[:8]))
