"""Summarise the --set full captures of a measurement pass (the *_details.csv
and *_raw.csv written by scripts/r02_final*.sh) into one text file.
usage: python scripts/ncu_final_summary.py <dir> > profiles/.../ncu_summary.txt"""
import csv
import os
import sys

D = sys.argv[1]
DET = ("SM Frequency", "Memory Throughput", "DRAM Throughput", "Duration",
       "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
       "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Theoretical Occupancy",
       "Achieved Occupancy")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum")
for tag in ("attn_llama", "attn_cogvideox", "quant_llama", "predict_128k"):
    det, raw = os.path.join(D, tag + "_details.csv"), os.path.join(D, tag + "_raw.csv")
    if not os.path.exists(det):
        continue
    print(f"## {tag} (ncu --set full --clock-control none, one launch each)")
    rows = list(csv.reader(open(det)))
    h = {k: i for i, k in enumerate(rows[0])}
    for r in rows[1:]:
        if len(r) > h["Metric Value"] and r[h["Metric Name"]] in DET:
            print(f"  [{r[h['ID']]}] {r[h['Kernel Name']][:48]:48s} {r[h['Metric Name']]:36s} "
                  f"{r[h['Metric Value']]} {r[h['Metric Unit']]}")
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        for m in RAW:
            if m in hdr:
                i = hdr.index(m)
                print(f"  [{r[hdr.index('ID')]}] {m} {r[i]} {units[i]}")
    print()
