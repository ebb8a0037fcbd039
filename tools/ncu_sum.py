"""Key metrics of one ncu report (dev tool): python tools/ncu_sum.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Executed Instructions", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "DRAM Throughput", "No Eligible"]
for row in csv.DictReader(io.StringIO(det)):
    if row["Metric Name"] in want:
        print(f"{row['Kernel Name'][:40]:40s} {row['Metric Name']:24s} {row['Metric Value']} {row['Metric Unit']}")
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h = raw[0]
for v in raw[2:]:
    for k, x in zip(h, v):
        if k in ("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
                 "sm__pipe_fma_cycles_active.sum.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active",
                 "dram__bytes_read.sum", "dram__bytes_write.sum"):
            print(f"  {k} {x}")
