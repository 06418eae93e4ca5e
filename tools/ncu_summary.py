"""Condense an `ncu --page raw --csv` export to the metrics the roofline uses
(one 'name value unit' line each; bench.py's ncu_traffic() reads these).
Usage: python tools/ncu_summary.py <raw.csv> > <summary.txt>"""
import csv
import sys

NAMES = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
         "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
         "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
         "launch__grid_size", "launch__block_size", "dram__bytes.sum.per_second",
         "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
         "launch__stack_size", "launch__shared_mem_per_block_dynamic",
         "launch__occupancy_limit_shared_mem", "launch__occupancy_per_block_size"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print("Kernel Name", r[hdr.index("Kernel Name")], "")
    for n in NAMES:
        if n in hdr:
            print(n, r[hdr.index(n)], units[hdr.index(n)])
