"""Summarise an ncu report: key throughput metrics per kernel and the top
stall-sampled SASS instructions (ncu --page source). Dev tool.
usage: python tools/ncu_top.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg"]
for r in rows[2:]:
    for w in want:
        if w in hdr:
            print(f"{w:70s} {r[hdr.index(w)]}")
    print()
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
k = 0
while k < len(rows):
    if rows[k] and rows[k][0] == "Address":
        hdr = rows[k]
        i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_ex = hdr.index("Instructions Executed")
        data = []
        k += 1
        while k < len(rows) and rows[k] and rows[k][0] != "Address" and rows[k][0] != "Kernel Name":
            r = rows[k]
            try:
                data.append((int(r[i_s] or 0), r[i_src][:100], r[i_ex]))
            except (ValueError, IndexError):
                pass
            k += 1
        tot = sum(d[0] for d in data) or 1
        print("stall samples", tot)
        for d in sorted(data, reverse=True)[:ntop]:
            print(f"{100*d[0]/tot:5.1f}%  {d[1]:100s} x{d[2]}")
        print()
    else:
        k += 1
