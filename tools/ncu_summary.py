"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
  python tools/ncu_summary.py full gpurun_out/x.ncu-rep profiles/r01_x.md [algo_bytes_or_flops unit]
"""
import csv
import collections
import subprocess
import sys


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    all_t = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary: {path}\n\n")
        f.write("gpu__time_duration.sum per kernel (cold-cache, serialised; compare SHARES)\n\n")
        f.write("| kernel | launches | total | share |\n|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"| `{k[:90]}` | {cnt[k]} | {v/1e3:.1f} us | {v/all_t*100:.1f}% |\n")
        f.write(f"\nTotal {all_t/1e3:.1f} us over {sum(cnt.values())} launches\n")
    print(open(out).read())


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path, out, algo=None, unit=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: {path}\n\n")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            f.write(f"## `{name[:160]}`\n\n| metric | value | unit |\n|---|---|---|\n")
            vals = {}
            for m in METRICS:
                if m in hdr:
                    i = hdr.index(m)
                    vals[m] = r[i]
                    f.write(f"| {m} | {r[i]} | {units[i]} |\n")
            try:
                dur_us = float(vals["gpu__time_duration.sum"].replace(",", ""))
                sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = float(vals["dram__bytes_read.sum"].replace(",", "")) * \
                    sc.get(units[hdr.index("dram__bytes_read.sum")], 1)
                wr = float(vals["dram__bytes_write.sum"].replace(",", "")) * \
                    sc.get(units[hdr.index("dram__bytes_write.sum")], 1)
                f.write(f"\nDRAM traffic {(rd + wr) / 1e6:.2f} MB in {dur_us:.1f} us\n")
                if algo:
                    f.write(f"Algorithmic {algo} {unit} per launch -> "
                            f"{float(algo) / (dur_us * 1e-6) / 1e12:.2f} T{unit}/s under ncu\n")
            except Exception:
                pass
            f.write("\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], *(sys.argv[4:6] if len(sys.argv) > 5 else []))
