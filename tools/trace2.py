"""Summarise a k_gconv_tc2 clock64 trace (SK_NVCC_EXTRA=-DSK_CONV_TRACE build,
SK_TRACE=<file>): per stage use n of CTA 0, producer warp 0 slots
0 (before empty wait) 1 (after) 2 (after cp.async + arrive), MMA slots
3 (before full wait) 4 (after) 5 (after issue), 6 last producer warp arrive.

  python tools/trace2.py trace.txt"""
import sys
import numpy as np

blocks, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("C "):
        continue
    if line.startswith("#"):
        cur = {"hdr": line.strip(), "rows": []}
        blocks.append(cur)
        continue
    v = [int(x) for x in line.split()]
    if v:
        cur["rows"].append(v)
for b in blocks:
    a = np.array(b["rows"], dtype=np.int64)
    if len(a) < 20:
        continue
    a = a[10:-5]
    t0 = a[:, 4]
    step = np.median(np.diff(t0))
    print(b["hdr"], f"stages {len(a)}")
    print(f"  MMA full->full per stage (median) {step:.0f} cyc, mean {np.mean(np.diff(t0)):.0f}")
    print(f"  producer w0: empty wait {np.median(a[:,1]-a[:,0]):.0f}, issue {np.median(a[:,2]-a[:,1]):.0f}, "
          f"loop {np.median(np.diff(a[:,0])):.0f}")
    print(f"  last producer arrive - w0 arrive {np.median(a[:,6]-a[:,2]):.0f}")
    print(f"  MMA: full wait {np.median(a[:,4]-a[:,3]):.0f}, issue {np.median(a[:,5]-a[:,4]):.0f}")
    print(f"  data latency (w0 arrive -> full seen) {np.median(a[:,4]-a[:,2]):.0f} "
          f"(last arrive -> full {np.median(a[:,4]-a[:,6]):.0f})")
    print(f"  empty->producer resume: (w0 empty done[n] - MMA issue done[n-stages]) see loop")

# per-CTA records (MMA warp: globaltimer start/end in ns, stages, smid)
for path in sys.argv[1:]:
    cs = [l.split() for l in open(path) if l.startswith("C ")]
    if not cs:
        continue
    a = np.array([[int(x) for x in c[1:]] for c in cs], dtype=np.int64)
    t0 = a[:, 1].min()
    dur = (a[:, 2] - a[:, 1]) / 1e3
    print(f"CTAs {len(a)}: kernel span {(a[:, 2].max() - t0) / 1e3:.1f} us; per-CTA busy us "
          f"p10/50/90/max {np.percentile(dur, 10):.1f}/{np.median(dur):.1f}/{np.percentile(dur, 90):.1f}/{dur.max():.1f}; "
          f"start spread {(a[:, 1].max() - t0) / 1e3:.1f} us")
    st = a[:, 3]
    print(f"  stages per CTA p10/50/90/max {np.percentile(st, 10):.0f}/{np.median(st):.0f}/"
          f"{np.percentile(st, 90):.0f}/{st.max()}; ns per stage median {np.median(dur * 1e3 / np.maximum(st, 1)):.0f}")

# slot 7: zero warp 1 arrival (k_gconv_tc2)
for path in sys.argv[1:]:
    rows = [[int(x) for x in l.split()] for l in open(path) if l.strip() and not l[0] in "#C"]
    a = np.array(rows, dtype=np.int64)[10:-5]
    if len(a) and a[:, 7].min() > 0:
        print(f"zero warp arrive - w0 arrive median {np.median(a[:, 7] - a[:, 2]):.0f}; "
              f"full seen - zero arrive {np.median(a[:, 4] - a[:, 7]):.0f}")

# k_gconv_tc2 producer warp 0 per step: cols 14,15 = before / after its fetch
for path in sys.argv[1:]:
    rows = [[int(x) for x in l.split()] for l in open(path) if l.strip() and not l[0] in "#C"]
    a = np.array(rows, dtype=np.int64)[10:-5]
    if len(a) and a[:, 14].min() > 0:
        print(f"w0 step start -> after fetch {np.median(a[:, 15] - a[:, 14]):.0f}; "
              f"after fetch -> slot0 {np.median(a[:, 0] - a[:, 15]):.0f}; "
              f"slot2 -> next step start {np.median(a[1:, 14] - a[:-1, 2]):.0f}")
