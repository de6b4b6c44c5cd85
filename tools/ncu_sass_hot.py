"""Top stall-sampled SASS lines per kernel from `ncu --page source --csv --print-source sass` (dev tool)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]; blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = r
    elif cur is not None:
        cur[2].append(r)
for name, hdr, data in blocks:
    if want not in name:
        continue
    iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
    iSrc = hdr.index("Source"); iA = hdr.index("Address")
    f = lambda x: float(x or 0)
    tot = sum(f(r[iS]) for r in data)
    print("==", name[:100], "samples", tot, "instructions", sum(f(r[iE]) for r in data))
    for r in sorted(data, key=lambda r: -f(r[iS]))[:ntop]:
        print(f"{r[iA]:>6} {f(r[iS]) / tot * 100:5.1f}% exec={r[iE]:>8} {r[iSrc][:100]}")
