"""Top warp-stall SASS lines of an ncu `--page source --csv --print-source sass` export."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    i_all = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for idx, r in enumerate(rows[2:]):
        try:
            data.append((int(r[i_all]), idx, r[1].strip()))
        except (ValueError, IndexError):
            pass
    total = sum(d[0] for d in data) or 1
    print(f"{path}: {total} samples, {len(data)} instructions")
    for s, idx, src in sorted(data, reverse=True)[:top]:
        print(f"{100.0 * s / total:5.1f}%  #{idx:5d}  {src[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
