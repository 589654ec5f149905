"""Top stalled SASS instructions of an ncu source-page export (ncu -i REP --page source --csv).

    python profiles/tools/stall_hotspots.py SOURCE_CSV [N]
"""
import csv
import sys
from collections import Counter


def main(path, n=15):
    rows = list(csv.reader(open(path)))
    k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    title = rows[k - 1][1] if k >= 1 and len(rows[k - 1]) > 1 else ""
    hdr, data = rows[k], []
    for r in rows[k + 1:]:  # first kernel section only
        if not r or r[0] in ("Kernel Name", "Address"):
            break
        if len(r) == len(hdr):
            data.append(r)
    sa = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "(Not Issued)" not in h]
    base = int(data[0][0], 16)
    tot = sum(int(r[sa]) for r in data) or 1
    print(f"# {title}")
    print(f"# stall samples: {tot}; share by reason:")
    agg = Counter({hdr[i][6:]: sum(int(r[i]) for r in data) / tot for i in cols})
    print("  " + ", ".join(f"{a} {b * 100:.1f}%" for a, b in agg.most_common(8)))
    print(f"# top {n} instructions by samples (offset, SASS, share, top reasons)")
    for r in sorted(data, key=lambda r: -int(r[sa]))[:n]:
        st = Counter({hdr[i][6:]: int(r[i]) for i in cols if int(r[i]) > 0}).most_common(2)
        print(f"  {int(r[0], 16) - base:#07x}  {r[1].strip()[:48]:48s} {int(r[sa]) / tot * 100:5.1f}%  {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)
